# chunk pipeline: counters zeroed ahead on the side stream (two sets) vs memset on the hot stream (FKS_PIPE_HOT_MEMSET)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_macro.py tests/test_gpu_step_parity.py -m gpu -x -q -k "pipelined or chunk or bench_configuration or two_streams or host" > gpurun_out/r2pm_tests.txt 2>&1; tail -1 gpurun_out/r2pm_tests.txt
for i in 1 2; do
for v in ahead hotmemset; do
  case $v in ahead) env="";; hotmemset) env="FKS_PIPE_HOT_MEMSET=1";; esac
  env $env timeout 400 python bench.py --no-e2e --cpu-seconds 1 > gpurun_out/r2pm_$v$i.json 2> gpurun_out/r2pm_$v$i.err
  python -c "
import json;d=json.load(open('gpurun_out/r2pm_$v$i.json'));print('$v', round(d['ms_per_step'],2), round(d['phases_ms_per_step']['term_loop'],2), round(d['roofline']['frac'],4))"
done; done
