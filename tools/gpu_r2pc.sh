# chunk pipeline: quarter-slot first / last chunks (FKS_PIPE_NO_CARVE = equal chunks), c3 and c4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_macro.py tests/test_gpu_step_parity.py -m gpu -x -q -k "pipelined or chunk or bench_configuration" > gpurun_out/r2pc_tests.txt 2>&1; tail -1 gpurun_out/r2pc_tests.txt
for i in 1 2; do
for v in carve nocarve; do
  case $v in carve) env="";; nocarve) env="FKS_PIPE_NO_CARVE=1";; esac
  env $env timeout 400 python bench.py --no-e2e --cpu-seconds 1 > gpurun_out/r2pc_c3$v$i.json 2> gpurun_out/r2pc_c3$v$i.err
  python -c "
import json;d=json.load(open('gpurun_out/r2pc_c3$v$i.json'));print('c3 $v', round(d['ms_per_step'],2), round(d['phases_ms_per_step']['term_loop'],2), round(d['roofline']['frac'],4), round(d['whole_step']['frac_of_fp64_peak'],4))"
  env $env timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-e2e --cpu-seconds 1 > gpurun_out/r2pc_c4$v$i.json 2> gpurun_out/r2pc_c4$v$i.err
  python -c "
import json;d=json.load(open('gpurun_out/r2pc_c4$v$i.json'));print('c4 $v', round(d['ms_per_step'],2), round(d['phases_ms_per_step']['term_loop'],2), round(d['roofline']['frac'],4), round(d['whole_step']['frac_of_fp64_peak'],4), d['clocks']['reasons'])"
done; done
