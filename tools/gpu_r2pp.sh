# chunk pipeline (transforms of neighbouring chunks beside the term loop): parity + bench A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_macro.py tests/test_gpu_step_parity.py -m gpu -x -q -k "pipelined or chunk or bench_configuration or two_streams" > gpurun_out/r2pp_tests.txt 2>&1; tail -3 gpurun_out/r2pp_tests.txt
for i in 1 2; do
timeout 400 python bench.py --no-e2e --cpu-seconds 1 > gpurun_out/r2pp_bench_pipe$i.json 2> gpurun_out/r2pp_bench_pipe$i.err
FKS_NO_PIPELINE=1 timeout 400 python bench.py --no-e2e --cpu-seconds 1 > gpurun_out/r2pp_bench_seq$i.json 2> gpurun_out/r2pp_bench_seq$i.err
done
for f in gpurun_out/r2pp_bench_*.json; do python -c "
import json,sys;d=json.load(open('$f'));print('$f', round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['phases_ms_per_step'].items()}, round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"; done
