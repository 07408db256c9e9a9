# chunk pipeline: side-stream transforms over sub-ranges (FKS_PIPE_SUB cells; 0 = whole chunks): parity + c3 / c4 A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_macro.py tests/test_gpu_step_parity.py -m gpu -x -q -k "pipelined or chunk or bench_configuration or host" > gpurun_out/r2sb_tests.txt 2>&1; tail -1 gpurun_out/r2sb_tests.txt
for i in 1 2; do
for v in 1024 0 256; do
  FKS_PIPE_SUB=$v timeout 400 python bench.py --no-e2e --cpu-seconds 1 > gpurun_out/r2sb_c3_$v$i.json 2> gpurun_out/r2sb_c3_$v$i.err
  python -c "
import json;d=json.load(open('gpurun_out/r2sb_c3_$v$i.json'));print('c3 sub $v', round(d['ms_per_step'],2), round(d['phases_ms_per_step']['term_loop'],2), round(d['roofline']['frac'],4), round(d['whole_step']['frac_of_fp64_peak'],4), d['clocks']['reasons'])"
done; done
for v in 1024 0; do
  FKS_PIPE_SUB=$v timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-e2e --cpu-seconds 1 > gpurun_out/r2sb_c4_$v.json 2> gpurun_out/r2sb_c4_$v.err
  python -c "
import json;d=json.load(open('gpurun_out/r2sb_c4_$v.json'));print('c4 sub $v', round(d['ms_per_step'],2), round(d['phases_ms_per_step']['term_loop'],2), round(d['roofline']['frac'],4), round(d['whole_step']['frac_of_fp64_peak'],4), d['clocks']['reasons'])"
done
