set -x
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fast or c2 or c3 or c4" > gpurun_out/r2u_tests.txt 2>&1
tail -1 gpurun_out/r2u_tests.txt
for i in 1 2 3; do
 for v in v4i bc2; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2u_ab.txt 2>&1; done
done
cat gpurun_out/r2u_ab.txt
timeout 400 python bench.py --steps 5 --warmup 3 --no-e2e > gpurun_out/r2u_bench.json 2> gpurun_out/r2u_bench.err
python -c "import json; d=json.load(open('gpurun_out/r2u_bench.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['operating_point'], d['phases_ms_per_step'])"
