set -x
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step_parity.py -m gpu -x -q -k "c0 or c1 or random_fields or pad_and or chunking or step_with_transport or edge or host" > gpurun_out/r2f_tests.txt 2>&1
tail -3 gpurun_out/r2f_tests.txt
for i in 1 2; do
 FKS_CFG=c1 FKS_LIB=build_variants/libfks_sm1.so timeout 100 python tools/ab_time_raw.py 64 10 >> gpurun_out/r2f_ab.txt 2>&1
 FKS_CFG=c1 FKS_LIB=build_variants/libfks_sm2.so timeout 100 python tools/ab_time_raw.py 64 10 >> gpurun_out/r2f_ab.txt 2>&1
done
cat gpurun_out/r2f_ab.txt
timeout 300 ncu --set full --import-source on --clock-control none -k regex:small_term_kernel -s 2 -c 1 -o gpurun_out/r2f_small python bench.py --config c1 --steps 2 --warmup 1 --cpu-seconds 1 --no-e2e > gpurun_out/r2f_ncu.log 2>&1
tail -1 gpurun_out/r2f_ncu.log
