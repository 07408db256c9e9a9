# small-N kernel: one run_phase call site (task bodies inlined once) vs four
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step_parity.py -m gpu -x -q -k "c1 or c0 or small or other_kernels" > gpurun_out/r2az_tests.txt 2>&1; tail -1 gpurun_out/r2az_tests.txt
for i in 1 2 3; do
 for v in smcur sm1site; do FKS_CFG=c1 FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 64 20 >> gpurun_out/r2az_ab.txt 2>&1; done
done
for v in smcur sm1site; do FKS_CFG=c0 FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8 50 >> gpurun_out/r2az_ab.txt 2>&1; done
cat gpurun_out/r2az_ab.txt
