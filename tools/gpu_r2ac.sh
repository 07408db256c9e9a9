# small-N kernel: bfly3 with the s3 products folded into FMAs (b3) vs before (b3base)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step_parity.py -m gpu -x -q -k "c1 or c0 or small or other_kernels" > gpurun_out/r2ac_tests.txt 2>&1; tail -1 gpurun_out/r2ac_tests.txt
for i in 1 2 3; do
 for v in b3base b3; do FKS_CFG=c1 FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 64 20 >> gpurun_out/r2ac_ab.txt 2>&1; done
done
cat gpurun_out/r2ac_ab.txt
