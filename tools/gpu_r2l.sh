set -x
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fast or c3 or c2 or c4" > gpurun_out/r2l_tests.txt 2>&1
tail -2 gpurun_out/r2l_tests.txt
for i in 1 2 3; do
 for v in base v4i; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2l_ab.txt 2>&1; done
done
cat gpurun_out/r2l_ab.txt
