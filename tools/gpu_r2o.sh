set -x
cd $GRAFT_REPO_ROOT
for v in zs12 zs16; do FKS_LIB=build_variants/libfks_$v.so timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c1 or random_fields" > gpurun_out/r2o_tests_$v.txt 2>&1; tail -1 gpurun_out/r2o_tests_$v.txt; done
for i in 1 2; do
 for v in sm5 zs12 zs16; do FKS_CFG=c1 FKS_LIB=build_variants/libfks_$v.so timeout 100 python tools/ab_time_raw.py 64 10 >> gpurun_out/r2o_ab.txt 2>&1; done
done
cat gpurun_out/r2o_ab.txt
