set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2i_tests.txt 2>&1
tail -3 gpurun_out/r2i_tests.txt
timeout 300 python tools/step_moments_time.py c3 3 > gpurun_out/r2i_stepmom.json 2>&1; cat gpurun_out/r2i_stepmom.json
for i in 1 2; do
 for v in sm2 sm4; do FKS_CFG=c1 FKS_LIB=build_variants/libfks_$v.so timeout 100 python tools/ab_time_raw.py 64 10 >> gpurun_out/r2i_ab.txt 2>&1; done
done
for i in 1 2; do
 for v in base sm4; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2i_ab.txt 2>&1; done
done
cat gpurun_out/r2i_ab.txt
