set -x
cd $GRAFT_REPO_ROOT
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step_parity.py -m gpu -x -q -k "fast or c2 or c3 or c4 or bench" > gpurun_out/r2y_tests.txt 2>&1
tail -1 gpurun_out/r2y_tests.txt
for i in 1 2 3; do
 for v in v4i gp; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2y_ab.txt 2>&1; done
done
cat gpurun_out/r2y_ab.txt
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"kb1" -c 4 --csv python tools/profile_hot.py c3 4096 2>/dev/null | grep kb1 | tail -2
