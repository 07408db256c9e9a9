set -x
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step_parity.py -m gpu -x -q -k "c0 or c1 or random_fields or pad_and or chunking or step_with_transport or edge or host" > gpurun_out/r2h_tests.txt 2>&1
tail -3 gpurun_out/r2h_tests.txt
for i in 1 2; do
 for v in sm2 sm3; do FKS_CFG=c1 FKS_LIB=build_variants/libfks_$v.so timeout 100 python tools/ab_time_raw.py 64 10 >> gpurun_out/r2h_ab.txt 2>&1; done
done
cat gpurun_out/r2h_ab.txt
timeout 120 python tools/phase_timing_small.py c1 > gpurun_out/r2h_phase.txt 2>&1; cat gpurun_out/r2h_phase.txt
