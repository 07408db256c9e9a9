# Y warps release the W1 buffer after the last combine (before the last FFT16): refill overlaps it (yearly)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step_parity.py -m gpu -x -q -k "fast or c2 or c3 or c4 or bench" > gpurun_out/r2r6_tests.txt 2>&1; tail -1 gpurun_out/r2r6_tests.txt
FKS_LIB=build_variants/libfks_ptyearly.so timeout 200 python tools/phase_timing_v4.py c3 1440 > gpurun_out/r2r6_phase.txt 2>&1; cat gpurun_out/r2r6_phase.txt
for i in 1 2; do
 for v in cur yearly; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2r6_ab.txt 2>&1; done
done
cat gpurun_out/r2r6_ab.txt
