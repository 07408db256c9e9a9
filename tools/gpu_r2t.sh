# Y warps read W1 straight from L2 (yl2: no bulk copy, no refill chain, 61 KB of shared memory freed) vs cur
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step_parity.py -m gpu -x -q -k "fast or c2 or c3 or c4 or bench" > gpurun_out/r2t_tests.txt 2>&1; tail -1 gpurun_out/r2t_tests.txt
FKS_LIB=build_variants/libfks_ptyl2.so timeout 200 python tools/phase_timing_v4.py c3 1440 > gpurun_out/r2t_phase.txt 2>&1; cat gpurun_out/r2t_phase.txt
for i in 1 2; do
 for v in cur yl2; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2t_ab.txt 2>&1; done
done
cat gpurun_out/r2t_ab.txt
