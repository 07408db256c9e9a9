# round-2 PFA experiment: fast-path parity, then A/B timing of the c3 collision (base vs Good-Thomas class tasks)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step_parity.py -m gpu -x -q -k "fast or c2 or c3 or c4 or bench" > gpurun_out/r2p_tests.txt 2>&1
tail -3 gpurun_out/r2p_tests.txt
for i in 1 2 3; do
 for v in base pfa; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2p_ab.txt 2>&1; done
done
cat gpurun_out/r2p_ab.txt
