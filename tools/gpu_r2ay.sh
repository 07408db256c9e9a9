# Good-Thomas Y warps: release the W1 buffer after the second combine (refill overlaps the last FFT16)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fast_path_vs_oracle or fast_path_random or project_mass" > gpurun_out/r2ay_tests.txt 2>&1; tail -1 gpurun_out/r2ay_tests.txt
for i in 1 2 3; do
 for v in cur yearly2; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2ay_ab.txt 2>&1; done
done
cat gpurun_out/r2ay_ab.txt
