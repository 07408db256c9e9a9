# PFA experiment, part 3: which role's class transform decides (Z only / Z+Y / Z+X / all), phase timing with X stamps
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fast_path_vs_oracle or fast_path_random" > gpurun_out/r2p3_tests.txt 2>&1; tail -1 gpurun_out/r2p3_tests.txt
for v in ptpfa ptpfaZ; do echo "== $v" >> gpurun_out/r2p3_phase.txt; FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/phase_timing_v4.py c3 1440 >> gpurun_out/r2p3_phase.txt 2>&1; done
cat gpurun_out/r2p3_phase.txt
for i in 1 2; do
 for v in base pfa pfaZ pfaZY pfaZX; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2p3_ab.txt 2>&1; done
done
cat gpurun_out/r2p3_ab.txt
