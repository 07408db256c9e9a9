# mbarrier hand-offs: which roles should use the Good-Thomas transform / the tangent FFT16
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
FKS_LIB=build_variants/libfks_ptmbwZ.so timeout 200 python tools/phase_timing_v4.py c3 1440 > gpurun_out/r2p6_phase.txt 2>&1
cat gpurun_out/r2p6_phase.txt
for i in 1 2; do
 for v in mbwZ mbwZX mbwZY mbwP16 mbwZP16 mbw; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2p6_ab.txt 2>&1; done
done
cat gpurun_out/r2p6_ab.txt
