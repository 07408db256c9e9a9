# PFA experiment, part 2: phase timing and ncu --set full of the base and Good-Thomas term-loop kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in ptbase ptpfa; do echo "== $v" >> gpurun_out/r2p2_phase.txt; FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/phase_timing_v4.py c3 1440 >> gpurun_out/r2p2_phase.txt 2>&1; done
cat gpurun_out/r2p2_phase.txt
for v in base pfa; do
FKS_LIB=build_variants/libfks_$v.so timeout 600 ncu --set full --import-source on --clock-control none -k regex:hot_kernel_v4 -s 1 -c 1 -o gpurun_out/r2p2_$v python tools/profile_hot.py c3 1440 > gpurun_out/r2p2_ncu_$v.log 2>&1
done
ls -la gpurun_out
