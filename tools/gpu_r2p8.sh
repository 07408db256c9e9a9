# mbwZ vs tangent FFT16 in the Y/X DIF transforms, global-counter poll interval 32 / 512 ns
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
 for v in mbwZ mbwZT mbwZp32 mbwZp512; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2p8_ab.txt 2>&1; done
done
cat gpurun_out/r2p8_ab.txt
