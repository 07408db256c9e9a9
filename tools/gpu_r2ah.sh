# code-layout sweep: a never-taken block of N instructions before the role split shifts every hot loop
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
 for n in 0 2 4 6 8 12 16 24; do FKS_LIB=build_variants/libfks_pad$n.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2ah_ab.txt 2>&1; done
done
cat gpurun_out/r2ah_ab.txt
