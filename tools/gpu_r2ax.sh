# Y: slot wait before the first transform (as in round 1) instead of after it
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
true
for i in 1 2 3; do
 for v in cur ywf; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2ax_ab.txt 2>&1; done
done
cat gpurun_out/r2ax_ab.txt
