# kb1 at 3 CTAs per SM (launch bounds; register spills) vs 2: 8640-cell c3 collision, sequential chunk
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2 3; do
 for v in cur kb1m3; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2kb_ab.txt 2>&1; done
done
cat gpurun_out/r2kb_ab.txt
