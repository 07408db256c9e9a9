# c0pf with a short publication poll (128 / 32 ns)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
 for v in cur c0pf128 c0pf32; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2r9_ab.txt 2>&1; done
done
cat gpurun_out/r2r9_ab.txt
