# Y warps transform both planes in one interleaved instruction stream (ydual; spills 740 B) vs current
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
 for v in zpub ydual; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2q5_ab.txt 2>&1; done
done
cat gpurun_out/r2q5_ab.txt
