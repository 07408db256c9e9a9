# relaxed polling of the team counters (one acquire when the target is seen) vs acquire polling (p*)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
 for v in p128 p2048 rx128 rx512 rx2048; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2p10_ab.txt 2>&1; done
done
cat gpurun_out/r2p10_ab.txt
