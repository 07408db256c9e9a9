# team-counter poll interval on the final kernel: 1 / 2 (cur) / 4 us
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2 3; do
 for v in cur p1k p4k; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2ar_ab.txt 2>&1; done
done
cat gpurun_out/r2ar_ab.txt
