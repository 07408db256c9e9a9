# mbarrier wait loop: suspend hint 20 us (cur), no hint, + nanosleep 32 / 128 ns between try_waits, hint 1 ms
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
 for v in cur twnh tws32 tws128 twh1m; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2w_ab.txt 2>&1; done
done
cat gpurun_out/r2w_ab.txt
