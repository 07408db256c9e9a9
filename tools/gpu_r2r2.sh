# ycnt ack without fence.sc (ackr), single acquire in the W1 prefetch check (pfacq), no G write-out (timing bound only)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
 for v in cur ackr pfacq nogout; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2r2_ab.txt 2>&1; done
done
cat gpurun_out/r2r2_ab.txt
