# the class-0 Y warp acquires W1(t+1)'s publication off the critical path; the last sibling then issues the refill
# without its own L2 round trip (pubok)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
 for v in cur pubok; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2t2_ab.txt 2>&1; done
done
cat gpurun_out/r2t2_ab.txt
