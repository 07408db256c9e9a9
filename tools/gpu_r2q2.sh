# Good-Thomas transform in the Y / X roles again, now with mbarrier hand-offs and relaxed polls
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
 for v in cur ygt xgt yxgt; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2q2_ab.txt 2>&1; done
done
cat gpurun_out/r2q2_ab.txt
