# do the X warps take issue slots from the critical Z warps? X sleeps 100 / 400 ns before each class task
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
 for v in zpub xs100 xs400; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2q7_ab.txt 2>&1; done
done
cat gpurun_out/r2q7_ab.txt
