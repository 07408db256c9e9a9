# on top of the Good-Thomas Y warps: X FFT16 in tangent form (xf16i); one refill call site in Y (onec2)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2 3; do
 for v in cur xf16i onec2; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2aq_ab.txt 2>&1; done
done
cat gpurun_out/r2aq_ab.txt
