# risk probe: x-pass of G in the X warps' end-of-cell write-out (gxprobe; results wrong until the back transform
# reads Gx) vs cur: does the term-loop kernel slow down?
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2 3; do
 for v in cur gxprobe; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2v_ab.txt 2>&1; done
done
cat gpurun_out/r2v_ab.txt
