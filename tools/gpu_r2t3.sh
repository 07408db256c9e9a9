# W1 ring depth NB = 3 / 4 (cur) / 5 / 6
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
 for v in cur nb3 nb5 nb6; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2t3_ab.txt 2>&1; done
done
cat gpurun_out/r2t3_ab.txt
