# forward / back transform kernels at 3 CTAs per SM (launch bounds) vs 2 (register-limited)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
 for v in xfcur mbkf mbkb3 mball; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 5 >> gpurun_out/r2aa_ab.txt 2>&1; done
done
cat gpurun_out/r2aa_ab.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"kf1|kf2|kb1|kb2|kb3" --csv python tools/profile_hot.py c3 4096 2>/dev/null | grep -E "kf1|kf2|kb1|kb2|kb3" | tail -5 > gpurun_out/r2aa_cur_k.txt
FKS_LIB=build_variants/libfks_mball.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"kf1|kf2|kb1|kb2|kb3" --csv python tools/profile_hot.py c3 4096 2>/dev/null | grep -E "kf1|kf2|kb1|kb2|kb3" | tail -5 > gpurun_out/r2aa_mball_k.txt
cat gpurun_out/r2aa_cur_k.txt gpurun_out/r2aa_mball_k.txt | cut -c1-250
