# instruction-cache hypothesis: ncu stall reasons of cur vs twc (Y combine with 3 compile-time class copies: +3 KB code)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in cur twc; do
FKS_LIB=build_variants/libfks_$v.so timeout 600 ncu --set full --clock-control none -k regex:hot_kernel_v4 -s 1 -c 1 -o gpurun_out/r2af_$v python tools/profile_hot.py c3 1440 > gpurun_out/r2af_ncu_$v.log 2>&1
done
ls gpurun_out | grep r2af
