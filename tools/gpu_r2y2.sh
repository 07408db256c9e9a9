# sensitivity probe: +16 dependent DFMA (+~8 % FP64) per class task in one role (Y / X / Z) vs cur
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
 for v in cur padY padX padZ; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2y2_ab.txt 2>&1; done
done
cat gpurun_out/r2y2_ab.txt
