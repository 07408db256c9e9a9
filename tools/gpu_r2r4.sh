# poll interval of the Y warps' W1 publication poll (128 / 512 ns; Z ring poll stays 2 us) and Z ring poll 8 us
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
 for v in cur y128 y512 z8k; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2r4_ab.txt 2>&1; done
done
cat gpurun_out/r2r4_ab.txt
