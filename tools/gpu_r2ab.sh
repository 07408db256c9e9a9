# kb1 with 4 / 2 / 1 px planes per CTA (more, smaller CTAs per SM)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fast_path_vs_oracle or fast_path_random or project_mass" > gpurun_out/r2ab_tests.txt 2>&1; tail -1 gpurun_out/r2ab_tests.txt
for v in pb4 pb2 pb1; do FKS_LIB=build_variants/libfks_$v.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"kb1" --csv python tools/profile_hot.py c3 4096 2>/dev/null | grep kb1 | tail -1 | awk -F'","' -v v=$v '{print v, $NF}' >> gpurun_out/r2ab_k.txt; done
cat gpurun_out/r2ab_k.txt
