set -x
cd $GRAFT_REPO_ROOT
for v in ys2 tabtma; do FKS_LIB=build_variants/libfks_$v.so timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fast_path_vs_oracle or random_and_ragged" 2>&1 | tail -1; done
for i in 1 2 3; do
 for v in cur ys2 tabtma; do FKS_LIB=build_variants/libfks_$v.so timeout 120 python tools/ab_time_raw.py 8640 3 2>&1 | tail -1; done
done
