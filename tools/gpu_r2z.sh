set -x
cd $GRAFT_REPO_ROOT
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step_parity.py tests/test_gpu_macro.py -m gpu -x -q -k "fast or c2 or c3 or c4 or bench or step_moments" > gpurun_out/r2z_tests.txt 2>&1
tail -1 gpurun_out/r2z_tests.txt
for v in gp kb2; do FKS_LIB=build_variants/libfks_$v.so timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k[bf]" -c 10 --csv python tools/profile_hot.py c3 4096 2>/dev/null | grep -E "\"k[bf][0-9]" | awk -F'","' '{print "'$v'", $5, $NF}' | sed 's/"//g' | sort | uniq | head -12; done
