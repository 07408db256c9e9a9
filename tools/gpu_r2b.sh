set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "step_parity or slab or macro" > gpurun_out/r2b_tests.txt 2>&1
tail -5 gpurun_out/r2b_tests.txt
timeout 600 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r2b_tests_all.txt 2>&1
tail -25 gpurun_out/r2b_tests_all.txt
