set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2e_tests.txt 2>&1
tail -5 gpurun_out/r2e_tests.txt
timeout 300 ncu --set full --import-source on --clock-control none -k regex:small_term_kernel -s 2 -c 1 -o gpurun_out/r2e_small python bench.py --config c1 --steps 2 --warmup 1 --cpu-seconds 1 --no-e2e > gpurun_out/r2e_ncu.log 2>&1
tail -3 gpurun_out/r2e_ncu.log
