set -x
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_slab.py tests/test_gpu_step_parity.py tests/test_gpu_macro.py -m gpu -x -q > gpurun_out/r2j_tests.txt 2>&1
tail -3 gpurun_out/r2j_tests.txt
timeout 300 python bench.py --decomposed --steps 3 --warmup 3 --cpu-seconds 2 --no-e2e > gpurun_out/r2j_dec.json 2> gpurun_out/r2j_dec.err
tail -2 gpurun_out/r2j_dec.err; cut -c1-400 gpurun_out/r2j_dec.json
