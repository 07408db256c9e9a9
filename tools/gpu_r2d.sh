set -x
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c0 or c1 or random_fields or pad_and or chunking or step_with_transport or edge" > gpurun_out/r2d_tests.txt 2>&1
tail -15 gpurun_out/r2d_tests.txt
timeout 200 python bench.py --config c1 --steps 5 --warmup 3 --cpu-seconds 3 > gpurun_out/r2d_c1.json 2> gpurun_out/r2d_c1.err
tail -3 gpurun_out/r2d_c1.err; cut -c1-600 gpurun_out/r2d_c1.json
timeout 200 python bench.py --config c0 --steps 5 --warmup 3 --cpu-seconds 3 > gpurun_out/r2d_c0.json 2> gpurun_out/r2d_c0.err
tail -3 gpurun_out/r2d_c0.err; cut -c1-600 gpurun_out/r2d_c0.json
