set -x
cd $GRAFT_REPO_ROOT
timeout 300 python tools/profile_hot.py c3 1440 > gpurun_out/r2k_plain.txt 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:hot_kernel_v4 -s 1 -c 1 -o gpurun_out/r2k_hot python tools/profile_hot.py c3 1440 > gpurun_out/r2k_ncu_hot.log 2>&1
tail -2 gpurun_out/r2k_ncu_hot.log
timeout 300 python tools/profile_hot.py c1 64 > gpurun_out/r2k_plain1.txt 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:small_term_kernel -s 1 -c 1 -o gpurun_out/r2k_small python tools/profile_hot.py c1 64 > gpurun_out/r2k_ncu_small.log 2>&1
tail -2 gpurun_out/r2k_ncu_small.log
FKS_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config c2 --steps 2 --warmup 1 --cpu-seconds 1 --no-e2e > gpurun_out/r2k_n2.json 2> gpurun_out/r2k_n2.err
tail -3 gpurun_out/r2k_n2.err; cut -c1-300 gpurun_out/r2k_n2.json
timeout 300 python bench.py > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err
tail -2 gpurun_out/r2k_bench.err
