# round-2 measurement point r2q: bench (c3 default, c2, c4), ncu launch list of the bench command, ncu --set full of the
# term-loop kernel on a 10 923-cell c3 launch
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2q_smi.txt
timeout 400 python bench.py > gpurun_out/r2q_bench.json 2> gpurun_out/r2q_bench.err
cut -c1-400 gpurun_out/r2q_bench.json
timeout 300 python bench.py --config c2 --steps 10 --warmup 3 > gpurun_out/r2q_bench_c2.json 2> gpurun_out/r2q_bench_c2.err
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/r2q_bench_c4.json 2> gpurun_out/r2q_bench_c4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2q_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --cpu-seconds 1 > gpurun_out/r2q_ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:hot_kernel_v4 -s 1 -c 1 -o gpurun_out/r2q_hot python tools/profile_hot.py c3 10923 > gpurun_out/r2q_ncu_hot.log 2>&1
tail -1 gpurun_out/r2q_ncu_hot.log
ls -la gpurun_out/ | grep r2q
