set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/r2f2_smi.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r2f2_tests.txt 2>&1
tail -2 gpurun_out/r2f2_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/r2f2_smoke.txt 2>&1
tail -1 gpurun_out/r2f2_smoke.txt
timeout 400 python bench.py > gpurun_out/r2f2_bench.json 2> gpurun_out/r2f2_bench.err
timeout 400 python bench.py --impl reference > gpurun_out/r2f2_ref.json 2> gpurun_out/r2f2_ref.err
timeout 300 python bench.py --config c1 --steps 100 --warmup 3 > gpurun_out/r2f2_bench_c1.json 2> gpurun_out/r2f2_bench_c1.err
timeout 300 python bench.py --config c0 --steps 200 --warmup 3 > gpurun_out/r2f2_bench_c0.json 2> gpurun_out/r2f2_bench_c0.err
timeout 300 python bench.py --config c2 --steps 20 --warmup 3 > gpurun_out/r2f2_bench_c2.json 2> gpurun_out/r2f2_bench_c2.err
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/r2f2_bench_c4.json 2> gpurun_out/r2f2_bench_c4.err
timeout 300 python bench.py --workload bgk > gpurun_out/r2f2_bgk.json 2> gpurun_out/r2f2_bgk.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2f2_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --cpu-seconds 1 > gpurun_out/r2f2_ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:hot_kernel_v4 -s 1 -c 1 -o gpurun_out/r2f2_hot python tools/profile_hot.py c3 10923 > gpurun_out/r2f2_ncu_hot.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:small_term_kernel -s 1 -c 1 -o gpurun_out/r2f2_small python tools/profile_hot.py c1 64 > gpurun_out/r2f2_ncu_small.log 2>&1
ls gpurun_out | grep r2f2
