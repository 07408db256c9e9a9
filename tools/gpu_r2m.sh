set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/r2m_smi.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r2m_tests.txt 2>&1
tail -3 gpurun_out/r2m_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/r2m_smoke.txt 2>&1
tail -1 gpurun_out/r2m_smoke.txt
timeout 400 python bench.py > gpurun_out/r2m_bench.json 2> gpurun_out/r2m_bench.err
timeout 400 python bench.py --impl reference > gpurun_out/r2m_ref.json 2> gpurun_out/r2m_ref.err
for c in c0 c1 c2; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r2m_bench_$c.json 2> gpurun_out/r2m_bench_$c.err; done
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/r2m_bench_c4.json 2> gpurun_out/r2m_bench_c4.err
timeout 300 python bench.py --workload bgk > gpurun_out/r2m_bgk.json 2> gpurun_out/r2m_bgk.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2m_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --cpu-seconds 1 > gpurun_out/r2m_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:hot_kernel_v4 -s 1 -c 1 -o gpurun_out/r2m_hot python tools/profile_hot.py c3 10923 > gpurun_out/r2m_ncu_hot.log 2>&1
tail -1 gpurun_out/r2m_ncu_hot.log
ls -la gpurun_out/ | grep r2m
