# round-2 measurement point r2s: GPU tests + smoke, bench (c3, c2, c4, c0, c1, bgk, reference arm), ncu launch list,
# ncu --set full of the term-loop kernel on a 10 923-cell c3 launch
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2s_smi.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r2s_tests.txt 2>&1; tail -2 gpurun_out/r2s_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/r2s_smoke.txt 2>&1; tail -1 gpurun_out/r2s_smoke.txt
timeout 400 python bench.py > gpurun_out/r2s_bench.json 2> gpurun_out/r2s_bench.err
cut -c1-300 gpurun_out/r2s_bench.json
timeout 300 python bench.py --config c2 --steps 10 --warmup 3 > gpurun_out/r2s_bench_c2.json 2> gpurun_out/r2s_bench_c2.err
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/r2s_bench_c4.json 2> gpurun_out/r2s_bench_c4.err
for c in c0 c1; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r2s_bench_$c.json 2> gpurun_out/r2s_bench_$c.err; done
timeout 400 python bench.py --impl reference > gpurun_out/r2s_ref.json 2> gpurun_out/r2s_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2s_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --cpu-seconds 1 > gpurun_out/r2s_ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:hot_kernel_v4 -s 1 -c 1 -o gpurun_out/r2s_hot python tools/profile_hot.py c3 10923 > gpurun_out/r2s_ncu_hot.log 2>&1
tail -1 gpurun_out/r2s_ncu_hot.log
ls gpurun_out | grep r2s
