# round-2 final measurement point: GPU tests + smoke, bench c3 / c1 / c2 / c4 / c0 / bgk, reference arm, ncu launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2fin2_smi.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r2fin2_tests.txt 2>&1; tail -2 gpurun_out/r2fin2_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/r2fin2_smoke.txt 2>&1; tail -1 gpurun_out/r2fin2_smoke.txt
timeout 400 python bench.py > gpurun_out/r2fin2_bench.json 2> gpurun_out/r2fin2_bench.err
for c in c1 c2 c0; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r2fin2_bench_$c.json 2> gpurun_out/r2fin2_bench_$c.err; done
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/r2fin2_bench_c4.json 2> gpurun_out/r2fin2_bench_c4.err
timeout 300 python bench.py --workload bgk > gpurun_out/r2fin2_bgk.json 2> gpurun_out/r2fin2_bgk.err
timeout 400 python bench.py --impl reference > gpurun_out/r2fin2_ref.json 2> gpurun_out/r2fin2_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2fin2_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --cpu-seconds 1 > gpurun_out/r2fin2_ncu_launch.log 2>&1
ls gpurun_out | grep r2fin2
timeout 900 ncu --set full --import-source on --clock-control none -k regex:hot_kernel_v4 -s 1 -c 1 -o gpurun_out/r2fin2_hot python tools/profile_hot.py c3 10923 > gpurun_out/r2fin2_ncu_hot.log 2>&1
tail -1 gpurun_out/r2fin2_ncu_hot.log
