# chunk pipeline also in fks_collision_batch_host: GPU suite, c3 bench (e2e incl. collision-only), c4 bench, ncu launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2pr_tests.txt 2>&1; tail -2 gpurun_out/r2pr_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/r2pr_smoke.txt 2>&1; tail -1 gpurun_out/r2pr_smoke.txt
timeout 400 python bench.py > gpurun_out/r2pr_bench.json 2> gpurun_out/r2pr_bench.err
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/r2pr_bench_c4.json 2> gpurun_out/r2pr_bench_c4.err
for f in gpurun_out/r2pr_bench*.json; do python -c "
import json,sys;d=json.load(open('$f'));print('$f', round(d['ms_per_step'],2), d['value'], round(d['roofline']['frac'],4), round(d['whole_step']['frac_of_fp64_peak'],4), d['clocks']['sm_mhz'], 'e2e', d['e2e']['value'], d['e2e'].get('collision_only'))"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2pr_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --cpu-seconds 1 > gpurun_out/r2pr_ncu_launch.log 2>&1
tail -2 gpurun_out/r2pr_ncu_launch.log
