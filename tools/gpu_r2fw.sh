# final point (r02r): GPU suite + smoke, bench c3 / c4 / c2 / c1, ncu launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r2fw_tests.txt 2>&1; tail -1 gpurun_out/r2fw_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/r2fw_smoke.txt 2>&1; tail -1 gpurun_out/r2fw_smoke.txt
timeout 400 python bench.py > gpurun_out/r2fw_bench.json 2> gpurun_out/r2fw_bench.err
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/r2fw_bench_c4.json 2> gpurun_out/r2fw_bench_c4.err
for c in c2 c1; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r2fw_bench_$c.json 2> gpurun_out/r2fw_bench_$c.err; done
for f in gpurun_out/r2fw_bench*.json; do python -c "
import json,sys;d=json.load(open('$f'));print('$f', round(d['ms_per_step'],4), '%.4g'%d['value'], round(d['roofline']['frac'],4), round(d['whole_step']['frac_of_fp64_peak'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'], 'e2e', '%.4g'%d['e2e']['value'], '%.4g'%d['e2e']['collision_only']['value'])"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2fw_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --cpu-seconds 1 > gpurun_out/r2fw_ncu_launch.log 2>&1
tail -1 gpurun_out/r2fw_ncu_launch.log | cut -c1-120
