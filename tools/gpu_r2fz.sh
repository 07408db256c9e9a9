# final suite after the pipeline / carve changes: GPU tests + smoke, c3 and c2 bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/r2fz_tests.txt 2>&1; tail -12 gpurun_out/r2fz_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/r2fz_smoke.txt 2>&1; tail -1 gpurun_out/r2fz_smoke.txt
timeout 400 python bench.py > gpurun_out/r2fz_bench.json 2> gpurun_out/r2fz_bench.err
timeout 300 python bench.py --config c2 --steps 10 --warmup 3 > gpurun_out/r2fz_bench_c2.json 2> gpurun_out/r2fz_bench_c2.err
for f in gpurun_out/r2fz_bench*.json; do python -c "
import json,sys;d=json.load(open('$f'));print('$f', round(d['ms_per_step'],4), '%.4g'%d['value'], round(d['roofline']['frac'],4), round(d['whole_step']['frac_of_fp64_peak'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'], 'e2e', '%.4g'%d['e2e']['value'], d['e2e'].get('collision_only',{}).get('value'))"; done
