# verification after the N = 16 term-chunk change: GPU suite + smoke, c0 / c1 bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r2fu_tests.txt 2>&1; tail -1 gpurun_out/r2fu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/r2fu_smoke.txt 2>&1; tail -1 gpurun_out/r2fu_smoke.txt
for c in c0 c1; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r2fu_bench_$c.json 2> gpurun_out/r2fu_bench_$c.err
python -c "
import json;d=json.load(open('gpurun_out/r2fu_bench_$c.json'));print('$c', round(d['ms_per_step'],4), '%.4g'%d['value'], round(d['roofline']['frac'],4), 'e2e', '%.4g'%d['e2e']['value'])"; done
