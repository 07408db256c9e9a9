# final verification of the committed code: GPU suite + smoke, c3 bench, BGK bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r2fv_tests.txt 2>&1; tail -1 gpurun_out/r2fv_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/r2fv_smoke.txt 2>&1; tail -1 gpurun_out/r2fv_smoke.txt
timeout 400 python bench.py > gpurun_out/r2fv_bench.json 2> gpurun_out/r2fv_bench.err
timeout 300 python bench.py --workload bgk > gpurun_out/r2fv_bgk.json 2> gpurun_out/r2fv_bgk.err
for f in gpurun_out/r2fv_bench.json gpurun_out/r2fv_bgk.json; do python -c "
import json,sys;d=json.load(open('$f'));print('$f', round(d['ms_per_step'],4), '%.4g'%d['value'], round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'], 'e2e', '%.4g'%d['e2e']['value'])"; done
