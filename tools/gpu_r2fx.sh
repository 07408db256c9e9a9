# final code check: GPU suite + smoke + c3 bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r2fx_tests.txt 2>&1; tail -1 gpurun_out/r2fx_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/r2fx_smoke.txt 2>&1; tail -1 gpurun_out/r2fx_smoke.txt
timeout 400 python bench.py > gpurun_out/r2fx_bench.json 2> gpurun_out/r2fx_bench.err
python -c "
import json;d=json.load(open('gpurun_out/r2fx_bench.json'));print(round(d['ms_per_step'],2), '%.4g'%d['value'], round(d['roofline']['frac'],4), round(d['whole_step']['frac_of_fp64_peak'],4), d['clocks'], '%.4g'%d['e2e']['value'])"
