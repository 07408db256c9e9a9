# end-of-round-2 measurement point with the chunk pipeline (r02p): GPU tests + smoke, bench c3 / c1 / c2 / c0 / c4 / bgk, reference arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2pz_smi.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r2pz_tests.txt 2>&1; tail -2 gpurun_out/r2pz_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/r2pz_smoke.txt 2>&1; tail -1 gpurun_out/r2pz_smoke.txt
timeout 400 python bench.py > gpurun_out/r2pz_bench.json 2> gpurun_out/r2pz_bench.err
for c in c1 c2 c0; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r2pz_bench_$c.json 2> gpurun_out/r2pz_bench_$c.err; done
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/r2pz_bench_c4.json 2> gpurun_out/r2pz_bench_c4.err
timeout 300 python bench.py --workload bgk > gpurun_out/r2pz_bgk.json 2> gpurun_out/r2pz_bgk.err
timeout 400 python bench.py --impl reference > gpurun_out/r2pz_ref.json 2> gpurun_out/r2pz_ref.err
for f in gpurun_out/r2pz_bench*.json; do python -c "
import json,sys;d=json.load(open('$f'));print('$f', round(d['ms_per_step'],4), '%.4g'%d['value'], round(d['roofline']['frac'],4), round(d['whole_step']['frac_of_fp64_peak'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'], 'e2e', '%.4g'%d['e2e']['value'])"; done
