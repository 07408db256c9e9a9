# final measurement point (r02q): GPU tests + smoke, bench c3 / c1 / c2 / c0 / c4 / bgk, reference arm, ncu launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2fy_smi.txt
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r2fy_tests.txt 2>&1; tail -1 gpurun_out/r2fy_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/r2fy_smoke.txt 2>&1; tail -1 gpurun_out/r2fy_smoke.txt
timeout 400 python bench.py > gpurun_out/r2fy_bench.json 2> gpurun_out/r2fy_bench.err
for c in c1 c2 c0; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r2fy_bench_$c.json 2> gpurun_out/r2fy_bench_$c.err; done
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/r2fy_bench_c4.json 2> gpurun_out/r2fy_bench_c4.err
timeout 300 python bench.py --workload bgk > gpurun_out/r2fy_bgk.json 2> gpurun_out/r2fy_bgk.err
timeout 400 python bench.py --impl reference > gpurun_out/r2fy_ref.json 2> gpurun_out/r2fy_ref.err
for f in gpurun_out/r2fy_bench*.json; do python -c "
import json,sys;d=json.load(open('$f'));print('$f', round(d['ms_per_step'],4), '%.4g'%d['value'], round(d['roofline']['frac'],4), round(d['whole_step']['frac_of_fp64_peak'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'], 'e2e', '%.4g'%d['e2e']['value'], '%.4g'%d['e2e']['collision_only']['value'])"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2fy_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --cpu-seconds 1 > gpurun_out/r2fy_ncu_launch.log 2>&1
tail -1 gpurun_out/r2fy_ncu_launch.log | cut -c1-200
