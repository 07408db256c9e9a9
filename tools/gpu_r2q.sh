set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r2q_tests.txt 2>&1
tail -2 gpurun_out/r2q_tests.txt
for c in c0 c1 c2; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r2q_bench_$c.json 2> gpurun_out/r2q_bench_$c.err; done
python - <<'PY'
import json
for c in ("c0", "c1", "c2"):
    d = json.load(open(f"gpurun_out/r2q_bench_{c}.json"))
    print(c, "%.4g" % d["value"], "ms %.3f" % d["ms_per_step"], "frac %.3f" % d["roofline"]["frac"], "e2e %.4g" % d["e2e"]["value"], "clk", d["clocks"]["sm_mhz"], "warmup", d["warmup"])
PY
