# small-N kernel: term-chunk size at c0 (8 cells, T + 1 = 17; FKS_SMALL_TPC terms per chunk)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
for t in 8 4 3 2; do
FKS_SMALL_TPC=$t timeout 200 python bench.py --config c0 --steps 50 --warmup 5 --no-e2e --cpu-seconds 1 > gpurun_out/r2c0_$t.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/r2c0_$t.json'));print('tpc $t', round(d['ms_per_step'],4), round(d['phases_ms_per_step']['term_loop'],4), round(d['roofline']['frac'],4))"
done; done
