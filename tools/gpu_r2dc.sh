# slab-decomposed step at N = 1 with the chunk pipeline (interior planes before the barrier)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 400 python bench.py --decomposed --no-e2e --cpu-seconds 1 > gpurun_out/r2dc_dec.json 2> gpurun_out/r2dc_dec.err
python -c "
import json;d=json.load(open('gpurun_out/r2dc_dec.json'));print('decomposed', round(d['ms_per_step'],2), '%.4g'%d['value'], round(d['roofline']['frac'],4), d['config']['workload'][-80:])"
tail -3 gpurun_out/r2dc_dec.err
