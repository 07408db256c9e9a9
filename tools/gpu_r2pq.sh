# chunk pipeline for the device step and the host-buffer step: full GPU suite + bench A/B (with e2e)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2pq_tests.txt 2>&1; tail -3 gpurun_out/r2pq_tests.txt
timeout 400 python bench.py --cpu-seconds 1 > gpurun_out/r2pq_bench_pipe1.json 2> gpurun_out/r2pq_bench_pipe1.err
FKS_NO_PIPELINE=1 timeout 400 python bench.py --cpu-seconds 1 > gpurun_out/r2pq_bench_seq1.json 2> gpurun_out/r2pq_bench_seq1.err
timeout 400 python bench.py --cpu-seconds 1 > gpurun_out/r2pq_bench_pipe2.json 2> gpurun_out/r2pq_bench_pipe2.err
for f in gpurun_out/r2pq_bench_*.json; do python -c "
import json,sys;d=json.load(open('$f'));print('$f', round(d['ms_per_step'],2), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], 'e2e', d['e2e']['value'], d['e2e'].get('collision_only'))"; done
