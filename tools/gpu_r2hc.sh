# host-buffer step: outer quarter of the first / last multi-plane slab as its own piece (c2 e2e)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "host" > gpurun_out/r2hc_tests.txt 2>&1; tail -1 gpurun_out/r2hc_tests.txt
for i in 1 2; do
for v in carve nocarve; do
  case $v in carve) env="";; nocarve) env="FKS_HOST_NO_CARVE=1";; esac
  env $env timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --cpu-seconds 1 > gpurun_out/r2hc_$v$i.json 2> gpurun_out/r2hc_$v$i.err
  python -c "
import json;d=json.load(open('gpurun_out/r2hc_$v$i.json'));print('$v', round(d['ms_per_step'],3), '%.4g'%d['value'], 'e2e', '%.4g'%d['e2e']['value'])"
done; done
for s in 8 16; do
  FKS_HOST_SLABS=$s timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --cpu-seconds 1 > gpurun_out/r2hc_s$s.json 2> gpurun_out/r2hc_s$s.err
  python -c "
import json;d=json.load(open('gpurun_out/r2hc_s$s.json'));print('slabs $s', round(d['ms_per_step'],3), 'e2e', '%.4g'%d['e2e']['value'])"
done
