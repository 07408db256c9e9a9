# fks_collision_batch_host: chunks by bytes (>= 32 MB) with carved ends vs the previous n/512 rule (FKS_HOST_NO_CARVE
# only turns the carve off here; the chunk count rule is new in both)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "host" > gpurun_out/r2hb_tests.txt 2>&1; tail -1 gpurun_out/r2hb_tests.txt
for i in 1 2; do
for v in carve nocarve; do
  case $v in carve) env="";; nocarve) env="FKS_HOST_NO_CARVE=1";; esac
  for c in c2 c3; do
  env $env timeout 300 python bench.py --config $c --steps 5 --warmup 3 --cpu-seconds 1 > gpurun_out/r2hb_$c$v$i.json 2> gpurun_out/r2hb_$c$v$i.err
  python -c "
import json;d=json.load(open('gpurun_out/r2hb_$c$v$i.json'));print('$c $v', round(d['ms_per_step'],3), 'e2e', '%.4g'%d['e2e']['value'], 'coll_only', '%.4g'%d['e2e']['collision_only']['value'])"
  done
done; done
