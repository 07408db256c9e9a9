# chunk pipeline variants: L2 persistence window on the W1 ring (FKS_L2_PERSIST), no stream priorities (FKS_PIPE_NOPRIO)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
for v in base persist noprio; do
  case $v in base) env="";; persist) env="FKS_L2_PERSIST=1";; noprio) env="FKS_PIPE_NOPRIO=1";; esac
  env $env timeout 400 python bench.py --no-e2e --cpu-seconds 1 > gpurun_out/r2pl_$v$i.json 2> gpurun_out/r2pl_$v$i.err
  python -c "
import json;d=json.load(open('gpurun_out/r2pl_$v$i.json'));print('$v', round(d['ms_per_step'],2), round(d['phases_ms_per_step']['term_loop'],2), round(d['roofline']['frac'],4))"
done; done
grep FKS_L2 gpurun_out/r2pl_persist1.err
