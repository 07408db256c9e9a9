# BGK / moments kernel: bulk (TMA) staging per constant-source kz run vs per-pair cp.async (FKS_MACRO_NO_BULK)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_macro.py -m gpu -x -q > gpurun_out/r2bk_tests.txt 2>&1; tail -3 gpurun_out/r2bk_tests.txt
for i in 1 2; do
for v in bulk nobulk; do
  case $v in bulk) env="";; nobulk) env="FKS_MACRO_NO_BULK=1";; esac
  env $env timeout 300 python bench.py --workload bgk --cpu-seconds 1 > gpurun_out/r2bk_$v$i.json 2> gpurun_out/r2bk_$v$i.err
  python -c "
import json;d=json.load(open('gpurun_out/r2bk_$v$i.json'));print('$v', round(d['ms_per_step'],3), '%.4g'%d['value'], round(d['roofline']['frac'],4), 'e2e', '%.4g'%d['e2e']['value'])" || tail -3 gpurun_out/r2bk_$v$i.err
done; done
