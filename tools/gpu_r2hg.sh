# host-buffer calls: consecutive pieces merged into ramped compute groups (FKS_HOST_GROUP cells, 0 = one launch per piece)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "host" > gpurun_out/r2hg_tests.txt 2>&1; tail -1 gpurun_out/r2hg_tests.txt
for i in 1 2; do
for v in 4096 0; do
  FKS_HOST_GROUP=$v timeout 400 python bench.py --cpu-seconds 1 > gpurun_out/r2hg_c3_$v$i.json 2> gpurun_out/r2hg_c3_$v$i.err
  python -c "
import json;d=json.load(open('gpurun_out/r2hg_c3_$v$i.json'));print('c3 group $v', round(d['ms_per_step'],2), 'e2e', '%.4g'%d['e2e']['value'], 'coll_only', '%.4g'%d['e2e']['collision_only']['value'], d['clocks']['reasons'])"
done; done
for v in 4096 0; do
  FKS_HOST_GROUP=$v timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --cpu-seconds 1 > gpurun_out/r2hg_c2_$v.json 2> gpurun_out/r2hg_c2_$v.err
  python -c "
import json;d=json.load(open('gpurun_out/r2hg_c2_$v.json'));print('c2 group $v', round(d['ms_per_step'],3), 'e2e', '%.4g'%d['e2e']['value'], 'coll_only', '%.4g'%d['e2e']['collision_only']['value'])"
done
