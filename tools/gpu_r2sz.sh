# side-stream sub-range size (FKS_PIPE_SUB): 1024 (shipped) / 2048 / 512, three passes, c3 bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2 3; do
for v in 1024 2048 512; do
  FKS_PIPE_SUB=$v timeout 400 python bench.py --no-e2e --cpu-seconds 1 > gpurun_out/r2sz_$v$i.json 2> gpurun_out/r2sz_$v$i.err
  python -c "
import json;d=json.load(open('gpurun_out/r2sz_$v$i.json'));print('sub $v', round(d['ms_per_step'],2), round(d['phases_ms_per_step']['term_loop'],2), d['clocks']['reasons'])"
done; done
