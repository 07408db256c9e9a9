# team-counter poll interval under the chunk pipeline (c3 bench): 1024 / 2048 (shipped) / 4096 ns
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
for v in cur p1024 p4096; do
  FKS_LIB=build_variants/libfks_$v.so timeout 400 python bench.py --no-e2e --cpu-seconds 1 > gpurun_out/r2pw_$v$i.json 2> gpurun_out/r2pw_$v$i.err
  python -c "
import json;d=json.load(open('gpurun_out/r2pw_$v$i.json'));print('$v', round(d['ms_per_step'],2), round(d['phases_ms_per_step']['term_loop'],2), round(d['roofline']['frac'],4), d['clocks']['reasons'])"
done; done
