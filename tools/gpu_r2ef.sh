# transforms with an L2 evict-first policy on their cp.async loads (FKS_SIDE_EVICT_FIRST) vs shipped, pipelined bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
for v in cur ef; do
  FKS_LIB=build_variants/libfks_$v.so timeout 400 python bench.py --no-e2e --cpu-seconds 1 > gpurun_out/r2ef_c3$v$i.json 2> gpurun_out/r2ef_c3$v$i.err
  python -c "
import json;d=json.load(open('gpurun_out/r2ef_c3$v$i.json'));print('c3 $v', round(d['ms_per_step'],2), round(d['phases_ms_per_step']['term_loop'],2), round(d['roofline']['frac'],4), round(d['whole_step']['frac_of_fp64_peak'],4))"
done; done
for v in cur ef; do
  FKS_LIB=build_variants/libfks_$v.so timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-e2e --cpu-seconds 1 > gpurun_out/r2ef_c4$v.json 2> gpurun_out/r2ef_c4$v.err
  python -c "
import json;d=json.load(open('gpurun_out/r2ef_c4$v.json'));print('c4 $v', round(d['ms_per_step'],2), round(d['phases_ms_per_step']['term_loop'],2), round(d['roofline']['frac'],4), round(d['whole_step']['frac_of_fp64_peak'],4), d['clocks']['reasons'])"
done
