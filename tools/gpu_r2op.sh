# operating-point / run-to-run spread of the shipped build: 4 default bench runs (c3), separate processes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2 3 4; do
  timeout 400 python bench.py --no-e2e --cpu-seconds 1 > gpurun_out/r2op_$i.json 2> gpurun_out/r2op_$i.err
  python -c "
import json;d=json.load(open('gpurun_out/r2op_$i.json'));r=d['roofline'];print('run $i', round(d['ms_per_step'],2), round(r['ms_per_launch'],2), round(r['frac'],4), r['operating_point'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
