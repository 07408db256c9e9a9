set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2t_tests.txt 2>&1
tail -3 gpurun_out/r2t_tests.txt
for i in 1 2 3; do
 for v in v4i bc; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2t_ab.txt 2>&1; done
done
cat gpurun_out/r2t_ab.txt
timeout 400 python bench.py --steps 5 --warmup 3 > gpurun_out/r2t_bench.json 2> gpurun_out/r2t_bench.err
python -c "import json; d=json.load(open('gpurun_out/r2t_bench.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['phases_ms_per_step'], d['e2e']['value'])"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"^k[bf]" -c 20 --csv --log-file gpurun_out/r2t_xf.csv python tools/profile_hot.py c3 10923 > gpurun_out/r2t_ncu.log 2>&1
tail -1 gpurun_out/r2t_ncu.log
