set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_tests.txt 2>&1
tail -3 gpurun_out/r2a_tests.txt
timeout 120 tools/microbench3 > gpurun_out/r2a_mb3.jsonl 2>&1
for i in 1 2; do
 FKS_LIB=build_variants/libfks_old.so timeout 120 python tools/ab_time_raw.py 8640 5 >> gpurun_out/r2a_ab.txt 2>&1
 timeout 120 python tools/ab_time_raw.py 8640 5 >> gpurun_out/r2a_ab.txt 2>&1
done
timeout 300 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:hot_kernel_v4 -s 1 -c 1 -o gpurun_out/r2a_hot python tools/profile_hot.py c3 1440 > gpurun_out/r2a_ncu.log 2>&1
echo done
