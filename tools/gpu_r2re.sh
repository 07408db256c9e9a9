# re-entry check of the committed state: GPU tests + smoke + c3 bench + A/B timing of the hot kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2re_smi.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r2re_tests.txt 2>&1; tail -2 gpurun_out/r2re_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/r2re_smoke.txt 2>&1; tail -1 gpurun_out/r2re_smoke.txt
timeout 400 python bench.py > gpurun_out/r2re_bench.json 2> gpurun_out/r2re_bench.err
cat gpurun_out/r2re_bench.json
for i in 1 2; do timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2re_ab.txt 2>&1; done
cat gpurun_out/r2re_ab.txt
