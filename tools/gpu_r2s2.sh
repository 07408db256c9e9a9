# round-2 end measurement point r2s2 (after the small-N Good-Thomas FFT12): GPU tests + smoke, c1 / c0 bench,
# ncu --set full of the small-N term kernel on c1
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r2s2_tests.txt 2>&1; tail -2 gpurun_out/r2s2_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/r2s2_smoke.txt 2>&1; tail -1 gpurun_out/r2s2_smoke.txt
for c in c1 c0; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r2s2_bench_$c.json 2> gpurun_out/r2s2_bench_$c.err; cut -c1-200 gpurun_out/r2s2_bench_$c.json; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:small_term_kernel -s 1 -c 1 -o gpurun_out/r2s2_small python tools/profile_hot.py c1 64 > gpurun_out/r2s2_ncu_small.log 2>&1
tail -1 gpurun_out/r2s2_ncu_small.log
