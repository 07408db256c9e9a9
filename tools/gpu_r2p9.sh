# full GPU suite on the new default (Good-Thomas Z tasks + mbarrier hand-offs); poll interval of the global counters
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2p9_tests.txt 2>&1; tail -2 gpurun_out/r2p9_tests.txt
for i in 1 2; do
 for v in p128 p512 p1024 p2048; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2p9_ab.txt 2>&1; done
done
cat gpurun_out/r2p9_ab.txt
