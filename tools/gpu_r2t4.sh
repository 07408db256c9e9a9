# X warps: class branch outside the element loops, DIF (xsplit) and Good-Thomas (xgt2) vs cur
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step_parity.py -m gpu -x -q -k "fast or c2 or c3 or c4 or bench" > gpurun_out/r2t4_tests.txt 2>&1; tail -1 gpurun_out/r2t4_tests.txt
for i in 1 2; do
 for v in cur xsplit xgt2; do FKS_LIB=build_variants/libfks_$v.so timeout 200 python tools/ab_time_raw.py 8640 3 >> gpurun_out/r2t4_ab.txt 2>&1; done
done
cat gpurun_out/r2t4_ab.txt
