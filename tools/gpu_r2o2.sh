set -x
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "host" > gpurun_out/r2o2_tests.txt 2>&1
tail -1 gpurun_out/r2o2_tests.txt
for v in w12 hs w12 hs; do FKS_LIB=build_variants/libfks_$v.so timeout 500 python bench.py --steps 3 --warmup 3 --e2e-steps 3 --cpu-seconds 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['e2e']['value'], d['e2e']['collision_only']['value'])"; done
