cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_jacobian.py tests/test_gpu_parity.py -q -p no:cacheprovider > gpurun_out/r02_adjmma_tests2.log 2>&1; echo "rc=$?" >> gpurun_out/r02_adjmma_tests2.log
for m in 1; do echo "== ADJ_MMA=$m"; GBOPT_ADJ_MMA=$m timeout 300 python tools/prof_outputs.py c2 j | grep -E "adj_cols|adj_reduce|total"; done > gpurun_out/r02_adjmma_ab2.log 2>&1
for m in 1 0; do GBOPT_ADJ_MMA=$m timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-sharded --no-e2e --no-parity | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$m', d['value'], json.dumps(d['hbm_paths']['jacobian_reverse']))"; done >> gpurun_out/r02_adjmma_ab2.log 2>&1
