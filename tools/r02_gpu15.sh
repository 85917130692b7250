cd $GRAFT_REPO_ROOT
python tools/prof_outputs.py c2 j > gpurun_out/r02_prof_c2_j2.txt 2>&1
GBOPT_ADJ_KW4_CTAS=100000 python tools/prof_outputs.py c2 j > gpurun_out/r02_prof_c2_j2_kw2.txt 2>&1
python -m pytest tests/test_gpu_jacobian.py tests/test_gpu_parity.py -q -p no:cacheprovider > gpurun_out/r02_jtest.log 2>&1
python bench.py --steps 10 --no-cpu-baseline --no-sharded > gpurun_out/r02_bench_j.json 2>&1
