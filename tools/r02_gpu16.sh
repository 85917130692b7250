cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_ldlt_ref.py tests/test_ldlt.py tests/test_kkt.py -q -p no:cacheprovider > gpurun_out/r02_ldlt_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_ldlt_tests.log
python tools/bench_ldlt.py 1000 4000 10000 20500 > gpurun_out/r02_ldlt_bench.jsonl 2> gpurun_out/r02_ldlt_bench.err
