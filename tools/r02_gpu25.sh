cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_gputest_full2.log 2>&1; echo "rc=$?" >> gpurun_out/r02_gputest_full2.log
timeout 600 python bench.py > gpurun_out/r02_bench_c2_final1.json 2> gpurun_out/r02_bench_c2_final1.err
