# full GPU suite + default bench + smoke (checkpoint)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_gputest_full2.log 2>&1; echo "rc=$?" >> gpurun_out/r02_gputest_full2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_smoke2.log 2>&1
timeout 900 python bench.py > gpurun_out/r02_bench_c2_final.json 2> gpurun_out/r02_bench_c2_final.err
