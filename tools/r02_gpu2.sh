cd $GRAFT_REPO_ROOT
python bench.py > gpurun_out/r02_bench_c2.json 2> gpurun_out/r02_bench_c2.err; echo "bench rc=$?" >> gpurun_out/r02_bench_c2.err
python -m pytest tests/test_gpu_multirank.py -x -q -p no:cacheprovider > gpurun_out/r02_multirank.log 2>&1; echo "rc=$?" >> gpurun_out/r02_multirank.log
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r02_ref_c2.json 2> gpurun_out/r02_ref_c2.err
