cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_multirank.py tests/test_gpu_multidevice.py tests/test_cpp_api.py -q -p no:cacheprovider > gpurun_out/r02_multi.log 2>&1; echo "rc=$?" >> gpurun_out/r02_multi.log
python bench.py --gpus 2 --dist-backend gloo --config c2 --steps 3 --warmup 1 > gpurun_out/r02_bench_gloo2.json 2> gpurun_out/r02_bench_gloo2.err
