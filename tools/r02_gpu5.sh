cd $GRAFT_REPO_ROOT
timeout 600 python tools/debug_multi.py 67 3 > gpurun_out/r02_debug_multi2.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_multidevice.py tests/test_gpu_multirank.py tests/test_cpp_api.py tests/test_reduced_space.py tests/test_gpu_dataflow.py tests/test_gpu_ldlt_ref.py tests/test_ldlt.py -q -p no:cacheprovider -m gpu > gpurun_out/r02_gpu5.log 2>&1; echo "rc=$?" >> gpurun_out/r02_gpu5.log
