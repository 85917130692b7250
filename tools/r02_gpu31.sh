cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_ldlt_ref.py tests/test_ldlt.py tests/test_kkt.py -x -q -m gpu > gpurun_out/r02_ldlt_suite.log 2>&1
echo "rc $?" >> gpurun_out/r02_ldlt_suite.log
