cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ldlt_ref.py tests/test_ldlt.py tests/test_kkt.py -x -q -m gpu > gpurun_out/r02_bkp_sync_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_bkp_sync_tests.log
rm -f gpurun_out/r02_bkp_sync.log
for rep in 1 2; do
  GBOPT_LDLT_KERNEL=panel GBOPT_LDLT_TIMING=1 timeout 300 python tools/ldlt_split.py 300 704 1150 2>&1 | grep -E "bkp_factor" >> gpurun_out/r02_bkp_sync.log
done
