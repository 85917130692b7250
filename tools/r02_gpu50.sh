cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ldlt_ref.py tests/test_ldlt.py tests/test_kkt.py -x -q -m gpu > gpurun_out/r02_bkq_slot_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_bkq_slot_tests.log
for rep in 1 2; do GBOPT_LDLT_KERNEL=cpanel GBOPT_LDLT_TIMING=1 timeout 300 python tools/ldlt_split.py 1500 4000 7100 2>&1 | grep -E "cpanel nb" ; done > gpurun_out/r02_bkq_slot.log
