cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
for lib in ab/lib_prev.so paper_2509_22462_b200/libgbopt_b200.so; do
  echo "== $lib" >> gpurun_out/r02_bkp_ilp.log
  GBOPT_LIB=$GRAFT_REPO_ROOT/$lib GBOPT_LDLT_KERNEL=panel GBOPT_LDLT_TIMING=1 timeout 300 python tools/ldlt_split.py 715 1500 2>&1 | grep -E "bkp_factor_kernel|factor .* ms solve" | awk 'NR%3!=1' >> gpurun_out/r02_bkp_ilp.log
done
done
timeout 900 python -m pytest tests/test_ldlt.py tests/test_gpu_ldlt_ref.py tests/test_kkt.py -x -q -m gpu > gpurun_out/r02_bkp_ilp_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_bkp_ilp_tests.log
