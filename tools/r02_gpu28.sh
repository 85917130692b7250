cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/r02_cpanel_split.log
timeout 600 python -m pytest tests/test_gpu_ldlt_ref.py -x -q -k panel > gpurun_out/r02_cpanel_tests.log 2>&1
echo "ref tests rc $?" >> gpurun_out/r02_cpanel_tests.log
GBOPT_LDLT_KERNEL=cpanel timeout 600 python -m pytest tests/test_gpu_ldlt_ref.py -x -q -k n4000 >> gpurun_out/r02_cpanel_tests.log 2>&1
echo "n4000 rc $?" >> gpurun_out/r02_cpanel_tests.log
GBOPT_LDLT_KERNEL=cpanel timeout 900 python -m pytest tests/test_ldlt.py -x -q -m gpu >> gpurun_out/r02_cpanel_tests.log 2>&1
echo "test_ldlt rc $?" >> gpurun_out/r02_cpanel_tests.log
for k in cpanel; do
  echo "== $k" >> gpurun_out/r02_cpanel_split.log
  GBOPT_LDLT_KERNEL=$k GBOPT_LDLT_TIMING=1 timeout 300 python tools/ldlt_split.py 300 704 1500 4000 10000 2>&1 | grep -E "bkp_|cpanel|bk_factor|^[0-9]" >> gpurun_out/r02_cpanel_split.log
done
