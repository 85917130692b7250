cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/r02_cpanel16.log
for c in 8 16; do
  GBOPT_LDLT_CPANEL_CTAS=$c GBOPT_LDLT_KERNEL=cpanel GBOPT_LDLT_TIMING=1 timeout 900 python tools/ldlt_split.py 4000 8000 10000 14000 20500 2>&1 | grep -E "cpanel nb|^[0-9]|rror" | sed "s/^/[$c] /" >> gpurun_out/r02_cpanel16.log
done
GBOPT_LDLT_KERNEL=grid GBOPT_LDLT_TIMING=1 timeout 900 python tools/ldlt_split.py 14000 20500 2>&1 | grep -E "bk_factor_kernel [0-9]|^[0-9]" | grep -v " 0.0[0-9][0-9] ms" | sed "s/^/[grid] /" >> gpurun_out/r02_cpanel16.log
