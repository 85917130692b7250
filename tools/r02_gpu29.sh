cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/r02_cpanel_cross.log
for k in "" cpanel panel grid; do
  GBOPT_LDLT_KERNEL=$k GBOPT_LDLT_TIMING=1 timeout 600 python tools/ldlt_split.py 300 704 1150 1500 4000 5400 7100 8000 10000 2>&1 | grep -E "cpanel nb|bkp_factor|bk_factor_kernel [0-9]|cpanel update" | grep -v " 0.0[0-9][0-9] ms" | sed "s/^/[${k:-default}] /" >> gpurun_out/r02_cpanel_cross.log
done
