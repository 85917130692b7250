cd $GRAFT_REPO_ROOT
for k in cpanel panel grid; do
  GBOPT_LDLT_KERNEL=$k GBOPT_LDLT_TIMING=1 timeout 600 python tools/ldlt_split.py 1150 1500 4000 7100 8000 2>&1 | grep -E "cpanel nb|bkp_factor|bk_factor_kernel [0-9]" | grep -v " 0.0[0-9][0-9] ms" | awk 'NR%2==1' | sed "s/^/[$k] /" | cut -c1-110
done
