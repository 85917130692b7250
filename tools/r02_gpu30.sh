cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/r02_bkp_ab.log
for rep in 1 2; do
for k in panel; do
  GBOPT_LDLT_KERNEL=$k GBOPT_LDLT_TIMING=1 timeout 300 python tools/ldlt_split.py 300 704 1500 2>&1 | grep -E "bkp|bkq" >> gpurun_out/r02_bkp_ab.log
done
done
