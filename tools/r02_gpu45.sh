cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
GBOPT_LDLT_KERNEL=panel timeout 600 ncu --set full --clock-control none --import-source on -k regex:bkp_factor -c 1 -f -o gpurun_out/r02_ncu_bkp python tools/ldlt_ncu_driver.py 704 > gpurun_out/r02_ncu_bkp.log 2>&1
echo rc=$? >> gpurun_out/r02_ncu_bkp.log
