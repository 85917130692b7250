cd $GRAFT_REPO_ROOT
GBOPT_LDLT_TIMING=1 timeout 300 python tools/ldlt_split.py 704 1500 > gpurun_out/r02_ldlt_split.log 2>&1
