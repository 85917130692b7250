cd $GRAFT_REPO_ROOT
timeout 300 python tools/jac_capture.py c2 > gpurun_out/r02_jac_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:adj_cols -c 2 -o gpurun_out/r02_adj_c2 python tools/jac_capture.py c2 > gpurun_out/r02_ncu_adj.log 2>&1
