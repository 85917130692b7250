cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for m in forward jacobian oracle; do timeout 300 python tools/ncu_paths.py $m c2 >> gpurun_out/r02_paths_plain.log 2>&1; done
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:fwd_row1 -c 6 -f -o gpurun_out/r02_ncu_fwd python tools/ncu_paths.py forward c2 > gpurun_out/r02_ncu_fwd.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:adj_ -c 12 -f -o gpurun_out/r02_ncu_jac python tools/ncu_paths.py jacobian c2 > gpurun_out/r02_ncu_jac.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:adj_cols -c 5 -f -o gpurun_out/r02_ncu_adj python tools/ncu_paths.py oracle c2 > gpurun_out/r02_ncu_adj.log 2>&1
ls -la gpurun_out/r02_ncu_*.ncu-rep >> gpurun_out/r02_paths_plain.log
