cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:nt_mma_kernel -c 3 -f -o gpurun_out/r02_ncu_c1 python tools/ncu_capture.py c1 > gpurun_out/r02_ncu_c1.log 2>&1
