cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/c1_launches.py c1 > gpurun_out/r02_c1_plain.log 2>&1 && \
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c1_launches.csv python tools/c1_launches.py c1 > gpurun_out/r02_c1_ncu.log 2>&1
echo "rc $?" >> gpurun_out/r02_c1_ncu.log
