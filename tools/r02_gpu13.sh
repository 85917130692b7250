cd $GRAFT_REPO_ROOT
python tools/df_trace.py c1 > gpurun_out/r02_dftrace_c1.txt 2>&1
python tools/timeline.py c4 64 > gpurun_out/r02_timeline_c4.txt 2>&1
python tools/timeline.py c2 > gpurun_out/r02_timeline_c2.txt 2>&1
