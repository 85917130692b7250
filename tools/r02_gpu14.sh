cd $GRAFT_REPO_ROOT
python tools/prof_outputs.py c2 j > gpurun_out/r02_prof_c2_j.txt 2>&1
python tools/prof_outputs.py c2 y > gpurun_out/r02_prof_c2_y.txt 2>&1
