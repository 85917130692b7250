cd $GRAFT_REPO_ROOT
for a in "96 3 1 0" "44 2 1 0" "64 3 1 0" "67 3 0 0" "67 3 1 1" "66 3 1 0" "23 1 1 0"; do timeout 300 python tools/debug_multi2.py $a 2>&1 | tail -2; done > gpurun_out/r02_debug_multi3.log
./tools/read_probe2.bin > gpurun_out/r02_read_probe2.log 2>&1
