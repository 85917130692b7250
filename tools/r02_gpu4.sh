cd $GRAFT_REPO_ROOT
for a in "64 2" "67 3" "64 1"; do echo "== $a"; timeout 300 python tools/debug_multi.py $a 2>&1 | tail -20; done > gpurun_out/r02_debug_multi.log
timeout 300 compute-sanitizer --tool memcheck python tools/debug_multi.py 64 2 > gpurun_out/r02_debug_multi_san.log 2>&1
python -m pytest tests/test_gpu_multirank.py -q -p no:cacheprovider -k c2 > gpurun_out/r02_multirank_c2.log 2>&1
