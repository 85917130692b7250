cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/r02_fwdy.log
for v in 0 1 0 1; do for c in c2 c5 c1; do GBOPT_FWD_STREAM=0 GBOPT_FWD_SMEM_Y=$v timeout 120 python tools/fwd_bench.py $c >> gpurun_out/r02_fwdy.log 2>&1; done; done
GBOPT_FWD_SMEM_Y=1 timeout 900 ncu --profile-from-start off --set full --clock-control none -k regex:fwd_row1 -c 6 -f -o gpurun_out/r02_ncu_fwd2 python tools/ncu_paths.py forward c2 > gpurun_out/r02_ncu_fwd2.log 2>&1
timeout 600 python -m pytest tests/test_gpu_forward_stream.py tests/test_gpu_parity.py -x -q > gpurun_out/r02_fwdy_tests.log 2>&1; echo "rc $?" >> gpurun_out/r02_fwdy_tests.log
