cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/r02_flaky.log
for i in 1 2; do
  timeout 600 python -m pytest tests/test_gpu_ref_parity.py -q -p no:cacheprovider 2>&1 | tail -1 | sed "s/^/[ref_parity alone $i] /" >> gpurun_out/r02_flaky.log
done
for f in test_gpu_multidevice test_gpu_multirank test_gpu_parity test_gpu_ldlt_ref test_gpu_jacobian test_gpu_gbnn_e2e test_gpu_forward_stream test_gpu_edges test_gpu_dataflow; do
  timeout 900 python -m pytest tests/$f.py tests/test_gpu_ref_parity.py -q -p no:cacheprovider 2>&1 | tail -1 | sed "s/^/[$f + ref_parity] /" >> gpurun_out/r02_flaky.log
done
