cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_forward_stream.py tests/test_gpu_multidevice.py tests/test_cpp_api.py tests/test_gpu_gbnn_e2e.py -q -s -p no:cacheprovider -m gpu > gpurun_out/r02_gpu7.log 2>&1; echo "rc=$?" >> gpurun_out/r02_gpu7.log
for c in c2 c5 c1; do GBOPT_FWD_STREAM=1 python tools/fwd_bench.py $c; GBOPT_FWD_STREAM=0 python tools/fwd_bench.py $c; done > gpurun_out/r02_fwd_bench.jsonl 2>&1
