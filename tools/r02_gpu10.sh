cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_forward_stream.py -q -p no:cacheprovider > gpurun_out/r02_fwdtest3.log 2>&1
for c in c2 c5 c1; do GBOPT_FWD_STREAM=1 python tools/fwd_bench.py $c; GBOPT_FWD_STREAM=0 python tools/fwd_bench.py $c; done > gpurun_out/r02_fwd_bench3.jsonl 2>&1
GBOPT_FWD_STREAM=1 python tools/fwd_bench.py c2 > gpurun_out/r02_fwd_plain3.json 2>&1 && \
GBOPT_FWD_STREAM=1 ncu --set full --clock-control none --import-source on -k regex:fwd_stream_kernel -c 1 -o gpurun_out/r02_fwd_stream3 python tools/fwd_bench.py c2 > gpurun_out/r02_ncu_fwd_stream3.log 2>&1
