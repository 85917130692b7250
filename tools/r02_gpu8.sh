cd $GRAFT_REPO_ROOT
GBOPT_FWD_STREAM=1 python tools/fwd_bench.py c2 > gpurun_out/r02_fwd_plain.json 2>&1 && \
GBOPT_FWD_STREAM=1 ncu --set full --clock-control none --import-source on -k regex:fwd_stream_kernel -c 1 -o gpurun_out/r02_fwd_stream python tools/fwd_bench.py c2 > gpurun_out/r02_ncu_fwd_stream.log 2>&1
