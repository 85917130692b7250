cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/bench_ldlt.py 1000 1500 4000 6000 > gpurun_out/r02_ldlt_bench2.jsonl 2> gpurun_out/r02_ldlt_bench2.err
