cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --config c1 --steps 10 --warmup 3 > gpurun_out/r02_bench_c1.json 2> gpurun_out/r02_bench_c1.err
