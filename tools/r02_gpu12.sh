cd $GRAFT_REPO_ROOT
python bench.py > gpurun_out/r02_bench_c2b.json 2> gpurun_out/r02_bench_c2b.err
python tools/sched_compare.py c1 c5 > gpurun_out/r02_sched_c1.log 2>&1
python tools/timeline.py c1 > gpurun_out/r02_timeline_c1.txt 2>&1
