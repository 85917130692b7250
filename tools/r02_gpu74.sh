# final validation of the last commit: GPU suite, smoke, default bench, c1 launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r02_gputest_last.log 2>&1; echo "rc=$?" >> gpurun_out/r02_gputest_last.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_smoke_last.log 2>&1
timeout 900 python bench.py > gpurun_out/r02_bench_last.json 2> gpurun_out/r02_bench_last.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/r02_launches_c1.csv python bench.py --config c1 --steps 2 --warmup 1 --no-cpu-baseline --no-sharded --no-e2e --no-parity > gpurun_out/r02_launches_c1.log 2>&1
