# final refresh: per-config bench records, reference arm, smoke, GPU suite, c2 launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02_bench_c2.json 2> gpurun_out/r02_bench_c2.err
for c in c1 c3 c4 c5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r02_bench_$c.json 2> gpurun_out/r02_bench_$c.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_ref_c2.json 2> gpurun_out/r02_ref_c2.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_smoke.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r02_gputest_full.log 2>&1; echo "rc=$?" >> gpurun_out/r02_gputest_full.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-sharded > gpurun_out/r02_launches_c2.log 2>&1
