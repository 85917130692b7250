cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r02_gputest_split2.log 2>&1; echo "rc=$?" >> gpurun_out/r02_gputest_split2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r02_bench_c2.json 2> gpurun_out/r02_bench_c2.err
timeout 900 python bench.py --config c1 --steps 10 --warmup 3 > gpurun_out/r02_bench_c1.json 2> gpurun_out/r02_bench_c1.err
for cfg in "c2 1 40" "c2 3 20"; do
  timeout 600 python tools/stress_oracle2.py $cfg >> gpurun_out/r02_stress_split2.log 2>&1; echo "$cfg rc=$?" >> gpurun_out/r02_stress_split2.log
done
