cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/r02_flaky3.log
timeout 600 python tools/stress_adj3.py 300 2>&1 | tail -1 | sed 's/^/[stress] /' >> gpurun_out/r02_flaky3.log
./tools/adj_mma_conc.bin 10 | tail -1 | sed 's/^/[repro] /' >> gpurun_out/r02_flaky3.log
for i in 1 2 3; do
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_full_$i.log 2>&1
  tail -1 gpurun_out/r02_full_$i.log | sed "s/^/[full $i] /" >> gpurun_out/r02_flaky3.log
  grep FAILED gpurun_out/r02_full_$i.log >> gpurun_out/r02_flaky3.log
done
timeout 900 python bench.py > gpurun_out/r02_bench_c2_after.json 2> gpurun_out/r02_bench_c2_after.err
