cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/r02_fence.log
./tools/adj_mma_conc.bin 30 | tail -1 | sed 's/^/[repro 2cta] /' >> gpurun_out/r02_fence.log
./tools/adj_mma_conc.bin 30 1 | tail -1 | sed 's/^/[repro 2cta + noise] /' >> gpurun_out/r02_fence.log
timeout 900 python tools/stress_adj3.py 500 2>&1 | tail -1 | sed 's/^/[stress J 500] /' >> gpurun_out/r02_fence.log
for c in "c5 4 60" "c3 4 30" "c4 256 40"; do timeout 900 python tools/stress_oracle2.py $c 2>&1 | tail -1 | sed 's/^/[stress oracle] /' >> gpurun_out/r02_fence.log; done
for i in 1 2 3; do
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_full_$i.log 2>&1
  tail -1 gpurun_out/r02_full_$i.log | sed "s/^/[full $i] /" >> gpurun_out/r02_fence.log
  grep FAILED gpurun_out/r02_full_$i.log >> gpurun_out/r02_fence.log
done
timeout 900 python bench.py > gpurun_out/r02_bench_c2_fence.json 2> gpurun_out/r02_bench_c2_fence.err
for c in c4 c5; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-sharded > gpurun_out/r02_bench_${c}_fence.json 2>/dev/null; done
