# Round-1 GPU session: other-config benches, the c2 launch list and one
# ncu --set full capture of the dominant kernel (nt_mma_kernel).
set -x
for c in c1 c3 c4 c5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $CMD > gpurun_out/ncu_launches.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:nt_mma -s 4 -c 2 -o gpurun_out/prof_nt_mma $CMD > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none -k regex:"fwd_rows|adj_cols" -s 22 -c 4 -o gpurun_out/prof_gemv $CMD > gpurun_out/ncu_gemv.log 2>&1
ls -la gpurun_out
