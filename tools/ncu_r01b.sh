# Round-1 (session 2) per-config launch metrics of one evaluation: DRAM bytes,
# duration and DMMA-pipe activity of every kernel launch (ncu replays each).
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,launch__grid_size
for c in c1 c2 c3 c4 c5; do
  timeout 900 ncu --profile-from-start off --clock-control none --metrics $M --csv \
    --log-file gpurun_out/ncu_launch_$c.csv python tools/ncu_capture.py $c > gpurun_out/ncu_launch_$c.log 2>&1
done
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:df_kernel -c 1 \
  -o gpurun_out/df_c5 python tools/ncu_capture.py c5 > gpurun_out/ncu_df_c5.log 2>&1
ls -la gpurun_out/*.csv gpurun_out/*.ncu-rep
