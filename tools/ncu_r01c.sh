# Session-2 final captures (c2, layer-by-layer schedule = the bench's auto pick):
# launch list of one evaluation, ncu --set full of one tangent GEMM and one SYRK.
CMD="python tools/ncu_capture.py c2"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,launch__grid_size
GBOPT_DATAFLOW=0 timeout 600 ncu --profile-from-start off --clock-control none --metrics $M --csv \
  --log-file gpurun_out/ncu_launch_c2_final.csv $CMD > gpurun_out/ncu_launch_c2_final.log 2>&1
GBOPT_DATAFLOW=0 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:nt_mma_kernel -c 3 -o gpurun_out/nt_c2_final $CMD > gpurun_out/ncu_full_c2_final.log 2>&1
ls -la gpurun_out/*final*
