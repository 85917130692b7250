# Round-1 final captures (c2): launch list + ncu --set full of nt_mma (GEMM and
# SYRK launches) and of the forward / adjoint GEMVs.
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2b.csv $CMD > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:nt_mma_kernel -s 6 -c 4 -o gpurun_out/prof_nt_mma_b $CMD > gpurun_out/ncu_full_b.log 2>&1
ncu --set full --clock-control none -k regex:"fwd_row1|adj_cols" -s 12 -c 4 -o gpurun_out/prof_gemv_b $CMD > gpurun_out/ncu_gemv_b.log 2>&1
ls -la gpurun_out/*.ncu-rep
