cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
# launch list of the nt_mma launches of one c4 evaluation, then a full-set capture of the first tangent GEMM (the first launch > 10 ms)
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -k regex:nt_mma_kernel --csv --log-file gpurun_out/r02_c4_ntmma_list.csv python tools/ncu_capture.py c4 > /dev/null 2>&1
SKIP=$(python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/r02_c4_ntmma_list.csv')) if len(r)>10]
hdr=rows[0]; ki=hdr.index('ID'); mi=hdr.index('Metric Name'); vi=hdr.index('Metric Value')
ids=[]
for r in rows[1:]:
    if r[mi]=='gpu__time_duration.sum':
        ids.append((int(r[ki]), float(r[vi].replace(',',''))))
ids.sort()
for k,(i,t) in enumerate(ids):
    if t > 10e3 or t > 10e6:
        print(k); break
PY
)
echo "skip=$SKIP" > gpurun_out/r02_ncu_c4gemm.log
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:nt_mma_kernel --launch-skip $SKIP -c 1 -f -o gpurun_out/r02_ncu_c4gemm python tools/ncu_capture.py c4 >> gpurun_out/r02_ncu_c4gemm.log 2>&1
