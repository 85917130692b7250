cd $GRAFT_REPO_ROOT
timeout 300 python tools/ncu_capture.py c2 > gpurun_out/r02_ncu_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:nt_mma -c 4 -o gpurun_out/r02_nt_c2 python tools/ncu_capture.py c2 > gpurun_out/r02_ncu_nt_c2.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-sharded --no-e2e --no-parity > gpurun_out/r02_b_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-sharded --no-e2e --no-parity > gpurun_out/r02_ncu_launches.log 2>&1
