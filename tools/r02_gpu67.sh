cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/r02_gemmfuse_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_gemmfuse_tests.log
for rep in 1 2 3; do
  for lib in ab/lib_prev.so paper_2509_22462_b200/libgbopt_b200.so; do
    for c in c2 c1; do
      GBOPT_LIB=$GRAFT_REPO_ROOT/$lib timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-sharded 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib $c', round(d['ms_per_step'],4), round(d['value'],1), 'resident', round(d.get('value_l2_resident') or 0,1), 'e2e', round(d['e2e']['value'],1), 'launches', d.get('gpu_launches'), 'clk', d.get('clocks',{}).get('sm_mhz'), d.get('clocks',{}).get('reasons'))" >> gpurun_out/r02_gemmfuse_ab.log 2>&1
    done
  done
done
timeout 400 python bench.py --config c4 --steps 10 --warmup 3 > gpurun_out/r02_bench_c4.json 2> gpurun_out/r02_bench_c4.err
