cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/r02_amfuse_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_amfuse_tests.log
for rep in 1 2; do
  for lib in ab/lib_prev.so paper_2509_22462_b200/libgbopt_b200.so; do
    GBOPT_LIB=$GRAFT_REPO_ROOT/$lib timeout 300 python bench.py --config c2 --steps 30 --warmup 5 --no-cpu-baseline --no-sharded 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib c2', round(d['value'],1), 'hbm_paths', {k: round(v['ms'],4) for k,v in (d.get('hbm_paths') or {}).items()})" >> gpurun_out/r02_amfuse_ab.log 2>&1
  done
done
