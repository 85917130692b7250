cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2 3; do
  for lib in ab/lib_prev.so paper_2509_22462_b200/libgbopt_b200.so; do
    GBOPT_LIB=$GRAFT_REPO_ROOT/$lib timeout 300 python bench.py --config c2 --steps 30 --warmup 5 --no-cpu-baseline --no-sharded --no-parity 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib c2', round(d['ms_per_step'],4), round(d['value'],2), 'rowepi', d['kernel_breakdown'].get('row_epilogue',{}).get('ms'))" >> gpurun_out/r02_s0vec_ab.log 2>&1
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r02_s0vec_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_s0vec_tests.log
