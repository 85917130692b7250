cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
  for v in 0 1; do
    for c in c4; do
      GBOPT_S0_PASS=$v timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-sharded 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('s0=$v $c', round(d['ms_per_step'],3), round(d['value'],1), 'eval', round(d['roofline_eval']['frac_of_peak'],4), 'e2e', round(d['e2e']['value'],1))" >> gpurun_out/r02_s0_ab2.log 2>&1
    done
  done
done
GBOPT_S0_PASS=1 timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r02_s0_tests2.log 2>&1; echo "rc=$?" >> gpurun_out/r02_s0_tests2.log
