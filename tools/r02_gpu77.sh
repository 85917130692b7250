cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
  for v in 0 1; do
    for c in c2 c1; do
      GBOPT_SIDE_HIGH=$v timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-sharded --no-parity --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('side_high=$v $c', round(d['ms_per_step'],4), round(d['value'],2))" >> gpurun_out/r02_sidehigh_ab.log 2>&1
    done
  done
done
