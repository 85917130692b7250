cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
  for v in 8 4 6 16; do
    GBOPT_SYRK_MIN_KB=$v timeout 300 python bench.py --config c1 --steps 30 --warmup 5 --no-cpu-baseline --no-sharded 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('minkb=$v c1', round(d['ms_per_step'],4), round(d['value'],1), 'resident', round(d.get('value_l2_resident') or 0,1))" >> gpurun_out/r02_minkb_ab.log 2>&1
  done
done
