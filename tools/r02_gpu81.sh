cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
  for v in 2 3 4; do
    for c in c2 c3; do
      GBOPT_SYRK_SPLIT_MUL=$v timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-sharded --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mul=$v $c', round(d['ms_per_step'],4), round(d['value'],2), d['parity']['pass'])" >> gpurun_out/r02_splitmul_ab2.log 2>&1
    done
  done
done
