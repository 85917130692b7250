cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
  for v in none gemm syrk; do
    E=""; [ $v = gemm ] && E="GBOPT_HACK_NOSCALE=1"; [ $v = syrk ] && E="GBOPT_HACK_NOSCALE_SYRK=1"
    for c in c4 c2; do
      env $E timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-sharded --no-parity --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('noscale=$v $c', round(d['ms_per_step'],3), round(d['value'],1), {k: round(v['ms'],3) for k,v in d['kernel_breakdown'].items() if k.startswith('nt_mma')})" >> gpurun_out/r02_noscale.log 2>&1
    done
  done
done
