cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/r02_pdl_ab.log
for v in 1 0 1 0; do
  for c in c1 c5 c2; do
    GBOPT_PDL=$v timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-sharded --no-parity --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl=$v', '$c', round(d['ms_per_step'],4), round(d['value'],1), d.get('schedule'))" >> gpurun_out/r02_pdl_ab.log 2>&1
  done
done
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02_pdl_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_pdl_tests.log
