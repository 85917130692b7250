cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/r02_small_ab.log
for v in 1 0 1 0; do
  GBOPT_SMALL_NET=$v timeout 300 python bench.py --config c1 --steps 30 --warmup 5 --no-cpu-baseline --no-sharded --no-parity 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('small=$v c1', round(d['ms_per_step'],4), round(d['value'],1), 'e2e', round(d['e2e']['value'],1))" >> gpurun_out/r02_small_ab.log 2>&1
  GBOPT_SMALL_NET=$v GBOPT_FWD_STREAM=0 timeout 120 python tools/fwd_bench.py c1 >> gpurun_out/r02_small_ab.log 2>&1
done
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02_small_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_small_tests.log
