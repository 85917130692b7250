cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
  for v in 0 1; do
    for c in c2 c3 c4; do
      st=30; [ $c != c2 ] && st=8
      GBOPT_FWD_ADJ3=$v timeout 400 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --no-sharded --no-parity --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fwdadj3=$v $c', round(d['ms_per_step'],4), round(d['value'],2))" >> gpurun_out/r02_fwdadj3_ab.log 2>&1
    done
  done
done
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/r02_fwdadj3_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_fwdadj3_tests.log
timeout 120 python tools/timeline.py c2 > gpurun_out/r02_timeline_c2_3s.txt 2>&1
