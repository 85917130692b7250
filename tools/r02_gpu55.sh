cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/r02_tail_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_tail_tests.log
for rep in 1 2; do
  for c in c1 c2; do
    timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-sharded 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],4), round(d['value'],1), 'resident', round(d.get('value_l2_resident') or 0,1), 'e2e', round(d['e2e']['value'],1), 'launches', d.get('gpu_launches'))" >> gpurun_out/r02_tail_ab.log 2>&1
  done
done
timeout 120 python tools/timeline.py c1 > gpurun_out/r02_timeline_c1_tail.txt 2>&1
