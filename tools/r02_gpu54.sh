cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/r02_gather_tests3.log 2>&1; echo "rc=$?" >> gpurun_out/r02_gather_tests3.log
for rep in 1 2; do
for v in "1 0" "1 1"; do
  set -- $v
  for c in c1 c2; do
    GBOPT_ADJ_FUSE=$1 GBOPT_SYRK_GATHER=$2 timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-sharded 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('adjfuse=$1 gather=$2 $c', round(d['ms_per_step'],4), round(d['value'],1), 'resident', round(d.get('value_l2_resident') or 0,1), 'e2e', round(d['e2e']['value'],1), 'launches', d.get('gpu_launches'), 'parity', d.get('parity',{}).get('max_rel') if isinstance(d.get('parity'),dict) else d.get('parity'))" >> gpurun_out/r02_gather_ab3.log 2>&1
  done
done
done
timeout 120 python tools/timeline.py c1 > gpurun_out/r02_timeline_c1_gather3.txt 2>&1
