cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/r02_chunks_ab.log
for ch in 4 8 16 4 8 16; do
  GBOPT_HOST_CHUNKS=$ch timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --no-sharded --no-parity 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chunks=$ch c4', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))" >> gpurun_out/r02_chunks_ab.log 2>&1
done
for ch in 2 4 2 4; do
  GBOPT_HOST_CHUNKS=$ch timeout 600 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline --no-sharded --no-parity 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chunks=$ch c5', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))" >> gpurun_out/r02_chunks_ab.log 2>&1
done
