# refresh the per-config bench records with the current build
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in c2 c1 c3 c4 c5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r02_bench_$c.json 2> gpurun_out/r02_bench_$c.err
done
timeout 600 python bench.py --impl reference --config c2 --steps 3 --warmup 1 > gpurun_out/r02_ref_c2.json 2> gpurun_out/r02_ref_c2.err
