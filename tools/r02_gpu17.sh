cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_gputest_full.log 2>&1; echo "rc=$?" >> gpurun_out/r02_gputest_full.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke2.log 2>&1
for c in c1 c3 c4 c5; do python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r02_bench_$c.json 2> gpurun_out/r02_bench_$c.err; done
python bench.py --impl reference --config c2 --steps 5 --warmup 1 > gpurun_out/r02_ref_c2b.json 2>&1
