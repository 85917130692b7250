cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in c2 c1 c5; do timeout 600 python tools/bench_reduced_space.py $c 10 3; done > gpurun_out/r02_reduced_space.jsonl 2> gpurun_out/r02_reduced_space.err
for c in c2 c1 c5; do timeout 900 python tools/bench_newton_step.py $c 5; done > gpurun_out/r02_newton.jsonl 2> gpurun_out/r02_newton.err
