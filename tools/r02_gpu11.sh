cd $GRAFT_REPO_ROOT
for c in c2 c5; do for m in 1 0; do GBOPT_FWD_EVENTS=1 GBOPT_FWD_STREAM=$m python tools/fwd_bench.py $c 2>&1 | sort | uniq -c | sort -rn | head -4; done; done > gpurun_out/r02_fwd_events.log 2>&1
