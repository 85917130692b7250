cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
  timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r02_suite_rep$rep.log 2>&1; echo "rc=$?" >> gpurun_out/r02_suite_rep$rep.log
done
# the single-point chain (gather, fused adjoint, forward tail) under two concurrent handles
for cfg in "c1 1 200" "c2 1 40" "c2 3 20"; do
  timeout 600 python tools/stress_oracle2.py $cfg >> gpurun_out/r02_stress_single.log 2>&1; echo "$cfg rc=$?" >> gpurun_out/r02_stress_single.log
done
