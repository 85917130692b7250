cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/r02_flaky2.log
for i in 1 2 3; do
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_full_$i.log 2>&1
  tail -1 gpurun_out/r02_full_$i.log | sed "s/^/[full $i] /" >> gpurun_out/r02_flaky2.log
  grep FAILED gpurun_out/r02_full_$i.log >> gpurun_out/r02_flaky2.log
done
