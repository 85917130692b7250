cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/sanitize_f3.py > gpurun_out/r02_san_plain.log 2>&1
for t in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python tools/sanitize_f3.py > gpurun_out/r02_san_$t.log 2>&1
  echo "$t rc $?" >> gpurun_out/r02_san_summary.log
done
