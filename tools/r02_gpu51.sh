cd $GRAFT_REPO_ROOT
for rep in 1 2; do
  for lib in tools/libab/a518.so paper_2509_22462_b200/libgbopt_b200.so; do
    echo "== $lib" ; GBOPT_LIB=$lib GBOPT_LDLT_KERNEL=cpanel GBOPT_LDLT_TIMING=1 timeout 300 python tools/ldlt_split.py 4000 2>&1 | grep -E "cpanel nb" | cut -c1-250
  done
done
