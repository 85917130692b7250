#!/bin/bash
# A/B of the grid factorisation kernel's panel width (GBOPT_LDLT_GRID_NB; 0 =
# unblocked left-looking): kernel time from GBOPT_LDLT_TIMING and the
# factor + solve residual from tools/bench_ldlt.py
dims=${*:-2500 4500 9000}
for nb in 0 32 64 96; do
  echo "== GBOPT_LDLT_GRID_NB=$nb"
  GBOPT_LDLT_KERNEL=grid GBOPT_LDLT_GRID_NB=$nb GBOPT_LDLT_TIMING=1 python tools/bench_ldlt.py $dims 2>&1 \
    | grep -E "bk_factor_kernel|residual" | grep -vE "^ldlt: .*panel"
done
