#!/bin/bash
# A/B of the three Bunch-Kaufman factorisation kernels (blocked / one-cluster / grid)
for c in panel cluster grid; do
  echo "== GBOPT_LDLT_KERNEL=$c"
  GBOPT_LDLT_KERNEL=$c GBOPT_LDLT_TIMING=1 python tools/ldlt_split.py "$@" 2>&1 | grep -E "bkp_factor|bkc_factor|bk_factor_kernel [0-9]|factor .*solve"
done
