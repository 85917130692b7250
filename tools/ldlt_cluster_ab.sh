#!/bin/bash
# A/B of the cluster-barrier vs cooperative-grid Bunch-Kaufman factorisation
for c in 1 0; do
  echo "== GBOPT_LDLT_CLUSTER=$c"
  GBOPT_LDLT_CLUSTER=$c GBOPT_LDLT_TIMING=1 python tools/ldlt_split.py "$@" 2>&1 | grep -E "bk_factor|factor .*solve"
done
