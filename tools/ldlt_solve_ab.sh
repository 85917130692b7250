#!/bin/bash
# substitution A/B: one CTA vs the grid-wide kernel
for sv in cta grid; do
  echo "== GBOPT_LDLT_SOLVE=$sv"
  GBOPT_LDLT_SOLVE=$sv python tools/ldlt_solve_probe.py "$@"
done
