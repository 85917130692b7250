"""Reduced-space ("gray box") embedding callbacks over the B200 oracle.

Python mirror of ``gbopt::b200::ReducedSpaceOracle`` (include/gbopt/nn_b200.hpp),
restating the reference's ``embed_reduced_space`` block
(proj/src/formulations.cpp:267-349):

* variables of the block are ``xb = [x (n inputs); y (m outputs)]``;
* residual ``r = y - NN(x)`` (formulations.cpp:317-319);
* Jacobian values: ``-J`` row-major over the inputs, then ``+1`` per output
  (formulations.cpp:320-331), pattern rows/cols from ``jac_pattern()``;
* Lagrangian-Hessian values over the dense lower triangle of the inputs,
  with the network oracle seeing ``-lambda`` because
  ``L = f + lambda^T (y - NN(x))`` (formulations.cpp:298-315, 332-340);
  local (r, c) are flipped where the host's input indices are not
  ascending, exactly like the reference.

Each callback does the least device work that answers it and caches per x,
and every quantity has exactly one producer, so a callback's value at x does
not depend on which callbacks ran before it: residual -> forward, Jacobian ->
reverse mode (m sweeps), Hessian -> the fused evaluation with the Hessian
only (its y and J are not kept).
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import numpy as np

from .gbopt import NeuralNet


class ReducedSpaceBlock:
    def __init__(self, net: NeuralNet, input_vars: Optional[Sequence[int]] = None):
        self.net = net
        self.n = net.input_dim
        self.m = net.output_dim
        self.input_vars = list(range(self.n)) if input_vars is None else list(input_vars)
        if len(self.input_vars) != self.n:
            raise ValueError("input_vars must have one host index per network input")
        self._y = self._yx = None
        self._j = self._jx = None
        self._h = self._hx = self._hl = None
        self.evaluations = 0
        hr, hc = [], []
        for a in range(self.n):
            for b in range(a + 1):
                r, c = a, b
                if self.input_vars[a] < self.input_vars[b]:
                    r, c = c, r
                hr.append(r)
                hc.append(c)
        self.hess_rows = np.array(hr, dtype=np.int64)
        self.hess_cols = np.array(hc, dtype=np.int64)

    # ---- sparsity patterns (formulations.cpp:286-315) ----
    def jac_pattern(self) -> Tuple[np.ndarray, np.ndarray]:
        rows = [i for i in range(self.m) for _ in range(self.n)] + list(range(self.m))
        cols = [j for _ in range(self.m) for j in range(self.n)] + [self.n + i for i in range(self.m)]
        return np.array(rows, dtype=np.int64), np.array(cols, dtype=np.int64)

    def hess_pattern(self) -> Tuple[np.ndarray, np.ndarray]:
        return self.hess_rows, self.hess_cols

    # ---- callbacks ----
    def residual(self, xb) -> np.ndarray:
        xb = np.asarray(xb, dtype=np.float64)
        x = xb[:self.n]
        if self._yx is None or not np.array_equal(x, self._yx):
            self._y = self.net.forward(x)
            self._yx = x.copy()
            self.evaluations += 1
        return xb[self.n:self.n + self.m] - self._y

    def jacobian(self, xb) -> np.ndarray:
        x = np.asarray(xb, dtype=np.float64)[:self.n]
        if self._jx is None or not np.array_equal(x, self._jx):
            self._j = self.net.jacobian(x)
            self._jx = x.copy()
            self.evaluations += 1
        return np.concatenate([-self._j.reshape(-1), np.ones(self.m)])

    def lag_hessian(self, xb, lam) -> np.ndarray:
        x = np.asarray(xb, dtype=np.float64)[:self.n]
        neg = -np.asarray(lam, dtype=np.float64)
        if self._hx is None or not np.array_equal(x, self._hx) or not np.array_equal(neg, self._hl):
            # the device packs the lower triangle in the pattern's value order
            # (a flipped (r, c) pattern entry has the same value: H is symmetric)
            _, _, hv = self.net.oracle_lower(x, neg, want_y=False, want_j=False)
            self._h = hv
            self._hx = x.copy()
            self._hl = neg.copy()
            self.evaluations += 1
        return self._h.copy()
