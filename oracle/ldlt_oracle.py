"""CPU oracle for the KKT factorisation row.

TEST INFRASTRUCTURE ONLY (see oracle/gbopt_oracle.py header).

Restates the reference ldlt_factor contract (proj/src/linalg.cpp:39-120,
393-438): the same checks, the same symmetric Ruiz equilibration
(linalg.cpp:72-99), a Bunch-Kaufman LDL^T of the equilibrated matrix
(scipy.linalg.ldl -- LAPACK sytrf, the same pivoting family as the
reference's blocked implementation, linalg.cpp:101-287) and the inertia from
the 1x1 / 2x2 pivot blocks with the zero threshold 1e-11 * max|SAS|.  The
solution is checked through residuals, not factor entries (pivot sequences
legitimately differ between blocked and unblocked Bunch-Kaufman).
"""
import numpy as np
import scipy.linalg


class OracleError(Exception):
    pass


def ruiz(A, rounds=20, tol=0.01):
    """linalg.cpp:72-99."""
    bal = np.array(A, dtype=np.float64, copy=True)
    n = bal.shape[0]
    equil = np.ones(n)
    for _ in range(rounds):
        cmax = np.abs(bal).max(axis=0) if n else np.zeros(0)
        rs = np.where(cmax > 0, 1.0 / np.sqrt(np.where(cmax > 0, cmax, 1.0)), 1.0)
        dev = np.abs(cmax[cmax > 0] - 1.0).max() if np.any(cmax > 0) else 0.0
        if dev <= tol:
            break
        bal = bal * rs[:, None] * rs[None, :]
        equil = equil * rs
    return bal, equil


def inertia(A):
    """(n_pos, n_neg, n_zero) as the reference classifies pivots."""
    A = np.asarray(A, dtype=np.float64)
    if not np.isfinite(A).all():
        raise OracleError("non-finite")
    bal, _ = ruiz(A)
    n = bal.shape[0]
    thresh = 1e-11 * (np.abs(bal).max() if n else 0.0)
    lu, d, perm = scipy.linalg.ldl(bal, lower=True)
    pos = neg = zero = 0
    k = 0
    while k < n:
        if k + 1 < n and d[k + 1, k] != 0.0:
            eigs = np.linalg.eigvalsh(d[k:k + 2, k:k + 2])
            k += 2
        else:
            eigs = [d[k, k]]
            k += 1
        for e in eigs:
            if abs(e) <= thresh:
                zero += 1
            elif e > 0:
                pos += 1
            else:
                neg += 1
    return pos, neg, zero


def matrix_with_spectrum(rng, eigs):
    """tests/test_util.hpp:46-67: Q diag(eigs) Q^T with a seeded orthogonal Q."""
    n = len(eigs)
    m = rng.uniform(-1, 1, (n, n))
    q, r = np.linalg.qr(m)
    q = q * np.sign(np.diag(r))[None, :]
    a = q @ np.diag(eigs) @ q.T
    return 0.5 * (a + a.T)
