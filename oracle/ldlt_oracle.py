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


# ---- KKT assembly and inertia correction (ipm.cpp:466-557) ----------------

K_DELTA_C = 1e-8      # ipm.cpp:23
K_DELTA_C_MAX = 1e-2  # ipm.cpp:24


def assemble_kkt(x, lower, z, lam, grad_f, g, jac_rows, jac_cols, jac_values, hess_rows, hess_cols, hess_values,
                 mu, delta_w=0.0, delta_c=0.0):
    """ipm.cpp:466-518, element by element in the reference's order: the
    Hessian triplets (mirrored off the diagonal), then Sigma and delta_w on
    the (1,1) diagonal, then the Jacobian triplets into both off-diagonal
    blocks, then -delta_c; rhs = [-grad_f - J^T lambda (+ mu / (x - lower));
    -g] with J^T lambda as jac_t_lambda (ipm.cpp:33-42).  Python floats:
    every operation rounds once, like the reference built without FMA
    contraction.  Returns (mat, rhs)."""
    x, lower, z = (np.asarray(v, dtype=np.float64) for v in (x, lower, z))
    n, m = x.size, np.asarray(g).size
    mat = [[0.0] * (n + m) for _ in range(n + m)]
    for r, c, v in zip(hess_rows, hess_cols, hess_values):
        mat[r][c] += float(v)
        if r != c:
            mat[c][r] += float(v)
    for i in range(n):
        if np.isfinite(lower[i]):
            mat[i][i] += float(z[i]) / (float(x[i]) - float(lower[i]))
        if delta_w != 0.0:
            mat[i][i] += delta_w
    for r, c, v in zip(jac_rows, jac_cols, jac_values):
        mat[n + r][c] += float(v)
        mat[c][n + r] += float(v)
    if delta_c != 0.0:
        for i in range(m):
            mat[n + i][n + i] -= delta_c
    jt = [0.0] * n
    for r, c, v in zip(jac_rows, jac_cols, jac_values):
        jt[c] += float(v) * float(lam[r])
    rhs = [-float(grad_f[i]) - jt[i] for i in range(n)]
    for i in range(n):
        if np.isfinite(lower[i]):
            rhs[i] += mu / (float(x[i]) - float(lower[i]))
    rhs += [-float(v) for v in g]
    return np.array(mat, dtype=np.float64).reshape(n + m, n + m), np.array(rhs, dtype=np.float64)


def inertia_correct(mat, n, m, delta0=1e-4, delta_growth=10.0, delta_max=1e40, delta_w_start=0.0,
                    inertia_fn=None):
    """ipm.cpp:520-557 with this module's inertia() (or `inertia_fn`, e.g. the
    reference's own ldlt_factor from oracle/ref.py): returns (delta_w,
    delta_c, inertia) of the first shifted matrix with inertia (n, m, 0)."""
    inertia_of = inertia_fn or inertia
    delta_w, delta_c = delta_w_start, 0.0
    while True:
        t = np.array(mat, dtype=np.float64, copy=True)
        if delta_w != 0.0:
            t[np.arange(n), np.arange(n)] += delta_w
        if delta_c != 0.0:
            t[n + np.arange(m), n + np.arange(m)] -= delta_c
        got = tuple(inertia_of(t))
        if got == (n, m, 0):
            return delta_w, delta_c, got
        if got[2] > 0 and m > 0 and delta_c < K_DELTA_C_MAX:
            delta_c = K_DELTA_C if delta_c == 0.0 else delta_c * 1e2
            continue
        delta_w = delta0 if delta_w == 0.0 else delta_w * delta_growth
        if delta_w > delta_max:
            raise OracleError("inertia correction: regularization exceeded the configured maximum")
