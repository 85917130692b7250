"""KKT factorisation row (f3): GPU LDL^T (gbopt_ldlt_factor + one refined
solve, host matrix in) against the reference's OWN linalg.cpp (oracle/_ref:
ldlt_factor with Ruiz equilibration + blocked Bunch-Kaufman, then solve with
iterative refinement; OpenBLAS products on all host threads) on seeded
IPM-like KKT matrices.  Both sides do the same work: one factorisation and
one refined solve.  python tools/bench_ldlt.py [n ...]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_22462_b200 as gb  # noqa: E402
from oracle import ref  # noqa: E402


def kkt(n, m, seed):
    rng = np.random.default_rng(seed)
    H = rng.uniform(-1, 1, (n, n))
    H = 0.5 * (H + H.T) + np.diag(10.0 ** rng.uniform(-2, 6, n))
    J = rng.uniform(-1, 1, (m, n))
    return np.block([[H, J.T], [J, -1e-8 * np.eye(m)]]), rng.uniform(-1, 1, n + m)


threads = os.cpu_count() or 1
ref.set_threads(threads)
out = []
for n in [int(v) for v in sys.argv[1:]] or [784, 2000, 4000]:
    K, b = kkt(n, n // 8, n)
    gb.ldlt_factor(K).solve(b)  # warm-up
    t0 = time.perf_counter()
    f = gb.ldlt_factor(K)
    x = f.solve(b)
    tg = time.perf_counter() - t0
    t0 = time.perf_counter()
    rf = ref.RefLdlt(K)
    xr = rf.solve(b)
    tc = time.perf_counter() - t0
    out.append({"dim": K.shape[0], "gpu_factor_solve_s": tg, "ref_linalg_factor_solve_s": tc,
                "inertia_gpu": f.inertia, "inertia_ref": rf.inertia,
                "residual_gpu": float(np.abs(K @ x - b).max()), "residual_ref": float(np.abs(K @ xr - b).max()),
                "cpu_threads": threads, "cpu": "reference linalg.cpp (oracle/_ref), OpenBLAS products"})
    print(json.dumps(out[-1]), flush=True)
