"""KKT factorisation row (f3): GPU LDL^T (gbopt_ldlt_factor + one solve)
against the CPU oracle path (Ruiz + LAPACK sytrf via scipy, all threads)
on seeded IPM-like KKT matrices.  python tools/bench_ldlt.py [n ...]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_22462_b200 as gb  # noqa: E402
from oracle import ldlt_oracle as lo  # noqa: E402


def kkt(n, m, seed):
    rng = np.random.default_rng(seed)
    H = rng.uniform(-1, 1, (n, n))
    H = 0.5 * (H + H.T) + np.diag(10.0 ** rng.uniform(-2, 6, n))
    J = rng.uniform(-1, 1, (m, n))
    return np.block([[H, J.T], [J, -1e-8 * np.eye(m)]]), rng.uniform(-1, 1, n + m)


out = []
for n in [int(v) for v in sys.argv[1:]] or [784, 2000, 4000]:
    K, b = kkt(n, n // 8, n)
    gb.ldlt_factor(K).solve(b)  # warm-up
    t0 = time.perf_counter()
    f = gb.ldlt_factor(K)
    x = f.solve(b)
    tg = time.perf_counter() - t0
    t0 = time.perf_counter()
    inert = lo.inertia(K)
    xc = np.linalg.solve(K, b)
    tc = time.perf_counter() - t0
    out.append({"dim": K.shape[0], "gpu_factor_solve_s": tg, "cpu_oracle_s": tc, "inertia_gpu": f.inertia,
                "inertia_cpu": inert, "residual": float(np.abs(K @ x - b).max()), "cpu_threads": os.cpu_count()})
    print(json.dumps(out[-1]), flush=True)
