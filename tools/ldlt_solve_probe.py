"""Solve-phase probe for the native LDL^T: substitution alone (keep_input=False)
vs with refinement, and the device kernel time per substitution."""
import sys, time
import numpy as np
sys.path.insert(0, '/root/repo')
import paper_2509_22462_b200 as gb
from ldlt_split import kkt  # noqa: E402
for n in [int(v) for v in sys.argv[1:]] or (784, 2000, 4000, 8000):
    K, b = kkt(n, n // 8, n)
    for keep in (False, True):
        f = gb.ldlt_factor(K, keep_input=keep)
        f.solve(b)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter(); x = f.solve(b); ts.append(time.perf_counter() - t0)
        print(K.shape[0], "keep" if keep else "plain", "solve %.2f ms" % (min(ts) * 1e3),
              "resid %.2e" % np.abs(K @ x - b).max(), flush=True)
