"""Repeat factorisations (cluster-panel / panel / grid kernels) of one KKT
matrix and check bitwise-identical inertia and solutions, single-threaded
and from two host threads at once.  python tools/stress_ldlt.py [n] [reps]"""
import os
import sys
import threading

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ldlt_split import kkt, gb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
K, b = kkt(n, n // 8, n)
f0 = gb.ldlt_factor(K)
x0 = f0.solve(b)
in0 = f0.inertia
bad = [0, 0, 0]
for r in range(reps):
    f = gb.ldlt_factor(K)
    x = f.solve(b)
    if f.inertia != in0 or not np.array_equal(x, x0):
        bad[0] += 1
        print("single rep", r, "differs", f.inertia, float(np.abs(x - x0).max()), flush=True)


def work(t):
    for r in range(reps):
        f = gb.ldlt_factor(K)
        x = f.solve(b)
        if f.inertia != in0 or not np.array_equal(x, x0):
            bad[1 + t] += 1
            print("thread", t, "rep", r, "differs", f.inertia, float(np.abs(x - x0).max()), flush=True)


ths = [threading.Thread(target=work, args=(t,)) for t in range(2)]
for th in ths:
    th.start()
for th in ths:
    th.join()
print("n", K.shape[0], "kernel", os.environ.get("GBOPT_LDLT_KERNEL", "default"), "bad", bad, flush=True)
