"""Repeat the reverse-mode Jacobian (adj_mma path) and the 4-point c3-shaped
oracle on the c2 shape and check bitwise repeatability; then compare once
with the reference build.  python tools/stress_adj.py [reps]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_22462_b200 as gb  # noqa: E402
from oracle import gbopt_oracle as o  # noqa: E402
from oracle import ref  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
ref.set_threads(os.cpu_count() or 1)
wl = ref.make_config("c3", batch=4, hidden=ref.TANH)
net = gb.NeuralNet.from_layers([w for w, _, _ in wl.layers], [b for _, b, _ in wl.layers],
                               [a for _, _, a in wl.layers]).bind_device(0)
x = wl.X[0]
J0 = net.jacobian(x)
bad = 0
for r in range(reps):
    J = net.jacobian(x)
    if not np.array_equal(J, J0):
        bad += 1
        print("rep", r, "J differs: max rel", o.rel_err(J, J0), flush=True)
print("jacobian: %d of %d repeats differ" % (bad, reps), flush=True)
Y0, Jt0, H0 = net.oracle_batched(wl.X, wl.Lam)
badh = 0
for r in range(reps):
    Y, Jt, H = net.oracle_batched(wl.X, wl.Lam)
    if not np.array_equal(H, H0):
        badh += 1
        print("rep", r, "H differs: max rel", max(o.rel_err(H[i], H0[i]) for i in range(4)), flush=True)
print("oracle_batched(4): %d of %d repeats differ" % (badh, reps), flush=True)
rn = wl.net()
RJ = rn.jacobian(x)
print("J vs reference:", o.rel_err(J0, RJ))
RY, RJ4, RH = rn.oracle_batched(wl.X, wl.Lam)
print("H vs reference:", [o.rel_err(H0[i], RH[i]) for i in range(4)])
RJb = rn.jacobian(x)
print("reference J repeat identical:", np.array_equal(RJ, RJb), o.rel_err(RJ, RJb))
