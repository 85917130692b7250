"""Two handles of one net evaluated concurrently from two host threads
(distinct workspaces / streams, shared GPU): every result must equal the
single-threaded result bitwise.  Exercises the tangent GEMM / SYRK
(nt_mma), forward and adjoint kernels under overlap.
python tools/stress_oracle2.py [config] [batch] [reps]"""
import os
import sys
import threading

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_22462_b200 as gb  # noqa: E402
from paper_2509_22462_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 4
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 30
wl = configs.make(name, batch=B)
layers = [wl.net.layer(l) for l in range(wl.net.layer_count)]
mk = lambda: gb.NeuralNet.from_layers([w for w, _, _ in layers], [b for _, b, _ in layers],  # noqa: E731
                                      [a for _, _, a in layers]).bind_device(0)
base = mk()
want = base.oracle_batched(wl.X, wl.Lam)
del base
nets = [mk(), mk()]
bad = [0, 0]


def work(t):
    for r in range(reps):
        got = nets[t].oracle_batched(wl.X, wl.Lam)
        for a, b, what in zip(got, want, "YJH"):
            if not np.array_equal(a, b):
                bad[t] += 1
                print("thread", t, "rep", r, what, "differs, max abs", float(np.abs(a - b).max()), flush=True)


ths = [threading.Thread(target=work, args=(t,)) for t in range(2)]
for th in ths:
    th.start()
for th in ths:
    th.join()
print(name, "B", B, "bad", bad, "of", 2 * reps, flush=True)
