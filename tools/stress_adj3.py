"""Two host threads, two handles of the c2-shaped net, reverse-mode J
(adj_mma) concurrently, each checked against a CUDA-core-sweep result."""
import os
import sys
import threading

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_22462_b200 as gb  # noqa: E402
from paper_2509_22462_b200 import configs  # noqa: E402
from oracle import gbopt_oracle as o  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
wl = configs.make("c2", batch=1)
Xs = [wl.X[0], np.clip(wl.X[0] + 0.01, 0, 1)]
layers = [wl.net.layer(l) for l in range(wl.net.layer_count)]
mk = lambda: gb.NeuralNet.from_layers([w for w, _, _ in layers], [b for _, b, _ in layers], [a for _, _, a in layers]).bind_device(0)
os.environ["GBOPT_ADJ_MMA"] = "0"
base = mk()
want = [base.jacobian(Xs[i]) for i in range(2)]
want4 = base.oracle_batched(np.repeat(wl.X[:1], 4, 0), np.repeat(wl.Lam[:1], 4, 0))[2]
del base
os.environ["GBOPT_ADJ_MMA"] = os.environ.get("STRESS_MMA", "1")
nets = [mk(), mk()]
bad = [0, 0]


def work(t):
    for r in range(reps):
        J = nets[t].jacobian(Xs[t])
        e = o.rel_err(J, want[t])
        if e > 1e-12:
            bad[t] += 1
            print("thread", t, "rep", r, "J rel", e, flush=True)
        if r % 10 == 0:
            H = nets[t].oracle_batched(np.repeat(wl.X[:1], 4, 0), np.repeat(wl.Lam[:1], 4, 0))[2]
            e = max(o.rel_err(H[i], want4[i]) for i in range(4))
            if e > 1e-12:
                bad[t] += 1
                print("thread", t, "rep", r, "H4 rel", e, flush=True)


ths = [threading.Thread(target=work, args=(t,)) for t in range(2)]
for th in ths:
    th.start()
for th in ths:
    th.join()
print("bad", bad, flush=True)
