"""Hunt the intermittent reverse-mode J error: the c2-shaped net's J through
the DMMA adjoint (adj_mma) against the CUDA-core sweep (GBOPT_ADJ_MMA=0 at
bind time) while other nets of other shapes are created, evaluated and
destroyed in between (memory reuse as in the full test session)."""
import gc
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_22462_b200 as gb  # noqa: E402
from paper_2509_22462_b200 import configs  # noqa: E402
from oracle import gbopt_oracle as o  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
rng = np.random.default_rng(1)
wl = configs.make("c2", batch=1)
x = wl.X[0]
bad = 0
for r in range(reps):
    os.environ["GBOPT_ADJ_MMA"] = "0"
    ref_net = gb.NeuralNet.from_layers(*[list(t) for t in zip(*[wl.net.layer(l) for l in range(wl.net.layer_count)])]).bind_device(0)
    J_ref = ref_net.jacobian(x)
    del ref_net
    gc.collect()
    os.environ["GBOPT_ADJ_MMA"] = "1"
    # churn: other shapes
    for sh in ([100, 300, 200, 7], [784, 512, 512, 10], [108, 1024, 1024, 1]):
        nn = gb.random_net(sh, "tanh", "linear", r).bind_device(0)
        X = rng.uniform(-1, 1, (5, sh[0])); L = rng.normal(size=(5, sh[-1]))
        nn.oracle_batched(X, L); nn.jacobian(X[0])
        del nn
    gc.collect()
    net = gb.NeuralNet.from_layers(*[list(t) for t in zip(*[wl.net.layer(l) for l in range(wl.net.layer_count)])]).bind_device(0)
    for k in range(3):
        J = net.jacobian(x)
        e = o.rel_err(J, J_ref)
        if e > 1e-12:
            bad += 1
            print("rep", r, "call", k, "J(mma) vs J(cols) rel", e, flush=True)
    del net
    gc.collect()
print("bad", bad, "of", 3 * reps, flush=True)
