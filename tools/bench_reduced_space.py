"""Reduced-space callback loop: per emulated IPM iteration
one residual + Jacobian + Lagrangian Hessian at the iterate (the order of
ipm.cpp:256,278,420) plus `ls` line-search residuals at trial points
(ipm.cpp:340-355).  GPU: paper_2509_22462_b200.reduced_space.ReducedSpaceBlock
(cached per x: forward, reverse-mode J, fused H).  CPU: the reference
callbacks (formulations.cpp:317-340) on the reference's own nn.cpp
(oracle/_ref, OpenBLAS products on all host threads), each recomputing its
own forward pass; softplus configs (c2, c3) time the same shape with tanh
hidden layers (nn.cpp has no softplus).
python tools/bench_reduced_space.py [config] [iters] [ls]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_22462_b200 import configs  # noqa: E402
from paper_2509_22462_b200.reduced_space import ReducedSpaceBlock  # noqa: E402
from oracle import ref  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
ls = int(sys.argv[3]) if len(sys.argv) > 3 else 3
wl = configs.make(name, batch=1)
net = wl.net.bind_device(0)
n, m = net.input_dim, net.output_dim
rng = np.random.default_rng(0)
xs = [np.concatenate([wl.X[0] + 0.01 * rng.normal(size=n), rng.normal(size=m)]) for _ in range(iters)]
lams = [rng.normal(size=m) for _ in range(iters)]
trials = [[x + 1e-3 * rng.normal(size=n + m) for _ in range(ls)] for x in xs]

blk = ReducedSpaceBlock(net)
blk.residual(xs[0]); blk.jacobian(xs[0]); blk.lag_hessian(xs[0], lams[0])  # warm-up (graphs)
t0 = time.perf_counter()
for x, lam, tr in zip(xs, lams, trials):
    blk.residual(x)
    blk.jacobian(x)
    blk.lag_hessian(x, lam)
    for t in tr:
        blk.residual(t)
gpu_s = (time.perf_counter() - t0) / iters

ref.set_threads(os.cpu_count() or 1)
rwl = ref.make_config(name, batch=1, hidden=ref.TANH if name in ("c2", "c3") else None)
rnet = rwl.net()
cpu_iters = max(1, min(iters, 3))
t0 = time.perf_counter()
for x, lam, tr in list(zip(xs, lams, trials))[:cpu_iters]:
    xb = x[:n]
    x[n:] - rnet.forward(xb)
    rnet.jacobian(xb)
    rnet.lagrangian_hessian(xb, -lam)
    for t in tr:
        t[n:] - rnet.forward(t[:n])
cpu_s = (time.perf_counter() - t0) / cpu_iters
print(json.dumps({"config": name, "line_search_residuals": ls, "gpu_s_per_ipm_iter": gpu_s,
                  "cpu_s_per_ipm_iter": cpu_s, "cpu_threads": os.cpu_count(), "cpu": "reference nn.cpp (oracle/_ref)", "speedup": cpu_s / gpu_s,
                  "device_evaluations": blk.evaluations}))
