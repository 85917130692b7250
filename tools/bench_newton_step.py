"""One interior-point Newton step on a reduced-space NN problem (SURVEY §8f
rows f1 + f3): the NN block's residual / Jacobian / Lagrangian-Hessian
callbacks at the iterate (ipm.cpp:256, 278, 420), KKT assembly
(ipm.cpp:291-293, 466-518), inertia correction (ipm.cpp:298-299, 520-557) and
the step solve (ipm.cpp:302).

Problem: min 0.5 |xb|^2 s.t. y - NN(x) = 0, xb = [x (n, bounded below by 0);
y (m, free)] -- the shape of the reference's reduced-space formulations
(formulations.cpp:267-349) with a separable objective.

GPU: ReducedSpaceBlock (device oracle) + KktPattern.assemble + inertia_correct
+ KktSystem.solve, the matrix never leaving the device.
CPU: the reference path on the reference's own code -- three callbacks each
recomputing the forward pass (nn.cpp, oracle/_ref; softplus configs timed
with tanh hidden layers, nn.cpp has none), numpy assembly from the triplets,
the inertia-correction loop (ipm.cpp:520-557) over the reference's
ldlt_factor (linalg.cpp) and its refined solve, all host threads.

python tools/bench_newton_step.py [config] [iters]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_22462_b200 as gb  # noqa: E402
from paper_2509_22462_b200 import configs  # noqa: E402
from paper_2509_22462_b200.reduced_space import ReducedSpaceBlock  # noqa: E402
from oracle import ldlt_oracle as lo  # noqa: E402
from oracle import ref as rf  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
wl = configs.make(name, batch=1)
net = wl.net.bind_device(0)
blk = ReducedSpaceBlock(net)
nin, m = blk.n, blk.m
n = nin + m
jr, jc = blk.jac_pattern()
hr, hc = blk.hess_pattern()
hr2, hc2 = np.r_[hr, np.arange(n)], np.r_[hc, np.arange(n)]   # + objective Hessian (identity)
lower = np.r_[np.zeros(nin), np.full(m, -np.inf)]
rng = np.random.default_rng(0)
pts = []
for _ in range(iters):
    x0 = np.clip(wl.X[0] + 0.01 * rng.normal(size=nin), 1e-3, None)
    xb = np.r_[x0, rng.normal(size=m)]
    pts.append((xb, rng.normal(size=m), rng.uniform(0.01, 1.0, nin), 10.0 ** rng.uniform(-4, -1)))

pat = gb.KktPattern(n, m, hr2, hc2, jr, jc)


def gpu_step(xb, lam, zin, mu):
    r = blk.residual(xb)
    jv = blk.jacobian(xb)
    hv = np.r_[blk.lag_hessian(xb, lam), np.ones(n)]
    z = np.r_[zin, np.zeros(m)]
    s = pat.assemble(xb, lower, z, lam, xb, r, jv, hv, mu)
    cf = gb.inertia_correct(s)
    return s.solve(cf.fact), cf


gpu_step(*pts[0])  # warm-up (graphs, autotune)
t0 = time.perf_counter()
for p in pts:
    sol, cf = gpu_step(*p)
gpu_s = (time.perf_counter() - t0) / iters
# phases of one step (wall clock, synchronous calls)
# (a second block, warmed at another point, so that the callbacks evaluate
# afresh at pts[-1] instead of hitting the first block's cache)
xb, lam, zin, mu = pts[-1]
ph = {}
blk2 = ReducedSpaceBlock(net)
xw, lw = pts[0][0], pts[0][1]
blk2.residual(xw); blk2.jacobian(xw); blk2.lag_hessian(xw, lw)
t = time.perf_counter()
r = blk2.residual(xb); jv = blk2.jacobian(xb); hv = np.r_[blk2.lag_hessian(xb, lam), np.ones(n)]
ph["callbacks"] = time.perf_counter() - t
t = time.perf_counter()
s = pat.assemble(xb, lower, np.r_[zin, np.zeros(m)], lam, xb, r, jv, hv, mu)
ph["assemble"] = time.perf_counter() - t
t = time.perf_counter()
cf = gb.inertia_correct(s)
ph["inertia_correct"] = time.perf_counter() - t
t = time.perf_counter()
s.solve(cf.fact)
ph["solve"] = time.perf_counter() - t

rf.set_threads(os.cpu_count() or 1)
ref = rf.make_config(name, batch=1, hidden=rf.TANH if name in ("c2", "c3") else None).net()
cpu_iters = max(1, min(iters, 2))
t0 = time.perf_counter()
for xb, lam, zin, mu in pts[:cpu_iters]:
    x = xb[:nin]
    r = xb[nin:] - ref.forward(x)                       # formulations.cpp:317-319
    J = ref.jacobian(x)                                  # :320-331
    H = ref.lagrangian_hessian(x, -lam)                  # :332-340
    K = np.zeros((n + m, n + m))
    K[:nin, :nin] = H
    K[np.arange(n), np.arange(n)] += 1.0
    K[np.arange(nin), np.arange(nin)] += zin / (x - lower[:nin])
    Jf = np.zeros((m, n))
    Jf[:, :nin] = -J
    Jf[np.arange(m), nin + np.arange(m)] = 1.0
    K[n:, :n] = Jf
    K[:n, n:] = Jf.T
    rhs = np.r_[-xb - Jf.T @ lam, -r]
    rhs[:nin] += mu / (x - lower[:nin])
    dw, dc, _ = lo.inertia_correct(K, n, m, inertia_fn=lambda A: rf.RefLdlt(A, keep_input=False).inertia)
    rf.RefLdlt(K + np.diag(np.r_[np.full(n, dw), np.full(m, -dc)])).solve(rhs)   # ipm.cpp:298-302
cpu_s = (time.perf_counter() - t0) / cpu_iters
print(json.dumps({"config": name, "kkt_dim": n + m, "gpu_s_per_newton_step": gpu_s, "cpu_s_per_newton_step": cpu_s,
                  "cpu_threads": os.cpu_count(), "cpu": "reference nn.cpp + linalg.cpp (oracle/_ref)", "speedup": cpu_s / gpu_s, "delta_w_last": cf.delta_w,
                  "inertia_last": cf.fact.inertia, "device_evaluations": blk.evaluations,
                  "phases_s_last_step": ph}))
