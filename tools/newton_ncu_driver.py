"""One reduced-space Newton step (callbacks, KKT assembly, inertia
correction, solve) after a warm-up, bracketed by cudaProfilerStart/Stop for
`ncu --profile-from-start off`:  python tools/newton_ncu_driver.py [config]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_22462_b200 as gb  # noqa: E402
from paper_2509_22462_b200 import configs  # noqa: E402
from paper_2509_22462_b200.reduced_space import ReducedSpaceBlock  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
wl = configs.make(name, batch=1)
net = wl.net.bind_device(0)
nin, m = net.input_dim, net.output_dim
n = nin + m
rng = np.random.default_rng(0)
jr = jc = hr = hc = None


def step(blk, pat, xb, lam):
    r = blk.residual(xb)
    jv = blk.jacobian(xb)
    hv = np.r_[blk.lag_hessian(xb, lam), np.ones(n)]
    lower = np.r_[np.zeros(nin), np.full(m, -np.inf)]
    z = np.r_[np.full(nin, 0.1), np.zeros(m)]
    s = pat.assemble(xb, lower, z, lam, xb, r, jv, hv, 0.01)
    cf = gb.inertia_correct(s)
    return s.solve(cf.fact)


blk = ReducedSpaceBlock(net)
jr, jc = blk.jac_pattern()
hr, hc = blk.hess_pattern()
pat = gb.KktPattern(n, m, np.r_[hr, np.arange(n)], np.r_[hc, np.arange(n)], jr, jc)
pts = [(np.r_[np.clip(wl.X[0] + 0.01 * rng.normal(size=nin), 1e-3, None), rng.normal(size=m)], rng.normal(size=m))
       for _ in range(2)]
step(blk, pat, *pts[0])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
step(blk, pat, *pts[1])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
