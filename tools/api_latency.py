"""Latency of the single-call C-ABI oracle entries on one point (host buffers,
synchronous, like the reference API and the IPM callbacks):
    python tools/api_latency.py c2"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_22462_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
wl = configs.make(name, batch=1)
net = wl.net.bind_device(0)
x, lam = wl.X[0], wl.Lam[0]
calls = {
    "forward": lambda: net.forward(x),
    "jacobian": lambda: net.jacobian(x),
    "lagrangian_gradient": lambda: net.lagrangian_gradient(x, lam),
    "lagrangian_hessian": lambda: net.lagrangian_hessian(x, lam),
    "oracle (y, J, H)": lambda: net.oracle(x, lam),
}
for k, f in calls.items():
    for _ in range(5):
        f()
    reps = 50 if k in ("forward", "jacobian", "lagrangian_gradient") else 20
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    dt = (time.perf_counter() - t0) / reps
    print(f"{name} {k:22s} {dt * 1e3:8.3f} ms/call  ({net.last_launch_count} kernels)")
