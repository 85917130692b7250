"""Reverse-mode Jacobian (gbopt_net_jacobian: m seed vectors swept through
the weights once) wall time per call for a BASELINE config.
python tools/jac_probe.py [config]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_22462_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
wl = configs.make(name, batch=1)
net = wl.net.bind_device(0)
x = wl.X[0]
for _ in range(5):
    net.jacobian(x)
t0 = time.perf_counter()
for _ in range(30):
    J = net.jacobian(x)
print(f"{name} jacobian: {(time.perf_counter() - t0) / 30 * 1e3:.3f} ms/call  J[0,0]={J[0, 0]!r}")
