"""Single-point forward (gbopt_net_forward path) of a BASELINE config: wall
time per call and, with GBOPT_FWD_ROWS set, the row-per-warp GEMV instead of
the per-SM balanced one.  python tools/fwd_probe.py [config]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_22462_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
wl = configs.make(name, batch=1)
net = wl.net.bind_device(0)
x = wl.X[0]
for _ in range(5):
    net.forward(x)
t0 = time.perf_counter()
for _ in range(50):
    y = net.forward(x)
dt = (time.perf_counter() - t0) / 50
print(f"{name} forward {'rows' if os.environ.get('GBOPT_FWD_ROWS') else 'flat'}: {dt * 1e3:.3f} ms/call  y[0]={y[0]!r}")
