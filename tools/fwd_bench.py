"""Standalone forward() (the IPM line-search residual, ipm.cpp:342-343) on
the c2 network through the host API: median wall time of 50 calls and the
HBM rate it implies (871.6 MB of weights per call).  Run twice, with
GBOPT_FWD_STREAM=1 (persistent TMA-streamed launch, default) and =0 (one GEMV
launch per layer).  python tools/fwd_bench.py [config]"""
import json
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
ts = []
for _ in range(50):
    t0 = time.perf_counter()
    net.forward(x)
    ts.append(time.perf_counter() - t0)
ts.sort()
med = ts[len(ts) // 2]
wbytes = 8.0 * net.param_count
print(json.dumps({"config": name, "fwd_stream": os.environ.get("GBOPT_FWD_STREAM", "1"), "median_ms": med * 1e3,
                  "best_ms": ts[0] * 1e3, "weight_bytes": wbytes, "gbs_median": wbytes / med / 1e9,
                  "gbs_best": wbytes / ts[0] / 1e9, "launches": net.last_launch_count}))
