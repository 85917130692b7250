"""Device-timed comparison of the two oracle schedules (layer-by-layer
launches vs the persistent dataflow launch) on BASELINE configs:
    python tools/sched_compare.py c2 c5 [--steps 30]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_22462_b200 import configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="+")
ap.add_argument("--steps", type=int, default=30)
ap.add_argument("--batch", type=int, default=None)
a = ap.parse_args()
dev = torch.device("cuda", 0)
for name in a.configs:
    wl = configs.make(name, batch=a.batch)
    net = wl.net.bind_device(0)
    B, n, m = wl.X.shape[0], wl.X.shape[1], wl.Lam.shape[1]
    X = torch.from_numpy(wl.X).to(dev)
    L = torch.from_numpy(wl.Lam).to(dev)
    Y = torch.empty(B, m, dtype=torch.float64, device=dev)
    J = torch.empty(B, m, n, dtype=torch.float64, device=dev)
    H = torch.empty(B, n, n, dtype=torch.float64, device=dev)
    s = torch.cuda.current_stream(dev)
    res = {}
    for sched in ("layered", "dataflow", "layered", "dataflow"):
        net.set_schedule(sched)
        for _ in range(3):
            net.oracle_batched_device(B, X.data_ptr(), L.data_ptr(), Y.data_ptr(), J.data_ptr(), H.data_ptr(),
                                      s.cuda_stream)
        torch.cuda.synchronize()
        used = net.last_schedule
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(a.steps):
            net.oracle_batched_device(B, X.data_ptr(), L.data_ptr(), Y.data_ptr(), J.data_ptr(), H.data_ptr(),
                                      s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        res.setdefault(sched, []).append(ms)
        print(f"{name} B={B} {sched:9s} (ran {used:9s}) {ms:8.3f} ms/step  {B / ms * 1e3:10.2f} evals/s", flush=True)
    del net
