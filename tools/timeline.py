"""Prints the two-stream launch timeline of one eager evaluation
(gbopt_net_profile_timeline) for a BASELINE config:  python tools/timeline.py c2"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_22462_b200 as gb  # noqa: E402
from paper_2509_22462_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
B = int(sys.argv[2]) if len(sys.argv) > 2 else None
wl = configs.make(name, batch=B)
net = wl.net.bind_device(0)
dev = torch.device("cuda", 0)
X = torch.from_numpy(wl.X).to(dev)
L = torch.from_numpy(wl.Lam).to(dev)
for _ in range(3):
    net.oracle_batched(wl.X, wl.Lam)
tl = gb.gbopt.profile_timeline(net, X.shape[0], X.data_ptr(), L.data_ptr())
tl = gb.gbopt.profile_timeline(net, X.shape[0], X.data_ptr(), L.data_ptr())
end = max(t[3] for t in tl)
print(f"{name}: {len(tl)} launches, eager two-stream evaluation {end:.3f} ms")
for k, s, a, b in tl:
    bar = [" "] * 100
    for i in range(int(100 * a / end), max(int(100 * b / end), int(100 * a / end) + 1)):
        bar[min(i, 99)] = "#" if s == 0 else "="
    print(f"{k:14s} s{s} {a:8.3f} {b:8.3f} {b - a:7.3f} |{''.join(bar)}|")
