"""Per-item trace of one dataflow evaluation for a BASELINE config:
    python tools/df_trace.py c2 [batch] [out.npy]
Prints per-kind statistics (count, busy time, dependency waits), SM
utilisation over time and the tail."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_22462_b200 as gb  # noqa: E402
from paper_2509_22462_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
B = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else None
wl = configs.make(name, batch=B)
net = wl.net.set_schedule("dataflow").bind_device(0)
dev = torch.device("cuda", 0)
X = torch.from_numpy(wl.X).to(dev)
L = torch.from_numpy(wl.Lam).to(dev)
for _ in range(3):
    net.oracle_batched(wl.X, wl.Lam)
tr = gb.gbopt.dataflow_trace(net, X.shape[0], X.data_ptr(), L.data_ptr())
tr = gb.gbopt.dataflow_trace(net, X.shape[0], X.data_ptr(), L.data_ptr())
if len(sys.argv) > 3:
    np.save(sys.argv[3], tr)
kind = tr[:, 0].astype(int)
claim, ready, begin, end = tr[:, 8], tr[:, 9], tr[:, 10], tr[:, 11]
span = end.max()
print(f"{name}: {len(tr)} items, kernel span {span / 1e3:.3f} ms, SMs {len(np.unique(tr[:, 7]))}")
names = ["fwd", "adj", "gemm", "syrk"]
for k in range(4):
    s = kind == k
    if not s.any():
        continue
    dur = end[s] - begin[s]
    wait = ready[s] - claim[s]
    print(f"  {names[k]:5s} n={s.sum():6d} busy {dur.sum() / 1e3:9.3f} SM-ms  mean {dur.mean():8.2f} us  "
          f"max {dur.max():8.2f}  dep-wait mean {wait.mean():8.2f} max {wait.max():8.2f} us  "
          f"first {begin[s].min() / 1e3:.3f} last-end {end[s].max() / 1e3:.3f} ms")
# SM occupancy by consumer-busy intervals, 20 bins
bins = 25
edges = np.linspace(0, span, bins + 1)
busy = np.zeros(bins)
for b0, e0 in zip(begin, end):
    for i in range(bins):
        lo, hi = max(b0, edges[i]), min(e0, edges[i + 1])
        if hi > lo:
            busy[i] += hi - lo
nsm = len(np.unique(tr[:, 7]))
print("  consumer-busy fraction per time bin:")
print("  " + " ".join(f"{x:.2f}" for x in busy / (nsm * (edges[1] - edges[0]))))
# per-SM idle: gaps between consecutive items on one SM (end -> next begin)
gaps = []
for smv in np.unique(tr[:, 7]):
    s = np.where(tr[:, 7] == smv)[0]
    s = s[np.argsort(begin[s])]
    gaps.extend(begin[s[1:]] - end[s[:-1]])
    gaps.append(begin[s[0]])
    gaps.append(span - end[s[-1]])
gaps = np.array(gaps)
print(f"  idle SM time {gaps.sum() / 1e3:.3f} SM-ms of {nsm * span / 1e3:.3f} ({gaps.sum() / (nsm * span):.3f})")
