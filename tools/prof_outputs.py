"""Per-launch CUDA-event profile of one evaluation with a chosen output set
(GBOPT_PROFILE_OUTPUTS = y / j / yjh ...):  python tools/prof_outputs.py c2 j"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["GBOPT_PROFILE_OUTPUTS"] = sys.argv[2] if len(sys.argv) > 2 else "yjh"
import torch  # noqa: E402

import paper_2509_22462_b200 as gb  # noqa: E402
from paper_2509_22462_b200 import configs  # noqa: E402

wl = configs.make(sys.argv[1] if len(sys.argv) > 1 else "c2", batch=1)
net = wl.net.bind_device(0)
X = torch.from_numpy(wl.X).cuda()
L = torch.from_numpy(wl.Lam).cuda()
for _ in range(2):
    recs = gb.gbopt.profile_launches(net, 1, X.data_ptr(), L.data_ptr())
tot = 0.0
for tag, ms, fl, by in recs:
    tot += ms
    print(f"{tag:14s} {ms * 1e3:9.2f} us  {by / 1e6:9.1f} MB  {by / (ms * 1e-3) / 1e9 if by else 0:8.1f} GB/s")
print(f"total {tot * 1e3:.1f} us (serialised, events around every launch)")
