"""One c1 oracle evaluation under ncu's launch list: warm up (graph capture),
then 3 evaluations bracketed by cudaProfilerStart/Stop so that
`ncu --profile-from-start off --metrics gpu__time_duration.sum` lists exactly
their kernels (serialised, per-kernel device time)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_22462_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
wl = configs.make(name, batch=1)
net = wl.net.bind_device(0)
x, lam = wl.X[0], wl.Lam[0]
for _ in range(5):
    net.oracle(x, lam)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(3):
    net.oracle(x, lam)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")
