"""One call of an HBM-bound path of a BASELINE config inside
cudaProfilerStart/Stop, for `ncu --profile-from-start off --set full -k ...`:
  forward   net.forward(x)          (fwd_row1_kernel per layer; IPM line search)
  jacobian  net.jacobian(x)         (reverse-mode J: adj_mma / adj_cols kernels)
  oracle    net.oracle(x, lam)      (the fused evaluation: its adjoint sweep)
python tools/ncu_paths.py <forward|jacobian|oracle> [config]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_22462_b200 import configs  # noqa: E402

mode = sys.argv[1]
name = sys.argv[2] if len(sys.argv) > 2 else "c2"
wl = configs.make(name, batch=1)
net = wl.net.bind_device(0)
x, lam = wl.X[0], wl.Lam[0]
call = {"forward": lambda: net.forward(x), "jacobian": lambda: net.jacobian(x),
        "oracle": lambda: net.oracle(x, lam)}[mode]
for _ in range(3):
    call()
torch.cuda.synchronize()
torch.cuda.profiler.start()
call()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(mode, name, "done")
