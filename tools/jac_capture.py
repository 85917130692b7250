"""Reverse-mode Jacobian of one c2 point inside cudaProfilerStart/Stop (for
ncu --profile-from-start off):  python tools/jac_capture.py [config]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_22462_b200 import configs  # noqa: E402

wl = configs.make(sys.argv[1] if len(sys.argv) > 1 else "c2", batch=1)
net = wl.net.bind_device(0)
X = torch.from_numpy(wl.X).cuda()
J = torch.empty(1, wl.Lam.shape[1], wl.X.shape[1], dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream()
for _ in range(3):
    net.oracle_batched_device(1, X.data_ptr(), 0, 0, J.data_ptr(), 0, s.cuda_stream)
torch.cuda.synchronize()
torch.cuda.profiler.start()
net.oracle_batched_device(1, X.data_ptr(), 0, 0, J.data_ptr(), 0, s.cuda_stream)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
