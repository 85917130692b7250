"""One evaluation of a BASELINE config inside cudaProfilerStart/Stop, for
ncu --profile-from-start off (warm-up and the auto-schedule measurement run
before the range):
    ncu --profile-from-start off --metrics ... python tools/ncu_capture.py c5"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_22462_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
wl = configs.make(name)
net = wl.net.bind_device(0)
dev = torch.device("cuda", 0)
B, n, m = wl.X.shape[0], wl.X.shape[1], wl.Lam.shape[1]
X = torch.from_numpy(wl.X).to(dev)
L = torch.from_numpy(wl.Lam).to(dev)
Y = torch.empty(B, m, dtype=torch.float64, device=dev)
J = torch.empty(B, m, n, dtype=torch.float64, device=dev)
H = torch.empty(B, n, n, dtype=torch.float64, device=dev)
s = torch.cuda.current_stream(dev)


def ev():
    net.oracle_batched_device(B, X.data_ptr(), L.data_ptr(), Y.data_ptr(), J.data_ptr(), H.data_ptr(), s.cuda_stream)


for _ in range(3):
    ev()
torch.cuda.synchronize()
torch.cuda.profiler.start()
ev()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(name, "schedule", net.last_schedule)
