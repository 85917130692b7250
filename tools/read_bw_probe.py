"""Achievable HBM read bandwidth for a 210 MB stream (the size of one
5120 x 5120 FP64 weight matrix): torch.sum and a float64 dot product, CUDA
events, best of 20.  The forward/adjoint GEMVs are compared with this, not
with the copy figure in MEASURED_PEAKS.json.  python tools/read_bw_probe.py"""
import torch

dev = torch.device("cuda", 0)
n = 5120 * 5120
a = torch.rand(n, dtype=torch.float64, device=dev)
b = torch.rand(5120, dtype=torch.float64, device=dev)
A = a.view(5120, 5120)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def best(fn):
    ts = []
    for _ in range(20):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return min(ts)


for name, fn in (("sum", lambda: a.sum()), ("mv (cuBLAS dgemv)", lambda: torch.mv(A, b)),
                 ("copy", lambda: a.clone())):
    t = best(fn)
    by = 8 * n * (2 if name == "copy" else 1)
    print(f"{name:20s} {t * 1e6:8.1f} us  {by / t / 1e9:8.1f} GB/s")
