"""Throwaway probe: cuBLAS DGEMM throughput (FP64 roofline denominator candidate),
host core count and numpy/OpenBLAS DGEMM speed on the GPU box."""
import os, time, json, subprocess
import numpy as np
import torch
res = {"nproc": os.cpu_count()}
try:
    res["lscpu"] = subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines()[:20]
except Exception as e:
    res["lscpu"] = str(e)
dev = torch.device("cuda:0")
for (m, n, k) in [(8192, 8192, 8192), (5120, 784, 5120), (5120, 50176, 5120)]:
    a = torch.randn(m, k, dtype=torch.float64, device=dev)
    b = torch.randn(k, n, dtype=torch.float64, device=dev)
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    res[f"cublas_dgemm_{m}x{n}x{k}_tflops"] = 2 * m * n * k / best / 1e12
    # sustained 4 s
    t0 = time.time(); cnt = 0
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() - t0 < 4:
        for _ in range(5):
            c = a @ b
        cnt += 5
        torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    res[f"cublas_dgemm_{m}x{n}x{k}_sustained_tflops"] = 2 * m * n * k * cnt / (e0.elapsed_time(e1) / 1e3) / 1e12
    del a, b, c
for threads in [1, os.cpu_count()]:
    try:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=threads):
            a = np.random.rand(5120, 5120); b = np.random.rand(5120, 784)
            a @ b
            t0 = time.perf_counter(); a @ b; dt = time.perf_counter() - t0
            res[f"numpy_dgemm_5120x784x5120_{threads}thr_gflops"] = 2 * 5120 * 5120 * 784 / dt / 1e9
    except Exception as e:
        res[f"numpy_err_{threads}"] = str(e)
print(json.dumps(res, indent=1))
