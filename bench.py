#!/usr/bin/env python
"""Benchmark of the B200 FP64 gray-box NN oracle (one JSON line on rank 0).

Metric (BASELINE.json): NN oracle evals/s, one eval = (y, J, H) at one
(x, lambda) of the 109M-parameter MLP 784-[5120]x5-10 (config c2), plus the
roofline fraction of the dominant kernel.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2]
  python bench.py --impl reference ...   # CPU arm: the reference's own nn.cpp

--gpus N > 1 runs one process per GPU: under torchrun it uses the launcher's
ranks; started directly it launches torchrun itself (127.0.0.1) and exits
with the ranks' status.

A "step" is one oracle evaluation of one c2 point per GPU (weak scaling:
each rank evaluates its own point, the shared weights are replicated); for
N > 1 the step ends with an NCCL gather of every rank's (y, J, H) to rank 0
(the only collective of the path).  `value` is timed with CUDA
events on the launching stream, inputs resident in HBM, max over ranks.
`e2e` is the same metric through the public host-buffer API: at N = 1
gbopt_net_oracle_batched (pinned host x/lambda in, y/J/H out); at N > 1
parallel.ShardedOracle (host shard in on every rank, H2D, device oracle,
NCCL gather, rank 0's D2H of all results).  `sharded` adds the batched (c3,
B = 64) and contingency (c4, K = 4096) workloads split over the N GPUs.

The CPU legs (`cpu_baseline`, `cpu_baseline_1t`, `--impl reference`) run the
reference's OWN oracle: proj/src/nn.cpp compiled unmodified into
oracle/_ref/libgbopt_ref.so (oracle/ref.py); they never load the product
library.  nn.cpp has no softplus, so on c2/c3 the reference times the same
shape with tanh hidden layers (identical GEMM chain; stated in `sample`).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "NN oracle evals/s (y+Jacobian+Lagrangian Hessian) at 109M params; % roofline"
UNIT = "evals/s"
THROTTLE_BITS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
    0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
    0x100: "display_clock_setting",
}

# BASELINE.json configs (pure data; the generators live in
# paper_2509_22462_b200/configs.py and, independently, oracle/ref.py).
WIDTHS = {"c1": [784, 512, 512, 10], "c2": [784] + [5120] * 5 + [10], "c3": [784] + [5120] * 5 + [10],
          "c4": [108, 1024, 1024, 1024, 1], "c5": [784] + [1024] * 20 + [10]}
SOFTPLUS_CONFIGS = ("c2", "c3")
CONFIG_DESC = {
    "c1": "c1: single-point FP64 oracle, MLP 784-512-512-10 tanh/identity (Xavier-uniform, seed 0)",
    "c2": "c2: single-point FP64 oracle, MLP 784-[5120]x5-10 softplus/identity, 108,948,490 params "
          "(Xavier-normal, seed 1)",
    "c3": "c3: batched FP64 oracle, c2's MLP, B=64 points (seed 2)",
    "c4": "c4: K=4096 contingency copies of MLP 108-[1024]x3-1 tanh/sigmoid (Xavier-uniform, seed 3)",
    "c5": "c5: deep-chain FP64 oracle, MLP 784-[1024]x20-10 sigmoid/identity, B=16 (N(0,1/fan_in), seed 4)",
}
L2_FLUSH = ("c1",)  # working set below the L2: flush between timed steps
L2_NOTE = {
    "c1": "L2 flushed between timed steps (a 256 MB write outside each step's CUDA events): the 5.4 MB "
          "of weights and 4.9 MB Hessian fit the 126 MB L2; value_l2_resident is the unflushed rate "
          "(weights L2-resident, as between IPM iterations)",
    "c2": "no flush needed: the weights streamed every step (871.6 MB) exceed the 126 MB L2",
    "c3": "no flush needed: the weights streamed every step (871.6 MB) exceed the 126 MB L2",
    "c4": "no flush needed: every step writes 4096 Hessians of 108^2 (382 MB), beyond the 126 MB L2",
    "c5": "no flush needed: the weights streamed every step (166.1 MB) exceed the 126 MB L2",
}
TOTAL_POINTS = {"c1": 1, "c2": 1, "c3": 64, "c4": 4096, "c5": 16}
SHARDED = ("c3", "c4", "c5")  # fixed point sets split over the ranks


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: correctness run of the N>1 path (e.g. 2 ranks on one GPU); not a perf number")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sharded", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    return ap.parse_args()


def params_of(widths):
    return sum(widths[l] * widths[l - 1] + widths[l] for l in range(1, len(widths)))


def points_per_gpu(name, world, rank=0):
    if name in SHARDED:
        P = TOTAL_POINTS[name]
        base, extra = divmod(P, world)
        return base + (1 if rank < extra else 0)
    return TOTAL_POINTS[name]


def config_dict(name, world):
    """The `config` object of both arms (identical by construction)."""
    P = TOTAL_POINTS[name]
    return {
        "workload": CONFIG_DESC[name],
        "points_per_step": P * world if name not in SHARDED else P,
        "points_per_step_per_gpu": points_per_gpu(name, world),
        "params": params_of(WIDTHS[name]),
        "l2": L2_NOTE[name],
        "parallelism": (f"replicated weights, points sharded over {world} GPUs, NCCL gather to rank 0"
                        if world > 1 else "1 GPU"),
    }


def flops_per_eval(name):
    w = WIDTHS[name]
    n = w[0]
    hidden_nonlinear = True
    f = 0.0
    L = len(w) - 1
    for l in range(1, L + 1):
        mac = w[l] * w[l - 1]
        f += 2 * mac
        if l >= 2:
            f += 2 * mac + 2 * mac * n
        nonlinear = hidden_nonlinear if l < L else (name == "c4")  # c4's output is sigmoid, others linear
        if nonlinear:
            f += w[l] * n * (n + 1)
    return f


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def maybe_launch_ranks(args):
    """--gpus N > 1 outside a launcher: start N ranks with torchrun."""
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    return None


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 3:
                try:
                    self.rows.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                except ValueError:
                    pass

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        busy = [r for r in self.rows if not (r[2] & 0x1)] or self.rows
        mhz = sorted(r[0] for r in busy)
        reasons = set()
        for r in busy:
            for bit, name in THROTTLE_BITS.items():
                if r[2] & bit and bit != 0x1:
                    reasons.add(name)
        return {"sm_mhz": mhz[len(mhz) // 2], "sm_max_mhz": max(r[1] for r in busy), "reasons": sorted(reasons),
                "samples": len(busy)}


# ---------------------------------------------------------------------------
# CPU arm: the reference's own nn.cpp (oracle/_ref), never the product
# ---------------------------------------------------------------------------
def reference_sample(name, threads: int, budget_s: float, min_evals: int = 1, max_steps: int = 10 ** 6,
                     warmup: int = 1, per_step=None):
    """Times forward + jacobian + lagrangian_hessian per point (the three
    reduced-space callbacks, formulations.cpp:317-340) with the reference
    build on `threads` host threads.  Returns (evals/s, evals, seconds,
    steps, description, per-step seconds).  A step is `per_step` points
    (point-parallel over the threads when it is >= the thread count, else
    one point at a time with the BLAS on all threads)."""
    from oracle import ref

    hidden = ref.TANH if name in SOFTPLUS_CONFIGS else None
    P = TOTAL_POINTS[name]
    if per_step is None:
        per_step = min(P, 4 * threads) if name == "c4" else 1
    pool = min(P, max(per_step, 4))
    wl = ref.make_config(name, batch=pool, hidden=hidden)
    rn = wl.net()
    point_parallel = per_step >= threads and threads > 1
    ref.set_threads(1 if point_parallel else threads)
    tthreads = threads if point_parallel else 1

    def step(k):
        idx = [(k * per_step + i) % pool for i in range(per_step)]
        rn.oracle_batched(wl.X[idx], wl.Lam[idx], threads=tthreads)

    for i in range(warmup):
        step(i)
    times = []
    t_start = time.perf_counter()
    k = 0
    while k < max_steps and (len(times) * per_step < min_evals or time.perf_counter() - t_start < budget_s):
        t0 = time.perf_counter()
        step(k)
        times.append(time.perf_counter() - t0)
        k += 1
        if len(times) * per_step >= min_evals and time.perf_counter() - t_start >= budget_s:
            break
    evals = len(times) * per_step
    tot = sum(times)
    how = (f"point-parallel on {threads} threads" if point_parallel else
           f"OpenBLAS on {threads} thread{'s' if threads > 1 else ''}")
    desc = (f"{evals} evals of {name} in {tot:.2f}s, {per_step} point(s) per step; reference nn.cpp "
            f"(proj/src/nn.cpp:113-292 compiled unmodified, oracle/_ref) forward+jacobian+lagrangian_hessian, "
            f"{how}")
    if hidden is not None:
        desc += "; tanh hidden layers in place of softplus (nn.cpp has none), same GEMM chain"
    return evals / tot, evals, tot, len(times), desc, times


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    from oracle import ref

    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (make -C oracle/ref_build)"}))
        return 0
    name = args.config
    cores = os.cpu_count() or 1
    v, evals, tot, steps, desc, times = reference_sample(name, cores, budget_s=150.0, min_evals=1,
                                                         max_steps=args.steps, warmup=min(args.warmup, 1))
    line = {
        "metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": world,
        "steps": steps, "warmup": min(args.warmup, 1), "ms_per_step": 1e3 * tot / steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(name, world),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "reference", "sample": desc},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if steps < args.steps:
        line["note"] = f"stopped after {steps} of {args.steps} steps (150 s CPU budget)"
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
def measure_fp64_peak(torch, dev):
    """Live FP64 denominator: cuBLAS DGEMM 8192^3, best of 5 (CUDA events).
    MEASURED_PEAKS.json carries no FP64 entry."""
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    for _ in range(2):
        a @ b
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    del a, b
    torch.cuda.empty_cache()
    return 2.0 * n ** 3 / best / 1e12


def load_traffic():
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu
    --set full capture summary (profiles/*traffic*.json), or None."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*traffic*.json")))
    if not files:
        return None, None
    try:
        d = json.load(open(files[-1]))
        return d, os.path.basename(files[-1])
    except Exception:
        return None, None


def hbm_peak_gbs():
    """Measured copy bandwidth of this pool's B200s (MEASURED_PEAKS.json,
    driver-written), else the profiling recipe's fallback."""
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy, read+write bytes)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md; MEASURED_PEAKS.json absent)"


def max_over_ranks(torch, dist, world, dev, t):
    if world <= 1:
        return t
    tt = torch.tensor([t], dtype=torch.float64, device=dev if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    return float(tt.item())


def oracle_parity(name, wl, X, Lam, Y, J, H, k):
    """(y, J, H) max rel err over the first k benchmarked points against the
    reference nn.cpp build (oracle/_ref), or, for softplus nets (which nn.cpp
    lacks), against the numpy restatement of nn.cpp (oracle/gbopt_oracle.py)."""
    from oracle import gbopt_oracle as orc
    from oracle import ref

    layers = [wl.net.layer(l) for l in range(wl.net.layer_count)]
    if name in SOFTPLUS_CONFIGS or not ref.available():
        on = orc.NeuralNet([orc.Layer(w, b, a) for w, b, a in layers])
        RY = [on.forward(X[i]) for i in range(k)]
        RJ = [on.jacobian(X[i]) for i in range(k)]
        RH = [on.lagrangian_hessian(X[i], Lam[i]) for i in range(k)]
        against = "oracle port (numpy restatement of nn.cpp:113-292; nn.cpp has no softplus)"
    else:
        ref.set_threads(os.cpu_count() or 1)
        rn = ref.RefNet.from_layers(layers)
        RY, RJ, RH = rn.oracle_batched(X[:k], Lam[:k])
        against = "reference nn.cpp compiled unmodified (oracle/_ref)"
    e = [max(orc.rel_err(Y[i], RY[i]) for i in range(k)), max(orc.rel_err(J[i], RJ[i]) for i in range(k)),
         max(orc.rel_err(H[i], RH[i]) for i in range(k))]
    return {"y": e[0], "J": e[1], "H": e[2], "points": k, "against": against, "bar": 1e-10,
            "pass": max(e) <= 1e-10}


def run_sharded(torch, dist, gb, configs, parallel, name, world, rank, dev, peak, steps, warmup, net=None):
    """One fixed point set of config `name` split over the ranks; every step
    evaluates the rank's shard (device-resident inputs) and gathers the
    results to rank 0.  Returns the record on rank 0."""
    wl = configs.make(name, net=net) if net is not None else configs.make(name)
    rnet = wl.net
    if net is None:
        rnet.bind_device(dev.index)
    P = wl.X.shape[0]
    start, count = parallel.shard(P, world, rank)
    rows = parallel.max_shard(P, world)
    n, m = rnet.input_dim, rnet.output_dim
    per = m + m * n + n * n
    Xd = torch.from_numpy(wl.X[start:start + count].copy()).to(dev)
    Ld = torch.from_numpy(wl.Lam[start:start + count].copy()).to(dev)
    Yd = torch.empty(count, m, dtype=torch.float64, device=dev)
    Jd = torch.empty(count, m, n, dtype=torch.float64, device=dev)
    Hd = torch.empty(count, n, n, dtype=torch.float64, device=dev)
    flat = torch.zeros(rows * per, dtype=torch.float64, device=dev) if world > 1 else None
    gloo = world > 1 and dist.get_backend() == "gloo"
    flat_c = flat.cpu() if gloo else flat
    gat = [torch.empty_like(flat_c) for _ in range(world)] if (world > 1 and rank == 0) else None
    stream = torch.cuda.current_stream(dev)

    def compute():
        rnet.oracle_batched_device(count, Xd.data_ptr(), Ld.data_ptr(), Yd.data_ptr(), Jd.data_ptr(),
                                   Hd.data_ptr(), stream.cuda_stream)

    def collect():
        if world > 1:
            parallel.pack(Yd, Jd, Hd, rows, m, n, flat)
            if gloo:
                flat_c.copy_(flat)
            dist.gather(flat_c, gather_list=gat, dst=0)

    for _ in range(warmup):
        compute()
        collect()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        compute()
        collect()
    e1.record(stream)
    torch.cuda.synchronize()
    t = max_over_ranks(torch, dist, world, dev, e0.elapsed_time(e1) / 1e3)
    # the gather alone (same buffers), to show its share
    tg = 0.0
    if world > 1:
        dist.barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(steps):
            collect()
        g1.record(stream)
        torch.cuda.synchronize()
        tg = max_over_ranks(torch, dist, world, dev, g0.elapsed_time(g1) / 1e3)
    if rank != 0:
        return None
    F = flops_per_eval(name)
    v = P * steps / t
    return {"config": name, "workload": CONFIG_DESC[name], "points_total": P, "points_per_gpu_max": rows,
            "n_gpus": world, "steps": steps, "evals_s": v, "ms_per_step": 1e3 * t / steps,
            "gather_ms_per_step": 1e3 * tg / steps, "gather_bytes_per_step": world * rows * per * 8 if world > 1 else 0,
            "achieved_tflops_per_gpu": F * v / world / 1e12,
            "frac_of_peak": (F * v / world / 1e12) / peak if peak else None,
            "schedule": rnet.last_schedule}


def run_b200(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    ndev = torch.cuda.device_count()
    gloo = args.dist_backend == "gloo"
    if local >= ndev and not gloo:
        print(f"bench.py: rank {rank} needs GPU {local} but only {ndev} visible", file=sys.stderr)
        return 2
    dev_index = local % ndev
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    if world > 1:
        if gloo:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    import paper_2509_22462_b200 as gb
    from paper_2509_22462_b200 import configs, parallel

    name = args.config
    P = TOTAL_POINTS[name]
    wl = configs.make(name)
    net = wl.net
    net.bind_device(dev_index)
    n, m = net.input_dim, net.output_dim
    # this rank's points: weak-scaling configs (c1, c2) evaluate point `rank`
    # of the seeded stream (wrapping); c3/c4/c5 split their fixed point set.
    if name in SHARDED:
        start, B = parallel.shard(P, world, rank)
        idx = list(range(start, start + B))
    else:
        B = P
        idx = [(rank * B + i) % wl.X.shape[0] for i in range(B)]
    rows = max(len(idx), 1) if name not in SHARDED else parallel.max_shard(P, world)
    Xd = torch.from_numpy(wl.X[idx]).to(dev)
    Ld = torch.from_numpy(wl.Lam[idx]).to(dev)
    Yd = torch.empty(B, m, dtype=torch.float64, device=dev)
    Jd = torch.empty(B, m, n, dtype=torch.float64, device=dev)
    Hd = torch.empty(B, n, n, dtype=torch.float64, device=dev)
    per = m + m * n + n * n
    flat = torch.zeros(rows * per, dtype=torch.float64, device=dev) if world > 1 else None
    flat_c = (flat.cpu() if gloo else flat) if world > 1 else None
    gather = [torch.empty_like(flat_c) for _ in range(world)] if (world > 1 and rank == 0) else None
    stream = torch.cuda.current_stream(dev)

    def step():
        net.oracle_batched_device(B, Xd.data_ptr(), Ld.data_ptr(), Yd.data_ptr(), Jd.data_ptr(), Hd.data_ptr(),
                                  stream.cuda_stream)
        if world > 1:
            # result gather to rank 0: the path's only collective
            parallel.pack(Yd, Jd, Hd, rows, m, n, flat)
            if gloo:
                flat_c.copy_(flat)
            dist.gather(flat_c, gather_list=gather, dst=0)

    peak = measure_fp64_peak(torch, dev) if rank == 0 else None

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    launches_per_step = net.last_launch_count
    schedule = net.last_schedule

    # working sets below the 126 MB L2 (c1): every timed step starts from a
    # flushed L2 (a 256 MB write between steps, outside the per-step events);
    # the L2-resident rate (as between IPM iterations) is reported beside it
    flush = name in L2_FLUSH
    flush_buf = torch.empty(256 << 18, dtype=torch.float32, device=dev) if flush else None
    resident = None
    if flush:
        torch.cuda.synchronize()
        r0 = torch.cuda.Event(enable_timing=True)
        r1 = torch.cuda.Event(enable_timing=True)
        r0.record(stream)
        for _ in range(args.steps):
            step()
        r1.record(stream)
        torch.cuda.synchronize()
        resident = max_over_ranks(torch, dist, world, dev, r0.elapsed_time(r1) / 1e3)
    with ClockSampler(dev_index) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step_evs = []
        for i in range(args.steps):
            if flush:
                flush_buf.fill_(float(i))  # evicts the L2 (not timed: outside this step's events)
                a_ev = torch.cuda.Event(enable_timing=True)
                b_ev = torch.cuda.Event(enable_timing=True)
                a_ev.record(stream)
                step()
                b_ev.record(stream)
                step_evs.append((a_ev, b_ev))
            else:
                step()
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    t_local = (sum(a_ev.elapsed_time(b_ev) for a_ev, b_ev in step_evs) if flush else e0.elapsed_time(e1)) / 1e3
    t = max_over_ranks(torch, dist, world, dev, t_local)
    total_points = (P * world if name not in SHARDED else P)
    value = total_points * args.steps / t
    clocks = clk.summary()

    # ---- the N>1 path end to end: gathered results == per-shard calls ----
    ok = bool(torch.isfinite(Hd).all().item()) and bool(torch.equal(Hd, Hd.transpose(1, 2)))
    shards = ([parallel.shard(P, world, r) for r in range(world)] if name in SHARDED else
              [(r * B, B) for r in range(world)])
    all_idx = [i % wl.X.shape[0] for s0, c in shards for i in range(s0, s0 + c)]
    multi = None
    if world > 1 and rank == 0:
        counts = [c for _, c in shards]
        GY, GJ, GH = parallel.unpack([g.cpu().numpy() for g in gather], counts, rows, m, n)
        # the same shards evaluated one after another by a single process on
        # this GPU through the same device entry and batch size each rank used
        # (batching may change the kernels, so the comparison is per shard):
        # bit for bit
        same = True
        o = 0
        for s0, c in shards:
            if c == 0:
                continue
            sel = all_idx[o:o + c]
            sX = torch.from_numpy(wl.X[sel]).to(dev)
            sL = torch.from_numpy(wl.Lam[sel]).to(dev)
            sY = torch.empty(c, m, dtype=torch.float64, device=dev)
            sJ = torch.empty(c, m, n, dtype=torch.float64, device=dev)
            sH = torch.empty(c, n, n, dtype=torch.float64, device=dev)
            net.oracle_batched_device(c, sX.data_ptr(), sL.data_ptr(), sY.data_ptr(), sJ.data_ptr(), sH.data_ptr(),
                                      stream.cuda_stream)
            SY, SJ, SH = sY.cpu().numpy(), sJ.cpu().numpy(), sH.cpu().numpy()
            same = same and np.array_equal(GY[o:o + c], SY) and np.array_equal(GJ[o:o + c], SJ) and \
                np.array_equal(GH[o:o + c], SH)
            o += c
        multi = {"gathered_points": int(GY.shape[0]), "bitwise_equal_to_single_process_shards": bool(same),
                 "backend": args.dist_backend}
        ok = ok and same

    # ---- roofline of the dominant kernel: per-launch CUDA events ----
    roof = None
    prof_summary = None
    if rank == 0:
        recs = gb.gbopt.profile_launches(net, B, Xd.data_ptr(), Ld.data_ptr())
        agg = {}
        for tag, ms, fl, by in recs:
            a = agg.setdefault(tag, [0, 0.0, 0.0, 0.0])
            a[0] += 1
            a[1] += ms
            a[2] += fl
            a[3] += by
        total_ms = sum(a[1] for a in agg.values())
        prof_summary = {k: {"launches": v[0], "ms": round(v[1], 4), "share": round(v[1] / total_ms, 4),
                            "tflops": round(v[2] / (v[1] / 1e3) / 1e12, 3) if v[2] and v[1] else None,
                            "gbs": round(v[3] / (v[1] / 1e3) / 1e9, 1) if v[3] and v[1] else None}
                        for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])}
        dom = max(agg.items(), key=lambda kv: kv[1][1])[0]
        cnt, ms, fl, _ = agg[dom]
        achieved = (fl / cnt) / (ms / cnt / 1e3) / 1e12
        traffic, tsrc = load_traffic()
        per_l = traffic.get("per_launch_dram_bytes", {}) if traffic else {}
        roof = {"kernel": dom, "bound": "tensor", "achieved": round(achieved, 3), "peak": round(peak, 3),
                "unit": "TFLOP/s", "frac": round(achieved / peak, 4), "traffic": per_l.get(f"{dom}@{name}"),
                "algorithmic_flops_per_launch": fl / cnt, "avg_launch_ms": ms / cnt,
                "peak_source": "cuBLAS DGEMM 8192^3 burst, measured live in this run (FP64; no FP64 entry in "
                               "MEASURED_PEAKS.json); DMMA issue ceiling 37.1 TFLOP/s (tools/fp64_probe.cu)",
                "traffic_source": tsrc}

    # ---- HBM-bound single-point paths of the IPM callbacks (rank 0) ----
    # the line-search residual (forward only, ipm.cpp:342-343) and the
    # Jacobian callback (reverse mode, m seed vectors in one adjoint sweep),
    # device-timed through the same device entry with only dY / only dJ
    hbm_paths = None
    if rank == 0 and name in ("c1", "c2"):
        hbm_peak, hbm_src = hbm_peak_gbs()
        wbytes = 8.0 * params_of(WIDTHS[name])
        hbm_paths = {}
        for tag, dy, dj, nbytes in (("line_search_forward", Yd.data_ptr(), 0, wbytes),
                                    ("jacobian_reverse", 0, Jd.data_ptr(), 2.0 * wbytes)):
            call = lambda: net.oracle_batched_device(1, Xd.data_ptr(), 0, dy, dj, 0, stream.cuda_stream)  # noqa: E731
            for _ in range(5):
                call()
            torch.cuda.synchronize()
            reps = 50
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record(stream)
            for _ in range(reps):
                call()
            f1.record(stream)
            torch.cuda.synchronize()
            ms = f0.elapsed_time(f1) / reps
            gbs = nbytes / (ms * 1e-3) / 1e9
            hbm_paths[tag] = {"ms": ms, "algorithmic_bytes": nbytes, "achieved_gbs": gbs, "peak_gbs": hbm_peak,
                              "frac": gbs / hbm_peak, "peak_source": hbm_src, "launches": net.last_launch_count}

    # ---- e2e through the public host-buffer API (pinned host memory) ----
    e2e = None
    Yh = Jh = Hh = None
    if not args.no_e2e:
        Xh = torch.from_numpy(wl.X[idx]).pin_memory().numpy()
        Lh = torch.from_numpy(wl.Lam[idx]).pin_memory().numpy()
        if world == 1:
            Yh = torch.empty(B, m, dtype=torch.float64).pin_memory().numpy()
            Jh = torch.empty(B, m, n, dtype=torch.float64).pin_memory().numpy()
            Hh = torch.empty(B, n, n, dtype=torch.float64).pin_memory().numpy()
            call = lambda: net.oracle_batched(Xh, Lh, out=(Yh, Jh, Hh))  # noqa: E731
            h2d, d2h, api = B * (n + m) * 8, B * per * 8, "gbopt_net_oracle_batched (host buffers, synchronous)"
        else:
            so = parallel.ShardedOracle(net, total_points if name in SHARDED else B * world, dist, rank, world, dev)
            call = lambda: so(Xh, Lh)  # noqa: E731
            h2d, d2h = total_points * (n + m) * 8, total_points * per * 8
            api = ("parallel.ShardedOracle (host shard in on every rank, H2D, device oracle, "
                   f"{args.dist_backend} gather, rank-0 D2H of all results)")
        for _ in range(2):
            call()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            out = call()
        torch.cuda.synchronize()
        te = max_over_ranks(torch, dist, world, dev, time.perf_counter() - t0)
        e2e = {"value": total_points * args.steps / te, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "api": api, "timer": "wall clock around the synchronous calls, max over ranks"}
        if world == 1:
            # the host-buffer call may evaluate the batch in chunks (c4: 4, so
            # its copy-out overlaps the next chunk), and split-K factors follow
            # the batch size: equal to rounding then, bit for bit otherwise
            Hdn = Hd.cpu().numpy()
            if np.array_equal(Hh, Hdn):
                e2e["matches_device"] = "bitwise"
            else:
                rel = float(np.abs(Hh - Hdn).max() / max(np.abs(Hdn).max(), 1e-300))
                e2e["matches_device"] = f"max rel {rel:.1e} (host path in sub-batches)"
                ok = ok and rel <= 1e-12
        elif rank == 0:
            Yh, Jh, Hh = out

    # ---- sharded workloads (batched c3 and contingency c4) ----
    sharded = None
    if not args.no_sharded and name == "c2":
        sharded = []
        sub_steps = max(2, min(args.steps, 5))
        r3 = run_sharded(torch, dist, gb, configs, parallel, "c3", world, rank, dev, peak, sub_steps, 2, net=net)
        r4 = run_sharded(torch, dist, gb, configs, parallel, "c4", world, rank, dev, peak, max(3, min(args.steps, 10)), 2)
        sharded = [r for r in (r3, r4) if r is not None]

    if world > 1:
        dist.barrier()

    # ---- CPU legs on rank 0, after the GPU phase: reference nn.cpp ----
    cpu = cpu1 = parity = None
    if rank == 0 and not args.no_cpu_baseline:
        from oracle import ref
        if ref.available():
            cores = os.cpu_count() or 1
            v, ne, tt, _, desc, _ = reference_sample(name, cores, budget_s=12.0)
            cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "reference", "sample": desc}
            v1, ne1, tt1, _, desc1, _ = reference_sample(name, 1, budget_s=3.0, per_step=1)
            cpu1 = {"value": v1, "unit": UNIT, "cores": 1, "kind": "reference",
                    "sample": desc1 + " (the reference build has no OpenMP, proj/CMakeLists.txt:17-20)"}
    if rank == 0 and not args.no_parity:
        if Yh is not None:      # e2e outputs: every point of the job (rank 0)
            PY, PJ, PH, sel = Yh, Jh, Hh, all_idx
        else:                   # device outputs of rank 0's own points
            PY, PJ, PH, sel = Yd.cpu().numpy(), Jd.cpu().numpy(), Hd.cpu().numpy(), idx
        k = min(2, PY.shape[0])
        parity = oracle_parity(name, wl, wl.X[sel[:k]], wl.Lam[sel[:k]], PY, PJ, PH, k)

    if rank == 0:
        F = flops_per_eval(name)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True,
            "scaling": "weak" if name not in SHARDED else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": config_dict(name, world),
            "roofline": roof,
            "roofline_eval": {"flops_per_eval": F, "achieved_tflops": F * value / world / 1e12,
                              "frac_of_peak": (F * value / world / 1e12) / peak if peak else None},
            "cpu_baseline": cpu,
            "cpu_baseline_1t": cpu1,
            "e2e": e2e,
            "parity": parity,
            "sharded": sharded,
            "hbm_paths": hbm_paths,
            "multi_rank": multi,
            "gpu_launches": int(launches_per_step * args.steps),
            "schedule": schedule,
            "clocks": clocks,
            "outputs_checked": bool(ok and (parity is None or parity["pass"])),
            "kernel_breakdown": prof_summary,
        }
        if resident is not None:
            line["value_l2_resident"] = total_points * args.steps / resident
        if gloo:
            line["note"] = ("gloo backend: a correctness run of the N>1 path (device oracle -> pack -> gather); "
                            "not a performance number")
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    rc = maybe_launch_ranks(args)
    if rc is not None:
        return rc
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
