#!/usr/bin/env python
"""Benchmark of the B200 FP64 gray-box NN oracle (one JSON line on rank 0).

Metric (BASELINE.json): NN oracle evals/s, one eval = (y, J, H) at one
(x, lambda) of the 109M-parameter MLP 784-[5120]x5-10 (config c2), plus the
roofline fraction of the dominant kernel.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2]
  python bench.py --impl reference ...   # CPU reference arm (oracle port)

A "step" is one oracle evaluation of one c2 point per GPU (weak scaling:
each rank evaluates its own points, the shared weights are replicated); for
N > 1 the step ends with an NCCL gather of every rank's (y, J, H) to rank 0
(the only collective of the path).  `value` is timed with CUDA
events on the launching stream, inputs resident in HBM, max over ranks.
`e2e` is the same metric through the public host-buffer API
(gbopt_net_oracle_batched): pinned host x/lambda in, y/J/H back out.
"""
from __future__ import annotations

import argparse
import json
import os
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--batch", type=int, default=None, help="points per GPU per step (default: config's own)")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


CONFIG_DESC = {
    "c1": "c1: single-point FP64 oracle, MLP 784-512-512-10 tanh/identity (Xavier-uniform, seed 0)",
    "c2": "c2: single-point FP64 oracle, MLP 784-[5120]x5-10 softplus/identity, 108,948,490 params "
          "(Xavier-normal, seed 1)",
    "c3": "c3: batched FP64 oracle, c2's MLP, B=64 points (seed 2)",
    "c4": "c4: K=4096 contingency copies of MLP 108-[1024]x3-1 tanh/sigmoid (Xavier-uniform, seed 3)",
    "c5": "c5: deep-chain FP64 oracle, MLP 784-[1024]x20-10 sigmoid/identity, B=16 (N(0,1/fan_in), seed 4)",
}
DEFAULT_BATCH = {"c1": 1, "c2": 1, "c3": 64, "c4": 4096, "c5": 16}


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
# CPU reference arm (the oracle port; reference nn.cpp:113-292 restated)
# ---------------------------------------------------------------------------
def oracle_net_from(net):
    from oracle import gbopt_oracle as orc
    layers = []
    for l in range(net.layer_count):
        w, b, a = net.layer(l)
        layers.append(orc.Layer(w, b, a))
    return orc.NeuralNet(layers)


def time_cpu_reference(wl, n_points: int, budget_s: float = 12.0, min_evals: int = 2):
    """Evals/s of the CPU oracle (reference algorithm: forward, reverse-mode
    Jacobian, forward-over-reverse Hessian) on all host threads, over a
    bounded sample: at least `min_evals` evaluations and about `budget_s`
    seconds of CPU work, cycling over the first `n_points` points."""
    ref = oracle_net_from(wl.net)
    t_total, evals = 0.0, 0
    t_start = time.perf_counter()
    i = 0
    while evals < min_evals or (time.perf_counter() - t_start < budget_s and evals < 2000):
        x, lam = wl.X[i % wl.X.shape[0]], wl.Lam[i % wl.X.shape[0]]
        t0 = time.perf_counter()
        ref.forward(x)
        ref.jacobian(x)
        ref.lagrangian_hessian(x, lam)
        t_total += time.perf_counter() - t0
        evals += 1
        i += 1
        if time.perf_counter() - t_start > budget_s:
            break
    return evals / t_total, evals, t_total


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_2509_22462_b200 import configs
    name = args.config
    B = args.batch or DEFAULT_BATCH[name]
    wl = configs.make(name, batch=min(B, 4))
    cores = os.cpu_count()
    # warmup W evals (bounded), then K steps each = one eval (bounded sample).
    ref = oracle_net_from(wl.net)
    for i in range(min(args.warmup, 1)):
        ref.lagrangian_hessian(wl.X[0], wl.Lam[0])
    times = []
    t_start = time.perf_counter()
    for k in range(args.steps):
        x, lam = wl.X[k % wl.X.shape[0]], wl.Lam[k % wl.X.shape[0]]
        t0 = time.perf_counter()
        ref.forward(x)
        ref.jacobian(x)
        ref.lagrangian_hessian(x, lam)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > 120:
            break
    val = len(times) / sum(times)
    line = {
        "metric": METRIC, "value": val, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": len(times), "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": CONFIG_DESC[name], "points_per_step": 1},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{len(times)} single-point evals of {name} (reference algorithm "
                                   f"nn.cpp:113-292, numpy/OpenBLAS on {cores} threads)"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if len(times) < args.steps:
        line["note"] = f"stopped after {len(times)} of {args.steps} steps (120 s CPU budget)"
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


def run_b200(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and rank == 0:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    import paper_2509_22462_b200 as gb
    from paper_2509_22462_b200 import configs, parallel

    name = args.config
    B = args.batch or DEFAULT_BATCH[name]
    if name == "c3" and world > 1:
        B = max(1, DEFAULT_BATCH["c3"] // world)  # 64 points sharded
    if name == "c4" and world > 1:
        B = max(1, DEFAULT_BATCH["c4"] // world)
    wl = configs.make(name)
    net = wl.net
    net.bind_device(local)
    n, m = net.input_dim, net.output_dim
    # this rank's points: a contiguous shard of the config's seeded stream
    # (c2: every rank evaluates point `rank` of the stream, wrapping).
    P = wl.X.shape[0]
    idx = [(rank * B + i) % P for i in range(B)]
    Xd = torch.from_numpy(wl.X[idx]).to(dev)
    Ld = torch.from_numpy(wl.Lam[idx]).to(dev)
    Yd = torch.empty(B, m, dtype=torch.float64, device=dev)
    Jd = torch.empty(B, m, n, dtype=torch.float64, device=dev)
    Hd = torch.empty(B, n, n, dtype=torch.float64, device=dev)
    flat = torch.empty(B * (m + m * n + n * n), dtype=torch.float64, device=dev) if world > 1 else None
    gather = [torch.empty_like(flat) for _ in range(world)] if (world > 1 and rank == 0) else None

    stream = torch.cuda.current_stream(dev)

    def step():
        net.oracle_batched_device(B, Xd.data_ptr(), Ld.data_ptr(), Yd.data_ptr(), Jd.data_ptr(), Hd.data_ptr(),
                                  stream.cuda_stream)
        if world > 1:
            # result gather to rank 0: the path's only collective
            # (paper_2509_22462_b200/parallel.py; CPU-tested over gloo)
            parallel.pack(Yd, Jd, Hd, B, m, n, flat)
            dist.gather(flat, gather_list=gather, dst=0)

    peak = measure_fp64_peak(torch, dev) if rank == 0 else None

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    launches_per_step = net.last_launch_count
    schedule = net.last_schedule  # auto: measured on the first evaluation (layer-by-layer graph or dataflow launch)

    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    t = e0.elapsed_time(e1) / 1e3
    if world > 1:
        tt = torch.tensor([t], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    value = world * B * args.steps / t
    clocks = clk.summary()

    # ---- parity spot check of the benchmarked outputs (rank 0) ----
    # (full parity lives in tests/; here: H symmetric and finite)
    ok = bool(torch.isfinite(Hd).all().item()) and bool(torch.equal(Hd, Hd.transpose(1, 2)))

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
        tr = None
        per = traffic.get("per_launch_dram_bytes", {}) if traffic else {}
        tr = per.get(f"{dom}@{args.config}")
        roof = {"kernel": dom, "bound": "tensor", "achieved": round(achieved, 3), "peak": round(peak, 3),
                "unit": "TFLOP/s", "frac": round(achieved / peak, 4), "traffic": tr,
                "algorithmic_flops_per_launch": fl / cnt, "avg_launch_ms": ms / cnt,
                "peak_source": "cuBLAS DGEMM 8192^3 burst, measured live in this run (FP64; no FP64 entry in "
                               "MEASURED_PEAKS.json)",
                "traffic_source": tsrc}

    # ---- e2e through the public host-buffer API (pinned host memory) ----
    e2e = None
    if not args.no_e2e:
        Xh = torch.from_numpy(wl.X[idx]).pin_memory().numpy()
        Lh = torch.from_numpy(wl.Lam[idx]).pin_memory().numpy()
        Yh = torch.empty(B, m, dtype=torch.float64).pin_memory().numpy()
        Jh = torch.empty(B, m, n, dtype=torch.float64).pin_memory().numpy()
        Hh = torch.empty(B, n, n, dtype=torch.float64).pin_memory().numpy()
        for _ in range(2):
            net.oracle_batched(Xh, Lh, out=(Yh, Jh, Hh))
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            net.oracle_batched(Xh, Lh, out=(Yh, Jh, Hh))
        te = time.perf_counter() - t0
        if world > 1:
            tt = torch.tensor([te], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt.item())
        e2e = {"value": world * B * args.steps / te, "unit": UNIT,
               "h2d_bytes_per_step": B * (n + m) * 8, "d2h_bytes_per_step": B * (m + m * n + n * n) * 8,
               "api": "gbopt_net_oracle_batched (host buffers, synchronous)"}
        ok = ok and bool(np.array_equal(Hh, Hd.cpu().numpy()))

    # ---- CPU baseline: oracle port on rank 0 at N=1 ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        wls = configs.make(name, batch=min(B, 4))
        v, ne, tt = time_cpu_reference(wls, n_points=min(B, 4), budget_s=12.0)
        cpu = {"value": v, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
               "sample": f"{ne} single-point evals of {name} in {tt:.1f}s (reference algorithm nn.cpp:113-292, "
                         f"numpy/OpenBLAS, all host threads)"}

    if rank == 0:
        F = configs.flops(name)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": CONFIG_DESC[name], "points_per_step_per_gpu": B,
                       "params": int(net.param_count),
                       "l2": "no flush needed: the weights streamed every step (%.1f MB) exceed the 126 MB L2"
                             % (8e-6 * net.param_count),
                       "parallelism": f"replicated weights, points sharded over {world} GPU(s), NCCL gather"
                       if world > 1 else "1 GPU"},
            "roofline": roof,
            "roofline_eval": {"flops_per_eval": F, "achieved_tflops": F * value / world / 1e12,
                              "frac_of_peak": (F * value / world / 1e12) / peak if peak else None},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches_per_step * args.steps),
            "schedule": schedule,
            "clocks": clocks,
            "outputs_checked": ok,
            "kernel_breakdown": prof_summary,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
