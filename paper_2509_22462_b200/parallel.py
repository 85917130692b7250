"""Multi-GPU data parallelism for the oracle: replicated weights, points
(or contingencies) sharded contiguously over ranks, one result gather.

The reference is single-process (no NCCL/MPI/threads); the
north_star asks for batched points and independent contingency copies to be
sharded across the GPUs of one box with no inter-GPU reduction, NCCL only to
gather results.  Each rank evaluates its shard with the device oracle
(``gbopt_net_oracle_batched_device``) and the (y, J, H) blocks are gathered
to ``dst`` with one ``torch.distributed.gather`` of a flat buffer per rank
(NCCL over NVLink on the GPU box; gloo in the CPU tests).  Shards may be
ragged (P not divisible by the world size): every rank pads its flat buffer
to the largest shard so the collective sees equal sizes, and the receiver
drops the padding.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Tuple

import numpy as np


def shard(points: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous shard [start, start+count) of `points` for `rank`;
    the first (points % world) ranks get one extra point."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("shard: bad world/rank")
    base, extra = divmod(points, world)
    count = base + (1 if rank < extra else 0)
    start = rank * base + min(rank, extra)
    return start, count


def max_shard(points: int, world: int) -> int:
    return -(-points // world)


def pack(y, j, h, rows: int, m: int, n: int, out):
    """Flatten (y, J, H) of `count` points into `out` (length rows*(m+mn+n^2));
    rows >= count, the tail stays as padding."""
    per = m + m * n + n * n
    count = y.shape[0]
    view = out.reshape(rows, per)
    view[:count, :m] = y.reshape(count, m)
    view[:count, m:m + m * n] = j.reshape(count, m * n)
    view[:count, m + m * n:] = h.reshape(count, n * n)
    return out


def unpack(flat_list, counts: List[int], rows: int, m: int, n: int, xp=np):
    """Concatenate gathered flat buffers into (Y, J, H) for all points."""
    per = m + m * n + n * n
    ys, js, hs = [], [], []
    for buf, c in zip(flat_list, counts):
        v = buf.reshape(rows, per)[:c]
        ys.append(v[:, :m])
        js.append(v[:, m:m + m * n].reshape(c, m, n))
        hs.append(v[:, m + m * n:].reshape(c, n, n))
    cat = xp.concatenate if xp is np else xp.cat
    return cat(ys), cat(js), cat(hs)


def evaluate_sharded(X, Lam, m: int, evaluate: Callable, dist, rank: int, world: int, dst: int = 0,
                     device: Optional[object] = None):
    """Evaluate all P points of X/Lam over `world` ranks and gather on `dst`.

    `evaluate(Xs, Ls) -> (Y, J, H)` computes one shard (torch tensors on
    `device`, or numpy arrays when device is None / CPU).  Returns the full
    (Y, J, H) on `dst` and None elsewhere.  Works with NCCL (CUDA tensors) and
    gloo (CPU tensors).
    """
    import torch

    P, n = X.shape
    start, count = shard(P, world, rank)
    rows = max_shard(P, world)
    per = m + m * n + n * n
    Y, J, H = evaluate(X[start:start + count], Lam[start:start + count])
    dev = device if device is not None else torch.device("cpu")
    flat = torch.zeros(rows * per, dtype=torch.float64, device=dev)
    Yt, Jt, Ht = (torch.as_tensor(a, device=dev) for a in (Y, J, H))
    pack(Yt, Jt, Ht, rows, m, n, flat)
    gather = [torch.empty_like(flat) for _ in range(world)] if rank == dst else None
    dist.gather(flat, gather_list=gather, dst=dst)
    if rank != dst:
        return None
    counts = [shard(P, world, r)[1] for r in range(world)]
    return unpack(gather, counts, rows, m, n, xp=torch)


class ShardedOracle:
    """The multi-GPU public API: one process per GPU, replicated weights,
    contiguous point shards, one result gather to ``dst``.

    Every rank constructs it with the same ``P`` (points per call) and calls
    it with its own shard of x/lambda (host arrays, ``shard(P, world, rank)``
    rows); rank ``dst`` receives (Y, J, H) of all P points in host buffers,
    the other ranks get None.  Per call: host->device copy of the shard,
    ``gbopt_net_oracle_batched_device`` on the rank's stream, pack, one
    ``torch.distributed.gather`` (NCCL over NVLink with CUDA tensors; with
    the gloo backend the flat buffer goes through host memory), and on
    ``dst`` one device->host copy of the gathered results.  No reduction.
    """

    def __init__(self, net, P: int, dist, rank: int, world: int, device, dst: int = 0, pinned: bool = True):
        import torch

        self.net, self.P, self.dist, self.rank, self.world, self.dst = net, P, dist, rank, world, dst
        self.dev = device
        self.n, self.m = net.input_dim, net.output_dim
        n, m = self.n, self.m
        self.start, self.count = shard(P, world, rank)
        self.rows = max_shard(P, world)
        self.per = m + m * n + n * n
        B = max(self.count, 1)
        self.Xd = torch.zeros(B, n, dtype=torch.float64, device=device)
        self.Ld = torch.zeros(B, m, dtype=torch.float64, device=device)
        self.Yd = torch.empty(B, m, dtype=torch.float64, device=device)
        self.Jd = torch.empty(B, m, n, dtype=torch.float64, device=device)
        self.Hd = torch.empty(B, n, n, dtype=torch.float64, device=device)
        self.backend = dist.get_backend() if world > 1 else "none"
        cdev = device if self.backend != "gloo" else torch.device("cpu")
        self.flat = torch.zeros(self.rows * self.per, dtype=torch.float64, device=device)
        self.flat_c = self.flat if cdev == device else torch.zeros_like(self.flat, device=cdev)
        self.gather = ([torch.empty_like(self.flat_c) for _ in range(world)]
                       if (rank == dst and world > 1) else None)
        if rank == dst:
            mk = (lambda *s: torch.empty(*s, dtype=torch.float64).pin_memory()) if pinned and \
                torch.cuda.is_available() else (lambda *s: torch.empty(*s, dtype=torch.float64))
            self.out_flat = mk(world * self.rows * self.per)
        self.stream = torch.cuda.current_stream(device)

    def h2d_bytes(self) -> int:
        return self.count * (self.n + self.m) * 8

    def d2h_bytes(self) -> int:
        return self.P * self.per * 8 if self.rank == self.dst else 0

    def __call__(self, X, Lam):
        import torch

        c = self.count
        if c:
            self.Xd[:c].copy_(torch.as_tensor(X), non_blocking=True)
            self.Ld[:c].copy_(torch.as_tensor(Lam), non_blocking=True)
            self.net.oracle_batched_device(c, self.Xd.data_ptr(), self.Ld.data_ptr(), self.Yd.data_ptr(),
                                           self.Jd.data_ptr(), self.Hd.data_ptr(), self.stream.cuda_stream)
            pack(self.Yd[:c], self.Jd[:c], self.Hd[:c], self.rows, self.m, self.n, self.flat)
        if self.world > 1:
            if self.flat_c is not self.flat:
                self.flat_c.copy_(self.flat)
            self.dist.gather(self.flat_c, gather_list=self.gather, dst=self.dst)
        if self.rank != self.dst:
            return None
        parts = self.gather if self.world > 1 else [self.flat]
        L = self.rows * self.per
        for r, buf in enumerate(parts):
            self.out_flat[r * L:(r + 1) * L].copy_(buf, non_blocking=True)
        torch.cuda.current_stream(self.dev).synchronize()
        counts = [shard(self.P, self.world, r)[1] for r in range(self.world)]
        flats = [self.out_flat[r * L:(r + 1) * L].numpy() for r in range(self.world)]
        return unpack(flats, counts, self.rows, self.m, self.n)
