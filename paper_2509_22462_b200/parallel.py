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
