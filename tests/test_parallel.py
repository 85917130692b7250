"""N > 1 path on the CPU: contiguous point sharding and the result gather
(paper_2509_22462_b200/parallel.py) over a world-size-2 (and 3) gloo group.

On the GPU box the same code runs over NCCL with the device oracle as the
per-shard evaluator; here the evaluator is the CPU oracle (a stand-in for
the compute, the logic under test is the sharding, padding and gather).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_22462_b200 import parallel


def test_shard_partitions_points():
    for P in (1, 2, 7, 64, 4096):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                s, c = parallel.shard(P, world, r)
                seen.extend(range(s, s + c))
                assert c <= parallel.max_shard(P, world)
            assert seen == list(range(P))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, P, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import gbopt_oracle as orc
    net = orc.random_net([6, 9, 8, 3], orc.TANH, orc.SOFTMAX, 77)
    rng = np.random.default_rng(1)
    X = rng.uniform(-1, 1, (P, 6))
    L = rng.uniform(-1, 1, (P, 3))

    def evaluate(Xs, Ls):
        ys = np.array([net.forward(x) for x in Xs]).reshape(len(Xs), 3)
        js = np.array([net.jacobian(x) for x in Xs]).reshape(len(Xs), 3, 6)
        hs = np.array([net.lagrangian_hessian(x, l) for x, l in zip(Xs, Ls)]).reshape(len(Xs), 6, 6)
        return torch.from_numpy(ys), torch.from_numpy(js), torch.from_numpy(hs)

    out = parallel.evaluate_sharded(X, L, 3, evaluate, dist, rank, world, dst=0)
    if rank == 0:
        Y, J, H = (t.numpy() for t in out)
        Ye, Je, He = (t.numpy() for t in evaluate(X, L))
        q.put(bool(np.array_equal(Y, Ye) and np.array_equal(J, Je) and np.array_equal(H, He) and Y.shape[0] == P))
    else:
        q.put(out is None)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,P", [(2, 5), (2, 8), (3, 7)])
def test_sharded_gather_matches_single_process(world, P):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, P, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    results = [q.get(timeout=5) for _ in range(world)]
    assert all(p.exitcode == 0 for p in procs)
    assert all(results)
