"""The five BASELINE.json configurations as seeded synthetic workloads.

The reference has no initialisers other than random_net (nn.cpp:336-367)
and no normal generator; the semantics below are the builder's, fixed in
SURVEY.md Appendix A and DESIGN.md:
  * one library Prng (mt19937_64, prng.hpp:11-23) per config seed;
  * per layer W row-major then b (nn.cpp:354-362), then all x (point-major),
    then all lambda;
  * normals: Box-Muller, both values of each pair used;
  * unspecified biases are 0 (no draws); c5's output layer is linear.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List

import numpy as np

from . import gbopt as g


@dataclass
class Workload:
    name: str
    widths: List[int]
    hidden: int
    final: int
    net: g.NeuralNet
    X: np.ndarray     # B x n
    Lam: np.ndarray   # B x m


def flops_per_eval(widths, acts) -> float:
    """Algorithmic FP64 flops of one (y, J, H) evaluation:
    F_fwd + F_adj + F_jac + F_hess with
      F_fwd  = sum_{l=1..L} 2 n_l n_{l-1}
      F_adj  = sum_{l=2..L} 2 n_l n_{l-1}
      F_jac  = sum_{l=2..L} 2 n_l n_{l-1} n
      F_hess = sum_{l nonlinear} n_l n (n+1)
    acts[l-1] is layer l's activation code."""
    n = widths[0]
    L = len(widths) - 1
    f = 0.0
    for l in range(1, L + 1):
        mac = widths[l] * widths[l - 1]
        f += 2 * mac
        if l >= 2:
            f += 2 * mac + 2 * mac * n
        if acts[l - 1] != g.LINEAR:
            f += widths[l] * n * (n + 1)
    return f


CONFIGS = {
    "c1": dict(widths=[784, 512, 512, 10], hidden=g.TANH, final=g.LINEAR, init=g.INIT_XAVIER_UNIFORM,
               bias=(-0.05, 0.05), seed=0, batch=1, xdist=("uniform", 0.0, 1.0), ldist=("normal", 0.0, 1.0)),
    "c2": dict(widths=[784] + [5120] * 5 + [10], hidden=g.SOFTPLUS, final=g.LINEAR, init=g.INIT_XAVIER_NORMAL,
               bias=(0.0, 0.0), seed=1, batch=1, xdist=("uniform", 0.0, 1.0), ldist=("normal", 0.0, 1.0)),
    "c3": dict(widths=[784] + [5120] * 5 + [10], hidden=g.SOFTPLUS, final=g.LINEAR, init=g.INIT_XAVIER_NORMAL,
               bias=(0.0, 0.0), seed=1, batch=64, input_seed=2, xdist=("uniform", 0.0, 1.0),
               ldist=("normal", 0.0, 1.0)),
    "c4": dict(widths=[108, 1024, 1024, 1024, 1], hidden=g.TANH, final=g.SIGMOID, init=g.INIT_XAVIER_UNIFORM,
               bias=(0.0, 0.0), seed=3, batch=4096, xdist=("normal", 1.0, 0.1), ldist=("uniform", 0.0, 1.0)),
    "c5": dict(widths=[784] + [1024] * 20 + [10], hidden=g.SIGMOID, final=g.LINEAR, init=g.INIT_NORMAL_FANIN,
               bias=(0.0, 0.0), seed=4, batch=16, xdist=("uniform", 0.0, 1.0), ldist=("normal", 0.0, 1.0)),
}


def _draw(rng: g.Prng, dist, n):
    kind, a, b = dist
    return rng.uniform(a, b, n) if kind == "uniform" else rng.normal(a, b, n)


def make(name: str, batch: int | None = None, widths_override=None, net: g.NeuralNet | None = None) -> Workload:
    """Build config `name`.  `batch` truncates the point set (the first B
    points of the full seeded stream, so subsamples are prefixes).  `net`
    reuses an already built network of the same seed for configs whose
    points come from their own seed (c3 shares c2's weights)."""
    c = CONFIGS[name]
    widths = widths_override or c["widths"]
    rng = g.Prng(c["seed"])
    if net is not None and "input_seed" not in c:
        raise ValueError(f"make: config {name} draws its points after the weights; cannot reuse a net")
    if net is None:
        net = g.random_net_ex(rng, widths, c["hidden"], c["final"], c["init"], *c["bias"])
    if "input_seed" in c:
        rng = g.Prng(c["input_seed"])
    B = c["batch"]
    n, m = widths[0], widths[-1]
    X = _draw(rng, c["xdist"], B * n).reshape(B, n)
    Lam = _draw(rng, c["ldist"], B * m).reshape(B, m)
    if batch is not None:
        X, Lam = X[:batch].copy(), Lam[:batch].copy()
    return Workload(name, list(widths), c["hidden"], c["final"], net, X, Lam)


def flops(name: str) -> float:
    c = CONFIGS[name]
    acts = [c["hidden"]] * (len(c["widths"]) - 2) + [c["final"]]
    return flops_per_eval(c["widths"], acts)
