"""GPU parity of the persistent dataflow schedule (dataflow.cuh): one launch
runs the forward chain, the adjoint chain, the tangent GEMMs and the Hessian
SYRKs as dependency-ordered tiles.  Checked against the CPU oracle
(oracle/gbopt_oracle.py, a restatement of proj/src/nn.cpp:113-292) and
against the layer-by-layer schedule on the same handle.

Parity metric: per array and per point,
max|GPU - CPU| / max|CPU| <= 1e-10 (north_star tolerance, FP64).
"""
import os

import numpy as np
import pytest

from conftest import has_gpu

pytestmark = pytest.mark.gpu

TOL = 1e-10

if has_gpu():
    import paper_2509_22462_b200 as gb
    from paper_2509_22462_b200 import configs
from oracle import gbopt_oracle as orc


def to_oracle(net):
    return orc.NeuralNet([orc.Layer(*net.layer(l)) for l in range(net.layer_count)])


def check_batch(net, ref, X, Lam, tol=TOL):
    Y, J, H = net.oracle_batched(X, Lam)
    for b in range(X.shape[0]):
        ry = ref.forward(X[b])
        rj = ref.jacobian(X[b])
        rh = ref.lagrangian_hessian(X[b], Lam[b])
        assert orc.rel_err(Y[b], ry) <= tol, ("y", b, orc.rel_err(Y[b], ry))
        assert orc.rel_err(J[b], rj) <= tol, ("J", b, orc.rel_err(J[b], rj))
        if np.abs(rh).max() > 0:
            assert orc.rel_err(H[b], rh) <= tol, ("H", b, orc.rel_err(H[b], rh))
        else:
            assert np.abs(H[b]).max() <= 1e-14
        assert np.array_equal(H[b], H[b].T)
    return Y, J, H


CASES = [
    # widths, hidden, final, seed, batch
    ([5, 7, 4], "tanh", "tanh", 1234, 1),
    ([4, 6, 6, 3], "sigmoid", "tanh", 3, 2),
    ([4, 6, 6, 3], "tanh", "linear", 5, 5),
    ([4, 6, 6, 3], "linear", "linear", 6, 1),           # no SYRK layer at all
    ([6, 9, 4], "softplus", "sigmoid", 41, 3),          # nonlinear output: small-K curvature
    ([3, 5], "tanh", "tanh", 1, 1),                     # one layer: no hidden layer, layered schedule
    ([3, 6, 5], "tanh", "tanh", 1, 2),                  # one hidden layer: T_0 only, no GEMM
    ([7, 4, 1], "softplus", "linear", 77, 4),           # scalar output
    ([9, 33, 17, 16], "tanh", "sigmoid", 8, 2),         # 16 outputs (skinny limit)
    ([130, 200, 150, 12], "softplus", "linear", 10, 3),  # n_pad > 112: several row blocks
    ([300, 257, 129, 3], "tanh", "tanh", 11, 2),
    ([113, 129, 300, 129, 5], "sigmoid", "linear", 12, 7),  # ragged K / tile edges
    ([64, 128, 96, 10], "softplus", "linear", 13, 16),
]


@pytest.mark.parametrize("widths,hid,fin,seed,B", CASES)
def test_dataflow_matches_oracle(widths, hid, fin, seed, B):
    net = gb.random_net(widths, hid, fin, seed).set_schedule("dataflow").bind_device(0)
    ref = to_oracle(net)
    rng = np.random.default_rng(seed)
    X = rng.uniform(-1, 1, (B, widths[0]))
    Lam = rng.normal(0, 1, (B, widths[-1]))
    check_batch(net, ref, X, Lam)
    assert net.last_schedule == ("dataflow" if len(widths) >= 3 else "layered")


@pytest.mark.parametrize("widths,hid,fin,seed,B", CASES[::3])
def test_dataflow_equals_layered(widths, hid, fin, seed, B):
    net = gb.random_net(widths, hid, fin, seed).bind_device(0)
    rng = np.random.default_rng(seed + 1)
    X = rng.uniform(-1, 1, (B, widths[0]))
    Lam = rng.normal(0, 1, (B, widths[-1]))
    net.set_schedule("layered")
    Y0, J0, H0 = net.oracle_batched(X, Lam)
    assert net.last_schedule == "layered"
    net.set_schedule("dataflow")
    Y1, J1, H1 = net.oracle_batched(X, Lam)
    assert net.last_schedule == "dataflow"
    # the forward / adjoint reductions differ (DMMA tiles vs GEMV sweeps):
    # equal to rounding
    for b in range(B):
        assert orc.rel_err(Y1[b], Y0[b]) <= 1e-13
        assert orc.rel_err(J1[b], J0[b]) <= 1e-13
        if np.abs(H0[b]).max() > 0:
            assert orc.rel_err(H1[b], H0[b]) <= 1e-13


def test_dataflow_deterministic_and_graph_invariant():
    widths = [130, 200, 150, 12]
    net = gb.random_net(widths, "softplus", "linear", 21).set_schedule("dataflow").bind_device(0)
    rng = np.random.default_rng(3)
    X = rng.uniform(-1, 1, (5, 130))
    Lam = rng.normal(0, 1, (5, 12))
    a = net.oracle_batched(X, Lam)
    for _ in range(3):
        b = net.oracle_batched(X, Lam)
        for u, v in zip(a, b):
            assert np.array_equal(u, v)
    net.set_graphs(False)
    c = net.oracle_batched(X, Lam)
    for u, v in zip(a, c):
        assert np.array_equal(u, v)


def test_dataflow_max_batch_and_fallback():
    widths = [40, 64, 48, 6]
    net = gb.random_net(widths, "tanh", "linear", 9).set_schedule("dataflow").bind_device(0)
    ref = to_oracle(net)
    rng = np.random.default_rng(4)
    X = rng.uniform(-1, 1, (112, 40))
    Lam = rng.normal(0, 1, (112, 6))
    Y, J, H = net.oracle_batched(X, Lam)
    assert net.last_schedule == "dataflow"
    for b in (0, 55, 111):
        assert orc.rel_err(H[b], ref.lagrangian_hessian(X[b], Lam[b])) <= TOL
        assert orc.rel_err(J[b], ref.jacobian(X[b])) <= TOL
    # 113 points do not fit one FWD/ADJ tile: layer-by-layer schedule
    X2 = rng.uniform(-1, 1, (113, 40))
    L2 = rng.normal(0, 1, (113, 6))
    _, _, H2 = net.oracle_batched(X2, L2)
    assert net.last_schedule == "layered"
    assert orc.rel_err(H2[112], ref.lagrangian_hessian(X2[112], L2[112])) <= TOL
    # a softmax output stays layer by layer
    sm = gb.random_net([4, 6, 6, 3], "tanh", "softmax", 2).set_schedule("dataflow").bind_device(0)
    sm.oracle(np.ones(4) * 0.1, np.ones(3))
    assert sm.last_schedule == "layered"


def test_auto_schedule_is_measured_and_sticky():
    """Auto mode times both schedules on the first evaluation of a shape and
    keeps the faster; the choice is reused, and either choice is correct."""
    widths = [300, 257, 129, 3]
    net = gb.random_net(widths, "tanh", "tanh", 11).bind_device(0)
    ref = to_oracle(net)
    rng = np.random.default_rng(12)
    X = rng.uniform(-1, 1, (2, 300))
    Lam = rng.normal(0, 1, (2, 3))
    Y, J, H = check_batch(net, ref, X, Lam)
    first = net.last_schedule
    assert first in ("layered", "dataflow")
    Y2, J2, H2 = net.oracle_batched(X, Lam)
    assert net.last_schedule == first
    assert np.array_equal(H, H2) and np.array_equal(J, J2)


def test_c2_dataflow_parity():
    """The 109M-parameter config through the dataflow launch."""
    wl = configs.make("c2")
    net = wl.net.set_schedule("dataflow").bind_device(0)
    ref = to_oracle(net)
    y, j, h = net.oracle(wl.X[0], wl.Lam[0])
    assert net.last_schedule == "dataflow"
    assert orc.rel_err(y, ref.forward(wl.X[0])) <= TOL
    assert orc.rel_err(j, ref.jacobian(wl.X[0])) <= TOL
    assert orc.rel_err(h, ref.lagrangian_hessian(wl.X[0], wl.Lam[0])) <= TOL
    assert np.array_equal(h, h.T)


@pytest.mark.parametrize("schedule", ["layered", "dataflow"])
@pytest.mark.parametrize("widths,hid,fin,seed", [
    ([5, 7, 4], "tanh", "tanh", 1),
    ([130, 200, 150, 12], "softplus", "linear", 2),
    ([113, 129, 300, 129, 5], "sigmoid", "linear", 3),
])
def test_oracle_lower_packs_the_full_hessian(schedule, widths, hid, fin, seed):
    """gbopt_net_oracle_lower: the Hessian packed on the device in the
    reduced-space callback's value order equals the full Hessian's lower
    triangle bit for bit (same kernels, only the epilogue differs), and y, J
    match the full call."""
    net = gb.random_net(widths, hid, fin, seed).set_schedule(schedule).bind_device(0)
    rng = np.random.default_rng(seed)
    x = rng.uniform(-1, 1, widths[0])
    lam = rng.normal(0, 1, widths[-1])
    y, j, h = net.oracle(x, lam)
    yl, jl, hl = net.oracle_lower(x, lam)
    n = widths[0]
    rows, cols = np.tril_indices(n)
    assert np.array_equal(hl, h[rows, cols])
    assert np.array_equal(yl, y) and np.array_equal(jl, j)
    ref = to_oracle(net).lagrangian_hessian(x, lam)
    assert orc.rel_err(hl, ref[rows, cols]) <= TOL
    # Hessian only
    _, _, hl2 = net.oracle_lower(x, lam, want_y=False, want_j=False)
    assert np.array_equal(hl2, hl)


@pytest.mark.parametrize("chunks", [2, 3, 7])
def test_host_call_in_chunks(monkeypatch, chunks):
    """Host-buffer batched calls evaluated in chunks whose device->host
    copies overlap the next chunk (GBOPT_HOST_CHUNKS forces the split):
    same results as one chunk (y, J bitwise; H to rounding) and as the
    oracle, pinned and pageable outputs."""
    import torch
    net = gb.random_net([40, 64, 48, 6], "tanh", "linear", 19).bind_device(0)
    ref = to_oracle(net)
    rng = np.random.default_rng(chunks)
    B = 7
    X = rng.uniform(-1, 1, (B, 40))
    Lam = rng.normal(0, 1, (B, 6))
    monkeypatch.setenv("GBOPT_HOST_CHUNKS", "1")
    Y0, J0, H0 = net.oracle_batched(X, Lam)
    monkeypatch.setenv("GBOPT_HOST_CHUNKS", str(chunks))
    Y1, J1, H1 = net.oracle_batched(X, Lam)
    pinned = [torch.empty(shape, dtype=torch.float64).pin_memory().numpy() for shape in ((B, 6), (B, 6, 40), (B, 40, 40))]
    Y2, J2, H2 = net.oracle_batched(X, Lam, out=tuple(pinned))
    for (Y, J, H) in ((Y1, J1, H1), (Y2, J2, H2)):
        for b in range(B):  # a one-point chunk takes the single-point kernels: equal to rounding
            assert orc.rel_err(Y[b], Y0[b]) <= 1e-14 and orc.rel_err(J[b], J0[b]) <= 1e-14
            assert orc.rel_err(H[b], H0[b]) <= 1e-14
            assert orc.rel_err(H[b], ref.lagrangian_hessian(X[b], Lam[b])) <= TOL


def test_auto_schedule_is_a_shape_rule():
    """The default schedule is a fixed rule on the shape (no timing), so
    c5 (21 layers, 13.5% idle waves) always takes the dataflow launch and
    c1 / c2 the layer-by-layer graph."""
    if not has_gpu():
        pytest.skip("no GPU")
    for name, batch, want in (("c5", 16, "dataflow"), ("c1", 1, "layered"), ("c4", 64, "layered")):
        wl = configs.make(name, batch=batch)
        net = wl.net.bind_device(0)
        net.oracle_batched(wl.X, wl.Lam)
        assert net.last_schedule == want, (name, net.last_schedule)


_HASH_SCRIPT = r"""
import hashlib, sys
sys.path.insert(0, {root!r})
from paper_2509_22462_b200 import configs
wl = configs.make("c5", batch=16)
net = wl.net.bind_device(0)
Y, J, H = net.oracle_batched(wl.X, wl.Lam)
print(net.last_schedule, hashlib.sha256(Y.tobytes() + J.tobytes() + H.tobytes()).hexdigest())
"""


def test_two_processes_give_bitwise_identical_outputs():
    if not has_gpu():
        pytest.skip("no GPU")
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = [subprocess.run([sys.executable, "-c", _HASH_SCRIPT.format(root=root)], capture_output=True, text=True,
                           timeout=600).stdout.strip() for _ in range(2)]
    assert outs[0] and outs[0] == outs[1], outs
