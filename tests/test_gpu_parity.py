"""GPU parity: the B200 oracle (through the C ABI) against the CPU oracle
restatement of the reference algorithm (oracle/gbopt_oracle.py, which
follows proj/src/nn.cpp:113-292 line by line).

Parity metric: per array and per point,
max|GPU - CPU| / max|CPU| <= 1e-10 (north_star tolerance, FP64).
"""
import numpy as np
import pytest

from conftest import has_gpu

pytestmark = pytest.mark.gpu

TOL = 1e-10

if has_gpu():
    import paper_2509_22462_b200 as gb
    from paper_2509_22462_b200 import configs
from oracle import gbopt_oracle as orc


def to_oracle(net) -> "orc.NeuralNet":
    layers = []
    for l in range(net.layer_count):
        w, b, a = net.layer(l)
        layers.append(orc.Layer(w, b, a))
    return orc.NeuralNet(layers)


def check_point(net, ref, x, lam, tol=TOL):
    y, j, h = net.oracle(x, lam)
    ry = ref.forward(x)
    rj = ref.jacobian(x)
    rh = ref.lagrangian_hessian(x, lam)
    assert orc.rel_err(y, ry) <= tol, ("y", orc.rel_err(y, ry))
    assert orc.rel_err(j, rj) <= tol, ("J", orc.rel_err(j, rj))
    if np.abs(rh).max() > 0:
        assert orc.rel_err(h, rh) <= tol, ("H", orc.rel_err(h, rh))
    else:
        assert np.abs(h).max() <= 1e-14
    assert np.array_equal(h, h.T)  # exactly symmetric (nn.cpp:291)
    return orc.rel_err(y, ry), orc.rel_err(j, rj), orc.rel_err(h, rh)


MIXES = [
    ([5, 7, 4], "tanh", "tanh", 1234),
    ([4, 6, 6, 3], "tanh", "softmax", 2),
    ([4, 6, 6, 3], "sigmoid", "tanh", 3),
    ([4, 6, 6, 3], "sigmoid", "softmax", 4),
    ([4, 6, 6, 3], "tanh", "linear", 5),
    ([4, 6, 6, 3], "linear", "linear", 6),
    ([5, 8, 7, 4], "sigmoid", "softmax", 999),
    ([6, 9, 4], "softplus", "sigmoid", 41),
    ([3, 5], "tanh", "tanh", 1),
    ([7, 4], "softplus", "softmax", 77),
    ([9, 33, 17, 40], "tanh", "sigmoid", 8),      # final width > 16 (big final path)
    ([9, 33, 17, 20], "sigmoid", "softmax", 9),    # softmax wider than 16
    ([130, 200, 150, 12], "softplus", "linear", 10),  # n_pad > 112, multiple M tiles
    ([300, 257, 129, 3], "tanh", "tanh", 11),
]


@pytest.mark.parametrize("widths,hid,fin,seed", MIXES)
def test_small_nets_match_oracle(widths, hid, fin, seed):
    net = gb.random_net(widths, hid, fin, seed)
    ref = to_oracle(net)
    rng = np.random.default_rng(seed)
    for _ in range(3):
        x = rng.uniform(-1.5, 1.5, widths[0])
        lam = rng.uniform(-2, 2, widths[-1])
        check_point(net, ref, x, lam)
        g = net.lagrangian_gradient(x, lam)
        assert orc.rel_err(g, ref.lagrangian_gradient(x, lam)) <= TOL


def test_acceptance_criterion1_nets():
    """acceptance.cpp:86-128: 25 nets, depth 1..5, widths 2..12, final softmax."""
    rng = np.random.default_rng(2026)
    hiddens = ["linear", "tanh", "sigmoid"]
    for k in range(25):
        depth = 1 + k % 5
        widths = [int(2 + rng.integers(0, 11)) for _ in range(depth + 1)]
        net = gb.random_net(widths, hiddens[k % 3], "softmax", 4000 + k)
        ref = to_oracle(net)
        x = rng.uniform(-0.9, 0.9, widths[0])
        lam = rng.uniform(-1, 1, widths[-1])
        check_point(net, ref, x, lam)
        # exact linearity in lambda (<= 1e-12)
        lam2 = rng.uniform(-1, 1, widths[-1])
        h1 = net.lagrangian_hessian(x, lam)
        h2 = net.lagrangian_hessian(x, lam2)
        hm = net.lagrangian_hessian(x, lam + 2.5 * lam2)
        assert np.abs(hm - (h1 + 2.5 * h2)).max() <= 1e-12


def test_known_answers_on_device():
    """test_nn.cpp:30-94, 151-167, 229-243 on the GPU path."""
    eye = gb.NeuralNet.from_layers([np.eye(2)], [np.zeros(2)], [gb.LINEAR])
    x = np.array([0.3, -0.7])
    assert np.array_equal(eye.forward(x), x)
    t = gb.NeuralNet.from_layers([np.eye(3)], [np.zeros(3)], [gb.TANH])
    assert np.abs(t.forward(np.zeros(3))).max() == 0.0
    assert np.array_equal(t.jacobian(np.zeros(3)), np.eye(3))
    assert np.abs(t.lagrangian_hessian(np.zeros(3), np.array([1.0, 0, 0]))).max() == 0.0
    rng = np.random.default_rng(17)
    w = rng.uniform(-1, 1, (3, 5))
    lin = gb.NeuralNet.from_layers([w], [rng.uniform(-1, 1, 3)], [gb.LINEAR])
    assert np.array_equal(lin.jacobian(rng.uniform(-1, 1, 5)), w)
    sm = gb.NeuralNet.from_layers([np.zeros((4, 4))], [np.zeros(4)], [gb.SOFTMAX])
    assert np.allclose(sm.forward(rng.uniform(-5, 5, 4)), 0.25, rtol=0, atol=1e-14)
    s = gb.NeuralNet.from_layers([np.eye(3)], [np.zeros(3)], [gb.SIGMOID])
    assert np.all(s.forward(np.zeros(3)) == 0.5)
    assert np.all(s.jacobian(np.zeros(3)) == 0.25 * np.eye(3))
    # linear net => zero Hessian
    ln = gb.random_net([4, 5, 3], "linear", "linear", 9)
    assert np.abs(ln.lagrangian_hessian(rng.uniform(-1, 1, 4), rng.uniform(-1, 1, 3))).max() <= 1e-14


def test_determinism_bitwise():
    net = gb.random_net([6, 8, 4], "tanh", "softmax", 21)
    x = np.random.default_rng(4).uniform(-1, 1, 6)
    lam = np.random.default_rng(5).uniform(-1, 1, 4)
    a = net.oracle(x, lam)
    b = net.oracle(x, lam)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)


def test_batched_equals_single():
    net = gb.random_net([20, 40, 30, 5], "sigmoid", "linear", 3)
    rng = np.random.default_rng(7)
    X = rng.uniform(-1, 1, (9, 20))
    L = rng.uniform(-1, 1, (9, 5))
    Y, J, H = net.oracle_batched(X, L)
    # batched and single-point calls use different GEMV reductions (the
    # single-point forward splits k across warps), so they agree to rounding;
    # points within one batched call are evaluated identically.
    for b in range(9):
        y, j, h = net.oracle(X[b], L[b])
        assert orc.rel_err(Y[b], y) <= 1e-14 and orc.rel_err(J[b], j) <= 1e-13 and orc.rel_err(H[b], h) <= 1e-13
    Y2, J2, H2 = net.oracle_batched(np.repeat(X[:1], 9, 0), np.repeat(L[:1], 9, 0))
    assert all(np.array_equal(Y2[0], Y2[b]) and np.array_equal(H2[0], H2[b]) for b in range(9))


def test_graphs_off_matches_graphs_on():
    net = gb.random_net([30, 64, 64, 7], "tanh", "softmax", 12)
    rng = np.random.default_rng(8)
    x, lam = rng.uniform(-1, 1, 30), rng.uniform(-1, 1, 7)
    a = net.oracle(x, lam)
    net.set_graphs(False)
    b = net.oracle(x, lam)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)


def test_config_c1_parity():
    wl = configs.make("c1")
    ref = to_oracle(wl.net)
    errs = check_point(wl.net, ref, wl.X[0], wl.Lam[0])
    print("c1 rel errs y/J/H:", errs)


@pytest.mark.slow
def test_config_c2_parity():
    wl = configs.make("c2")
    ref = to_oracle(wl.net)
    errs = check_point(wl.net, ref, wl.X[0], wl.Lam[0])
    print("c2 rel errs y/J/H:", errs)


@pytest.mark.slow
def test_config_c3_batched_parity():
    """c3: B=64 points of c2's net in one batched call; the first, a middle
    and the last point are checked against the oracle; every point's H is
    exactly symmetric."""
    wl = configs.make("c3")
    ref = to_oracle(wl.net)
    Y, J, H = wl.net.oracle_batched(wl.X, wl.Lam)
    assert Y.shape == (64, 10) and J.shape == (64, 10, 784) and H.shape == (64, 784, 784)
    for b in (0, 31, 63):
        assert orc.rel_err(Y[b], ref.forward(wl.X[b])) <= TOL
        assert orc.rel_err(J[b], ref.jacobian(wl.X[b])) <= TOL
        assert orc.rel_err(H[b], ref.lagrangian_hessian(wl.X[b], wl.Lam[b])) <= TOL
    assert np.array_equal(H, H.transpose(0, 2, 1))


def test_config_c4_contingency_parity():
    """c4: K=4096 contingencies (shared 108-[1024]x3-1 net) in one call;
    a sample of contingencies against the oracle."""
    wl = configs.make("c4")
    ref = to_oracle(wl.net)
    Y, J, H = wl.net.oracle_batched(wl.X, wl.Lam)
    assert Y.shape == (4096, 1) and J.shape == (4096, 1, 108) and H.shape == (4096, 108, 108)
    for k in (0, 1, 777, 2048, 4095):
        assert orc.rel_err(Y[k], ref.forward(wl.X[k])) <= TOL
        assert orc.rel_err(J[k], ref.jacobian(wl.X[k])) <= TOL
        assert orc.rel_err(H[k], ref.lagrangian_hessian(wl.X[k], wl.Lam[k])) <= TOL


def test_config_c5_deep_chain_parity():
    wl = configs.make("c5")
    ref = to_oracle(wl.net)
    Y, J, H = wl.net.oracle_batched(wl.X, wl.Lam)
    for b in (0, 15):
        assert orc.rel_err(Y[b], ref.forward(wl.X[b])) <= TOL
        assert orc.rel_err(J[b], ref.jacobian(wl.X[b])) <= TOL
        assert orc.rel_err(H[b], ref.lagrangian_hessian(wl.X[b], wl.Lam[b])) <= TOL


@pytest.mark.slow
def test_c2_full_size_properties():
    """Size-independent properties at BASELINE's full size (c2): linearity in
    lambda, gradient = J^T lambda, exact symmetry, batch == single."""
    wl = configs.make("c2")
    net = wl.net
    x = wl.X[0]
    rng = np.random.default_rng(3)
    l1, l2 = rng.normal(0, 1, 10), rng.normal(0, 1, 10)
    a, b = 0.37, -2.25
    h1 = net.lagrangian_hessian(x, l1)
    h2 = net.lagrangian_hessian(x, l2)
    hc = net.lagrangian_hessian(x, a * l1 + b * l2)
    assert orc.rel_err(hc, a * h1 + b * h2) <= 1e-12
    assert np.array_equal(hc, hc.T)
    j = net.jacobian(x)
    g = net.lagrangian_gradient(x, l1)
    assert orc.rel_err(g, j.T @ l1) <= 1e-12
    # Batching may change the SYRK's split-K factor (and so the summation
    # order of H at the rounding level); y and J are batch-invariant bitwise.
    # (net.jacobian is the reverse-mode sweep; the fused oracle's J comes from
    # the forward tangents: equal to rounding, compare fused with fused.)
    _, jf, _ = net.oracle(x, l1)
    assert orc.rel_err(jf, j) <= 1e-12
    Y, J, H = net.oracle_batched(np.stack([x, x]), np.stack([l1, l1]))
    assert np.array_equal(J[0], J[1]) and orc.rel_err(J[0], jf) <= 1e-13
    assert np.array_equal(H[0], H[1]) and orc.rel_err(H[0], h1) <= 1e-13


def test_device_pointer_entry_and_launch_count():
    import torch
    net = gb.random_net([40, 64, 48, 6], "softplus", "sigmoid", 5).bind_device(0)
    rng = np.random.default_rng(2)
    X = rng.uniform(0, 1, (3, 40))
    L = rng.normal(0, 1, (3, 6))
    Y, J, H = net.oracle_batched(X, L)
    dev = torch.device("cuda", 0)
    Xd, Ld = torch.from_numpy(X).to(dev), torch.from_numpy(L).to(dev)
    Yd = torch.empty(3, 6, dtype=torch.float64, device=dev)
    Jd = torch.empty(3, 6, 40, dtype=torch.float64, device=dev)
    Hd = torch.empty(3, 40, 40, dtype=torch.float64, device=dev)
    s = torch.cuda.current_stream(dev)
    net.oracle_batched_device(3, Xd.data_ptr(), Ld.data_ptr(), Yd.data_ptr(), Jd.data_ptr(), Hd.data_ptr(),
                              s.cuda_stream)
    torch.cuda.synchronize()
    assert np.array_equal(Yd.cpu().numpy(), Y) and np.array_equal(Jd.cpu().numpy(), J)
    assert np.array_equal(Hd.cpu().numpy(), H)
    assert net.last_launch_count > 5


def test_nonfinite_input_propagates_like_reference():
    """The reference oracle does not check x (nn.cpp:105-111 checks only the
    length): a NaN input yields NaN outputs, not an error."""
    net = gb.random_net([4, 5, 2], "tanh", "linear", 3)
    y = net.forward(np.array([np.nan, 0, 0, 0]))
    assert np.isnan(y).all()


def test_batched_intermediates_match_single(monkeypatch):
    """White-box: the batched (GEMM) forward/adjoint chains give the same
    per-layer z, y, sigma', sigma'', ybar, gz, d as the single-point GEMV
    chains (regression: stream-ordering of the W^T build / zero fills).
    The workspace holds the whole batch only when the host call is not
    split into chunks."""
    monkeypatch.setenv("GBOPT_HOST_CHUNKS", "1")
    widths = [784, 2048, 2048, 2048, 10]
    ref = gb.random_net(widths, "softplus", "linear", 3)
    rng = np.random.default_rng(0)
    X = rng.uniform(-1, 1, (40, 784))
    L = rng.uniform(-1, 1, (40, 10))
    net = gb.random_net(widths, "softplus", "linear", 3)
    net.oracle_batched(X, L)
    for b in (0, 17, 39):
        ref.oracle_batched(X[b:b + 1], L[b:b + 1])
        for name in ("z", "y", "s1", "s2", "ybar", "gz", "d"):
            for l in range(len(widths) - 1):
                got = net.intermediate(name, l, 40)[b]
                want = ref.intermediate(name, l, 1)[0]
                if np.abs(want).max() == 0:
                    assert np.abs(got).max() == 0, (name, l)
                else:
                    assert orc.rel_err(got, want) <= 1e-13, (name, l, b)


@pytest.mark.parametrize("widths,hid,fin", [([5, 7, 4], "tanh", "softmax"), ([784, 512, 512, 10], "tanh", "linear"),
                                             ([20, 64, 48, 3], "softplus", "sigmoid"), ([3, 2], "sigmoid", "tanh")])
def test_forward_trace_matches_oracle(widths, hid, fin):
    """forward_trace (nn.cpp:127-146): per-layer z and y of the device
    forward chain against the oracle restatement; the last y is the forward
    output (softmax applied)."""
    net = gb.random_net(widths, hid, fin, 12)
    ref = orc.NeuralNet([orc.Layer(*net.layer(l)) for l in range(net.layer_count)])
    x = np.random.default_rng(1).uniform(-1, 1, widths[0])
    zs, ys = net.forward_trace(x)
    rz, ry = ref.forward_trace(x)
    assert len(zs) == len(rz) == net.layer_count
    for l in range(net.layer_count):
        assert orc.rel_err(zs[l], rz[l]) <= 1e-13, ("z", l)
        assert orc.rel_err(ys[l], ry[l]) <= 1e-13, ("y", l)
    assert np.array_equal(ys[-1], net.forward(x))
    with pytest.raises(gb.ArgumentError):
        net.forward_trace(x[:-1])


# one-tile points with a batch that fills the GPU: every hidden layer's
# curvature in one multi-segment SYRK launch (nt_syrk_segs_kernel) -- up to
# four nonlinear hidden layers, a linear hidden layer skipped, and five
# (beyond the segment limit: the per-layer SYRKs)
SEG_NETS = [
    ([40, 64, 48, 1], "tanh", "sigmoid", 21),
    ([30, 32, 32, 32, 32, 2], "sigmoid", "linear", 22),
    ([30, 32, 32, 32, 32, 32, 2], "softplus", "tanh", 23),
    ([112, 50, 3], "tanh", "softmax", 24),
]


@pytest.mark.parametrize("widths,hid,fin,seed", SEG_NETS)
def test_multi_segment_syrk_batches(widths, hid, fin, seed):
    net = gb.random_net(widths, hid, fin, seed).bind_device(0)
    ref = to_oracle(net)
    rng = np.random.default_rng(seed)
    B = 300  # >= the SM count
    X = rng.uniform(-1, 1, (B, widths[0]))
    L = rng.normal(size=(B, widths[-1]))
    Y, J, H = net.oracle_batched(X, L)
    for k in (0, 1, 150, B - 1):
        assert orc.rel_err(Y[k], ref.forward(X[k])) <= TOL
        assert orc.rel_err(J[k], ref.jacobian(X[k])) <= TOL
        assert orc.rel_err(H[k], ref.lagrangian_hessian(X[k], L[k])) <= TOL
        assert np.array_equal(H[k], H[k].T)


def test_multi_segment_syrk_matches_per_layer():
    """The one-launch curvature against the per-layer SYRKs
    (GBOPT_SYRK_FUSE=0, separate process): same values to rounding."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import json, sys; sys.path.insert(0, %r)\n"
        "import numpy as np, paper_2509_22462_b200 as gb\n"
        "net = gb.random_net([40, 64, 48, 1], 'tanh', 'sigmoid', 21).bind_device(0)\n"
        "rng = np.random.default_rng(5)\n"
        "X = rng.uniform(-1, 1, (300, 40)); L = rng.normal(size=(300, 1))\n"
        "print(json.dumps(net.oracle_batched(X, L)[2][::37].tolist()))\n" % root)
    outs = []
    for v in ("1", "0"):
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                           env=dict(os.environ, GBOPT_SYRK_FUSE=v))
        assert r.returncode == 0, r.stderr
        outs.append(np.array(json.loads(r.stdout.strip().splitlines()[-1])))
    assert orc.rel_err(outs[0], outs[1]) <= 1e-13


def test_fused_reductions_are_bitwise_identical():
    """The single-point launch savings -- per-layer SYRK partials gathered in
    one launch (GBOPT_SYRK_GATHER), the adjoint chunk reduction in the sweep's
    last CTA (GBOPT_ADJ_FUSE) -- add in the same order as the separate
    reductions: Y, J, H (full and packed) bit for bit, separate processes."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import json, sys; sys.path.insert(0, %r)\n"
        "import numpy as np, paper_2509_22462_b200 as gb\n"
        "out = []\n"
        "for widths, hid, fin, B in (([784, 512, 512, 10], 'tanh', 'linear', 1),\n"
        "                            ([130, 200, 150, 12], 'softplus', 'sigmoid', 3),\n"
        "                            ([40, 64, 64, 64, 20], 'sigmoid', 'softmax', 2)):\n"
        "    net = gb.random_net(widths, hid, fin, 5).bind_device(0)\n"
        "    rng = np.random.default_rng(6)\n"
        "    X = rng.uniform(-1, 1, (B, widths[0])); L = rng.normal(size=(B, widths[-1]))\n"
        "    Y, J, H = net.oracle_batched(X, L)\n"
        "    out += [Y.tolist(), J.tolist(), H.tolist()]\n"
        "    out.append(net.oracle_lower(X[0], L[0])[2].tolist())\n"
        "print(json.dumps(out))\n" % root)
    outs = []
    for env in ({}, {"GBOPT_SYRK_GATHER": "0"}, {"GBOPT_ADJ_FUSE": "0"}, {"GBOPT_SYRK_GATHER": "0", "GBOPT_ADJ_FUSE": "0"}):
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                           env=dict(os.environ, **env))
        assert r.returncode == 0, r.stderr
        outs.append([np.array(a) for a in json.loads(r.stdout.strip().splitlines()[-1])])
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            assert np.array_equal(a, b)


def test_s0_pass_batch_beyond_grid_y_limit():
    """S_0 = T_0 diag(sigma'_0) materialised for a wide second layer with
    points x n_pad > 65535 rows (the grid-y limit of one launch)."""
    net = gb.random_net([784, 2048, 2048, 10], "softplus", "linear", 31).bind_device(0)
    ref = to_oracle(net)
    rng = np.random.default_rng(31)
    B = 90  # 90 x 784 = 70560 rows
    X = rng.uniform(0, 1, (B, 784))
    L = rng.normal(size=(B, 10))
    Y, J, H = net.oracle_batched(X, L)
    for k in (0, 89):
        assert orc.rel_err(Y[k], ref.forward(X[k])) <= TOL
        assert orc.rel_err(J[k], ref.jacobian(X[k])) <= TOL
        assert orc.rel_err(H[k], ref.lagrangian_hessian(X[k], L[k])) <= TOL


def test_batch_above_chunk_limit():
    """70000 contingency-style points in one call (> DeviceNet::kMaxChunk and
    > the 65535 grid-y/z limit of the per-point launches): consecutive
    sub-batches, every point still matches the oracle."""
    net = gb.random_net([8, 16, 16, 1], "tanh", "sigmoid", 37).bind_device(0)
    ref = to_oracle(net)
    rng = np.random.default_rng(37)
    B = 70000
    X = rng.normal(1.0, 0.1, (B, 8))
    L = rng.uniform(0, 1, (B, 1))
    Y, J, H = net.oracle_batched(X, L)
    for k in (0, 32767, 32768, 65535, 65536, B - 1):
        assert orc.rel_err(Y[k], ref.forward(X[k])) <= TOL
        assert orc.rel_err(J[k], ref.jacobian(X[k])) <= TOL
        assert orc.rel_err(H[k], ref.lagrangian_hessian(X[k], L[k])) <= TOL
