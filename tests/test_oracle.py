"""Pins the CPU oracle (oracle/gbopt_oracle.py) against the reference's own
tests for this path -- known answers, finite differences and properties from
proj/tests/test_nn.cpp, proj/tests/acceptance.cpp (criterion 1) and
proj/tests/test_nn_io.cpp -- and against a second, independent formulation
(the SYRK form the GPU implements).  The reference itself cannot be built
here (Eigen3 absent), so these are the pins.
"""
import numpy as np
import pytest

from oracle import gbopt_oracle as o


def single_layer(w, b, act):
    return o.NeuralNet([o.Layer(np.asarray(w, float), np.asarray(b, float), act)])


def rv(rng, n, lo=-1.0, hi=1.0):
    return np.array([rng.uniform(lo, hi) for _ in range(n)])


# ---- PRNG (prng.hpp:11-23; test_util.hpp:16-22) --------------------------
def test_mt19937_64_known_answer():
    # C++ standard [rand.predef]: the 10000th output of a default-constructed
    # std::mt19937_64 is 9981545732273789042.
    m = o.Mt19937_64(5489)
    for _ in range(9999):
        m()
    assert m() == 9981545732273789042


def test_uniform01_mapping():
    m = o.Mt19937_64(7)
    p = o.Prng(7)
    for _ in range(100):
        raw = m()
        assert p.uniform01() == (raw >> 11) * 2.0 ** -53


# ---- known answers (test_nn.cpp) -----------------------------------------
def test_known_answers():
    nn = single_layer(np.eye(2), np.zeros(2), o.LINEAR)
    x = np.array([0.3, -0.7])
    assert np.abs(nn.forward(x) - x).max() == 0.0                      # 30-36
    nn = single_layer(np.eye(3), np.zeros(3), o.TANH)
    assert np.abs(nn.forward(np.zeros(3))).max() == 0.0                  # 38-42
    nn = single_layer(np.zeros((4, 4)), np.zeros(4), o.SOFTMAX)
    y = nn.forward(np.random.default_rng(3).uniform(-5, 5, 4))
    assert np.allclose(y, 0.25, rtol=1e-14, atol=0)                      # 44-50
    rng = o.Prng(17)
    w = np.array([[rng.uniform(-1, 1) for _ in range(5)] for _ in range(3)])
    nn = single_layer(w, rv(rng, 3), o.LINEAR)
    assert np.abs(nn.jacobian(rv(rng, 5)) - w).max() == 0.0              # 80-87
    nn = single_layer(np.eye(4), np.zeros(4), o.TANH)
    assert np.abs(nn.jacobian(np.zeros(4)) - np.eye(4)).max() == 0.0     # 89-94
    lin = o.random_net([4, 5, 3], o.LINEAR, o.LINEAR, 9)
    assert np.abs(lin.lagrangian_hessian(rv(rng, 4), rv(rng, 3))).max() <= 1e-14  # 151-158
    nn = single_layer(np.eye(3), np.zeros(3), o.TANH)
    assert np.abs(nn.lagrangian_hessian(np.zeros(3), np.array([1.0, 0, 0]))).max() == 0.0  # 160-167
    v, d1, d2 = o.activation_elementwise(o.SIGMOID, np.zeros(3))          # 229-243
    assert np.all(v == 0.5) and np.all(d1 == 0.25) and np.abs(d2).max() <= 1e-16
    v, d1, d2 = o.activation_elementwise(o.TANH, np.zeros(3))
    assert np.all(v == 0) and np.all(d1 == 1) and np.all(d2 == 0)


def test_softmax_huge_preactivations():
    # test_nn.cpp:52-68
    rng = np.random.default_rng(11)
    for _ in range(10):
        nn = single_layer(np.eye(5) * 10.0, np.full(5, 720.0), o.SOFTMAX)
        y = nn.forward(rng.uniform(0, 3, 5))
        assert np.isfinite(y).all() and abs(y.sum() - 1) <= 1e-12 and (y > 0).all() and (y < 1).all()


def test_forward_deterministic():
    nn = o.random_net([6, 8, 4], o.TANH, o.SOFTMAX, 21)
    x = np.random.default_rng(4).uniform(-1, 1, 6)
    assert np.array_equal(nn.forward(x), nn.forward(x))


# ---- finite-difference agreement -----------------------------------------
def test_jacobian_fd_spec_case():
    nn = o.random_net([5, 7, 4], o.TANH, o.TANH, 1234)                   # test_nn.cpp:96-108
    rng = np.random.default_rng(55)
    for _ in range(20):
        x = rng.uniform(-2, 2, 5)
        assert np.abs(nn.jacobian(x) - o.fd_jacobian(nn.forward, x, 1e-5)).max() <= 1e-6


@pytest.mark.parametrize("hid,fin,seed", [(o.TANH, o.SOFTMAX, 2), (o.SIGMOID, o.TANH, 3), (o.SIGMOID, o.SOFTMAX, 4),
                                          (o.TANH, o.LINEAR, 5), (o.LINEAR, o.LINEAR, 6), (o.SOFTPLUS, o.LINEAR, 7),
                                          (o.SOFTPLUS, o.SOFTMAX, 8)])
def test_jacobian_fd_mixes(hid, fin, seed):
    nn = o.random_net([4, 6, 6, 3], hid, fin, seed)                       # test_nn.cpp:110-133
    x = np.random.default_rng(seed).uniform(-1.5, 1.5, 4)
    assert np.abs(nn.jacobian(x) - o.fd_jacobian(nn.forward, x, 1e-5)).max() <= 1e-6


def test_hessian_fd_contraction():
    nn = o.random_net([4, 6, 3], o.TANH, o.TANH, 4321)                   # test_nn.cpp:169-186
    rng = np.random.default_rng(12)
    x, lam = rng.uniform(-1, 1, 4), rng.uniform(-2, 2, 3)
    expected = sum(lam[i] * o.fd_hessian(lambda v, i=i: nn.forward(v)[i], x, 1e-4) for i in range(3))
    assert np.abs(nn.lagrangian_hessian(x, lam) - expected).max() <= 1e-5


@pytest.mark.parametrize("hid,fin", [(o.SIGMOID, o.SOFTMAX), (o.SOFTPLUS, o.SIGMOID), (o.TANH, o.SOFTPLUS)])
def test_hessian_fd_of_gradient(hid, fin):
    nn = o.random_net([5, 8, 7, 4], hid, fin, 999)                       # test_nn.cpp:188-200
    rng = np.random.default_rng(13)
    x, lam = rng.uniform(-1, 1, 5), rng.uniform(-1, 1, 4)
    fd = o.fd_jacobian(lambda v: nn.lagrangian_gradient(v, lam), x, 1e-6)
    assert np.abs(nn.lagrangian_hessian(x, lam) - 0.5 * (fd + fd.T)).max() <= 1e-7


def test_hessian_linear_in_lambda_and_symmetric():
    nn = o.random_net([4, 7, 5], o.TANH, o.SOFTMAX, 31)                  # test_nn.cpp:202-216
    rng = np.random.default_rng(14)
    x, l1, l2 = rng.uniform(-1, 1, 4), rng.uniform(-1, 1, 5), rng.uniform(-1, 1, 5)
    a, b = 0.37, -2.25
    hc = nn.lagrangian_hessian(x, a * l1 + b * l2)
    assert np.abs(hc - (a * nn.lagrangian_hessian(x, l1) + b * nn.lagrangian_hessian(x, l2))).max() <= 1e-12
    assert np.abs(hc - hc.T).max() == 0.0


def test_gradient_is_jt_lambda():
    nn = o.random_net([6, 9, 4], o.TANH, o.SOFTMAX, 41)                  # test_nn.cpp:218-227
    rng = np.random.default_rng(15)
    x, lam = rng.uniform(-1, 1, 6), rng.uniform(-1, 1, 4)
    assert np.abs(nn.lagrangian_gradient(x, lam) - nn.jacobian(x).T @ lam).max() <= 1e-13


def test_acceptance_criterion1():
    """acceptance.cpp:86-128 on the oracle: 25 nets, J <= 1e-6, H <= 1e-5,
    multiplier linearity <= 1e-12."""
    rng = np.random.default_rng(2026)
    hiddens = [o.LINEAR, o.TANH, o.SIGMOID]
    je = he = le = 0.0
    for k in range(25):
        depth = 1 + k % 5
        widths = [int(2 + rng.integers(0, 11)) for _ in range(depth + 1)]
        nn = o.random_net(widths, hiddens[k % 3], o.SOFTMAX, 4000 + k)
        x = rng.uniform(-0.9, 0.9, widths[0])
        lam = rng.uniform(-1, 1, widths[-1])
        je = max(je, np.abs(nn.jacobian(x) - o.fd_jacobian(nn.forward, x, 1e-5)).max())
        h = nn.lagrangian_hessian(x, lam)
        he = max(he, np.abs(h - o.fd_hessian(lambda p: lam @ nn.forward(p), x, 1e-4)).max())
        lam2 = rng.uniform(-1, 1, widths[-1])
        le = max(le, np.abs(nn.lagrangian_hessian(x, lam + 2.5 * lam2) - (h + 2.5 * nn.lagrangian_hessian(x, lam2))).max())
    assert je <= 1e-6 and he <= 1e-5 and le <= 1e-12


@pytest.mark.parametrize("seed", range(12))
def test_syrk_form_agrees_with_reference_algorithm(seed):
    """The SYRK formulation the GPU implements equals the reference's
    forward-over-reverse Hessian (nn.cpp:198-292) to rounding."""
    rng = np.random.default_rng(seed)
    L = 1 + seed % 4
    widths = [int(rng.integers(2, 30)) for _ in range(L + 1)]
    acts = [o.LINEAR, o.TANH, o.SIGMOID, o.SOFTPLUS]
    fin = [o.LINEAR, o.TANH, o.SIGMOID, o.SOFTMAX, o.SOFTPLUS][seed % 5]
    nn = o.random_net(widths, acts[seed % 4], fin, 100 + seed)
    x, lam = rng.uniform(-1, 1, widths[0]), rng.normal(0, 1, widths[-1])
    assert o.rel_err(nn.lagrangian_hessian_syrk(x, lam), nn.lagrangian_hessian(x, lam)) <= 1e-13


def test_softplus_extension_formulas():
    z = np.linspace(-40, 40, 161)
    v, d1, d2 = o.activation_elementwise(o.SOFTPLUS, z)
    assert np.allclose(v, np.logaddexp(0, z), rtol=1e-15, atol=1e-300)
    assert np.allclose(d1, 1 / (1 + np.exp(-z)), rtol=1e-14, atol=1e-300)
    fd2 = (o.activation_elementwise(o.SOFTPLUS, z + 1e-6)[1] - o.activation_elementwise(o.SOFTPLUS, z - 1e-6)[1]) / 2e-6
    assert np.abs(d2 - fd2).max() <= 1e-8


def test_random_net_deterministic_and_bounded():
    a = o.random_net([6, 10, 3], o.TANH, o.SOFTMAX, 7)                   # test_nn.cpp:294-312
    b = o.random_net([6, 10, 3], o.TANH, o.SOFTMAX, 7)
    c = o.random_net([6, 10, 3], o.TANH, o.SOFTMAX, 8)
    for la, lb in zip(a.layers, b.layers):
        assert np.array_equal(la.weight, lb.weight) and np.array_equal(la.bias, lb.bias)
        bound = 1 / np.sqrt(la.weight.shape[1])
        assert np.abs(la.weight).max() <= bound and np.abs(la.bias).max() <= bound
    assert np.abs(a.layers[0].weight - c.layers[0].weight).max() > 0
    assert a.param_count == 6 * 10 + 10 + 10 * 3 + 3


def test_validation_errors():
    with pytest.raises(o.StructuralError):
        o.NeuralNet([])
    with pytest.raises(o.StructuralError):
        o.NeuralNet([o.Layer(np.eye(3, 2), np.zeros(3)), o.Layer(np.eye(2, 4), np.zeros(2))])
    with pytest.raises(o.StructuralError):
        o.NeuralNet([o.Layer(np.eye(3), np.zeros(2))])
    with pytest.raises(o.StructuralError):
        o.NeuralNet([o.Layer(np.eye(3), np.zeros(3), o.SOFTMAX), o.Layer(np.eye(3), np.zeros(3))])
    w = np.eye(2)
    w[0, 0] = np.nan
    with pytest.raises(o.NumericError):
        o.NeuralNet([o.Layer(w, np.zeros(2))])
    nn = o.random_net([4, 3], o.TANH, o.TANH, 1)
    with pytest.raises(o.StructuralError):
        nn.forward(np.zeros(5))
    with pytest.raises(o.StructuralError):
        nn.jacobian(np.zeros(3))
    with pytest.raises(o.StructuralError):
        nn.lagrangian_hessian(np.zeros(4), np.zeros(4))


# ---- GBNN v1 (nn_io.cpp; test_nn_io.cpp) ----------------------------------
def valid_file_bytes():
    import struct
    b = b"GBNN" + struct.pack("<III", 1, 1, 2) + struct.pack("<IB", 2, 1)
    b += np.array([0.25 * i for i in range(4)], "<f8").tobytes() + np.array([-1.0 * i for i in range(2)], "<f8").tobytes()
    return b


def test_gbnn_oracle_reader():
    nn = o.load_weights_bytes(valid_file_bytes())
    assert nn.input_dim == 2 and nn.output_dim == 2 and nn.layers[0].activation == o.TANH
    assert nn.layers[0].weight[0, 1] == 0.25 and nn.layers[0].weight[1, 0] == 0.5
    net = o.random_net([5, 9, 7, 3], o.TANH, o.SOFTMAX, 2024)
    back = o.load_weights_bytes(o.save_weights_bytes(net))
    for a, b in zip(net.layers, back.layers):
        assert np.array_equal(a.weight, b.weight) and np.array_equal(a.bias, b.bias) and a.activation == b.activation
    vb = valid_file_bytes()
    for bad, err in [(b"", o.FormatError), (b"X" + vb[1:], o.FormatError), (vb[:4] + b"\x02" + vb[5:], o.FormatError),
                     (vb[:-19], o.TruncatedError), (vb[:-9], o.TruncatedError), (vb[:14], o.TruncatedError),
                     (vb + b"\0", o.FormatError), (vb[:20] + b"\x09" + vb[21:], o.FormatError)]:
        with pytest.raises(err):
            o.load_weights_bytes(bad)
