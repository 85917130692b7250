"""Edge cases of the device oracle: degenerate widths, ragged n (padding
boundaries of the 112-row tiles), saturated activations, zero multipliers,
wide single layers, batch edge sizes -- each against the CPU oracle."""
import numpy as np
import pytest

from conftest import has_gpu
from oracle import gbopt_oracle as orc

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(autouse=True)
def _gpu():
    if not has_gpu():
        pytest.skip("no GPU")


def ref_of(net):
    return orc.NeuralNet([orc.Layer(*net.layer(l)) for l in range(net.layer_count)])


def check(net, X, L):
    ref = ref_of(net)
    Y, J, H = net.oracle_batched(X, L)
    for b in range(X.shape[0]):
        ry, rj, rh = ref.forward(X[b]), ref.jacobian(X[b]), ref.lagrangian_hessian(X[b], L[b])
        assert orc.rel_err(Y[b], ry) <= TOL
        assert orc.rel_err(J[b], rj) <= TOL if np.abs(rj).max() > 0 else np.abs(J[b]).max() <= 1e-300
        if np.abs(rh).max() > 0:
            assert orc.rel_err(H[b], rh) <= TOL
        else:
            assert np.abs(H[b]).max() <= 1e-14
        assert np.array_equal(H[b], H[b].T)


@pytest.mark.parametrize("widths", [[1, 1], [1, 3, 1], [2, 1, 2], [1, 5, 5, 1], [3, 1, 1, 1, 2]])
def test_degenerate_widths(widths):
    import paper_2509_22462_b200 as gb
    for hid, fin in (("tanh", "sigmoid"), ("softplus", "softmax"), ("sigmoid", "linear")):
        net = gb.random_net(widths, hid, fin, 13)
        rng = np.random.default_rng(1)
        check(net, rng.uniform(-2, 2, (3, widths[0])), rng.uniform(-1, 1, (3, widths[-1])))


@pytest.mark.parametrize("n", [111, 112, 113, 223, 225, 336, 785])
def test_ragged_input_dims_around_tile_boundaries(n):
    import paper_2509_22462_b200 as gb
    net = gb.random_net([n, 130, 129, 7], "tanh", "softplus", n)
    rng = np.random.default_rng(n)
    check(net, rng.uniform(-1, 1, (2, n)), rng.normal(0, 1, (2, 7)))


def test_hidden_widths_around_tile_boundaries():
    import paper_2509_22462_b200 as gb
    net = gb.random_net([40, 127, 128, 129, 255, 257, 3], "sigmoid", "tanh", 5)
    rng = np.random.default_rng(5)
    check(net, rng.uniform(-1, 1, (3, 40)), rng.normal(0, 1, (3, 3)))


def test_saturated_activations_and_zero_multipliers():
    """In deep saturation the reference's own formula sigma' = 1 - tanh(z)^2
    (nn.cpp:55) is at the rounding level (tanh(z) rounds to +-1 within an
    ulp), so two correct FP64 implementations agree only absolutely there:
    derivatives are checked to 1e-15 absolute, y relatively."""
    import paper_2509_22462_b200 as gb
    net = gb.random_net([6, 8, 8, 3], "tanh", "sigmoid", 2)
    X = np.array([[80.0, -90.0, 50.0, 70.0, -60.0, 100.0]])
    L = np.array([[0.7, -1.2, 0.3]])
    ref = ref_of(net)
    Y, J, H = net.oracle_batched(X, L)
    assert orc.rel_err(Y[0], ref.forward(X[0])) <= TOL
    assert np.abs(J[0] - ref.jacobian(X[0])).max() <= 1e-15
    assert np.abs(H[0] - ref.lagrangian_hessian(X[0], L[0])).max() <= 1e-15
    assert np.array_equal(H[0], H[0].T)
    # lambda = 0 => H = 0 exactly; unsaturated point: the usual relative bar
    X2 = np.array([[0.1, 0.2, -0.3, 0.0, 0.5, -0.4]])
    _, _, H0 = net.oracle_batched(X2, np.zeros((1, 3)))
    assert np.all(H0 == 0.0)
    check(net, X2, np.array([[0.7, -1.2, 0.3]]))
    # softplus: the stable formulas keep relative accuracy on both tails
    sp = gb.random_net([5, 6, 2], "softplus", "linear", 3)
    check(sp, np.array([[700.0, -700.0, 30.0, -40.0, 1e-3]]), np.array([[1.0, -1.0]]))


def test_wide_output_single_layer_and_softmax():
    import paper_2509_22462_b200 as gb
    rng = np.random.default_rng(9)
    for fin in ("sigmoid", "softmax", "linear", "tanh"):
        net = gb.random_net([17, 150], "tanh", fin, 4)
        check(net, rng.uniform(-1, 1, (2, 17)), rng.normal(0, 1, (2, 150)))
    net = gb.random_net([17, 64, 150], "tanh", "softmax", 4)
    check(net, rng.uniform(-1, 1, (2, 17)), rng.normal(0, 1, (2, 150)))


@pytest.mark.parametrize("B", [1, 2, 31, 32, 33, 113])
def test_batch_sizes_around_gemm_threshold(B):
    """The forward/adjoint switch from GEMV sweeps to batched GEMMs at 32
    points, and the 112-row tiles of the batched GEMMs."""
    import paper_2509_22462_b200 as gb
    net = gb.random_net([20, 48, 36, 4], "softplus", "sigmoid", 8)
    rng = np.random.default_rng(B)
    X = rng.uniform(-1, 1, (B, 20))
    L = rng.normal(0, 1, (B, 4))
    ref = ref_of(net)
    Y, J, H = net.oracle_batched(X, L)
    for b in sorted({0, B // 2, B - 1}):
        assert orc.rel_err(Y[b], ref.forward(X[b])) <= TOL
        assert orc.rel_err(J[b], ref.jacobian(X[b])) <= TOL
        assert orc.rel_err(H[b], ref.lagrangian_hessian(X[b], L[b])) <= TOL


def test_workspace_growth_and_reuse():
    """Growing the batch reallocates the workspace; results stay identical."""
    import paper_2509_22462_b200 as gb
    net = gb.random_net([30, 40, 5], "tanh", "linear", 1)
    rng = np.random.default_rng(0)
    X = rng.uniform(-1, 1, (50, 30))
    L = rng.normal(0, 1, (50, 5))
    a = net.oracle_batched(X[:3], L[:3])
    net.oracle_batched(X, L)
    b = net.oracle_batched(X[:3], L[:3])
    for u, v in zip(a, b):
        assert np.array_equal(u, v)
