"""Reduced-space embedding callbacks (paper_2509_22462_b200/reduced_space.py)
against the reference's reduced-space tests (proj/tests/test_formulations.cpp:
215-274): residual exactly 0 at the forward image, block derivatives vs
finite differences, and the -lambda sign convention."""
import numpy as np
import pytest

from conftest import has_gpu
from oracle import gbopt_oracle as orc

pytestmark = pytest.mark.gpu


def mixed_net():
    import paper_2509_22462_b200 as gb
    rng = np.random.default_rng(31)
    ws = [rng.uniform(-1, 1, (5, 4)), rng.uniform(-1, 1, (6, 5)), rng.uniform(-1, 1, (3, 6))]
    bs = [rng.uniform(-1, 1, 5), rng.uniform(-1, 1, 6), rng.uniform(-1, 1, 3)]
    return gb.NeuralNet.from_layers(ws, bs, [gb.TANH, gb.SIGMOID, gb.SOFTMAX])


@pytest.fixture(autouse=True)
def _gpu():
    if not has_gpu():
        pytest.skip("no GPU")


def dense_jac(blk, xb):
    rows, cols = blk.jac_pattern()
    J = np.zeros((blk.m, blk.n + blk.m))
    np.add.at(J, (rows, cols), blk.jacobian(xb))
    return J


def dense_hess(blk, xb, lam):
    rows, cols = blk.hess_pattern()
    L = np.zeros((blk.n, blk.n))
    np.add.at(L, (rows, cols), blk.lag_hessian(xb, lam))
    return L + L.T - np.diag(np.diag(L))


def test_residual_zero_at_forward_image():
    from paper_2509_22462_b200.reduced_space import ReducedSpaceBlock
    net = mixed_net()
    blk = ReducedSpaceBlock(net)
    x = np.random.default_rng(32).uniform(-0.4, 0.4, 4)
    xb = np.concatenate([x, net.forward(x)])
    assert np.all(blk.residual(xb) == 0.0)


def test_block_derivatives_match_finite_differences():
    from paper_2509_22462_b200.reduced_space import ReducedSpaceBlock
    net = mixed_net()
    blk = ReducedSpaceBlock(net)
    rng = np.random.default_rng(43)
    xb = rng.uniform(-0.5, 0.5, 7)
    lam = rng.uniform(-1, 1, 3)
    fdj = orc.fd_jacobian(blk.residual, xb, 1e-6)
    assert np.abs(dense_jac(blk, xb) - fdj).max() <= 1e-6
    fdh = orc.fd_hessian(lambda v: lam @ blk.residual(v), xb, 1e-4)
    full = np.zeros((7, 7))
    full[:4, :4] = dense_hess(blk, xb, lam)
    assert np.abs(full - fdh).max() <= 1e-5


def test_multipliers_reach_the_oracle_negated():
    from paper_2509_22462_b200.reduced_space import ReducedSpaceBlock
    net = mixed_net()
    blk = ReducedSpaceBlock(net)
    rng = np.random.default_rng(53)
    xb = rng.uniform(-0.5, 0.5, 7)
    lam = rng.uniform(-1, 1, 3)
    got = dense_hess(blk, xb, lam)
    expected = net.lagrangian_hessian(xb[:4], -lam)
    wrong = net.lagrangian_hessian(xb[:4], lam)
    assert np.abs(got - expected).max() <= 1e-12
    assert np.abs(got + wrong).max() <= 1e-12


def test_non_ascending_inputs_flip_the_pattern_and_caching():
    from paper_2509_22462_b200.reduced_space import ReducedSpaceBlock
    net = mixed_net()
    blk = ReducedSpaceBlock(net, input_vars=[3, 1, 2, 0])
    r, c = blk.hess_pattern()
    # global coordinates stay lower triangular (formulations.cpp:298-312)
    g = np.array([3, 1, 2, 0])
    assert np.all(g[r] >= g[c])
    xb = np.random.default_rng(1).uniform(-0.5, 0.5, 7)
    lam = np.array([0.3, -0.2, 0.9])
    blk.residual(xb)
    blk.jacobian(xb)
    blk.lag_hessian(xb, lam)
    n0 = blk.evaluations
    blk.residual(xb)
    blk.jacobian(xb)
    blk.lag_hessian(xb, lam)
    assert blk.evaluations == n0


@pytest.mark.parametrize("order", [("r", "j", "h"), ("h", "j", "r"), ("j", "h", "r"), ("h", "r", "j")])
def test_callback_values_do_not_depend_on_call_order(order):
    """The reference callbacks are pure functions of x (formulations.cpp:
    317-340 call forward / jacobian / lagrangian_hessian afresh); each cached
    quantity here has one producer, so the values are bitwise independent of
    the order the IPM asks for them."""
    from paper_2509_22462_b200.reduced_space import ReducedSpaceBlock
    import paper_2509_22462_b200 as gb
    net = gb.random_net([30, 40, 40, 4], "tanh", "linear", 5).bind_device(0)
    rng = np.random.default_rng(1)
    xb = rng.uniform(-1, 1, 34)
    lam = rng.uniform(-1, 1, 4)
    ref = ReducedSpaceBlock(net)
    want = {"r": ref.residual(xb), "j": ref.jacobian(xb), "h": ref.lag_hessian(xb, lam)}
    blk = ReducedSpaceBlock(net)
    got = {}
    for c in order:
        got[c] = {"r": lambda: blk.residual(xb), "j": lambda: blk.jacobian(xb),
                  "h": lambda: blk.lag_hessian(xb, lam)}[c]()
    for c in "rjh":
        assert np.array_equal(got[c], want[c]), c
    # and once more after the caches are warm, in reverse
    for c in reversed(order):
        again = {"r": blk.residual(xb), "j": blk.jacobian(xb), "h": blk.lag_hessian(xb, lam)}[c]
        assert np.array_equal(again, want[c])
