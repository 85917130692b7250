"""J-only calls run the reverse-mode sweep (m seed vectors per point, like
the reference jacobian, nn.cpp:148-170); J from the fused oracle comes from
the forward tangents.  Both must match the oracle and each other."""
import numpy as np
import pytest

from conftest import has_gpu
from oracle import gbopt_oracle as orc

pytestmark = pytest.mark.gpu

CASES = [([5, 7, 4], "tanh", "tanh"), ([4, 6, 6, 3], "sigmoid", "softmax"), ([7, 4], "softplus", "softmax"),
         ([9, 33, 17, 40], "tanh", "sigmoid"), ([130, 200, 150, 12], "softplus", "linear"),
         ([784, 512, 512, 10], "tanh", "linear"), ([108, 1024, 1024, 1], "tanh", "sigmoid")]


@pytest.mark.parametrize("widths,hid,fin", CASES)
def test_reverse_mode_jacobian(widths, hid, fin):
    if not has_gpu():
        pytest.skip("no GPU")
    import paper_2509_22462_b200 as gb
    net = gb.random_net(widths, hid, fin, 5)
    ref = orc.NeuralNet([orc.Layer(*net.layer(l)) for l in range(net.layer_count)])
    rng = np.random.default_rng(3)
    X = rng.uniform(-1, 1, (5, widths[0]))
    L = rng.uniform(-1, 1, (5, widths[-1]))
    for x in X[:2]:
        j = net.jacobian(x)
        assert orc.rel_err(j, ref.jacobian(x)) <= 1e-12
    # batched J-only (reverse mode over 5 * m seed vectors) vs fused (tangents)
    _, Jr, _ = net.oracle_batched(X, None, want_h=False)
    _, Jt, _ = net.oracle_batched(X, L)
    for b in range(5):
        assert orc.rel_err(Jr[b], ref.jacobian(X[b])) <= 1e-12
        assert orc.rel_err(Jr[b], Jt[b]) <= 1e-12
