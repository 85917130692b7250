"""GPU parity against the REFERENCE'S OWN nn.cpp (oracle/_ref, built from
/root/reference/proj/src unmodified; see oracle/ref.py and
tests/test_ref_pin.py for how that build is itself pinned).

Two legs:
  * committed golden outputs of the reference (tests/golden/ref_nets.npz):
    the nets and points of proj/tests/test_nn.cpp, the 25 nets of
    acceptance criterion 1 (acceptance.cpp:86-128), two c4 contingencies;
  * the reference build evaluated live on the GPU box's host, at full
    BASELINE sizes: c1, c4 (32 contingencies of one batched call), c5 (two
    points of a batched call), the c2 shape with tanh hidden layers (nn.cpp
    has no softplus), and four c3-shaped points (tanh).

Bar (north_star): per array and per point max|GPU - REF| / max|REF| <= 1e-10.
"""
import os

import numpy as np
import pytest

from conftest import has_gpu
from oracle import gbopt_oracle as o
from oracle import ref

pytestmark = pytest.mark.gpu

TOL = 1e-10
HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
G = np.load(os.path.join(HERE, "ref_nets.npz"))
SMALL = sorted({k.split("/")[0] for k in G.files if k.endswith("/W0")})

if has_gpu():
    import paper_2509_22462_b200 as gb
    from paper_2509_22462_b200 import configs


@pytest.fixture(autouse=True)
def _need_gpu():
    if not has_gpu():
        pytest.skip("no GPU")


def assert_close(got, want, what):
    if np.abs(want).max() == 0:
        assert np.abs(got).max() <= 1e-14, what
    else:
        e = o.rel_err(got, want)
        assert e <= TOL, (what, e)


def device_net(layers):
    return gb.NeuralNet.from_layers([w for w, _, _ in layers], [b for _, b, _ in layers],
                                    [a for _, _, a in layers]).bind_device(0)


@pytest.mark.parametrize("name", SMALL)
def test_gpu_matches_reference_golden(name):
    acts = [int(a) for a in G[f"{name}/acts"]]
    layers = [(G[f"{name}/W{l}"], G[f"{name}/b{l}"], acts[l]) for l in range(len(acts))]
    net = device_net(layers)
    X, Lam = G[f"{name}/X"], G[f"{name}/Lam"]
    Y, J, H = net.oracle_batched(X, Lam)
    for i in range(X.shape[0]):
        assert_close(Y[i], G[f"{name}/Y"][i], ("y", name, i))
        assert_close(J[i], G[f"{name}/J"][i], ("J", name, i))
        assert_close(H[i], G[f"{name}/H"][i], ("H", name, i))
        assert np.array_equal(H[i], H[i].T)
        # single-point entry points of the C ABI
        y1, j1, h1 = net.oracle(X[i], Lam[i])
        assert_close(y1, G[f"{name}/Y"][i], ("y1", name))
        assert_close(j1, G[f"{name}/J"][i], ("J1", name))
        assert_close(h1, G[f"{name}/H"][i], ("H1", name))
        assert_close(net.jacobian(X[i]), G[f"{name}/J"][i], ("J reverse", name))
        assert_close(net.lagrangian_gradient(X[i], Lam[i]), G[f"{name}/G"][i], ("g", name))
        if f"{name}/H2" in G.files:
            assert_close(net.lagrangian_hessian(X[i], G[f"{name}/Lam2"][i]), G[f"{name}/H2"][i], ("H2", name))


def test_gpu_matches_reference_golden_c4():
    p = configs.make("c4", batch=2)
    net = p.net.bind_device(0)
    Y, J, H = net.oracle_batched(p.X, p.Lam)
    for i in range(2):
        assert_close(Y[i], G["c4_pts/Y"][i], "y")
        assert_close(J[i], G["c4_pts/J"][i], "J")
        assert_close(H[i], G["c4_pts/H"][i], "H")


needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not shipped")


@needs_ref
@pytest.mark.parametrize("name,batch,check,hidden", [
    ("c1", 1, 1, None),
    ("c4", 32, 32, None),
    ("c5", 2, 2, None),
    ("c2", 1, 1, ref.TANH),
    ("c3", 4, 4, ref.TANH),
])
def test_gpu_matches_reference_build_full_size(name, batch, check, hidden):
    ref.set_threads(os.cpu_count() or 1)
    wl = ref.make_config(name, batch=batch, hidden=hidden)
    rn = wl.net()
    net = device_net(wl.layers)
    Y, J, H = net.oracle_batched(wl.X, wl.Lam)
    RY, RJ, RH = rn.oracle_batched(wl.X[:check], wl.Lam[:check])
    worst = [0.0, 0.0, 0.0]
    for i in range(check):
        for k, (got, want) in enumerate(((Y[i], RY[i]), (J[i], RJ[i]), (H[i], RH[i]))):
            assert_close(got, want, (name, i, "yJH"[k]))
            worst[k] = max(worst[k], o.rel_err(got, want))
        assert np.array_equal(H[i], H[i].T)
    print(f"{name}: max rel err vs reference nn.cpp  y {worst[0]:.2e}  J {worst[1]:.2e}  H {worst[2]:.2e}")


@needs_ref
def test_gpu_forward_and_gradient_match_reference_build_c2_shape():
    """The standalone forward (line-search residual) and the lambda-gradient
    (nn.cpp:113-125, 172-196) on the 109M-parameter shape."""
    ref.set_threads(os.cpu_count() or 1)
    wl = ref.make_config("c2", batch=1, hidden=ref.TANH)
    rn = wl.net()
    net = device_net(wl.layers)
    x, lam = wl.X[0], wl.Lam[0]
    assert_close(net.forward(x), rn.forward(x), "forward")
    assert_close(net.lagrangian_gradient(x, lam), rn.lagrangian_gradient(x, lam), "gradient")
    assert_close(net.jacobian(x), rn.jacobian(x), "jacobian (reverse mode)")
    z_ref, y_ref = rn.forward_trace(x)
    z_gpu, y_gpu = net.forward_trace(x)
    for l in range(len(z_ref)):
        assert_close(z_gpu[l], z_ref[l], ("z", l))
        assert_close(y_gpu[l], y_ref[l], ("y", l))


@needs_ref
def test_gpu_loads_reference_written_gbnn(tmp_path):
    """f2: a file written by the reference's save_weights (nn_io.cpp:223-247)
    is loaded by the product and evaluated on the device."""
    rn = ref.RefNet.random([40, 64, 64, 6], ref.SIGMOID, ref.SOFTMAX, 123)
    p = str(tmp_path / "ref.gbnn")
    rn.save(p)
    net = gb.load_weights(p).bind_device(0)
    rng = np.random.default_rng(0)
    X, Lam = rng.uniform(-1, 1, (3, 40)), rng.normal(0, 1, (3, 6))
    Y, J, H = net.oracle_batched(X, Lam)
    RY, RJ, RH = rn.oracle_batched(X, Lam)
    for i in range(3):
        assert_close(Y[i], RY[i], "y")
        assert_close(J[i], RJ[i], "J")
        assert_close(H[i], RH[i], "H")
