"""Committed golden fixtures (tests/golden/make_golden.py): the oracle must
reproduce them bit-for-bit, the C++ library must regenerate their weights
bit-for-bit, and the GPU oracle must match them to the 1e-10 parity bar."""
import os

import numpy as np
import pytest

from conftest import has_gpu
from oracle import gbopt_oracle as o

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
G = np.load(os.path.join(HERE, "small_nets.npz"))
NAMES = sorted({k.split("/")[0] for k in G.files})


def case(name):
    meta = G[f"{name}/meta"]
    widths = [int(v) for v in meta[:-3]]
    hid, fin, seed = (int(v) for v in meta[-3:])
    layers = [o.Layer(G[f"{name}/W{l}"], G[f"{name}/b{l}"], hid if l + 1 < len(widths) - 1 else fin)
              for l in range(len(widths) - 1)]
    return widths, hid, fin, seed, layers


@pytest.mark.parametrize("name", NAMES)
def test_oracle_reproduces_golden(name):
    widths, hid, fin, seed, layers = case(name)
    net = o.NeuralNet(layers)
    for i, (x, lam) in enumerate(zip(G[f"{name}/X"], G[f"{name}/Lam"])):
        assert np.array_equal(net.forward(x), G[f"{name}/Y"][i])
        assert np.array_equal(net.jacobian(x), G[f"{name}/J"][i])
        assert np.array_equal(net.lagrangian_hessian(x, lam), G[f"{name}/H"][i])
        assert np.array_equal(net.lagrangian_gradient(x, lam), G[f"{name}/G"][i])


@pytest.mark.parametrize("name", NAMES)
def test_library_regenerates_golden_weights(name):
    import paper_2509_22462_b200 as gb
    widths, hid, fin, seed, layers = case(name)
    names = {v: k for k, v in gb.ACTIVATIONS.items()}
    net = gb.random_net(widths, names[hid], names[fin], seed)
    for l, lay in enumerate(layers):
        w, b, a = net.layer(l)
        assert np.array_equal(w, lay.weight) and np.array_equal(b, lay.bias) and a == lay.activation


def test_golden_gbnn_file_loads():
    import paper_2509_22462_b200 as gb
    net = gb.load_weights(os.path.join(HERE, "valid_2x2_tanh.gbnn"))
    w, b, a = net.layer(0)
    assert w[0, 1] == 0.25 and w[1, 0] == 0.5 and a == gb.TANH


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_matches_golden(name):
    if not has_gpu():
        pytest.skip("no GPU")
    import paper_2509_22462_b200 as gb
    widths, hid, fin, seed, layers = case(name)
    net = gb.NeuralNet.from_layers([l.weight for l in layers], [l.bias for l in layers], [l.activation for l in layers])
    Y, J, H = net.oracle_batched(G[f"{name}/X"], G[f"{name}/Lam"])
    for i in range(Y.shape[0]):
        assert o.rel_err(Y[i], G[f"{name}/Y"][i]) <= 1e-10
        assert o.rel_err(J[i], G[f"{name}/J"][i]) <= 1e-10
        ref_h = G[f"{name}/H"][i]
        if np.abs(ref_h).max() > 0:
            assert o.rel_err(H[i], ref_h) <= 1e-10
        else:
            assert np.abs(H[i]).max() <= 1e-14
        g = net.lagrangian_gradient(G[f"{name}/X"][i], G[f"{name}/Lam"][i])
        assert o.rel_err(g, G[f"{name}/G"][i]) <= 1e-10
