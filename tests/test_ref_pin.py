"""Parity pinned to the REFERENCE'S OWN CODE.

oracle/_ref/libgbopt_ref.so is proj/src/{nn,nn_io,linalg}.cpp compiled
unmodified (oracle/ref_build/Makefile, Eigen restated as a subset).  These
CPU tests check, in order:
  1. the reference's own doctest suites (test_nn.cpp, test_nn_io.cpp,
     test_linalg.cpp) pass against that build -- which validates the shims;
  2. the committed golden outputs of the reference (tests/golden/ref_nets.npz,
     make_ref_golden.py) are reproduced by the numpy oracle to 1e-13 and by
     the reference build bit for bit;
  3. the product's generators make the reference's weights and the BASELINE
     workloads bit for bit, and its GBNN reader/writer is byte- and
     error-compatible with nn_io.cpp;
  4. at full BASELINE sizes (c1, c4, c5, and the c2 shape with tanh -- the
     reference has no softplus) the numpy oracle equals the reference build
     to 1e-13;
  5. the reference LDL^T (linalg.cpp) agrees with the f3 oracle's inertia.
The GPU side of the pin is tests/test_gpu_ref_parity.py.
"""
import os
import struct
import subprocess

import numpy as np
import pytest

from oracle import gbopt_oracle as o
from oracle import ref

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
G = np.load(os.path.join(HERE, "ref_nets.npz"))
CASES = sorted({k.split("/")[0] for k in G.files})
SMALL = [c for c in CASES if f"{c}/W0" in G.files]
needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built (make -C oracle/ref_build)")

TOL = 1e-13


def layers_of(name):
    meta = G[f"{name}/meta"]
    widths = [int(v) for v in meta[:-1]]
    acts = [int(a) for a in G[f"{name}/acts"]]
    return widths, acts, int(meta[-1]), [(G[f"{name}/W{l}"], G[f"{name}/b{l}"], acts[l])
                                         for l in range(len(widths) - 1)]


def numpy_net(layers):
    return o.NeuralNet([o.Layer(w, b, a) for w, b, a in layers])


@needs_ref
def test_reference_doctest_suites_pass_against_the_build():
    r = subprocess.run([ref.TESTS_PATH], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "| 0 failed" in r.stdout and "test cases: 52" in r.stdout, r.stdout


@pytest.mark.parametrize("name", SMALL)
def test_numpy_oracle_matches_reference_golden(name):
    _, _, _, layers = layers_of(name)
    net = numpy_net(layers)
    for i, (x, lam) in enumerate(zip(G[f"{name}/X"], G[f"{name}/Lam"])):
        assert o.rel_err(net.forward(x), G[f"{name}/Y"][i]) <= TOL
        assert o.rel_err(net.jacobian(x), G[f"{name}/J"][i]) <= TOL
        h_ref = G[f"{name}/H"][i]
        h = net.lagrangian_hessian(x, lam)
        assert (o.rel_err(h, h_ref) <= TOL) if np.abs(h_ref).max() > 0 else np.abs(h).max() <= 1e-14
        assert o.rel_err(net.lagrangian_gradient(x, lam), G[f"{name}/G"][i]) <= TOL
        if f"{name}/H2" in G.files:
            assert o.rel_err(net.lagrangian_hessian(x, G[f"{name}/Lam2"][i]), G[f"{name}/H2"][i]) <= TOL


@pytest.mark.parametrize("name", SMALL)
def test_product_random_net_regenerates_reference_weights(name):
    import paper_2509_22462_b200 as gb
    widths, acts, seed, layers = layers_of(name)
    names = {v: k for k, v in gb.ACTIVATIONS.items()}
    hidden = acts[0] if len(acts) > 1 else acts[-1]
    net = gb.random_net(widths, names[hidden], names[acts[-1]], seed)
    for l, (w, b, a) in enumerate(layers):
        pw, pb, pa = net.layer(l)
        assert np.array_equal(pw, w) and np.array_equal(pb, b) and pa == a


def test_numpy_oracle_matches_reference_golden_c4_full_size():
    wl = ref.make_config("c4", batch=2) if ref.available() else None
    if wl is None:
        from paper_2509_22462_b200 import configs
        p = configs.make("c4", batch=2)
        layers = [p.net.layer(l) for l in range(p.net.layer_count)]
        X, Lam = p.X, p.Lam
    else:
        layers, X, Lam = wl.layers, wl.X, wl.Lam
    assert np.array_equal(X, G["c4_pts/X"]) and np.array_equal(Lam, G["c4_pts/Lam"])
    net = numpy_net(layers)
    for i in range(2):
        assert o.rel_err(net.forward(X[i]), G["c4_pts/Y"][i]) <= TOL
        assert o.rel_err(net.jacobian(X[i]), G["c4_pts/J"][i]) <= TOL
        assert o.rel_err(net.lagrangian_hessian(X[i], Lam[i]), G["c4_pts/H"][i]) <= TOL


@needs_ref
@pytest.mark.parametrize("name", SMALL)
def test_reference_build_reproduces_its_golden_bitwise(name):
    widths, acts, seed, layers = layers_of(name)
    hidden = acts[0] if len(acts) > 1 else acts[-1]
    net = ref.RefNet.random(widths, hidden, acts[-1], seed)
    for l, (w, b, a) in enumerate(layers):
        rw, rb, ra = net.layer(l)
        assert np.array_equal(rw, w) and np.array_equal(rb, b) and ra == a
    X, Lam = G[f"{name}/X"], G[f"{name}/Lam"]
    Y, J, H = net.oracle_batched(X, Lam)
    assert np.array_equal(Y, G[f"{name}/Y"]) and np.array_equal(J, G[f"{name}/J"])
    assert np.array_equal(H, G[f"{name}/H"])


@needs_ref
@pytest.mark.parametrize("name,batch", [("c1", 1), ("c4", 8), ("c5", 2), ("c3", 3)])
def test_baseline_workloads_identical_to_product(name, batch):
    """The reference-side restatement of BASELINE configs (oracle/ref.py)
    and the product's configs.make produce the same bytes."""
    from paper_2509_22462_b200 import configs
    r = ref.make_config(name, batch=batch)
    p = configs.make(name, batch=batch)
    assert np.array_equal(r.X, p.X) and np.array_equal(r.Lam, p.Lam)
    for l, (w, b, a) in enumerate(r.layers):
        pw, pb, pa = p.net.layer(l)
        assert np.array_equal(pw, w) and np.array_equal(pb, b) and pa == a


@needs_ref
@pytest.mark.parametrize("name,hidden", [("c1", None), ("c4", None), ("c5", None), ("c2", ref.TANH)])
def test_numpy_oracle_equals_reference_at_full_size(name, hidden):
    """Full BASELINE shapes: the restated algorithm and the reference's own
    nn.cpp agree to 1e-13 (one point; c2's shape with tanh hidden layers
    because nn.cpp has no softplus)."""
    wl = ref.make_config(name, batch=1, hidden=hidden)
    rn = wl.net()
    on = numpy_net(wl.layers)
    x, lam = wl.X[0], wl.Lam[0]
    Y, J, H = rn.oracle_batched(wl.X, wl.Lam)
    assert o.rel_err(on.forward(x), Y[0]) <= TOL
    assert o.rel_err(on.jacobian(x), J[0]) <= TOL
    assert o.rel_err(on.lagrangian_hessian(x, lam), H[0]) <= TOL
    assert o.rel_err(on.lagrangian_gradient(x, lam), rn.lagrangian_gradient(x, lam)) <= TOL


@needs_ref
def test_forward_trace_matches_reference():
    net = ref.RefNet.random([7, 9, 8, 3], ref.SIGMOID, ref.SOFTMAX, 5)
    on = numpy_net([net.layer(l) for l in range(3)])
    x = np.linspace(-1, 1, 7)
    zr, yr = net.forward_trace(x)
    zo, yo = on.forward_trace(x)
    for a, b in zip(zr + yr, zo + yo):
        assert o.rel_err(b, a) <= TOL


@needs_ref
@pytest.mark.parametrize("kind", [ref.LINEAR, ref.TANH, ref.SIGMOID])
def test_activation_formulas_match_reference(kind):
    z = np.concatenate([np.linspace(-40, 40, 801), [-1e-300, 0.0, 1e-300, 700.0, -700.0]])
    r = ref.activation_elementwise(kind, z)
    n = o.activation_elementwise(kind, z)
    for a, b in zip(r, n):   # normwise; glibc tanh(-19) and numpy differ by 1 ulp, amplified in 1 - t^2
        assert np.abs(a - b).max() <= 2e-15 * max(np.abs(b).max(), 1e-300)


@needs_ref
def test_reference_rejects_softplus_code():
    """nn.cpp has no softplus (nn.hpp:12-17): the reference build refuses a
    code-4 layer when it evaluates it, which is why c2/c3 are pinned by FD and
    the independent SYRK form instead."""
    net = ref.RefNet.from_layers([(np.eye(2), np.zeros(2), ref.SOFTPLUS)])
    with pytest.raises(ref.RefError) as e:
        net.forward(np.zeros(2))
    assert e.value.status == 1


# ---- GBNN v1 interoperability (nn_io.cpp:144-247) ---------------------------

@needs_ref
@pytest.mark.parametrize("ext", ["gbnn", "json"])
def test_gbnn_files_interchange_with_reference(tmp_path, ext):
    import paper_2509_22462_b200 as gb
    rnet = ref.RefNet.random([6, 11, 5, 3], ref.TANH, ref.SOFTMAX, 77)
    p_ref = str(tmp_path / f"r.{ext}")
    p_prod = str(tmp_path / f"p.{ext}")
    rnet.save(p_ref)
    pnet = gb.load_weights(p_ref)
    for l in range(3):
        rw, rb, ra = rnet.layer(l)
        pw, pb, pa = pnet.layer(l)
        assert rw.tobytes() == pw.tobytes() and rb.tobytes() == pb.tobytes() and ra == pa
    gb.save_weights(pnet, p_prod)
    if ext == "gbnn":
        assert open(p_ref, "rb").read() == open(p_prod, "rb").read()
    back = ref.RefNet.load(p_prod)
    for l in range(3):
        assert back.layer(l)[0].tobytes() == rnet.layer(l)[0].tobytes()


def _corrupt_files():
    vb = (b"GBNN" + struct.pack("<III", 1, 1, 2) + struct.pack("<IB", 2, 1) +
          np.array([0.25 * i for i in range(4)], "<f8").tobytes() + np.array([0.0, -1.0], "<f8").tobytes())
    bad_chain = (b"GBNN" + struct.pack("<II", 1, 2) + struct.pack("<IIB", 2, 2, 1) + b"\0" * 48 +
                 struct.pack("<IIB", 2, 3, 0) + b"\0" * 64)
    return [
        ("empty.gbnn", b""), ("magic.gbnn", b"X" + vb[1:]), ("version.gbnn", vb[:4] + b"\x02" + vb[5:]),
        ("cut_w.gbnn", vb[:len(vb) - 19]), ("cut_b.gbnn", vb[:len(vb) - 9]), ("cut_h.gbnn", vb[:14]),
        ("trail.gbnn", vb + b"\0"), ("zero.gbnn", b"GBNN" + struct.pack("<II", 1, 0)),
        ("chain.gbnn", bad_chain), ("act9.gbnn", vb[:20] + b"\x09" + vb[21:]),
        ("rows0.gbnn", b"GBNN" + struct.pack("<II", 1, 1) + struct.pack("<IIB", 0, 2, 1)),
        ("notjson.json", b"{ definitely not json"),
        ("nomagic.json", b'{"magic": "XXXX", "version": 1, "layers": []}'),
        ("nolayers.json", b'{"magic": "GBNN", "version": 1, "layers": []}'),
        ("missing.json", b'{"magic": "GBNN", "version": 1, "layers": [{"rows": 1}]}'),
        ("biaslen.json", b'{"magic": "GBNN", "version": 1, "layers": [{"rows": 2, "cols": 2, "activation": 1, '
                         b'"weights": [[1.0, 0.0], [0.0, 1.0]], "biases": [0.0]}]}'),
    ]


@needs_ref
@pytest.mark.parametrize("fname,data", _corrupt_files())
def test_loader_errors_match_reference(tmp_path, fname, data):
    """Same gbopt_status class and the same message text as nn_io.cpp."""
    import paper_2509_22462_b200 as gb
    p = str(tmp_path / fname)
    open(p, "wb").write(data)
    with pytest.raises(ref.RefError) as er:
        ref.RefNet.load(p)
    with pytest.raises(gb.GboptError) as ep:
        gb.load_weights(p)
    assert ep.value.status == er.value.status, (str(ep.value), er.value.msg)
    if fname.endswith(".gbnn"):
        assert str(ep.value) == er.value.msg


@needs_ref
def test_missing_file_error_matches_reference():
    import paper_2509_22462_b200 as gb
    with pytest.raises(ref.RefError) as er:
        ref.RefNet.load("/nonexistent/x.gbnn")
    with pytest.raises(gb.GboptError) as ep:
        gb.load_weights("/nonexistent/x.gbnn")
    assert ep.value.status == er.value.status == 4


# ---- dense LDL^T (linalg.cpp) -----------------------------------------------

@needs_ref
@pytest.mark.parametrize("n", [5, 33, 97, 160])
def test_f3_oracle_inertia_matches_reference_ldlt(n):
    from oracle import ldlt_oracle as lo
    rng = np.random.default_rng(n)
    a = rng.uniform(-1, 1, (n, n))
    a = 0.5 * (a + a.T)
    f = ref.RefLdlt(a)
    assert f.inertia == tuple(lo.inertia(a))
    b = rng.uniform(-1, 1, n)
    x = f.solve(b)
    assert np.abs(a @ x - b).max() <= 1e-10 * (1 + np.abs(b).max())
    assert np.abs(f.reconstruct() - a).max() <= 1e-10
