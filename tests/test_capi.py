"""CPU tests of the C-ABI library (no GPU compute): exports, host-side
generation, GBNN I/O and its error classes, argument/validation errors.

Restates proj/tests/test_nn_io.cpp, the network cases of
proj/tests/test_capi.cpp and the validation cases of proj/tests/test_nn.cpp
against libgbopt_b200.so.
"""
import os
import re
import struct

import numpy as np
import pytest

import paper_2509_22462_b200 as gb
from oracle import gbopt_oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "gbopt_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gbopt_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    import ctypes
    lib = ctypes.CDLL(gb.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_version_and_device_count():
    assert "sm_100a" in gb.version()
    assert gb.device_count() >= 0


# ---- generation -------------------------------------------------------------
def test_prng_matches_reference_generator():
    p = gb.Prng(5489)
    r = p.raw(10000)
    assert int(r[-1]) == 9981545732273789042
    m = orc.Mt19937_64(42)
    p = gb.Prng(42)
    u = p.uniform(-2.0, 3.0, 50)
    for v in u:
        assert v == -2.0 + 5.0 * ((m() >> 11) * 2.0 ** -53)


def test_prng_normal_is_box_muller_pairs():
    m = orc.Mt19937_64(9)
    z = gb.Prng(9).normal(1.0, 2.0, 6)
    for i in range(3):
        u1 = 1.0 - (m() >> 11) * 2.0 ** -53
        u2 = (m() >> 11) * 2.0 ** -53
        r = np.sqrt(-2 * np.log(u1))
        assert abs(z[2 * i] - (1 + 2 * r * np.cos(2 * np.pi * u2))) <= 1e-14
        assert abs(z[2 * i + 1] - (1 + 2 * r * np.sin(2 * np.pi * u2))) <= 1e-14


@pytest.mark.parametrize("widths,hid,fin,seed", [([6, 10, 3], "tanh", "softmax", 7), ([5, 9, 7, 3], "sigmoid", "linear", 1),
                                                 ([4, 2], "softplus", "tanh", 123)])
def test_random_net_bit_identical_to_reference_semantics(widths, hid, fin, seed):
    net = gb.random_net(widths, hid, fin, seed)
    ref = orc.random_net(widths, gb.ACTIVATIONS[hid], gb.ACTIVATIONS[fin], seed)
    assert net.param_count == ref.param_count
    for l in range(net.layer_count):
        w, b, a = net.layer(l)
        assert np.array_equal(w, ref.layers[l].weight) and np.array_equal(b, ref.layers[l].bias)
        assert a == ref.layers[l].activation


def test_random_net_ex_initialisers():
    rng = gb.Prng(3)
    net = gb.random_net_ex(rng, [50, 40, 30], gb.TANH, gb.LINEAR, gb.INIT_XAVIER_UNIFORM, -0.05, 0.05)
    w, b, _ = net.layer(0)
    assert np.abs(w).max() <= np.sqrt(6 / 90) and np.abs(b).max() <= 0.05 and np.abs(b).max() > 0
    rng = gb.Prng(3)
    net = gb.random_net_ex(rng, [400, 300], gb.SOFTPLUS, gb.LINEAR, gb.INIT_XAVIER_NORMAL, 0.0, 0.0)
    w, b, _ = net.layer(0)
    assert abs(w.std() - np.sqrt(2 / 700)) < 0.01 * np.sqrt(2 / 700) and np.all(b == 0)
    rng = gb.Prng(4)
    net = gb.random_net_ex(rng, [400, 300], gb.SIGMOID, gb.LINEAR, gb.INIT_NORMAL_FANIN, 0.0, 0.0)
    assert abs(net.layer(0)[0].std() - 1 / 20) < 0.01 / 20
    # draw order: W row-major then b, then the next layer (nn.cpp:354-362)
    m = orc.Mt19937_64(11)
    net = gb.random_net_ex(gb.Prng(11), [3, 2], gb.TANH, gb.TANH, gb.INIT_XAVIER_UNIFORM, -1.0, 1.0)
    w, b, _ = net.layer(0)
    bound = np.sqrt(6 / 5)
    seq = [((m() >> 11) * 2.0 ** -53) for _ in range(8)]
    assert np.array_equal(w.reshape(-1), np.array([-bound + 2 * bound * u for u in seq[:6]]))
    assert np.array_equal(b, np.array([-1 + 2 * u for u in seq[6:]]))


def test_configs_flops_match_survey():
    from paper_2509_22462_b200 import configs
    expect = {"c1": 1.051, "c2": 180.68, "c3": 180.68, "c4": 0.498, "c5": 43.94}
    for k, v in expect.items():
        assert abs(configs.flops(k) / 1e9 - v) / v < 2e-3


def test_config_c1_generation_deterministic():
    from paper_2509_22462_b200 import configs
    a, b = configs.make("c1"), configs.make("c1")
    assert np.array_equal(a.X, b.X) and np.array_equal(a.Lam, b.Lam)
    assert a.net.widths() == [784, 512, 512, 10]
    wa, ba, _ = a.net.layer(0)
    wb, bb, _ = b.net.layer(0)
    assert np.array_equal(wa, wb) and np.array_equal(ba, bb)
    assert 0 <= a.X.min() and a.X.max() < 1


# ---- GBNN I/O (test_nn_io.cpp) ---------------------------------------------
def valid_file_bytes():
    b = b"GBNN" + struct.pack("<III", 1, 1, 2) + struct.pack("<IB", 2, 1)
    b += np.array([0.25 * i for i in range(4)], "<f8").tobytes() + np.array([-1.0 * i for i in range(2)], "<f8").tobytes()
    return b


def write(tmp_path, name, data):
    p = tmp_path / name
    p.write_bytes(data) if isinstance(data, bytes) else p.write_text(data)
    return str(p)


def nets_equal(a, b):
    if a.layer_count != b.layer_count:
        return False
    for l in range(a.layer_count):
        wa, ba, aa = a.layer(l)
        wb, bb, ab = b.layer(l)
        if aa != ab or wa.shape != wb.shape or wa.tobytes() != wb.tobytes() or ba.tobytes() != bb.tobytes():
            return False
    return True


def test_binary_round_trip_bit_exact(tmp_path):
    net = gb.random_net([5, 9, 7, 3], "tanh", "softmax", 2024)
    p = str(tmp_path / "rt.gbnn")
    gb.save_weights(net, p)
    assert nets_equal(net, gb.load_weights(p))
    # the bytes are exactly the GBNN v1 layout (nn_io.cpp:223-247)
    ref = orc.random_net([5, 9, 7, 3], orc.TANH, orc.SOFTMAX, 2024)
    assert open(p, "rb").read() == orc.save_weights_bytes(ref)


def test_json_round_trip_bit_exact(tmp_path):
    net = gb.random_net([4, 6, 2], "sigmoid", "linear", 99)
    p = str(tmp_path / "rt.json")
    gb.save_weights(net, p)
    assert nets_equal(net, gb.load_weights(p))


def test_softplus_code_round_trips(tmp_path):
    net = gb.random_net([4, 6, 2], "softplus", "linear", 5)
    for name in ("sp.gbnn", "sp.json"):
        p = str(tmp_path / name)
        gb.save_weights(net, p)
        assert nets_equal(net, gb.load_weights(p))


def test_handcrafted_file_is_row_major(tmp_path):
    net = gb.load_weights(write(tmp_path, "v.gbnn", valid_file_bytes()))
    assert net.input_dim == 2 and net.output_dim == 2
    w, b, a = net.layer(0)
    assert a == gb.TANH and w[0, 1] == 0.25 and w[1, 0] == 0.5 and b[1] == -1.0


def corrupt_cases():
    vb = valid_file_bytes()
    two_layer_bad_chain = (b"GBNN" + struct.pack("<II", 1, 2) + struct.pack("<IIB", 2, 2, 1) + b"\0" * 48 +
                           struct.pack("<IIB", 2, 3, 0) + b"\0" * 64)
    return [
        ("empty", b"", gb.FormatError),
        ("magic", b"X" + vb[1:], gb.FormatError),
        ("version", vb[:4] + b"\x02" + vb[5:], gb.FormatError),
        ("cut_weights", vb[:len(vb) - 2 * 8 - 3], gb.TruncatedError),
        ("cut_biases", vb[:len(vb) - 9], gb.TruncatedError),
        ("cut_header", vb[:14], gb.TruncatedError),
        ("trailing", vb + b"\0", gb.FormatError),
        ("zero_layers", b"GBNN" + struct.pack("<II", 1, 0), gb.DimensionError),
        ("bad_chain", two_layer_bad_chain, gb.DimensionError),
        ("act_code_9", vb[:20] + b"\x09" + vb[21:], gb.FormatError),
        ("act_code_5", vb[:20] + b"\x05" + vb[21:], gb.FormatError),
        ("zero_rows", b"GBNN" + struct.pack("<II", 1, 1) + struct.pack("<IIB", 0, 2, 1), gb.DimensionError),
    ]


@pytest.mark.parametrize("name,data,err", corrupt_cases())
def test_corrupt_files_raise_distinct_errors(tmp_path, name, data, err):
    with pytest.raises(err):
        gb.load_weights(write(tmp_path, name + ".gbnn", data))


def test_truncation_is_not_a_format_error(tmp_path):
    with pytest.raises(gb.TruncatedError) as e:
        gb.load_weights(write(tmp_path, "t.gbnn", valid_file_bytes()[:14]))
    assert not isinstance(e.value, gb.FormatError)


def test_json_errors(tmp_path):
    bad_bias = ('{"magic": "GBNN", "version": 1, "layers": [{"rows": 2, "cols": 2, "activation": 1, '
                '"weights": [[1.0, 0.0], [0.0, 1.0]], "biases": [0.0]}]}')
    with pytest.raises(gb.DimensionError):
        gb.load_weights(write(tmp_path, "bb.json", bad_bias))
    with pytest.raises(gb.FormatError):
        gb.load_weights(write(tmp_path, "nj.json", "{ definitely not json"))
    with pytest.raises(gb.FormatError):
        gb.load_weights(write(tmp_path, "nm.json", '{"magic": "XXXX", "version": 1, "layers": []}'))
    with pytest.raises(gb.DimensionError):
        gb.load_weights(write(tmp_path, "nl.json", '{"magic": "GBNN", "version": 1, "layers": []}'))
    with pytest.raises(gb.FormatError):
        gb.load_weights(write(tmp_path, "mf.json", '{"magic": "GBNN", "version": 1, "layers": [{"rows": 1}]}'))
    ok = ('{"magic": "GBNN", "version": 1, "layers": [{"rows": 2, "cols": 2, "activation": 1, '
          '"weights": [[1.0, 0.5e-1], [0.0, 1.0]], "biases": [0.0, -2]}]}')
    net = gb.load_weights(write(tmp_path, "ok.json", ok))
    w, b, a = net.layer(0)
    assert w[0, 1] == 0.05 and b[1] == -2.0 and a == gb.TANH


def test_missing_file_is_io_error():
    with pytest.raises(gb.IoError) as e:
        gb.load_weights("/nonexistent/dir/net.gbnn")
    assert type(e.value) is gb.IoError


# ---- C-ABI argument conventions (test_capi.cpp:57-74) ------------------------
def test_argument_and_name_errors():
    import ctypes
    h = ctypes.c_void_p()
    assert gb.gbopt._net_load(None, ctypes.byref(h)) == gb.gbopt.ERR_ARGUMENT
    assert len(gb.last_error()) > 0
    with pytest.raises(gb.StructuralError):
        gb.random_net([4, 3], "tanh", "sideways", 1)
    net = gb.random_net([4, 3], "tanh", "softmax", 1)
    assert gb.last_error() == ""
    with pytest.raises(gb.ArgumentError):
        net.forward(np.zeros(3))          # wrong input length (capi.cpp:168-172)
    with pytest.raises(gb.ArgumentError):
        net.lagrangian_hessian(np.zeros(4), np.zeros(4))
    with pytest.raises(gb.ArgumentError):
        net.oracle_batched(np.zeros((2, 4)), np.zeros((3, 3)))


def test_from_layers_validation():
    with pytest.raises(gb.StructuralError):
        gb.NeuralNet.from_layers([np.eye(3, 2), np.eye(2, 4)], [np.zeros(3), np.zeros(2)], [1, 1])
    with pytest.raises(gb.StructuralError):
        gb.NeuralNet.from_layers([np.eye(3)], [np.zeros(2)], [1])
    with pytest.raises(gb.StructuralError):
        gb.NeuralNet.from_layers([np.eye(3), np.eye(3)], [np.zeros(3), np.zeros(3)], [gb.SOFTMAX, gb.LINEAR])
    w = np.eye(2)
    w[0, 0] = np.nan
    with pytest.raises(gb.NumericError):
        gb.NeuralNet.from_layers([w], [np.zeros(2)], [gb.LINEAR])
    with pytest.raises(gb.StructuralError):
        gb.NeuralNet.from_layers([np.eye(2)], [np.zeros(2)], [7])
    import ctypes
    h = ctypes.c_void_p()
    assert gb.gbopt._net_from_layers(0, None, None, None, None, ctypes.byref(h)) == gb.gbopt.ERR_STRUCTURAL
    net = gb.NeuralNet.from_layers([np.ones((3, 2)), np.ones((1, 3))], [np.zeros(3), np.zeros(1)], [gb.TANH, gb.LINEAR])
    assert net.widths() == [2, 3, 1] and net.param_count == 6 + 3 + 3 + 1


@pytest.mark.skipif(gb.device_count() > 0, reason="checks the no-device error path")
def test_compute_without_device_fails_loudly():
    net = gb.random_net([4, 3], "tanh", "tanh", 1)
    with pytest.raises(gb.DeviceError):
        net.forward(np.zeros(4))
    with pytest.raises(gb.DeviceError):
        net.bind_device(0)
    assert net.device == -1


def test_large_gbnn_round_trip_and_truncation(tmp_path):
    """Payloads >= 16 MB take the parallel pread path (nn_io.cpp): identical
    weights after a round trip, TruncatedError on a cut file."""
    import paper_2509_22462_b200 as gb
    net = gb.random_net([300, 2100, 8], "tanh", "linear", 5)  # 2100 x 300 and 8 x 2100
    big = gb.random_net([2100, 2100, 3], "sigmoid", "linear", 6)  # 35 MB first layer
    for k, n in (("a", net), ("b", big)):
        path = str(tmp_path / f"{k}.gbnn")
        gb.save_weights(n, path)
        back = gb.load_weights(path)
        for l in range(n.layer_count):
            w0, b0, a0 = n.layer(l)
            w1, b1, a1 = back.layer(l)
            assert np.array_equal(w0, w1) and np.array_equal(b0, b1) and a0 == a1
    path = str(tmp_path / "b.gbnn")
    data = open(path, "rb").read()
    cut = str(tmp_path / "cut.gbnn")
    open(cut, "wb").write(data[: len(data) // 2])
    with pytest.raises(gb.TruncatedError):
        gb.load_weights(cut)
