"""Generates tests/golden/small_nets.npz: seeded small nets (weights from the
pure-Python restatement of the reference random_net, nn.cpp:336-367, and
Prng, prng.hpp:11-23) with oracle outputs y, J, H, grad computed by the
reference algorithm restated in oracle/gbopt_oracle.py (nn.cpp:113-292).

These are regression pins of the oracle and cross-language pins of the
generator (the C++ library must regenerate identical weights); they are not
outputs of the reference binary, which cannot be built here.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import gbopt_oracle as o  # noqa: E402

CASES = [
    ("tanh_5_7_4", [5, 7, 4], o.TANH, o.TANH, 1234),
    ("sigmoid_softmax", [5, 8, 7, 4], o.SIGMOID, o.SOFTMAX, 999),
    ("softplus_linear", [12, 16, 16, 3], o.SOFTPLUS, o.LINEAR, 41),
    ("tanh_sigmoid_1out", [9, 20, 20, 20, 1], o.TANH, o.SIGMOID, 3),
    ("linear_linear", [4, 5, 3], o.LINEAR, o.LINEAR, 9),
    ("single_softmax", [7, 4], o.TANH, o.SOFTMAX, 77),
]


def main():
    out = {}
    for name, widths, hid, fin, seed in CASES:
        net = o.random_net(widths, hid, fin, seed)
        rng = o.Prng(seed + 1)
        pts = []
        for _ in range(3):
            x = np.array([rng.uniform(-1.0, 1.0) for _ in range(widths[0])])
            lam = np.array([rng.uniform(-2.0, 2.0) for _ in range(widths[-1])])
            pts.append((x, lam))
        out[f"{name}/meta"] = np.array(widths + [hid, fin, seed], dtype=np.int64)
        for l, lay in enumerate(net.layers):
            out[f"{name}/W{l}"] = lay.weight
            out[f"{name}/b{l}"] = lay.bias
        out[f"{name}/X"] = np.array([p[0] for p in pts])
        out[f"{name}/Lam"] = np.array([p[1] for p in pts])
        out[f"{name}/Y"] = np.array([net.forward(x) for x, _ in pts])
        out[f"{name}/J"] = np.array([net.jacobian(x) for x, _ in pts])
        out[f"{name}/H"] = np.array([net.lagrangian_hessian(x, l) for x, l in pts])
        out[f"{name}/G"] = np.array([net.lagrangian_gradient(x, l) for x, l in pts])
    np.savez_compressed(os.path.join(HERE, "small_nets.npz"), **out)
    # handcrafted GBNN v1 file of proj/tests/test_nn_io.cpp:34-45
    import struct
    b = b"GBNN" + struct.pack("<III", 1, 1, 2) + struct.pack("<IB", 2, 1)
    b += np.array([0.25 * i for i in range(4)], "<f8").tobytes() + np.array([-1.0 * i for i in range(2)], "<f8").tobytes()
    open(os.path.join(HERE, "valid_2x2_tanh.gbnn"), "wb").write(b)
    print("wrote", len(CASES), "cases")


if __name__ == "__main__":
    main()
