"""Generates tests/golden/ref_nets.npz from the REFERENCE ITSELF: every output
in it is computed by /root/reference/proj/src/nn.cpp (compiled unmodified
into oracle/_ref/libgbopt_ref.so by oracle/ref_build/Makefile), on nets made
by the reference's own random_net (nn.cpp:336-367).

Cases (inputs drawn exactly as the reference's tests draw them, with the
pure-Python mt19937_64 of oracle/gbopt_oracle.py standing in for
std::mt19937_64 + testutil::random_vec, test_util.hpp:16-30):
  * tnn_*   -- the nets and points of proj/tests/test_nn.cpp:96-227;
  * acc1_*  -- the 25 nets of acceptance criterion 1 (acceptance.cpp:86-128),
               with x, lambda and the second multiplier lambda2;
  * c4_pts  -- two points of BASELINE config c4 at full size (weights are
               regenerated from the seed by the tests, so only the outputs
               are stored).

Run in the build container (needs /root/reference for oracle/_ref):
    make -C oracle/ref_build && python tests/golden/make_ref_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import gbopt_oracle as o  # noqa: E402
from oracle import ref  # noqa: E402


class Rng:
    """std::mt19937_64 + testutil::uniform (test_util.hpp:16-22)."""

    def __init__(self, seed):
        self.eng = o.Mt19937_64(seed)

    def raw(self):
        return self.eng()

    def vec(self, n, lo=-1.0, hi=1.0):
        return np.array([lo + (hi - lo) * (float(self.eng() >> 11) * 2.0 ** -53) for _ in range(n)])


def record(out, name, net, widths, acts, seed, X, Lam, Lam2=None, store_weights=True):
    out[f"{name}/meta"] = np.array(list(widths) + [seed], dtype=np.int64)
    out[f"{name}/acts"] = np.array(acts, dtype=np.int64)
    if store_weights:
        for l in range(net.layer_count):
            w, b, _ = net.layer(l)
            out[f"{name}/W{l}"] = w
            out[f"{name}/b{l}"] = b
    X, Lam = np.atleast_2d(X), np.atleast_2d(Lam)
    out[f"{name}/X"] = X
    out[f"{name}/Lam"] = Lam
    out[f"{name}/Y"] = np.array([net.forward(x) for x in X])
    out[f"{name}/J"] = np.array([net.jacobian(x) for x in X])
    out[f"{name}/H"] = np.array([net.lagrangian_hessian(x, l) for x, l in zip(X, Lam)])
    out[f"{name}/G"] = np.array([net.lagrangian_gradient(x, l) for x, l in zip(X, Lam)])
    if Lam2 is not None:
        Lam2 = np.atleast_2d(Lam2)
        out[f"{name}/Lam2"] = Lam2
        out[f"{name}/H2"] = np.array([net.lagrangian_hessian(x, l) for x, l in zip(X, Lam2)])


def main():
    T, S, SM, LI = ref.TANH, ref.SIGMOID, ref.SOFTMAX, ref.LINEAR
    out = {}

    def rnet(widths, hid, fin, seed):
        return ref.RefNet.random(widths, hid, fin, seed), [hid] * (len(widths) - 2) + [fin]

    # test_nn.cpp:96-111 -- tanh 5-7-4, seed 1234, points from rng(55) on [-2, 2]
    net, acts = rnet([5, 7, 4], T, T, 1234)
    r = Rng(55)
    X = np.array([r.vec(5, -2.0, 2.0) for _ in range(3)])
    Lam = Rng(1055).vec(4 * 3).reshape(3, 4)
    record(out, "tnn_fd_spec", net, [5, 7, 4], acts, 1234, X, Lam)
    # test_nn.cpp:113-133 -- activation mixes on 4-6-6-3, points from rng(66)
    r = Rng(66)
    for hid, fin, seed in [(T, SM, 2), (S, T, 3), (S, SM, 4), (T, LI, 5), (LI, LI, 6)]:
        net, acts = rnet([4, 6, 6, 3], hid, fin, seed)
        x = r.vec(4, -1.5, 1.5)
        lam = Rng(2000 + seed).vec(3)
        record(out, f"tnn_mix_{seed}", net, [4, 6, 6, 3], acts, seed, x, lam)
    # test_nn.cpp:164-180 -- 4-6-3 tanh, seed 4321, rng(12)
    net, acts = rnet([4, 6, 3], T, T, 4321)
    r = Rng(12)
    x = r.vec(4)
    lam = r.vec(3, -2.0, 2.0)
    record(out, "tnn_fd_contraction", net, [4, 6, 3], acts, 4321, x, lam)
    # test_nn.cpp:182-196 -- 5-8-7-4 sigmoid/softmax, seed 999, rng(13)
    net, acts = rnet([5, 8, 7, 4], S, SM, 999)
    r = Rng(13)
    x = r.vec(5)
    lam = r.vec(4)
    record(out, "tnn_sigmoid_softmax", net, [5, 8, 7, 4], acts, 999, x, lam)
    # test_nn.cpp:198-212 -- 4-7-5 tanh/softmax, seed 31, rng(14): x, l1, l2
    net, acts = rnet([4, 7, 5], T, SM, 31)
    r = Rng(14)
    x = r.vec(4)
    l1 = r.vec(5)
    l2 = r.vec(5)
    record(out, "tnn_linearity", net, [4, 7, 5], acts, 31, x, l1, l2)
    # test_nn.cpp:214-223 -- 6-9-4 tanh/softmax, seed 41, rng(15)
    net, acts = rnet([6, 9, 4], T, SM, 41)
    r = Rng(15)
    x = r.vec(6)
    lam = r.vec(4)
    record(out, "tnn_grad_jt", net, [6, 9, 4], acts, 41, x, lam)

    # acceptance.cpp:86-128 -- criterion 1
    r = Rng(2026)
    hiddens = [LI, T, S]
    for k in range(25):
        depth = 1 + k % 5
        widths = [2 + r.raw() % 11 for _ in range(depth + 1)]
        net, acts = rnet(widths, hiddens[k % 3], SM, 4000 + k)
        x = r.vec(widths[0], -0.9, 0.9)
        lam = r.vec(widths[-1])
        lam2 = r.vec(widths[-1])
        record(out, f"acc1_{k:02d}", net, widths, acts, 4000 + k, x, lam, lam2)

    # BASELINE config c4 (full-size net), two contingencies
    wl = ref.make_config("c4", batch=2)
    net = wl.net()
    acts = [a for _, _, a in wl.layers]
    record(out, "c4_pts", net, wl.widths, acts, 3, wl.X, wl.Lam, store_weights=False)

    np.savez_compressed(os.path.join(HERE, "ref_nets.npz"), **out)
    print("wrote", len({k.split('/')[0] for k in out}), "cases")


if __name__ == "__main__":
    main()
