"""The reference's own oracle, compiled from its sources (oracle/_ref).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
the CPU legs of ``bench.py`` (``cpu_baseline`` and ``--impl reference``) may
import this module, and only as the checker / the timed CPU arm.  The
product package never imports it.

``oracle/_ref/libgbopt_ref.so`` is ``proj/src/nn.cpp``, ``nn_io.cpp`` and
``linalg.cpp`` from /root/reference, compiled unmodified by
``oracle/ref_build/Makefile`` against a restated Eigen subset
(``oracle/ref_build/eigen_subset``; Eigen3 is not installed here or on the
GPU box) with OpenBLAS for the matrix products.  The same build runs the
reference's own doctest suites (``oracle/_ref/ref_tests``: test_nn.cpp,
test_nn_io.cpp, test_linalg.cpp, all green), which is what pins the shim.

This module also restates the five BASELINE.json workloads (``make_config``)
with the reference's Prng, so the CPU arms never load the product library
to obtain their inputs; tests/test_ref_pin.py checks bit-identity with the
product's ``configs.make``.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libgbopt_ref.so")
TESTS_PATH = os.path.join(HERE, "_ref", "ref_tests")

LINEAR, TANH, SIGMOID, SOFTMAX, SOFTPLUS = 0, 1, 2, 3, 4

_i64p = ctypes.POINTER(ctypes.c_int64)
_dp = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p


class RefError(Exception):
    """A non-zero gbopt_status from the reference build (code, message)."""

    def __init__(self, status: int, msg: str):
        super().__init__(f"[{status}] {msg}")
        self.status = status
        self.msg = msg


_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run `make -C oracle/ref_build` "
                               "(needs /root/reference; __graft_entry__.build() does it)")
        L = ctypes.CDLL(LIB_PATH)
        L.gbref_last_error.restype = ctypes.c_char_p
        L.gbref_set_threads.argtypes = [ctypes.c_int]
        L.gbref_net_create.argtypes = [ctypes.c_int, _i64p, ctypes.POINTER(ctypes.c_uint8), _dp,
                                       ctypes.POINTER(_vp)]
        L.gbref_net_random.argtypes = [ctypes.c_int, _i64p, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_uint64, ctypes.POINTER(_vp)]
        L.gbref_net_load.argtypes = [ctypes.c_char_p, ctypes.POINTER(_vp)]
        L.gbref_net_save.argtypes = [_vp, ctypes.c_char_p]
        L.gbref_net_free.argtypes = [_vp]
        L.gbref_net_free.restype = None
        L.gbref_net_dims.argtypes = [_vp, _i64p]
        L.gbref_net_dims.restype = None
        L.gbref_net_layer.argtypes = [_vp, ctypes.c_int, _i64p, _i64p, ctypes.POINTER(ctypes.c_int),
                                      _dp, _dp]
        for name in ("gbref_forward", "gbref_jacobian"):
            getattr(L, name).argtypes = [_vp, _dp, ctypes.c_int64, _dp]
        L.gbref_forward_trace.argtypes = [_vp, _dp, ctypes.c_int64, _dp, _dp]
        for name in ("gbref_lagrangian_gradient", "gbref_lagrangian_hessian"):
            getattr(L, name).argtypes = [_vp, _dp, ctypes.c_int64, _dp, ctypes.c_int64, _dp]
        L.gbref_oracle_batched.argtypes = [_vp, ctypes.c_int64, _dp, _dp, _dp, _dp, _dp, ctypes.c_int]
        L.gbref_activation_elementwise.argtypes = [ctypes.c_int, _dp, ctypes.c_int64, _dp, _dp, _dp]
        L.gbref_ldlt_factor.argtypes = [_dp, ctypes.c_int64, ctypes.c_int, ctypes.POINTER(_vp),
                                        ctypes.POINTER(ctypes.c_int)]
        L.gbref_ldlt_solve.argtypes = [_vp, _dp, ctypes.c_int64, _dp]
        L.gbref_ldlt_reconstruct.argtypes = [_vp, _dp]
        L.gbref_ldlt_free.argtypes = [_vp]
        L.gbref_ldlt_free.restype = None
        L.gbref_prng_new.argtypes = [ctypes.c_uint64]
        L.gbref_prng_new.restype = _vp
        L.gbref_prng_free.argtypes = [_vp]
        L.gbref_prng_free.restype = None
        for name in ("gbref_prng_uniform", "gbref_prng_normal"):
            getattr(L, name).argtypes = [_vp, ctypes.c_double, ctypes.c_double, ctypes.c_int64, _dp]
            getattr(L, name).restype = None
        _lib = L
    return _lib


def _check(st: int):
    if st != 0:
        raise RefError(st, lib().gbref_last_error().decode())


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def set_threads(n: int) -> int:
    """OpenBLAS threads used inside the reference's matrix products."""
    return lib().gbref_set_threads(int(n))


class RefNet:
    """gbopt::NeuralNet (nn.hpp:40-81) from the reference's own nn.cpp."""

    def __init__(self, handle):
        self._h = handle
        dims = np.zeros(4, dtype=np.int64)
        lib().gbref_net_dims(self._h, dims.ctypes.data_as(_i64p))
        self.input_dim, self.output_dim, self.layer_count, self.param_count = (int(v) for v in dims)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.gbref_net_free(self._h)
            self._h = None

    # ---- construction
    @classmethod
    def from_layers(cls, layers) -> "RefNet":
        """layers: iterable of (W out x in, b, act)."""
        layers = [(_f64(w), _f64(b).reshape(-1), int(a)) for w, b, a in layers]
        widths = np.array([layers[0][0].shape[1]] + [w.shape[0] for w, _, _ in layers], dtype=np.int64)
        acts = np.array([a for _, _, a in layers], dtype=np.uint8)
        params = np.concatenate([np.concatenate([w.reshape(-1), b]) for w, b, _ in layers])
        h = _vp()
        _check(lib().gbref_net_create(len(layers), widths.ctypes.data_as(_i64p),
                                      acts.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)),
                                      _ptr(params), ctypes.byref(h)))
        return cls(h)

    @classmethod
    def random(cls, widths, hidden: int, final: int, seed: int) -> "RefNet":
        """random_net (nn.cpp:336-367)."""
        w = np.array(widths, dtype=np.int64)
        h = _vp()
        _check(lib().gbref_net_random(len(w), w.ctypes.data_as(_i64p), hidden, final, seed, ctypes.byref(h)))
        return cls(h)

    @classmethod
    def load(cls, path: str) -> "RefNet":
        """load_weights (nn_io.cpp:144-221, JSON mirror for *.json)."""
        h = _vp()
        _check(lib().gbref_net_load(path.encode(), ctypes.byref(h)))
        return cls(h)

    def save(self, path: str) -> None:
        _check(lib().gbref_net_save(self._h, path.encode()))

    def layer(self, l: int):
        r, c, a = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int()
        _check(lib().gbref_net_layer(self._h, l, ctypes.byref(r), ctypes.byref(c), ctypes.byref(a), None, None))
        w = np.empty((r.value, c.value))
        b = np.empty(r.value)
        _check(lib().gbref_net_layer(self._h, l, ctypes.byref(r), ctypes.byref(c), ctypes.byref(a),
                                     _ptr(w), _ptr(b)))
        return w, b, a.value

    # ---- the oracle (nn.cpp:113-292)
    def forward(self, x) -> np.ndarray:
        x = _f64(x)
        y = np.empty(self.output_dim)
        _check(lib().gbref_forward(self._h, _ptr(x), x.size, _ptr(y)))
        return y

    def forward_trace(self, x):
        x = _f64(x)
        widths = [self.layer(l)[0].shape[0] for l in range(self.layer_count)]
        z = np.empty(sum(widths))
        y = np.empty(sum(widths))
        _check(lib().gbref_forward_trace(self._h, _ptr(x), x.size, _ptr(z), _ptr(y)))
        cuts = np.cumsum(widths)[:-1]
        return np.split(z, cuts), np.split(y, cuts)

    def jacobian(self, x) -> np.ndarray:
        x = _f64(x)
        j = np.empty((self.output_dim, self.input_dim))
        _check(lib().gbref_jacobian(self._h, _ptr(x), x.size, _ptr(j)))
        return j

    def lagrangian_gradient(self, x, lam) -> np.ndarray:
        x, lam = _f64(x), _f64(lam)
        g = np.empty(self.input_dim)
        _check(lib().gbref_lagrangian_gradient(self._h, _ptr(x), x.size, _ptr(lam), lam.size, _ptr(g)))
        return g

    def lagrangian_hessian(self, x, lam) -> np.ndarray:
        x, lam = _f64(x), _f64(lam)
        h = np.empty((self.input_dim, self.input_dim))
        _check(lib().gbref_lagrangian_hessian(self._h, _ptr(x), x.size, _ptr(lam), lam.size, _ptr(h)))
        return h

    def oracle_batched(self, X, Lam, threads: int = 1, want=(True, True, True)):
        """forward + jacobian + lagrangian_hessian per point (the three
        reduced-space callbacks, formulations.cpp:317-340)."""
        X, Lam = _f64(X), _f64(Lam)
        B, n, m = X.shape[0], self.input_dim, self.output_dim
        Y = np.empty((B, m)) if want[0] else None
        J = np.empty((B, m, n)) if want[1] else None
        H = np.empty((B, n, n)) if want[2] else None
        _check(lib().gbref_oracle_batched(self._h, B, _ptr(X), _ptr(Lam),
                                          _ptr(Y) if Y is not None else None,
                                          _ptr(J) if J is not None else None,
                                          _ptr(H) if H is not None else None, int(threads)))
        return Y, J, H


def activation_elementwise(kind: int, z):
    """nn.cpp:43-72 (value, d1, d2)."""
    z = _f64(z)
    y, d1, d2 = np.empty_like(z), np.empty_like(z), np.empty_like(z)
    _check(lib().gbref_activation_elementwise(kind, _ptr(z), z.size, _ptr(y), _ptr(d1), _ptr(d2)))
    return y, d1, d2


# ---------------------------------------------------------------- LDL^T
class RefLdlt:
    """LdltFactorization (linalg.hpp:24-78) from the reference's linalg.cpp."""

    def __init__(self, a, keep_input: bool = True):
        a = _f64(a)
        n = a.shape[0]
        self.n = n
        h = _vp()
        inertia = (ctypes.c_int * 3)()
        _check(lib().gbref_ldlt_factor(_ptr(a), n, 1 if keep_input else 0, ctypes.byref(h), inertia))
        self._h = h
        self.inertia = (inertia[0], inertia[1], inertia[2])

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.gbref_ldlt_free(self._h)
            self._h = None

    def solve(self, b) -> np.ndarray:
        b = _f64(b)
        x = np.empty(self.n)
        _check(lib().gbref_ldlt_solve(self._h, _ptr(b), self.n, _ptr(x)))
        return x

    def reconstruct(self) -> np.ndarray:
        a = np.empty((self.n, self.n))
        _check(lib().gbref_ldlt_reconstruct(self._h, _ptr(a)))
        return a


# ------------------------------------------------------------- workloads
class Prng:
    """The reference Prng (prng.hpp:11-23) + the Appendix-A Box-Muller."""

    def __init__(self, seed: int):
        self._g = lib().gbref_prng_new(seed)

    def __del__(self):
        if getattr(self, "_g", None) and _lib is not None:
            _lib.gbref_prng_free(self._g)
            self._g = None

    def uniform(self, lo, hi, n) -> np.ndarray:
        out = np.empty(int(n))
        lib().gbref_prng_uniform(self._g, lo, hi, out.size, _ptr(out))
        return out

    def normal(self, mean, sd, n) -> np.ndarray:
        out = np.empty(int(n))
        lib().gbref_prng_normal(self._g, mean, sd, out.size, _ptr(out))
        return out


# BASELINE.json configs[0..4], restated independently of the product's
# paper_2509_22462_b200/configs.py (semantics: SURVEY Appendix A):
# one Prng per seed; per layer W row-major then b; then x (point-major), then
# lambda; unspecified biases 0 without draws; c5's output linear.
XU, XN, NF = "xavier_uniform", "xavier_normal", "normal_fanin"
CONFIGS = {
    "c1": dict(widths=[784, 512, 512, 10], hidden=TANH, final=LINEAR, init=XU, bias=(-0.05, 0.05),
               seed=0, batch=1, x=("uniform", 0.0, 1.0), lam=("normal", 0.0, 1.0)),
    "c2": dict(widths=[784] + [5120] * 5 + [10], hidden=SOFTPLUS, final=LINEAR, init=XN, bias=(0.0, 0.0),
               seed=1, batch=1, x=("uniform", 0.0, 1.0), lam=("normal", 0.0, 1.0)),
    "c3": dict(widths=[784] + [5120] * 5 + [10], hidden=SOFTPLUS, final=LINEAR, init=XN, bias=(0.0, 0.0),
               seed=1, input_seed=2, batch=64, x=("uniform", 0.0, 1.0), lam=("normal", 0.0, 1.0)),
    "c4": dict(widths=[108, 1024, 1024, 1024, 1], hidden=TANH, final=SIGMOID, init=XU, bias=(0.0, 0.0),
               seed=3, batch=4096, x=("normal", 1.0, 0.1), lam=("uniform", 0.0, 1.0)),
    "c5": dict(widths=[784] + [1024] * 20 + [10], hidden=SIGMOID, final=LINEAR, init=NF, bias=(0.0, 0.0),
               seed=4, batch=16, x=("uniform", 0.0, 1.0), lam=("normal", 0.0, 1.0)),
}


@dataclass
class RefWorkload:
    name: str
    widths: List[int]
    layers: list          # [(W, b, act)]
    X: np.ndarray
    Lam: np.ndarray

    def net(self) -> RefNet:
        """The reference NeuralNet (rejects softplus, which nn.cpp lacks)."""
        return RefNet.from_layers(self.layers)


def _draw(rng: Prng, dist, n):
    kind, a, b = dist
    return rng.uniform(a, b, n) if kind == "uniform" else rng.normal(a, b, n)


def make_config(name: str, batch: Optional[int] = None, hidden: Optional[int] = None) -> RefWorkload:
    """Weights and points of BASELINE config `name`; `batch` keeps the first
    B points of the full seeded stream; `hidden` overrides the hidden
    activation (same bytes otherwise) -- e.g. the c2 shape with tanh, which
    the reference's nn.cpp can evaluate."""
    c = CONFIGS[name]
    widths = c["widths"]
    rng = Prng(c["seed"])
    layers = []
    L = len(widths) - 1
    for l in range(1, L + 1):
        fi, fo = widths[l - 1], widths[l]
        if c["init"] == XU:
            bound = np.sqrt(6.0 / (fi + fo))
            w = rng.uniform(-bound, bound, fo * fi)
        elif c["init"] == XN:
            w = rng.normal(0.0, np.sqrt(2.0 / (fi + fo)), fo * fi)
        else:
            w = rng.normal(0.0, 1.0 / np.sqrt(fi), fo * fi)
        lo, hi = c["bias"]
        b = np.full(fo, lo) if lo == hi else rng.uniform(lo, hi, fo)
        act = c["final"] if l == L else (c["hidden"] if hidden is None else hidden)
        layers.append((w.reshape(fo, fi), b, act))
    if "input_seed" in c:
        rng = Prng(c["input_seed"])
    B, n, m = c["batch"], widths[0], widths[-1]
    X = _draw(rng, c["x"], B * n).reshape(B, n)
    Lam = _draw(rng, c["lam"], B * m).reshape(B, m)
    if batch is not None:
        X, Lam = X[:batch].copy(), Lam[:batch].copy()
    return RefWorkload(name, list(widths), layers, X, Lam)


def flops_per_eval(widths, acts) -> float:
    """SURVEY §8d algorithmic flops of one (y, J, H) evaluation."""
    n = widths[0]
    f = 0.0
    for l in range(1, len(widths)):
        mac = widths[l] * widths[l - 1]
        f += 2 * mac
        if l >= 2:
            f += 2 * mac + 2 * mac * n
        if acts[l - 1] != LINEAR:
            f += widths[l] * n * (n + 1)
    return f
