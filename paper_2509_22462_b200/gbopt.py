"""Python mirror of the reference ``gbopt::NeuralNet`` oracle API over the
B200 C ABI (``include/gbopt_b200.h``, ``libgbopt_b200.so``).

Method names, argument meaning and error classes follow the reference
C++ interface (``proj/include/gbopt/nn.hpp:40-110``) and its error taxonomy
(``proj/include/gbopt/errors.hpp``); every call goes through the shared
library -- there is no Python or CPU compute path.  If the library has not
been built, importing this module raises ``ImportError``.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GBOPT_LIB") or os.path.join(_HERE, "libgbopt_b200.so")  # GBOPT_LIB: A/B builds

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make -C {_HERE}/csrc` "
        "(or __graft_entry__.build()); there is no fallback path")

_lib = ctypes.CDLL(LIB_PATH)

_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_sz = ctypes.c_size_t
_dp = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p


def _fn(name, restype, *argtypes):
    f = getattr(_lib, name)
    f.restype = restype
    f.argtypes = list(argtypes)
    return f


_status = ctypes.c_int
_last_error = _fn("gbopt_last_error", ctypes.c_char_p)
_version = _fn("gbopt_version", ctypes.c_char_p)
_device_count = _fn("gbopt_device_count", ctypes.c_int)
_prng_new = _fn("gbopt_prng_new", _status, _u64, ctypes.POINTER(_vp))
_prng_free = _fn("gbopt_prng_free", None, _vp)
_prng_raw = _fn("gbopt_prng_raw", _status, _vp, ctypes.POINTER(_u64), _sz)
_prng_uniform = _fn("gbopt_prng_uniform", _status, _vp, ctypes.c_double, ctypes.c_double, _dp, _sz)
_prng_normal = _fn("gbopt_prng_normal", _status, _vp, ctypes.c_double, ctypes.c_double, _dp, _sz)
_net_load = _fn("gbopt_net_load", _status, ctypes.c_char_p, ctypes.POINTER(_vp))
_net_save = _fn("gbopt_net_save", _status, _vp, ctypes.c_char_p)
_net_random = _fn("gbopt_net_random", _status, ctypes.POINTER(_i64), _sz, ctypes.c_char_p, ctypes.c_char_p, _u64,
                  ctypes.POINTER(_vp))
_net_random_ex = _fn("gbopt_net_random_ex", _status, _vp, ctypes.POINTER(_i64), _sz, ctypes.c_int, ctypes.c_int,
                     ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.POINTER(_vp))
_net_from_layers = _fn("gbopt_net_from_layers", _status, _sz, ctypes.POINTER(_i64), ctypes.POINTER(ctypes.c_int32),
                       ctypes.POINTER(_dp), ctypes.POINTER(_dp), ctypes.POINTER(_vp))
_net_free = _fn("gbopt_net_free", None, _vp)
_net_input_dim = _fn("gbopt_net_input_dim", _i64, _vp)
_net_output_dim = _fn("gbopt_net_output_dim", _i64, _vp)
_net_param_count = _fn("gbopt_net_param_count", _i64, _vp)
_net_layer_count = _fn("gbopt_net_layer_count", _i64, _vp)
_net_layer_info = _fn("gbopt_net_layer_info", _status, _vp, _i64, ctypes.POINTER(_i64), ctypes.POINTER(_i64),
                      ctypes.POINTER(ctypes.c_int32))
_net_layer_copy = _fn("gbopt_net_layer_copy", _status, _vp, _i64, _dp, _sz, _dp, _sz)
_net_bind_device = _fn("gbopt_net_bind_device", _status, _vp, ctypes.c_int)
_net_device = _fn("gbopt_net_device", ctypes.c_int, _vp)
_net_forward = _fn("gbopt_net_forward", _status, _vp, _dp, _sz, _dp, _sz)
_net_jacobian = _fn("gbopt_net_jacobian", _status, _vp, _dp, _sz, _dp, _sz)
_net_lag_grad = _fn("gbopt_net_lagrangian_gradient", _status, _vp, _dp, _sz, _dp, _sz, _dp, _sz)
_net_lag_hess = _fn("gbopt_net_lagrangian_hessian", _status, _vp, _dp, _sz, _dp, _sz, _dp, _sz)
_net_oracle = _fn("gbopt_net_oracle", _status, _vp, _dp, _sz, _dp, _sz, _dp, _dp, _dp)
_net_oracle_batched = _fn("gbopt_net_oracle_batched", _status, _vp, _sz, _dp, _sz, _dp, _sz, _dp, _dp, _dp)
_net_oracle_batched_device = _fn("gbopt_net_oracle_batched_device", _status, _vp, _sz, _vp, _sz, _vp, _sz, _vp, _vp,
                                 _vp, _vp)
_net_oracle_multi = _fn("gbopt_net_oracle_batched_multi", _status, _vp, ctypes.POINTER(ctypes.c_int), _sz, _sz, _dp,
                        _sz, _dp, _sz, _dp, _dp, _dp)
_net_oracle_multi_gather = _fn("gbopt_net_oracle_batched_multi_gather", _status, _vp, ctypes.POINTER(ctypes.c_int),
                               _sz, _sz, _vp, _sz, _vp, _sz, _vp, _vp, _vp)
_net_forward_trace = _fn("gbopt_net_forward_trace", _status, _vp, _dp, _sz, _dp, _dp, _sz)
_net_oracle_lower = _fn("gbopt_net_oracle_lower", _status, _vp, _sz, _dp, _sz, _dp, _sz, _dp, _dp, _dp, _sz)
_net_last_launch_count = _fn("gbopt_net_last_launch_count", _i64, _vp)
_net_set_schedule = _fn("gbopt_net_set_schedule", _status, _vp, ctypes.c_int)
_net_last_schedule = _fn("gbopt_net_last_schedule", ctypes.c_int, _vp)
_net_dataflow_trace = _fn("gbopt_net_dataflow_trace", _status, _vp, _sz, _vp, _vp, _dp, _sz, ctypes.POINTER(_sz))
_net_set_graphs = _fn("gbopt_net_set_graphs", _status, _vp, ctypes.c_int)
_net_profile = _fn("gbopt_net_profile", _status, _vp, _sz, _vp, _vp, ctypes.POINTER(ctypes.c_int32),
                   ctypes.POINTER(ctypes.c_float), _dp, _dp, _sz, ctypes.POINTER(_sz))
_kernel_tag_name = _fn("gbopt_kernel_tag_name", ctypes.c_char_p, ctypes.c_int)
_net_profile_timeline = _fn("gbopt_net_profile_timeline", _status, _vp, _sz, _vp, _vp, ctypes.POINTER(ctypes.c_int32),
                            ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_float),
                            ctypes.POINTER(ctypes.c_float), _sz, ctypes.POINTER(_sz))
_ldlt_factor = _fn("gbopt_ldlt_factor", _status, _dp, _sz, ctypes.c_int, ctypes.POINTER(_vp))
_ldlt_inertia = _fn("gbopt_ldlt_inertia", _status, _vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64), ctypes.POINTER(_i64))
_ldlt_solve = _fn("gbopt_ldlt_solve", _status, _vp, _dp, _sz, _dp)
_ldlt_free = _fn("gbopt_ldlt_free", None, _vp)
_i64p = ctypes.POINTER(_i64)
_kkt_create = _fn("gbopt_kkt_create", _status, _sz, _sz, _i64p, _i64p, _sz, _i64p, _i64p, _sz, ctypes.POINTER(_vp))
_kkt_assemble = _fn("gbopt_kkt_assemble", _status, _vp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, ctypes.c_double,
                    ctypes.c_double, ctypes.c_double)
_kkt_matrix = _fn("gbopt_kkt_matrix", _status, _vp, _dp, _sz)
_kkt_rhs = _fn("gbopt_kkt_rhs", _status, _vp, _dp, _sz)
_kkt_inertia_correct = _fn("gbopt_kkt_inertia_correct", _status, _vp, ctypes.c_double, ctypes.c_double,
                           ctypes.c_double, ctypes.c_double, ctypes.POINTER(_vp), _dp, _dp)
_kkt_solve = _fn("gbopt_kkt_solve", _status, _vp, _vp, _dp, _sz)
_kkt_free = _fn("gbopt_kkt_free", None, _vp)
_net_debug_intermediate = _fn("gbopt_net_debug_intermediate", _status, _vp, ctypes.c_char_p, _i64, _sz, _dp, _sz)

# ---------------------------------------------------------------------------
# Error taxonomy (reference errors.hpp:10-71; status codes gbopt.h:19-31)
# ---------------------------------------------------------------------------
OK, ERR_STRUCTURAL, ERR_NUMERIC, ERR_SINGULAR, ERR_IO, ERR_FORMAT, ERR_DIMENSION, ERR_TRUNCATED, ERR_RANGE, \
    ERR_ARGUMENT, ERR_INTERNAL, ERR_DEVICE = range(12)


class GboptError(Exception):
    status = ERR_INTERNAL


class StructuralError(GboptError):
    status = ERR_STRUCTURAL


class NumericError(GboptError):
    status = ERR_NUMERIC


class SingularError(GboptError):
    status = ERR_SINGULAR


class IoError(GboptError):
    status = ERR_IO


class FormatError(IoError):
    status = ERR_FORMAT


class DimensionError(IoError):
    status = ERR_DIMENSION


class TruncatedError(IoError):
    status = ERR_TRUNCATED


class RangeError(GboptError):
    status = ERR_RANGE


class ArgumentError(GboptError):
    status = ERR_ARGUMENT


class DeviceError(GboptError):
    status = ERR_DEVICE


_BY_STATUS = {c.status: c for c in (StructuralError, NumericError, SingularError, IoError, FormatError,
                                    DimensionError, TruncatedError, RangeError, ArgumentError, DeviceError)}


def _check(status: int):
    if status != OK:
        msg = _last_error().decode(errors="replace")
        raise _BY_STATUS.get(status, GboptError)(msg)


def last_error() -> str:
    return _last_error().decode(errors="replace")


def version() -> str:
    return _version().decode()


def device_count() -> int:
    return int(_device_count())


LINEAR, TANH, SIGMOID, SOFTMAX, SOFTPLUS = 0, 1, 2, 3, 4
ACTIVATIONS = {"linear": LINEAR, "tanh": TANH, "sigmoid": SIGMOID, "softmax": SOFTMAX, "softplus": SOFTPLUS}
INIT_UNIFORM_FANIN, INIT_XAVIER_UNIFORM, INIT_XAVIER_NORMAL, INIT_NORMAL_FANIN = 0, 1, 2, 3


def _dptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(_dp)


def _vec(a, n=None) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1))
    return a


class Prng:
    """Seeded generator (reference prng.hpp:11-23) living in the library."""

    def __init__(self, seed: int):
        h = _vp()
        _check(_prng_new(_u64(seed & (2 ** 64 - 1)), ctypes.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _prng_free(h)
            self._h = None

    def raw(self, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint64)
        _check(_prng_raw(self._h, out.ctypes.data_as(ctypes.POINTER(_u64)), n))
        return out

    def uniform(self, lo: float, hi: float, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.float64)
        _check(_prng_uniform(self._h, lo, hi, _dptr(out), n))
        return out

    def normal(self, mean: float, std: float, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.float64)
        _check(_prng_normal(self._h, mean, std, _dptr(out), n))
        return out


class NeuralNet:
    """Handle over a ``gbopt_net`` (immutable; weights HBM-resident once bound).

    Mirrors ``gbopt::NeuralNet`` (reference nn.hpp:40-81): ``forward``,
    ``jacobian`` (m x n), ``lagrangian_gradient``, ``lagrangian_hessian``
    (n x n, symmetric), plus the fused ``oracle`` / ``oracle_batched`` this
    build adds.  Dimension mismatches raise ``ArgumentError`` at the C
    boundary (reference capi.cpp:168-172).
    """

    def __init__(self, handle):
        self._h = handle

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _net_free(h)
            self._h = None

    # ---- constructors -------------------------------------------------
    @classmethod
    def from_layers(cls, weights: Sequence[np.ndarray], biases: Sequence[np.ndarray],
                    activations: Sequence[int]) -> "NeuralNet":
        """'Load MLP weights and activations' from memory (row-major W_l)."""
        if len(weights) != len(biases) or len(weights) != len(activations):
            raise ArgumentError("from_layers: weights, biases and activations differ in length")
        ws = [np.ascontiguousarray(np.asarray(w, dtype=np.float64)) for w in weights]
        bs = [np.ascontiguousarray(np.asarray(b, dtype=np.float64).reshape(-1)) for b in biases]
        for w in ws:
            if w.ndim != 2:
                raise StructuralError("from_layers: weights must be 2-D")
        widths = [ws[0].shape[1] if ws else 0] + [w.shape[0] for w in ws]
        for l in range(1, len(ws)):
            if ws[l].shape[1] != ws[l - 1].shape[0]:
                raise StructuralError(f"NeuralNet: layer {l} input width does not chain")
        for l, (w, b) in enumerate(zip(ws, bs)):
            if b.size != w.shape[0]:
                raise StructuralError(f"NeuralNet: layer {l} weight rows != bias length")
        L = len(ws)
        warr = (_i64 * (L + 1))(*widths)
        aarr = (ctypes.c_int32 * max(L, 1))(*[int(a) for a in activations])
        wp = (_dp * max(L, 1))(*[_dptr(w) for w in ws])
        bp = (_dp * max(L, 1))(*[_dptr(b) for b in bs])
        h = _vp()
        _check(_net_from_layers(L, warr, aarr, wp, bp, ctypes.byref(h)))
        return cls(h)

    # ---- dimensions ----------------------------------------------------
    @property
    def input_dim(self) -> int:
        return int(_net_input_dim(self._h))

    @property
    def output_dim(self) -> int:
        return int(_net_output_dim(self._h))

    @property
    def param_count(self) -> int:
        return int(_net_param_count(self._h))

    @property
    def layer_count(self) -> int:
        return int(_net_layer_count(self._h))

    def layer(self, l: int):
        """(W row-major, b, activation code) of layer l (host copy)."""
        rows, cols, act = _i64(), _i64(), ctypes.c_int32()
        _check(_net_layer_info(self._h, l, ctypes.byref(rows), ctypes.byref(cols), ctypes.byref(act)))
        w = np.empty((rows.value, cols.value))
        b = np.empty(rows.value)
        _check(_net_layer_copy(self._h, l, _dptr(w), w.size, _dptr(b), b.size))
        return w, b, act.value

    def widths(self):
        return [self.input_dim] + [self.layer(l)[0].shape[0] for l in range(self.layer_count)]

    # ---- device ----------------------------------------------------------
    def bind_device(self, ordinal: int = 0) -> "NeuralNet":
        _check(_net_bind_device(self._h, ordinal))
        return self

    @property
    def device(self) -> int:
        return int(_net_device(self._h))

    def set_graphs(self, enabled: bool):
        _check(_net_set_graphs(self._h, 1 if enabled else 0))

    @property
    def last_launch_count(self) -> int:
        return int(_net_last_launch_count(self._h))

    def set_schedule(self, schedule: str) -> "NeuralNet":
        """'auto' (shape rule), 'layered', 'dataflow' or 'measured'
        (gbopt_net_set_schedule)."""
        code = {"auto": -1, "layered": 0, "dataflow": 1, "measured": -2}[schedule]
        _check(_net_set_schedule(self._h, code))
        return self

    @property
    def last_schedule(self) -> str:
        return {-1: "unbound", 0: "layered", 1: "dataflow"}[int(_net_last_schedule(self._h))]

    # ---- oracle ----------------------------------------------------------
    def forward(self, x) -> np.ndarray:
        x = _vec(x)
        y = np.empty(self.output_dim)
        _check(_net_forward(self._h, _dptr(x), x.size, _dptr(y), y.size))
        return y

    def jacobian(self, x) -> np.ndarray:
        x = _vec(x)
        m = self.output_dim
        j = np.empty((m, x.size))
        _check(_net_jacobian(self._h, _dptr(x), x.size, _dptr(j), j.size))
        return j

    def lagrangian_gradient(self, x, lam) -> np.ndarray:
        x, lam = _vec(x), _vec(lam)
        g = np.empty(x.size)
        _check(_net_lag_grad(self._h, _dptr(x), x.size, _dptr(lam), lam.size, _dptr(g), g.size))
        return g

    def lagrangian_hessian(self, x, lam) -> np.ndarray:
        x, lam = _vec(x), _vec(lam)
        h = np.empty((x.size, x.size))
        _check(_net_lag_hess(self._h, _dptr(x), x.size, _dptr(lam), lam.size, _dptr(h), h.size))
        return h

    def oracle(self, x, lam, want_y=True, want_j=True, want_h=True):
        """Fused (y, J, H) at one point from one forward pass."""
        x = _vec(x)
        lam = None if lam is None else _vec(lam)
        n, m = self.input_dim, self.output_dim
        y = np.empty(m) if want_y else None
        j = np.empty((m, n)) if want_j else None
        h = np.empty((n, n)) if want_h else None
        _check(_net_oracle(self._h, _dptr(x), x.size, _dptr(lam), m if lam is None else lam.size,
                           _dptr(y), _dptr(j), _dptr(h)))
        return y, j, h

    def forward_trace(self, x):
        """Per-layer (z_l, y_l) of one forward pass (reference
        NeuralNet::forward_trace, nn.cpp:127-146): two lists of vectors."""
        x = _vec(x)
        rows = [self.layer(l)[0].shape[0] for l in range(self.layer_count)]
        z = np.empty(sum(rows))
        y = np.empty(sum(rows))
        _check(_net_forward_trace(self._h, _dptr(x), x.size, _dptr(z), _dptr(y), z.size))
        cuts = np.cumsum(rows)[:-1]
        return list(np.split(z, cuts)), list(np.split(y, cuts))

    def oracle_lower(self, x, lam, want_y=True, want_j=True):
        """(y, J, Hl) at one point with the Hessian as its packed lower triangle in
        row order (Hl[a (a + 1) / 2 + c] = H[a, c], c <= a): the value order of the
        reduced-space Lagrangian-Hessian callback, packed on the device."""
        x, lam = _vec(x), _vec(lam)
        n, m = self.input_dim, self.output_dim
        y = np.empty(m) if want_y else None
        j = np.empty((m, n)) if want_j else None
        hl = np.empty(n * (n + 1) // 2)
        _check(_net_oracle_lower(self._h, 1, _dptr(x), x.size, _dptr(lam), lam.size, _dptr(y), _dptr(j), _dptr(hl),
                                 hl.size))
        return y, j, hl

    def oracle_batched(self, X, Lam, want_y=True, want_j=True, want_h=True, out=None):
        """B independent points with the shared weights: X (B x n), Lam (B x m).
        ``out`` may supply preallocated (Y, J, H) arrays (e.g. pinned)."""
        X = np.ascontiguousarray(np.asarray(X, dtype=np.float64))
        if X.ndim != 2:
            raise ArgumentError("oracle_batched: X must be B x n")
        B = X.shape[0]
        n, m = self.input_dim, self.output_dim
        Lam = None if Lam is None else np.ascontiguousarray(np.asarray(Lam, dtype=np.float64))
        if out is not None:
            Y, J, H = out
        else:
            Y = np.empty((B, m)) if want_y else None
            J = np.empty((B, m, n)) if want_j else None
            H = np.empty((B, n, n)) if want_h else None
        for arr, shape in ((Y, (B, m)), (J, (B, m, n)), (H, (B, n, n))):
            if arr is not None and (arr.shape != shape or arr.dtype != np.float64 or not arr.flags.c_contiguous):
                raise ArgumentError("oracle_batched: output buffer has the wrong shape or layout")
        if Lam is not None and Lam.shape != (B, m):
            raise ArgumentError("oracle_batched: Lambda must be B x m")
        _check(_net_oracle_batched(self._h, B, _dptr(X), X.shape[1], _dptr(Lam), m, _dptr(Y), _dptr(J), _dptr(H)))
        return Y, J, H

    def oracle_batched_multi(self, devices: Sequence[int], X, Lam, want_y=True, want_j=True, want_h=True):
        """B points split into contiguous shards over `devices` (one replica of
        the weights and one host thread per entry; duplicates allowed), each
        device writing its rows straight into the host outputs
        (gbopt_net_oracle_batched_multi)."""
        X = np.ascontiguousarray(np.asarray(X, dtype=np.float64))
        Lam = None if Lam is None else np.ascontiguousarray(np.asarray(Lam, dtype=np.float64))
        B, n, m = X.shape[0], self.input_dim, self.output_dim
        Y = np.empty((B, m)) if want_y else None
        J = np.empty((B, m, n)) if want_j else None
        H = np.empty((B, n, n)) if want_h else None
        devs = (ctypes.c_int * len(devices))(*devices)
        _check(_net_oracle_multi(self._h, devs, len(devices), B, _dptr(X), X.shape[1], _dptr(Lam), m, _dptr(Y),
                                 _dptr(J), _dptr(H)))
        return Y, J, H

    def oracle_batched_multi_gather(self, devices: Sequence[int], batch: int, dX: int, dLam: int, dY: int, dJ: int,
                                    dH: int):
        """Device buffers on devices[0] (raw CUDA addresses); the other devices
        pull their shards and push their results back with peer copies
        (gbopt_net_oracle_batched_multi_gather).  Synchronous."""
        devs = (ctypes.c_int * len(devices))(*devices)
        _check(_net_oracle_multi_gather(self._h, devs, len(devices), batch, dX, self.input_dim, dLam,
                                        self.output_dim, dY, dJ, dH))

    def intermediate(self, name: str, layer: int, batch: int = 1) -> np.ndarray:
        """Per-layer vector of the last evaluation (white-box tests; the last
        chunk's when a host-buffer batch ran in chunks, see GBOPT_HOST_CHUNKS)."""
        rows = self.layer(layer)[0].shape[0]
        out = np.empty((batch, rows))
        _check(_net_debug_intermediate(self._h, name.encode(), layer, batch, _dptr(out), out.size))
        return out

    def oracle_batched_device(self, batch: int, dX: int, dLam: int, dY: int, dJ: int, dH: int, stream: int = 0):
        """Device-pointer entry (raw CUDA addresses, e.g. torch ``data_ptr()``);
        enqueued on ``stream`` without a host synchronisation."""
        _check(_net_oracle_batched_device(self._h, batch, dX or None, self.input_dim, dLam or None, self.output_dim,
                                          dY or None, dJ or None, dH or None, stream or None))


def profile_launches(net: "NeuralNet", batch: int, dX: int, dLam: int):
    """Per-launch (kernel, ms, flops, bytes) of one eager evaluation, timed
    with CUDA events on the launching stream (gbopt_net_profile)."""
    cap = 4096
    tags = (ctypes.c_int32 * cap)()
    ms = (ctypes.c_float * cap)()
    fl = (ctypes.c_double * cap)()
    by = (ctypes.c_double * cap)()
    cnt = _sz()
    _check(_net_profile(net._h, batch, dX, dLam, tags, ms, fl, by, cap, ctypes.byref(cnt)))
    return [(_kernel_tag_name(tags[i]).decode(), float(ms[i]), float(fl[i]), float(by[i]))
            for i in range(min(cnt.value, cap))]


def profile_timeline(net: "NeuralNet", batch: int, dX: int, dLam: int):
    """(kernel, stream, start_ms, end_ms) of every launch of one eager
    evaluation that keeps the two-stream concurrency."""
    cap = 4096
    tags = (ctypes.c_int32 * cap)()
    st = (ctypes.c_int32 * cap)()
    t0 = (ctypes.c_float * cap)()
    t1 = (ctypes.c_float * cap)()
    cnt = _sz()
    _check(_net_profile_timeline(net._h, batch, dX, dLam, tags, st, t0, t1, cap, ctypes.byref(cnt)))
    return [(_kernel_tag_name(tags[i]).decode(), int(st[i]), float(t0[i]), float(t1[i]))
            for i in range(min(cnt.value, cap))]


def dataflow_trace(net: "NeuralNet", batch: int, dX: int, dLam: int) -> np.ndarray:
    """Per-item trace of one eager dataflow evaluation (gbopt_net_dataflow_trace):
    rows {kind, job, point, tm, tn, kb0, kb1, sm, t_claimed, t_ready, t_begin,
    t_end} in claim order, times in microseconds."""
    cnt = _sz()
    _check(_net_dataflow_trace(net._h, batch, dX, dLam, None, 0, ctypes.byref(cnt)))
    out = np.empty(12 * cnt.value, dtype=np.float64)
    _check(_net_dataflow_trace(net._h, batch, dX, dLam, out.ctypes.data_as(_dp), out.size, ctypes.byref(cnt)))
    return out.reshape(-1, 12)


class LdltFactorization:
    """GPU LDL^T of a symmetric (KKT) matrix: reference ldlt_factor /
    LdltFactorization (proj/include/gbopt/linalg.hpp:24-78)."""

    def __init__(self, A, keep_input: bool = True):
        A = np.ascontiguousarray(np.asarray(A, dtype=np.float64))
        if A.ndim != 2 or A.shape[0] != A.shape[1]:
            raise StructuralError(f"ldlt_factor: matrix is not square {A.shape}")
        h = _vp()
        _check(_ldlt_factor(_dptr(A), A.shape[0], 1 if keep_input else 0, ctypes.byref(h)))
        self._h = h
        self.dim = A.shape[0]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _ldlt_free(h)
            self._h = None

    @property
    def inertia(self):
        p, n, z = _i64(), _i64(), _i64()
        _check(_ldlt_inertia(self._h, ctypes.byref(p), ctypes.byref(n), ctypes.byref(z)))
        return p.value, n.value, z.value

    def solve(self, b):
        b = _vec(b)
        x = np.empty_like(b)
        _check(_ldlt_solve(self._h, _dptr(b), b.size, _dptr(x)))
        return x


def ldlt_factor(A, keep_input: bool = True) -> LdltFactorization:
    return LdltFactorization(A, keep_input)


def _idx(v):
    return np.ascontiguousarray(np.asarray(v, dtype=np.int64).reshape(-1))


def _ip(a):
    return a.ctypes.data_as(_i64p) if a.size else None


class KktPattern:
    """One NLP's KKT sparsity (Lagrangian-Hessian and Jacobian triplets),
    analysed once; assemble() then builds each IPM iteration's dense Newton
    system on the device (gbopt_kkt_*; reference assemble_kkt,
    proj/src/ipm.cpp:466-518)."""

    def __init__(self, n: int, m: int, hess_rows, hess_cols, jac_rows, jac_cols):
        hr, hc, jr, jc = _idx(hess_rows), _idx(hess_cols), _idx(jac_rows), _idx(jac_cols)
        if hr.size != hc.size or jr.size != jc.size:
            raise StructuralError("kkt: row and column triplet lists differ in length")
        h = _vp()
        _check(_kkt_create(n, m, _ip(hr), _ip(hc), hr.size, _ip(jr), _ip(jc), jr.size, ctypes.byref(h)))
        self._h = h
        self.n_var, self.n_con = int(n), int(m)
        self.nnz_h, self.nnz_j = hr.size, jr.size

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _kkt_free(h)
            self._h = None

    def assemble(self, x, lower, z, lam, grad_f, g, jac_values, hess_values, mu, delta_w=0.0, delta_c=0.0):
        n, m = self.n_var, self.n_con
        args = []
        for name, v, size in (("x", x, n), ("lower", lower, n), ("z", z, n), ("lambda", lam, m),
                              ("grad_f", grad_f, n), ("g", g, m), ("jac_values", jac_values, self.nnz_j),
                              ("hess_values", hess_values, self.nnz_h)):
            a = np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(-1))
            if a.size != size:
                raise StructuralError(f"assemble_kkt: {name} has size {a.size}, expected {size}")
            args.append(a)
        self._keep = args
        _check(_kkt_assemble(self._h, *[_dptr(a) if a.size else None for a in args], float(mu), float(delta_w),
                             float(delta_c)))
        return KktSystem(self)


class KktSystem:
    """The assembled system, resident on the device (reference KktSystem,
    proj/include/gbopt/ipm.hpp:80-87); .mat / .rhs copy it out."""

    def __init__(self, pattern: KktPattern):
        self.pattern = pattern
        self.n_var, self.n_con = pattern.n_var, pattern.n_con

    @property
    def mat(self):
        d = self.n_var + self.n_con
        out = np.empty((d, d))
        _check(_kkt_matrix(self.pattern._h, _dptr(out), out.size))
        return out

    @property
    def rhs(self):
        out = np.empty(self.n_var + self.n_con)
        _check(_kkt_rhs(self.pattern._h, _dptr(out), out.size))
        return out

    def solve(self, fact: "LdltFactorization"):
        """fact.solve(rhs) with the device-resident right-hand side."""
        out = np.empty(self.n_var + self.n_con)
        _check(_kkt_solve(self.pattern._h, fact._h, _dptr(out), out.size))
        return out


def assemble_kkt(x, lower, z, lam, grad_f, g, jac_rows, jac_cols, jac_values, hess_rows, hess_cols, hess_values, mu,
                 delta_w=0.0, delta_c=0.0) -> KktSystem:
    """Reference assemble_kkt (proj/include/gbopt/ipm.hpp:89-102) with the
    same argument order; the pattern analysis is redone per call (use
    KktPattern across iterations)."""
    n, m = np.asarray(x).size, np.asarray(g).size
    pat = KktPattern(n, m, hess_rows, hess_cols, jac_rows, jac_cols)
    return pat.assemble(x, lower, z, lam, grad_f, g, jac_values, hess_values, mu, delta_w, delta_c)


class IpmOptions:
    """The regularisation fields of the reference IpmOptions
    (proj/include/gbopt/ipm.hpp:21-23)."""

    def __init__(self, delta0=1e-4, delta_growth=10.0, delta_max=1e40):
        self.delta0, self.delta_growth, self.delta_max = delta0, delta_growth, delta_max


class CorrectedFactorization:
    def __init__(self, fact, delta_w, delta_c):
        self.fact, self.delta_w, self.delta_c = fact, delta_w, delta_c


def inertia_correct(kkt: KktSystem, opts: IpmOptions = None, delta_w_start: float = 0.0) -> CorrectedFactorization:
    """Reference inertia_correct (proj/src/ipm.cpp:520-557) on the device-
    resident matrix: SingularError once delta_w exceeds opts.delta_max."""
    opts = opts or IpmOptions()
    h = _vp()
    dw, dc = ctypes.c_double(), ctypes.c_double()
    _check(_kkt_inertia_correct(kkt.pattern._h, opts.delta0, opts.delta_growth, opts.delta_max, delta_w_start,
                                ctypes.byref(h), ctypes.byref(dw), ctypes.byref(dc)))
    f = LdltFactorization.__new__(LdltFactorization)
    f._h = h
    f.dim = kkt.n_var + kkt.n_con
    return CorrectedFactorization(f, dw.value, dc.value)


def load_weights(path: str) -> NeuralNet:
    """GBNN v1 binary / JSON mirror (reference nn_io.cpp:144-221)."""
    h = _vp()
    _check(_net_load(os.fsencode(path), ctypes.byref(h)))
    return NeuralNet(h)


def save_weights(nn: NeuralNet, path: str):
    """reference nn_io.cpp:223-247."""
    _check(_net_save(nn._h, os.fsencode(path)))


def random_net(widths: Sequence[int], hidden: str, final_act: str, seed: int) -> NeuralNet:
    """reference random_net (nn.cpp:336-367): U(+-1/sqrt(fan_in)) W and b."""
    warr = (_i64 * len(widths))(*[int(w) for w in widths])
    h = _vp()
    _check(_net_random(warr, len(widths), hidden.encode(), final_act.encode(), _u64(seed & (2 ** 64 - 1)),
                       ctypes.byref(h)))
    return NeuralNet(h)


def random_net_ex(rng: Prng, widths: Sequence[int], hidden: int, final_act: int, init: int,
                  bias_lo: float = 0.0, bias_hi: float = 0.0) -> NeuralNet:
    """Seeded net drawn from an existing stream (BASELINE initialisers)."""
    warr = (_i64 * len(widths))(*[int(w) for w in widths])
    h = _vp()
    _check(_net_random_ex(rng._h, warr, len(widths), int(hidden), int(final_act), int(init), float(bias_lo),
                          float(bias_hi), ctypes.byref(h)))
    return NeuralNet(h)
