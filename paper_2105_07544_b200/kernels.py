"""Dense Krylov primitives on the GPU (reference: pkg/src/mpkrylov/kernels.py).

Same names, argument meaning and errors as the reference; every operation
runs in libmpkb200 (``mpk_dot``/``mpk_norm2``/``mpk_axpy``/``mpk_scale``,
``mpk_cgs2_append``, ``mpk_lsq_*``).  Reductions are deterministic two-stage
trees accumulated in the vectors' own precision.  numpy in -> numpy out,
CUDA tensors in -> CUDA tensors out.  Inside the solvers these objects are
not used: the cycle runs the fused kernels of ``mpk_cycle_run`` directly.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from . import device as D
from .errors import (
    ColumnOrderError,
    DimensionMismatchError,
    PrecisionMismatchError,
    TriangularBreakdownError,
)
from .precision import Precision

__all__ = ["dot", "norm2", "axpy", "scale", "KrylovBasis", "cgs2_append", "HessenbergSystem"]


def _check_pair(x, y):
    if D.shape(x) != D.shape(y) or len(D.shape(x)) != 1:
        raise DimensionMismatchError("vectors must be 1-d and of equal length")
    if D.np_dtype(x) != D.np_dtype(y):
        raise PrecisionMismatchError("vector dtypes differ: %s vs %s" % (D.np_dtype(x), D.np_dtype(y)))


def _scalar_out(dt):
    return D.empty(1, Precision.from_dtype(dt).torch_dtype)


def _reduce(kind, x, y=None):
    dt = D.np_dtype(x)
    prec = Precision.from_dtype(dt)
    xd = D.to_device(x)
    out = _scalar_out(dt)
    lib = D.lib()
    ws = D.ReduceWorkspace.shared()
    n = xd.shape[0]
    if kind == "dot":
        yd = D.to_device(y)
        _lib.check(lib.mpk_dot(prec.code, n, D.ptr(xd), D.ptr(yd), D.ptr(out), ws.ptr, D.stream()))
    else:
        _lib.check(lib.mpk_norm2(prec.code, n, D.ptr(xd), D.ptr(out), ws.ptr, D.stream()))
    return dt.type(out.item())


def dot(x, y):
    """Inner product in the vectors' common precision (reference kernels.py:31-34)."""
    _check_pair(x, y)
    return _reduce("dot", x, y)


def norm2(x):
    """Euclidean norm accumulated in x's precision (reference kernels.py:37-41)."""
    if len(D.shape(x)) != 1:
        raise DimensionMismatchError("norm2 expects a 1-d vector")
    return _reduce("norm", x)


def _axpy(alpha, x, y):
    host = not D.is_tensor(x)
    prec = Precision.from_dtype(D.np_dtype(x))
    xd = D.to_device(x)
    yd = D.to_device(y) if y is not None else None
    out = D.empty(xd.shape[0], prec.torch_dtype)
    if xd.shape[0]:
        _lib.check(D.lib().mpk_axpy(prec.code, xd.shape[0], float(alpha), D.ptr(xd),
                                    D.ptr(yd) if yd is not None else None, D.ptr(out), D.stream()))
    return D.like_input(out, host)


def axpy(alpha, x, y):
    """y + alpha * x, inputs untouched (reference kernels.py:44-47)."""
    _check_pair(x, y)
    return _axpy(alpha, x, y)


def scale(alpha, x):
    """alpha * x in x's precision (reference kernels.py:50-52)."""
    return _axpy(alpha, x, None)


class KrylovBasis:
    """Fixed-capacity basis stored column-major in HBM (reference kernels.py:55-95).

    Columns are contiguous with a leading dimension padded to 64 elements.
    ``column``/``columns`` return device views, or host copies when the basis
    is fed numpy vectors (the reference's numpy-view contract)."""

    __slots__ = ("length", "capacity", "precision", "count", "ld", "_data", "_host")

    def __init__(self, length, capacity, precision: Precision):
        if capacity < 1 or length < 1:
            raise DimensionMismatchError("basis needs positive length and capacity")
        self.length = int(length)
        self.capacity = int(capacity)
        self.precision = precision
        self.count = 0
        self.ld = D.ld_for(self.length)
        self._data = D.torch().zeros((self.capacity, self.ld), dtype=precision.torch_dtype,
                                     device=D.device())
        self._host = False

    def append(self, v):
        if self.count >= self.capacity:
            raise DimensionMismatchError("basis is full (capacity %d)" % self.capacity)
        if D.shape(v) != (self.length,):
            raise DimensionMismatchError("vector length does not match basis")
        if D.np_dtype(v) != self.precision.dtype:
            raise PrecisionMismatchError(
                "basis stores %s but vector is %s" % (self.precision.dtype, D.np_dtype(v)))
        self._host = self._host or not D.is_tensor(v)
        self._data[self.count, : self.length].copy_(D.to_device(v))
        self.count += 1

    def _view(self, k):
        return self._data[:k, : self.length].t()

    def column(self, j):
        if not 0 <= j < self.count:
            raise DimensionMismatchError("column %d not in basis of size %d" % (j, self.count))
        col = self._data[j, : self.length]
        return D.to_host(col) if self._host else col

    def columns(self, k=None):
        if k is None:
            k = self.count
        if not 0 <= k <= self.count:
            raise DimensionMismatchError("requested %d columns, have %d" % (k, self.count))
        if self._host:
            return np.asfortranarray(D.to_host(self._data[:k, : self.length]).T)
        return self._view(k)


def cgs2_append(basis: KrylovBasis, w, rule: str = "n_u"):
    """Two classical Gram-Schmidt passes, then append w/beta unless
    beta <= n*u*||w|| (reference kernels.py:98-126; ``rule="u"`` is the
    documented non-reference threshold u*||w||).

    Returns (coeffs, beta, appended) like the reference."""
    if basis.count < 1:
        raise DimensionMismatchError("basis must hold at least one vector")
    if D.shape(w) != (basis.length,):
        raise DimensionMismatchError("vector length does not match basis")
    dt = basis.precision.dtype
    if D.np_dtype(w) != dt:
        raise PrecisionMismatchError("basis stores %s but vector is %s" % (dt, D.np_dtype(w)))
    if basis.count >= basis.capacity:
        # the reference only fails when it appends; keep a spare column
        spare = D.torch().zeros((1, basis.ld), dtype=basis.precision.torch_dtype, device=D.device())
        basis._data = D.torch().cat([basis._data, spare], 0)
    host = not D.is_tensor(w)
    wd = D.to_device(w)
    t = basis.precision.torch_dtype
    n, cnt = basis.length, basis.count
    coeffs = D.empty(cnt, t)
    out = D.empty(2, t)
    app = D.torch().zeros(1, dtype=D.torch().int32, device=D.device())
    tmp = D.empty(2 * n, t)
    ws = D.ReduceWorkspace.shared()
    _lib.check(D.lib().mpk_cgs2_append(
        basis.precision.code, n, basis.ld, cnt, D.ptr(basis._data), D.ptr(wd),
        _lib.RULE_U if rule == "u" else _lib.RULE_NU, D.ptr(coeffs), D.ptr(out), D.ptr(app),
        D.ptr(tmp), ws.ptr, D.stream()))
    appended = bool(app.item())
    beta = dt.type(out[0].item())
    if basis._data.shape[0] > basis.capacity:
        basis._data = basis._data[: basis.capacity].contiguous()
        if appended:
            raise DimensionMismatchError("basis is full (capacity %d)" % basis.capacity)
    if appended:
        basis.count += 1
    return (D.to_host(coeffs) if host else coeffs), beta, appended


class HessenbergSystem:
    """Givens-rotated least-squares state for min ||gamma e1 - Hbar d||
    (reference kernels.py:139-216), held in HBM; rotations run on one CTA."""

    def __init__(self, m, gamma, norm_scale=None, precision=Precision.binary64):
        if m < 1:
            raise DimensionMismatchError("need room for at least one column")
        self.m = int(m)
        if self.m > _lib.MAX_STEPS - 1:
            raise DimensionMismatchError("at most %d columns supported" % (_lib.MAX_STEPS - 1))
        self.precision = precision
        self.gamma = float(gamma)
        self.norm_scale = float(gamma if norm_scale is None else norm_scale)
        if self.norm_scale <= 0:
            raise DimensionMismatchError("norm_scale must be positive")
        self.count = 0
        lib = D.lib()
        self._hess = D.torch().zeros(int(lib.mpk_cycle_hess_bytes(self.m, precision.code)),
                                     dtype=D.torch().uint8, device=D.device())
        self._ctl = D.torch().zeros(ctypes.sizeof(_lib.MpkCycleCtl), dtype=D.torch().uint8,
                                    device=D.device())
        _lib.check(lib.mpk_lsq_init(precision.code, self.m, float(gamma), self.norm_scale,
                                    D.ptr(self._hess), D.ptr(self._ctl), D.stream()))

    def _arrays(self):
        m = self.m
        t = self.precision.torch_dtype
        sz = (m + 1) * m + m + m + (m + 1) + m + (m + 1) * m
        flat = self._hess[: sz * (4 if self.precision is Precision.binary32 else 8)].view(t)
        o = 0
        h = flat[o:o + (m + 1) * m].view(m, m + 1).t()
        o += (m + 1) * m
        cs = flat[o:o + m]
        o += m
        sn = flat[o:o + m]
        o += m
        g = flat[o:o + m + 1]
        o += m + 1
        d = flat[o:o + m]
        return h, cs, sn, g, d

    @property
    def h(self):
        return D.to_host(self._arrays()[0])

    @property
    def g(self):
        return D.to_host(self._arrays()[3])

    def update(self, j, coeffs, beta):
        """Fold in column j (1-based); returns the implicit relative residual."""
        if j != self.count + 1:
            raise ColumnOrderError("expected column %d, got %d" % (self.count + 1, j))
        if j > self.m:
            raise DimensionMismatchError("system already holds %d columns" % self.m)
        if D.shape(coeffs) != (j,):
            raise DimensionMismatchError("column %d needs %d coefficients" % (j, j))
        if D.np_dtype(coeffs) != self.precision.dtype:
            raise PrecisionMismatchError("coefficients must be %s" % self.precision.dtype)
        t = self.precision.torch_dtype
        cd = D.to_device(coeffs)
        bd = D.torch().tensor([float(beta)], dtype=D.torch().float64).to(t).to(D.device())
        ws = D.ReduceWorkspace.shared()
        _lib.check(D.lib().mpk_lsq_update(self.precision.code, self.m, j, D.ptr(cd), D.ptr(bd),
                                          D.ptr(self._hess), D.ptr(self._ctl), ws.ptr, D.stream()))
        self.count = j
        ctl = _lib.MpkCycleCtl.from_buffer_copy(D.to_host(self._ctl).tobytes())
        return float(ctl.implicit_relres[j - 1])

    def residual_norm(self):
        """Absolute implicit residual |g_count|."""
        return float(abs(self.g[self.count]))

    def solve(self, k=None):
        """Back-substitute the first k coefficients (reference kernels.py:202-216)."""
        if self.count == 0:
            raise ColumnOrderError("no columns processed yet")
        if k is None:
            k = self.count
        if not 1 <= k <= self.count:
            raise DimensionMismatchError("cannot solve for %d of %d columns" % (k, self.count))
        _lib.check(D.lib().mpk_lsq_solve(self.precision.code, self.m, int(k), D.ptr(self._hess),
                                         D.ptr(self._ctl), D.stream()))
        ctl = _lib.MpkCycleCtl.from_buffer_copy(D.to_host(self._ctl).tobytes())
        if ctl.tri_err:
            self._ctl[12:16].zero_()    # clear tri_err so a later solve(k') can run
            raise TriangularBreakdownError(ctl.tri_index, ctl.tri_entry, ctl.tri_threshold)
        return D.to_host(self._arrays()[4][:k])
