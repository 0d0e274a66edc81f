"""Per-solve device state and the host side of one restarted-GMRES cycle.

One :class:`CycleWorkspace` per (device, n, m, precision) holds the Krylov
basis (column-major, ld padded to 64), the three work vectors, the rotated
Hessenberg state, the reduction scratch and a control block.  A cycle is ONE
native call (``mpk_cycle_run``) that enqueues every kernel of the cycle; the
explicit residual of the restart follows on the same stream, and the host
reads the whole control block back with a single pinned copy + sync per
cycle (per refinement for GMRES-IR).
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from . import device as D
from .errors import TriangularBreakdownError
from .precision import Precision

# optional host-side accounting (tools/dist_check.py): seconds spent waiting
# in the per-cycle control-block sync, number of reads, host collectives
HOST_STATS = {"on": False, "sync_s": 0.0, "reads": 0, "host_collectives": 0}

CTL_BYTES = ctypes.sizeof(_lib.MpkCycleCtl)
OFF_RN2 = (CTL_BYTES + 63) // 64 * 64      # r.r in the cycle dtype (or fp64 outer)
OFF_RN2_LOW = OFF_RN2 + 8                 # fp32 r_low.r_low (refinement)
OFF_CHANGED = OFF_RN2 + 16                # int32 "x moved" flag (refinement)
OFF_BN2 = OFF_RN2 + 24                    # b.b (zero right-hand side check)
CTLBUF_BYTES = OFF_RN2 + 64


@dataclass
class Readout:
    steps: int
    implicit: list
    breakdown: bool
    rn2: float
    rn2_low: float
    changed: bool


class CycleWorkspace:
    _cache: dict = {}

    def __init__(self, n: int, m: int, prec: Precision, basis: str = "working"):
        t = D.torch()
        lib = D.lib()
        self.n, self.m, self.prec, self.basis = int(n), int(m), prec, basis
        self.ld = D.ld_for(n)
        td = prec.torch_dtype
        dev = D.device()
        # zero-initialised: rows [n, ld) of every column stay zero (the fused
        # kernel's 16-byte row groups and chunk tails read them).  A binary16
        # basis (SolverConfig.basis_precision) halves its bytes.
        vdt = {"binary16": t.float16, "bfloat16": t.bfloat16}.get(basis, td)
        self.V = t.zeros((self.m + 1) * self.ld, dtype=vdt, device=dev)
        # + 512 elements: 1-D bulk copies of a 256-row tile may run past w''s ld
        self.work = t.zeros(4 * self.ld + 512, dtype=td, device=dev)
        self.hess = t.zeros(int(lib.mpk_cycle_hess_bytes(self.m, prec.code)), dtype=t.uint8, device=dev)
        self.ws = D.ReduceWorkspace()
        self.ctlbuf = t.zeros(CTLBUF_BYTES, dtype=t.uint8, device=dev)
        self.host = t.empty(CTLBUF_BYTES, dtype=t.uint8, pin_memory=True)
        self.desc = _lib.MpkCycleDesc()
        self._pins = []
        self.flags = 0

    @classmethod
    def get(cls, n, m, prec, basis: str = "working") -> "CycleWorkspace":
        key = (D.torch().cuda.current_device(), int(n), int(m), prec, basis)
        ws = cls._cache.get(key)
        if ws is None:
            if len(cls._cache) > 8:
                cls._cache.clear()
            ws = cls._cache[key] = CycleWorkspace(n, m, prec, basis)
        return ws

    # -- pointers into the control buffer ----------------------------------
    @property
    def ctl_ptr(self) -> int:
        return D.ptr(self.ctlbuf)

    def at(self, off: int) -> int:
        return D.ptr(self.ctlbuf) + off

    # -- launches -----------------------------------------------------------
    def residual(self, A, b, x, r, r_low=None):
        """r = b - A x and r.r (+ fp32 copy and its r.r) into the control buffer."""
        lib = D.lib()
        _lib.check(lib.mpk_residual(ctypes.byref(A.descriptor()), D.ptr(b), D.ptr(x), D.ptr(r),
                                    self.at(OFF_RN2), D.ptr(r_low) if r_low is not None else None,
                                    self.at(OFF_RN2_LOW) if r_low is not None else None,
                                    self.ws.ptr, D.stream()))

    def bnorm2(self, b, prec: Precision):
        _lib.check(D.lib().mpk_dot(prec.code, b.shape[0], D.ptr(b), D.ptr(b), self.at(OFF_BN2),
                                   self.ws.ptr, D.stream()))

    def cycle(self, A, M, r0, rnorm2_off, x0, x_out, steps_cap, exit_tol, norm_scale, rule, orth="cgs2",
              basis="working"):
        """Enqueue one whole cycle (gmres.py:134-205) via mpk_cycle_run."""
        d = self.desc
        self._pins = [A.descriptor()]
        d.A = ctypes.pointer(self._pins[0])
        nat = M.native() if M is not None else None
        if nat is not None:
            self._pins.append(nat)
            d.M = ctypes.pointer(nat)
        else:
            d.M = None
        d.dtype = self.prec.code
        d.m = self.m
        d.steps_cap = int(steps_cap)
        d.rule = _lib.RULE_U if rule == "u" else _lib.RULE_NU
        d.exit_tol = float(exit_tol)
        d.norm_scale = float(norm_scale) if norm_scale is not None else -1.0
        d.n = self.n
        d.ld = self.ld
        d.V = D.ptr(self.V)
        d.r0 = D.ptr(r0)
        d.rnorm2 = self.at(rnorm2_off)
        d.x0 = D.ptr(x0)
        d.x_out = D.ptr(x_out)
        d.work = D.ptr(self.work)
        d.hess = D.ptr(self.hess)
        d.ws = self.ws.ptr
        d.ctl = self.ctl_ptr
        d.nranks = 1
        if basis != self.basis:
            raise ValueError("workspace holds a %s basis, cycle asked for %s" % (self.basis, basis))
        d.flags = self.flags | (16 if orth == "dcgs2" else 0) | {"binary16": 32, "bfloat16": 64}.get(basis, 0)
        _lib.check(D.lib().mpk_cycle_run(ctypes.byref(d), D.stream()))

    # -- readback -----------------------------------------------------------
    def read(self, rn2_dtype=np.float64, with_cycle=True) -> Readout:
        """One pinned D2H copy of the control block + stream sync."""
        self.host.copy_(self.ctlbuf, non_blocking=True)
        if HOST_STATS["on"]:
            t0 = time.perf_counter()
            D.sync()
            HOST_STATS["sync_s"] += time.perf_counter() - t0
            HOST_STATS["reads"] += 1
        else:
            D.sync()
        raw = self.host.numpy()
        rn2 = float(np.frombuffer(raw, dtype=rn2_dtype, count=1, offset=OFF_RN2)[0])
        rn2_low = float(np.frombuffer(raw, dtype=np.float32, count=1, offset=OFF_RN2_LOW)[0])
        changed = bool(np.frombuffer(raw, dtype=np.int32, count=1, offset=OFF_CHANGED)[0])
        if not with_cycle:
            return Readout(0, [], False, rn2, rn2_low, changed)
        head = np.frombuffer(raw, dtype=np.int32, count=6, offset=0)
        steps = int(head[1])
        if head[3]:
            tri = np.frombuffer(raw, dtype=np.float64, count=2, offset=24)
            raise TriangularBreakdownError(int(head[4]), float(tri[0]), float(tri[1]))
        imp = np.frombuffer(raw, dtype=np.float64, count=steps, offset=56).tolist()
        return Readout(steps, imp, bool(head[2]), rn2, rn2_low, changed)

    def bn2(self, dtype) -> float:
        return float(np.frombuffer(self.host.numpy(), dtype=dtype, count=1, offset=OFF_BN2)[0])

    def basis_host(self, k):
        """First k+... columns of V as an (n, k) Fortran array (diagnostics)."""
        V = self.V.view(self.m + 1, self.ld)[:k, : self.n]
        return np.asfortranarray(D.to_host(V).T)

    def raw_hessenberg(self, k):
        m = self.m
        t = self.prec.torch_dtype
        sv = 4 if self.prec is Precision.binary32 else 8
        off = ((m + 1) * m + m + m + (m + 1) + m)
        flat = self.hess[: (off + (m + 1) * m) * sv].view(t)
        raw = flat[off: off + (m + 1) * m].view(m, m + 1)   # [col][row]
        return D.to_host(raw[:k, : k + 1].t()).astype(np.float64)


def releases_l2(fn):
    """Solve-driver decorator: after the solve, return the L2 lines the cycle
    kernels' access-policy window marked persisting to normal status
    (mpk_l2_release), so the set-aside is free for whatever runs next."""
    import functools

    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        try:
            return fn(*args, **kwargs)
        finally:
            try:
                D.lib().mpk_l2_release()
            except _lib.NativeUnavailable:
                pass

    return wrapper


def sqrt_in(prec: Precision, v: float) -> float:
    """float(np.sqrt(v)) with the square root taken in prec (norm2's rounding)."""
    return float(np.sqrt(prec.dtype.type(v)))
