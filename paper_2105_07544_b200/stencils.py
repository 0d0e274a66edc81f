"""Regular-grid test problems (reference: pkg/src/mpkrylov/stencils.py).

Assembly is host setup (outside the timed region, as in the reference
harness); it reproduces the reference's arrays bit for bit (pinned by
tests/golden/stencils.json).  The returned matrix also carries its stencil
description, so the device applies it matrix-free with the same arithmetic.
Node (ix, iy[, iz]) is row ix + nx*iy (+ nx^2*iz); columns of a row follow
the displacement order, and out-of-grid neighbours are dropped (Dirichlet).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .sparse import CsrMatrix, StencilInfo

__all__ = ["PRESETS", "ProblemSpec", "generate_stencil", "stencil_dimensions"]

PRESETS = ("Laplace2D", "Laplace3D", "UniFlow2D", "BentPipe2D", "Stretched2D")


@dataclass(frozen=True)
class ProblemSpec:
    """Preset name, interior points per axis and physics parameters."""

    preset: str
    nx: int
    diffusion: float = 1.0
    velocity: float = 1.0
    convection_strength: float = 100.0
    stretch_factor: float = 50.0

    def __post_init__(self):
        if self.preset not in PRESETS:
            raise ValueError("unknown preset %r (choose from %s)" % (self.preset, ", ".join(PRESETS)))
        if int(self.nx) != self.nx or self.nx < 2:
            raise ValueError("nx must be an integer >= 2")
        if self.preset == "UniFlow2D" and self.diffusion <= 0:
            raise ValueError("diffusion must be positive")
        if self.preset == "Stretched2D" and self.stretch_factor <= 0:
            raise ValueError("stretch_factor must be positive")

    @property
    def n(self) -> int:
        return self.nx ** 3 if self.preset == "Laplace3D" else self.nx ** 2


def _layout(spec: ProblemSpec):
    """(displacements, validity mask [n, w]) of the preset's stencil."""
    nx = spec.nx
    n = spec.n
    node = np.arange(n, dtype=np.int64)
    ix = node % nx
    if spec.preset == "Laplace3D":
        iy, iz = (node // nx) % nx, node // (nx * nx)
        disp = np.array([-nx * nx, -nx, -1, 0, 1, nx, nx * nx], dtype=np.int64)
        cols = [iz > 0, iy > 0, ix > 0, None, ix < nx - 1, iy < nx - 1, iz < nx - 1]
    else:
        iy = node // nx
        w, e, s, nn = ix > 0, ix < nx - 1, iy > 0, iy < nx - 1
        if spec.preset == "Stretched2D":
            disp = np.array([-nx - 1, -nx, -nx + 1, -1, 0, 1, nx - 1, nx, nx + 1], dtype=np.int64)
            cols = [w & s, s, e & s, w, None, e, w & nn, nn, e & nn]
        else:
            disp = np.array([-nx, -1, 0, 1, nx], dtype=np.int64)
            cols = [s, w, None, e, nn]
    full = np.ones(n, dtype=bool)
    mask = np.column_stack([full if c is None else c for c in cols])
    return node, ix, disp, mask


def _values(spec: ProblemSpec, node, ix):
    """Per-entry coefficients [n, w] in binary64, reference formulas and order."""
    nx, n = spec.nx, spec.n
    if spec.preset == "Laplace3D":
        return np.broadcast_to(np.array([-1.0, -1.0, -1.0, 6.0, -1.0, -1.0, -1.0]), (n, 7))
    if spec.preset == "Laplace2D":
        return np.broadcast_to(np.array([-1.0, -1.0, 4.0, -1.0, -1.0]), (n, 5))
    h = 1.0 / (nx + 1)
    if spec.preset == "Stretched2D":
        a, b = 1.0 / spec.stretch_factor, float(spec.stretch_factor)
        k, ew, ns = -(a + b) / 2.0, b - 2.0 * a, a - 2.0 * b
        return np.broadcast_to(np.array([k, ns, k, ew, 4.0 * (a + b), ew, k, ns, k]), (n, 9))
    if spec.preset == "UniFlow2D":
        d = spec.diffusion
        vel = spec.velocity / np.sqrt(2.0)
        lo, hi = -d - 0.5 * h * vel, -d + 0.5 * h * vel
        return np.broadcast_to(np.array([lo, lo, 4.0 * d, hi, hi]), (n, 5))
    # BentPipe2D: v = c * (2y(1 - x^2), -2x(1 - y^2)) sampled at the node
    c = spec.convection_strength
    px = (ix + 1) * h
    py = (node // nx + 1) * h
    ux = c * 2.0 * py * (1.0 - px * px)
    uy = -c * 2.0 * px * (1.0 - py * py)
    out = np.empty((n, 5))
    out[:, 0] = -1.0 - 0.5 * h * uy
    out[:, 1] = -1.0 - 0.5 * h * ux
    out[:, 2] = 4.0
    out[:, 3] = -1.0 + 0.5 * h * ux
    out[:, 4] = -1.0 + 0.5 * h * uy
    return out


def stencil_dimensions(spec: ProblemSpec):
    """(n, nnz) from the validity masks alone (reference stencils.py:182-189)."""
    _, _, _, mask = _layout(spec)
    return spec.n, int(mask.sum())


def generate_stencil(spec: ProblemSpec, on_device: bool = False) -> CsrMatrix:
    """Assemble the preset in binary64 (reference stencils.py:192-207).

    on_device=True assembles on the GPU (``mpk_stencil_assemble``: entry
    counts, a scan, then every row's entries with the operator's own
    coefficient arithmetic) and keeps the device copy; the host arrays are
    the same bits as the numpy assembly (tests/test_gpu_assembly.py)."""
    if on_device:
        return _generate_on_device(spec)
    node, ix, disp, mask = _layout(spec)
    vals = _values(spec, node, ix)
    keep = mask.ravel()
    col_idx = (node[:, None] + disp[None, :]).ravel()[keep]
    values = np.ascontiguousarray(np.asarray(vals).ravel()[keep], dtype=np.float64)
    row_ptr = np.zeros(spec.n + 1, dtype=np.int64)
    np.cumsum(mask.sum(axis=1), out=row_ptr[1:])
    A = CsrMatrix(spec.n, row_ptr, col_idx, values, validate=False)
    A.stencil = StencilInfo(spec.preset, spec.nx, spec.diffusion, spec.velocity,
                            spec.convection_strength, spec.stretch_factor)
    return A


_WIDTH = {"Laplace2D": 5, "Laplace3D": 7, "UniFlow2D": 5, "BentPipe2D": 5, "Stretched2D": 9}


def _generate_on_device(spec: ProblemSpec) -> CsrMatrix:
    import ctypes

    from . import _lib
    from . import device as D
    from .sparse import _DeviceCsr

    t = D.torch()
    n = spec.n
    info = StencilInfo(spec.preset, spec.nx, spec.diffusion, spec.velocity, spec.convection_strength,
                       spec.stretch_factor)
    d = _lib.MpkMatrix()
    d.kind, d.dtype, d.n, d.row0 = _lib.STENCIL, _lib.F64, n, 0
    d.preset, d.nx = _lib.PRESET_IDS[spec.preset], spec.nx
    d.diffusion, d.velocity, d.convection, d.stretch = info.diffusion, info.velocity, info.convection, info.stretch
    cap = _WIDTH[spec.preset] * n
    rp = D.empty(n + 1, t.int64)
    ci = D.empty(cap, t.int32)
    va = D.empty(cap, t.float64)
    lib = D.lib()
    ws = D.empty(int(lib.mpk_stencil_assemble_ws_bytes(n)), t.uint8)
    _lib.check(lib.mpk_stencil_assemble(ctypes.byref(d), D.ptr(rp), D.ptr(ci), D.ptr(va), D.ptr(ws), D.stream()))
    row_ptr = D.to_host(rp)
    nnz = int(row_ptr[-1])
    ci, va = ci[:nnz], va[:nnz]
    A = CsrMatrix(n, row_ptr, D.to_host(ci).astype(np.int64), D.to_host(va), validate=False)
    A.stencil = info
    A._dev = _DeviceCsr(rp.to(t.int32), ci, va)
    return A
