"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

CPU restatement of the reference solve path.  Each function names the
reference lines it restates.  Dense BLAS-1/2 work goes through numpy (the
reference's own third-party arithmetic: OpenBLAS ``?dot``/``?gemv``); the
sparse product is the sequential C restatement of SciPy ``csr_matvec`` in
``csr_seq.c`` (bit-exact), with a vectorised numpy restatement of the same
row-sequential order as a fallback.

Breakdown rule: ``rule="n_u"`` is the reference's
``beta <= n*u*||w||`` test (pkg/src/mpkrylov/kernels.py:122-123); ``rule="u"``
is the documented non-reference option ``beta <= u*||w||`` used only for the
large fp32 configurations.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

U32 = 2.0 ** -24
U64 = 2.0 ** -53


def unit_roundoff(dtype) -> float:
    return U32 if np.dtype(dtype) == np.float32 else U64


# ---------------------------------------------------------------------------
# sparse product (sparse.py:190-206 -> scipy csr_matvec)
# ---------------------------------------------------------------------------

def _load_c():
    global _LIB
    if _LIB is not None:
        return _LIB
    path = os.path.join(HERE, "_build", "liboracle_spmv.so")
    if not os.path.exists(path):
        try:
            subprocess.run(["make", "-s", "-C", HERE], check=True,
                           stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except Exception:
            _LIB = False
            return _LIB
    lib = ctypes.CDLL(path)
    for name in ("oracle_spmv_f64", "oracle_spmv_f32"):
        fn = getattr(lib, name)
        fn.restype = None
        fn.argtypes = [ctypes.c_int64] + [ctypes.c_void_p] * 5
    _LIB = lib
    return _LIB


def spmv_seq(row_ptr, col_idx, vals, x):
    """y = A x with scipy's row-sequential, round-every-op order."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int64)
    vals = np.ascontiguousarray(vals)
    x = np.ascontiguousarray(x, dtype=vals.dtype)
    n = rp.shape[0] - 1
    y = np.empty(n, dtype=vals.dtype)
    lib = _load_c()
    if lib:
        fn = lib.oracle_spmv_f64 if vals.dtype == np.float64 else lib.oracle_spmv_f32
        fn(n, rp.ctypes.data, ci.ctypes.data, vals.ctypes.data, x.ctypes.data, y.ctypes.data)
        return y
    return spmv_seq_numpy(rp, ci, vals, x)


def spmv_seq_numpy(row_ptr, col_idx, vals, x):
    """Same order, vectorised across rows: position p of every row at once."""
    rp = np.asarray(row_ptr, dtype=np.int64)
    n = rp.shape[0] - 1
    lens = np.diff(rp)
    acc = np.zeros(n, dtype=vals.dtype)
    for p in range(int(lens.max(initial=0))):
        live = np.flatnonzero(lens > p)
        at = rp[live] + p
        acc[live] = acc[live] + vals[at] * x[col_idx[at]]
    return acc


# ---------------------------------------------------------------------------
# problem assembly (stencils.py:73-207) and COO compression (sparse.py:128-170)
# ---------------------------------------------------------------------------

def stencil_csr(preset, nx, diffusion=1.0, velocity=1.0, convection=100.0, stretch=50.0):
    """(row_ptr int64, col_idx int64, values f64) of a preset, x-fastest."""
    if preset == "Laplace3D":
        n = nx ** 3
        node = np.arange(n, dtype=np.int64)
        gx, gy, gz = node % nx, (node // nx) % nx, node // (nx * nx)
        offs = np.array([-nx * nx, -nx, -1, 0, 1, nx, nx * nx], dtype=np.int64)
        keep = np.column_stack([gz > 0, gy > 0, gx > 0, np.ones(n, bool),
                                gx < nx - 1, gy < nx - 1, gz < nx - 1])
        coef = np.broadcast_to(np.array([-1.0, -1.0, -1.0, 6.0, -1.0, -1.0, -1.0]), (n, 7))
    else:
        n = nx * nx
        node = np.arange(n, dtype=np.int64)
        gx, gy = node % nx, node // nx
        h = 1.0 / (nx + 1)
        if preset == "Stretched2D":
            a = 1.0 / stretch
            b = float(stretch)
            cc = -(a + b) / 2.0
            ew = b - 2.0 * a
            ns = a - 2.0 * b
            offs = np.array([-nx - 1, -nx, -nx + 1, -1, 0, 1, nx - 1, nx, nx + 1], dtype=np.int64)
            W, E, S, N = gx > 0, gx < nx - 1, gy > 0, gy < nx - 1
            keep = np.column_stack([W & S, S, E & S, W, np.ones(n, bool), E, W & N, N, E & N])
            coef = np.broadcast_to(np.array([cc, ns, cc, ew, 4.0 * (a + b), ew, cc, ns, cc]), (n, 9))
        else:
            offs = np.array([-nx, -1, 0, 1, nx], dtype=np.int64)
            keep = np.column_stack([gy > 0, gx > 0, np.ones(n, bool), gx < nx - 1, gy < nx - 1])
            if preset == "Laplace2D":
                coef = np.broadcast_to(np.array([-1.0, -1.0, 4.0, -1.0, -1.0]), (n, 5))
            elif preset == "UniFlow2D":
                d = diffusion
                vxy = velocity / np.sqrt(2.0)
                coef = np.broadcast_to(np.array([-d - 0.5 * h * vxy, -d - 0.5 * h * vxy, 4.0 * d,
                                                 -d + 0.5 * h * vxy, -d + 0.5 * h * vxy]), (n, 5))
            elif preset == "BentPipe2D":
                c = convection
                px = (gx + 1) * h
                py = (gy + 1) * h
                ux = c * 2.0 * py * (1.0 - px * px)
                uy = -c * 2.0 * px * (1.0 - py * py)
                coef = np.empty((n, 5))
                coef[:, 0] = -1.0 - 0.5 * h * uy
                coef[:, 1] = -1.0 - 0.5 * h * ux
                coef[:, 2] = 4.0
                coef[:, 3] = -1.0 + 0.5 * h * ux
                coef[:, 4] = -1.0 + 0.5 * h * uy
            else:
                raise ValueError(preset)
    flat = keep.reshape(-1)
    cols = (node[:, None] + offs[None, :]).reshape(-1)[flat]
    vals = np.ascontiguousarray(np.asarray(coef).reshape(-1)[flat], dtype=np.float64)
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(keep.sum(axis=1), out=rp[1:])
    return rp, cols, vals


def coo_compress(rows, cols, vals, n):
    """Sort by (row, col), sum duplicates in the value dtype (sparse.py:155-170)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals)
    if rows.size == 0:
        return np.zeros(n + 1, np.int64), np.zeros(0, np.int64), np.zeros(0, vals.dtype)
    order = np.lexsort((cols, rows))
    r, c, v = rows[order], cols[order], vals[order]
    head = np.ones(r.size, dtype=bool)
    head[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
    starts = np.flatnonzero(head)
    summed = np.add.reduceat(v, starts).astype(v.dtype, copy=False)
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(r[starts], minlength=n), out=rp[1:])
    return rp, c[starts], summed


# ---------------------------------------------------------------------------
# CGS2 and the rotated least-squares state (kernels.py:98-216)
# ---------------------------------------------------------------------------

def nrm(x):
    """sqrt(x.x) in x's dtype (kernels.py:37-41)."""
    return np.sqrt(np.dot(x, x))


def cgs2_step(V, count, w, rule="n_u"):
    """Two classical Gram-Schmidt passes against V[:, :count] (kernels.py:114-126).

    Returns (coeffs, beta, appended, new_column_or_None)."""
    n = w.shape[0]
    u = unit_roundoff(w.dtype)
    w_norm = nrm(w)
    Q = V[:, :count]
    c1 = Q.T @ w
    w = w - Q @ c1
    c2 = Q.T @ w
    w = w - Q @ c2
    beta = nrm(w)
    limit = (n * u if rule == "n_u" else u) * float(w_norm)
    ok = float(beta) > limit
    return c1 + c2, beta, ok, (w / beta if ok else None)


class RotatedLsq:
    """Givens-rotated Hessenberg state (kernels.py:139-216), one dtype throughout."""

    def __init__(self, m, gamma, scale, dtype):
        self.t = np.dtype(dtype)
        self.R = np.zeros((m + 1, m), dtype=self.t)
        self.cs = np.zeros(m, dtype=self.t)
        self.sn = np.zeros(m, dtype=self.t)
        self.g = np.zeros(m + 1, dtype=self.t)
        self.g[0] = gamma
        self.scale = float(scale)
        self.k = 0

    def push(self, coeffs, beta):
        """Fold the next column in; returns |g_k| / scale (kernels.py:166-196)."""
        j = self.k + 1
        t = self.t
        col = np.zeros(self.R.shape[0], dtype=t)
        col[:j] = coeffs
        col[j] = beta
        for i in range(j - 1):
            top = self.cs[i] * col[i] + self.sn[i] * col[i + 1]
            col[i + 1] = -self.sn[i] * col[i] + self.cs[i] * col[i + 1]
            col[i] = top
        a, b = col[j - 1], col[j]
        if b == 0:
            c, s, r = t.type(1.0), t.type(0.0), a
        else:
            r = np.hypot(a, b)
            c, s = a / r, b / r
        self.cs[j - 1], self.sn[j - 1] = c, s
        col[j - 1], col[j] = r, 0
        self.g[j] = -s * self.g[j - 1]
        self.g[j - 1] = c * self.g[j - 1]
        self.R[:, j - 1] = col
        self.k = j
        return float(np.abs(self.g[j])) / self.scale

    def back_solve(self, k):
        """Upper-triangular solve with the k*u*max|diag| guard (kernels.py:202-216).

        Returns (d, None) or (None, (index, entry, threshold))."""
        import scipy.linalg

        T = self.R[:k, :k]
        dg = np.abs(np.diagonal(T))
        lim = k * unit_roundoff(self.t) * float(dg.max(initial=0.0))
        if dg.size == 0 or float(dg.min()) <= lim:
            i = int(np.argmin(dg))
            return None, (i, float(dg[i]), lim)
        return scipy.linalg.solve_triangular(T, self.g[:k], lower=False), None


# ---------------------------------------------------------------------------
# preconditioners (preconditioners.py:96-305)
# ---------------------------------------------------------------------------

@dataclass
class Jacobi:
    starts: np.ndarray
    factors: list
    dtype: np.dtype

    def __call__(self, v):
        import scipy.linalg

        out = np.empty_like(v)
        for i, (lu, piv) in enumerate(self.factors):
            s, e = int(self.starts[i]), int(self.starts[i + 1])
            out[s:e] = scipy.linalg.lu_solve((lu, piv), v[s:e], check_finite=False)
        return out


def jacobi_build(rp, ci, vals, k, dtype):
    """Dense k-by-k diagonal blocks, LU with partial pivoting (preconditioners.py:96-130).

    Returns Jacobi or raises ValueError('singular', block, pivot, threshold)."""
    import warnings

    import scipy.linalg

    n = rp.shape[0] - 1
    dtype = np.dtype(dtype)
    starts = np.append(np.arange(0, n, k, dtype=np.int64), n)
    facs = []
    for bi in range(starts.size - 1):
        s, e = int(starts[bi]), int(starts[bi + 1])
        blk = np.zeros((e - s, e - s), dtype=dtype)
        for row in range(s, e):
            lo, hi = rp[row], rp[row + 1]
            cc = ci[lo:hi]
            a0, a1 = np.searchsorted(cc, s), np.searchsorted(cc, e)
            blk[row - s, cc[a0:a1] - s] = vals[lo + a0:lo + a1].astype(dtype, copy=False)
        lim = (e - s) * unit_roundoff(dtype) * float(np.abs(blk).sum(axis=1).max())
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            lu, piv = scipy.linalg.lu_factor(blk, check_finite=False)
        piv_abs = np.abs(np.diagonal(lu))
        if float(piv_abs.min()) <= lim:
            raise ValueError("singular", bi, float(piv_abs.min()), lim)
        facs.append((lu, piv))
    return Jacobi(starts, facs, dtype)


def harmonic_ritz(hbar):
    """preconditioners.py:171-185."""
    d = hbar.shape[1]
    H = hbar[:d, :]
    e = np.zeros(d)
    e[-1] = 1.0
    f = np.linalg.solve(H.T, e)
    aug = H.copy()
    aug[:, -1] += (hbar[d, d - 1] ** 2) * f
    return np.linalg.eigvals(aug)


def leja_order(roots):
    """Modified Leja order, conjugate pairs adjacent, +imag first (preconditioners.py:188-223)."""
    pool = list(np.asarray(roots, dtype=np.complex128))
    out = []

    def pick(i):
        z = pool.pop(i)
        if z.imag == 0:
            out.append(z)
            return
        if z.imag < 0:
            z = np.conj(z)
        out.append(z)
        mate = np.conj(z)
        j = min(range(len(pool)), key=lambda t: abs(pool[t] - mate))
        pool.pop(j)
        out.append(mate)

    pick(int(np.argmax(np.abs(pool))))
    while pool:
        arr = np.asarray(pool)
        with np.errstate(divide="ignore"):
            score = np.zeros(arr.shape[0])
            for z in out:
                score += np.log(np.abs(arr - z))
        pick(int(np.argmax(score)))
    return np.asarray(out, dtype=np.complex128)


@dataclass
class Poly:
    roots: np.ndarray
    degree: int
    requested: int
    truncated: bool
    rp: np.ndarray
    ci: np.ndarray
    vals: np.ndarray

    def __call__(self, v):
        """Product form p(A) v (preconditioners.py:276-305)."""
        acc = np.zeros_like(v)
        work = v.copy()
        i = 0
        while i < self.degree:
            z = self.roots[i]
            if z.imag == 0:
                inv = float(1.0 / z.real)
                acc += inv * work
                work = work - inv * spmv_seq(self.rp, self.ci, self.vals, work)
                i += 1
            else:
                tr = float(2.0 * z.real)
                m2 = float(z.real * z.real + z.imag * z.imag)
                t = spmv_seq(self.rp, self.ci, self.vals, work)
                acc += (tr * work - t) / m2
                work = work - (tr * t - spmv_seq(self.rp, self.ci, self.vals, t)) / m2
                i += 2
        return acc


def poly_build(rp, ci, vals, degree, seed, rule="n_u"):
    """d Arnoldi steps in the matrix dtype, then harmonic Ritz + Leja (preconditioners.py:226-273)."""
    n = rp.shape[0] - 1
    dt = vals.dtype
    gam = nrm(seed)
    V = np.zeros((n, degree + 1), dtype=dt, order="F")
    V[:, 0] = seed / gam
    cnt = 1
    cols = []
    trunc = False
    for j in range(degree):
        w = spmv_seq(rp, ci, vals, V[:, j])
        coeffs, beta, ok, q = cgs2_step(V, cnt, w, rule)
        cols.append((np.asarray(coeffs, dtype=np.float64), float(beta)))
        if not ok:
            trunc = True
            break
        V[:, cnt] = q
        cnt += 1
    d = len(cols)
    hbar = np.zeros((d + 1, d))
    for i, (cf, bt) in enumerate(cols):
        hbar[: i + 1, i] = cf
        hbar[i + 1, i] = bt
    roots = leja_order(harmonic_ritz(hbar))
    return Poly(roots, d, degree, trunc, rp, ci, vals)


def cast_wrap(inner, low, high):
    """CastApplyPreconditioner._apply (multiprecision.py:306-308)."""
    return lambda v: inner(v.astype(low)).astype(high)


# ---------------------------------------------------------------------------
# solvers (gmres.py:134-308, multiprecision.py:120-288)
# ---------------------------------------------------------------------------

@dataclass
class Outcome:
    converged: bool
    iters: int
    restarts: int
    relres: float
    history: list            # (iteration, phase, implicit, explicit)
    loss: bool
    x: np.ndarray
    baseline: float
    stalled: bool = False
    phases: dict = field(default_factory=dict)


@dataclass
class CycleOut:
    steps: int
    implicit: list
    scale: float
    breakdown: bool


def basis16_scale(n):
    """Power-of-two scale of the binary16 basis: 2^round(log2(sqrt(n)))."""
    return float(2.0 ** np.rint(0.5 * np.log2(max(n, 1))))


def round16(v, s):
    """Stored value of a binary16 basis entry: half(v*s) read back as v' = half/s
    (this repo's third precision, SolverConfig.basis_precision; not in the
    reference -- PAPER.md:441 future work)."""
    return ((v * np.float32(s)).astype(np.float16).astype(np.float32) / np.float32(s)).astype(v.dtype)


def round_bf16(v, s):
    """Stored value of a bfloat16 basis entry (round to nearest even on the
    upper 16 bits of the float32 v*s), read back as v' = bf16/s."""
    f = (v * np.float32(s)).astype(np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return ((r.astype(np.uint32).view(np.float32)) / np.float32(s)).astype(v.dtype)


def one_cycle(A, M, b, x0, m, tol, r0=None, scale=None, cap=None, rule="n_u", basis16=False):
    """gmres_cycle (gmres.py:134-205). A = (rp, ci, vals); M callable or None.
    basis16: store the basis columns rounded to binary16 (True / "binary16",
    round16) or bfloat16 ("bfloat16", round_bf16)."""
    rp, ci, vals = A
    dt = vals.dtype
    Mf = M if M is not None else (lambda v: v)
    if float(nrm(b)) == 0.0:
        raise ZeroDivisionError("zero rhs")
    r = b - spmv_seq(rp, ci, vals, x0) if r0 is None else r0
    gam = nrm(r)
    sc = float(gam) if scale is None else float(scale)
    steps_cap = m if cap is None else max(1, min(m, int(cap)))
    if float(gam) == 0.0:
        return x0.copy(), CycleOut(0, [], sc if sc > 0 else 1.0, False)
    n = b.shape[0]
    s16 = basis16_scale(n)
    V = np.zeros((n, steps_cap + 1), dtype=dt, order="F")
    rnd = (lambda v: round_bf16(v, s16)) if basis16 == "bfloat16" else (lambda v: round16(v, s16))
    V[:, 0] = rnd(r / gam) if basis16 else r / gam
    cnt = 1
    lsq = RotatedLsq(steps_cap, gam, sc, dt)
    rels = []
    brk = False
    k = 0
    while k < steps_cap:
        w = spmv_seq(rp, ci, vals, Mf(V[:, k]))
        coeffs, beta, ok, q = cgs2_step(V, cnt, w, rule)
        if ok:
            V[:, cnt] = rnd(q) if basis16 else q
            cnt += 1
        rel = lsq.push(coeffs, beta)
        rels.append(rel)
        k += 1
        if not ok:
            brk = True
            break
        if rel <= tol:
            break
    d, err = lsq.back_solve(k)
    if err is not None:
        raise ArithmeticError("triangular breakdown", *err)
    x = x0 + Mf(V[:, :k] @ d)
    return x, CycleOut(k, rels, sc, brk)


def dcgs2_cycle(A, M, b, x0, m, tol, r0=None, scale=None, cap=None, rule="n_u", basis16=False):
    """gmres_cycle with this repo's lagged one-reduction CGS2
    (SolverConfig.orthogonalization = "dcgs2"; not a reference feature: the
    reference's CGS2 of kernels.py:98-126 reordered so each step needs one
    reduction, fused_dcgs2.cuh).  Step j, with Q_j final and the candidate
    u = w_{j-1} - Q_j c after its first pass:
      z = A u ; X0 = Q_j^T u ; X1 = Q_j^T z ; a = u.u ; b = u.z
      rho = sqrt(a - X0.X0)      (clamped at 1e-3 a / 1e-11 a: cycle ends)
      H[:, j-1] = [c + X0; rho]  (the append test on ||w_{j-1}||^2 = a + c.c)
      t = (b - X0.X1)/rho, tau = t/rho, c' = ([X1; t] - H X0)/rho
      q_j = (u - Q_j X0)/rho ; u' = (z - Q_j (X1 - X0 tau) - u tau)/rho
    (the last two scaled by 1/rho, as the kernel does)
    basis16 as in one_cycle (q_j stored rounded); M must be None."""
    assert M is None, "dcgs2 restatement: identity preconditioner"
    rp, ci, vals = A
    dt = vals.dtype
    sp = lambda x: spmv_seq(rp, ci, vals, x)
    r = b - sp(x0) if r0 is None else r0
    gam = nrm(r)
    sc = float(gam) if scale is None else float(scale)
    steps_cap = m if cap is None else max(1, min(m, int(cap)))
    if float(gam) == 0.0:
        return x0.copy(), CycleOut(0, [], sc if sc > 0 else 1.0, False)
    n = b.shape[0]
    u_rnd = unit_roundoff(dt)
    s16 = basis16_scale(n)
    rnd = (lambda v: round_bf16(v, s16)) if basis16 == "bfloat16" else (lambda v: round16(v, s16))
    store = rnd if basis16 else (lambda v: v)
    eta = dt.type(1e-3 if dt == np.float32 else 1e-11)
    Q = np.zeros((n, steps_cap + 1), dtype=dt, order="F")
    H = np.zeros((steps_cap + 1, steps_cap), dtype=dt)
    Q[:, 0] = store(r / gam)
    w = sp(Q[:, 0])
    c = Q[:, :1].T @ w
    u = w - Q[:, :1] @ c
    lsq = RotatedLsq(steps_cap, gam, sc, dt)
    rels = []
    brk = False
    k = 0
    for j in range(1, steps_cap + 1):
        z = sp(u)
        X0 = Q[:, :j].T @ u
        X1 = Q[:, :j].T @ z
        a, bb = np.dot(u, u), np.dot(u, z)
        rho2 = a - np.dot(X0, X0)
        trunc = not rho2 > eta * a
        if trunc:
            rho2 = eta * a
        rho = np.sqrt(rho2)
        H[:j, j - 1] = c + X0
        H[j, j - 1] = rho
        limit = (n * u_rnd if rule == "n_u" else u_rnd) * float(np.sqrt(a + np.dot(c, c)))
        ok = float(rho) > limit
        rel = lsq.push(H[:j, j - 1], rho)
        rels.append(rel)
        k = j
        if not ok:
            brk = True
            break
        if rel <= tol or trunc or j == steps_cap:
            break
        t = (bb - np.dot(X0, X1)) / rho
        tau = t / rho
        c = (np.append(X1, t) - H[:j + 1, :j] @ X0) / rho
        ri = dt.type(1) / rho   # the kernel scales q and u' by 1/rho (fused_dcgs2.cuh dc_phase_u)
        Q[:, j] = store((u - Q[:, :j] @ X0) * ri)
        u = (z - Q[:, :j] @ (X1 - X0 * tau) - u * tau) * ri
    d, err = lsq.back_solve(k)
    if err is not None:
        raise ArithmeticError("triangular breakdown", *err)
    return x0 + Q[:, :k] @ d, CycleOut(k, rels, sc, brk)


def restarted(A, M, b, x0, m=50, rtol=1e-10, max_iters=100_000, max_restarts=1_000_000,
              baseline=None, restart_on_loss=True, phase=None, rule="n_u"):
    """gmres_restarted (gmres.py:221-308)."""
    rp, ci, vals = A
    dt = vals.dtype
    if float(nrm(b)) == 0.0:
        raise ZeroDivisionError("zero rhs")
    if phase is None:
        phase = "double" if dt == np.float64 else "single"
    x = x0.astype(dt, copy=True)
    r = b - spmv_seq(rp, ci, vals, x)
    own = float(nrm(r))
    sc = own if baseline is None else float(baseline)
    hist = [(0, phase, None, own / sc if sc else 0.0)]
    if own == 0.0:
        return Outcome(True, 0, 0, 0.0, hist, False, x, sc, phases={phase: 0})
    total = restarts = 0
    loss = conv = False
    expl = own / sc
    while True:
        if expl <= rtol:
            conv = True
            break
        left = max_iters - total
        if left <= 0 or restarts >= max_restarts:
            break
        x, st = one_cycle(A, M, b, x, m, rtol, r0=r, scale=sc, cap=left, rule=rule)
        hist.extend((total + i + 1, phase, rel, None) for i, rel in enumerate(st.implicit))
        total += st.steps
        restarts += 1
        r = b - spmv_seq(rp, ci, vals, x)
        expl = float(nrm(r)) / sc
        if st.steps:
            it, ph, imp, _ = hist[-1]
            hist[-1] = (it, ph, imp, expl)
        fin = st.implicit[-1] if st.implicit else 0.0
        now = fin <= rtol and expl > 10.0 * rtol
        loss = loss or now
        if now and not restart_on_loss:
            break
    return Outcome(conv, total, restarts, expl, hist, loss, x, sc, phases={phase: total})


def refine(A64, b, x0, m=50, rtol=1e-10, inner_max_iters=100_000, max_refinements=1_000_000,
           M=None, A32=None, rule="n_u", basis16=False, orth="cgs2"):
    """gmres_ir (multiprecision.py:120-233): fp64 outer, fp32 inner cycles
    (orth="dcgs2": inner cycles with dcgs2_cycle)."""
    cycle = dcgs2_cycle if orth == "dcgs2" else one_cycle
    rp, ci, v64 = A64
    if A32 is None:
        A32 = (rp, ci, v64.astype(np.float32))
    if float(nrm(b)) == 0.0:
        raise ZeroDivisionError("zero rhs")
    x = x0.astype(np.float64, copy=True)
    r = b - spmv_seq(rp, ci, v64, x)
    base = float(nrm(r))
    hist = [(0, "outer", None, 1.0 if base else 0.0)]
    if base == 0.0:
        return Outcome(True, 0, 0, 0.0, hist, False, x, base, phases={"inner": 0, "outer": 0})
    floor = 10.0 * U32
    z32 = np.zeros(b.shape[0], dtype=np.float32)
    expl = 1.0
    total = refs = streak = 0
    stalled = conv = False
    while True:
        if expl <= rtol:
            conv = True
            break
        if refs >= max_refinements:
            break
        left = inner_max_iters - total
        if left <= 0:
            break
        r32 = r.astype(np.float32)
        r32n = float(nrm(r32))
        if r32n == 0.0:
            refs += 1
            streak += 1
            if streak >= 2:
                stalled = True
                break
            continue
        u32, st = cycle(A32, M, r32, z32, m, floor, r0=r32, cap=left, rule=rule, basis16=basis16)
        hist.extend((total + i + 1, "inner", rel * r32n / base, None)
                    for i, rel in enumerate(st.implicit))
        total += st.steps
        refs += 1
        xn = x + u32.astype(np.float64)
        streak = streak + 1 if np.array_equal(xn, x) else 0
        x = xn
        r = b - spmv_seq(rp, ci, v64, x)
        expl = float(nrm(r)) / base
        hist.append((total, "outer", None, expl))
        if streak >= 2:
            stalled = True
            break
    return Outcome(conv, total, refs, expl, hist, False, x, base, stalled,
                   phases={"inner": total, "outer": refs})


def switch(A64, b, x0, switch_iter, m=50, rtol=1e-10, max_iters=100_000,
           M_low=None, M_high=None, A32=None, rule="n_u"):
    """gmres_fd (multiprecision.py:236-288)."""
    rp, ci, v64 = A64
    if switch_iter == 0:
        out = restarted(A64, M_high, b, x0, m, rtol, max_iters, rule=rule)
        out.phases = {"single": 0, "double": out.iters}
        return out
    if float(nrm(b)) == 0.0:
        raise ZeroDivisionError("zero rhs")
    base = float(nrm(b - spmv_seq(rp, ci, v64, x0)))
    if A32 is None:
        A32 = (rp, ci, v64.astype(np.float32))
    lo = restarted(A32, M_low, b.astype(np.float32), x0.astype(np.float32), m, rtol,
                   switch_iter, phase="single", rule=rule)
    hi = restarted(A64, M_high, b, lo.x.astype(np.float64), m, rtol, max_iters,
                   baseline=base, phase="double", rule=rule)
    off = lo.iters
    hist = list(lo.history) + [(it + off, ph, a, e) for it, ph, a, e in hi.history]
    return Outcome(hi.converged, off + hi.iters, lo.restarts + hi.restarts, hi.relres, hist,
                   lo.loss or hi.loss, hi.x, base, phases={"single": off, "double": hi.iters})


# ---------------------------------------------------------------------------
# BASELINE config 5: synthetic irregular nonsymmetric CSR (no reference generator)
# ---------------------------------------------------------------------------

def synthetic_irregular(n, seed=20240817, mean_len=49, max_len=1000, band=2000,
                        far_frac=0.01, dominance=1.1, shift=1.0, signs="random"):
    """Config-5 matrix as specified in SURVEY §8(d) (calibrated far_frac default).

    Row length 1 + Geometric(1/mean_len) clipped to max_len; off-diagonal
    columns clip(i + U[-band, band]) or, with probability far_frac, U[0, n);
    values N(0,1) (or -|N(0,1)| for signs="negative"); duplicates summed by
    COO compression; diagonal = dominance * sum|offdiag| + shift.  Returns
    (row_ptr, col_idx, values f64)."""
    rng = np.random.default_rng(seed)
    lens = np.minimum(1 + rng.geometric(1.0 / mean_len, size=n), max_len).astype(np.int64)
    off = lens - 1
    rows = np.repeat(np.arange(n, dtype=np.int64), off)
    tot = rows.size
    near = np.clip(rows + rng.integers(-band, band + 1, size=tot), 0, n - 1)
    far = rng.integers(0, n, size=tot)
    cols = np.where(rng.random(tot) < far_frac, far, near)
    vals = rng.standard_normal(tot)
    if signs == "negative":
        vals = -np.abs(vals)
    diag_mask = cols == rows
    rows, cols, vals = rows[~diag_mask], cols[~diag_mask], vals[~diag_mask]
    rp, ci, vv = coo_compress(rows, cols, vals, n)
    owner = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
    rowsum = np.bincount(owner, weights=np.abs(vv), minlength=n)
    diag = dominance * rowsum + shift
    allr = np.concatenate([owner, np.arange(n, dtype=np.int64)])
    allc = np.concatenate([ci, np.arange(n, dtype=np.int64)])
    allv = np.concatenate([vv, diag])
    return coo_compress(allr, allc, allv, n)
