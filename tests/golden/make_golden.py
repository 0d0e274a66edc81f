"""Generate the golden fixtures in tests/golden/ by running the UNMODIFIED
reference (mpkrylov, imported from /root/reference/pkg/src) in the survey
container.  The GPU box has no /root/reference, so the outputs are committed.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--big]

Writes:
  stencils.json   sha256 of (row_ptr int64, col_idx int64, values f64) per preset/nx
                  (``--big`` adds the BASELINE benchmark sizes C1-C4)
  spmv.npz        seeded SpMV inputs/outputs (fp64 and fp32) from mpkrylov.spmv
  runs.json       solver runs: counts, flags, full residual histories
  runs_x.npz      final iterates of the small runs
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)
import mpkrylov as mk  # noqa: E402
from mpkrylov import gmres as _g, kernels as _k, preconditioners as _p  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def stencil_fixture(big):
    cases = [("Laplace2D", 4), ("Laplace2D", 16), ("Laplace2D", 32), ("Laplace3D", 5),
             ("Laplace3D", 12), ("UniFlow2D", 30), ("BentPipe2D", 64), ("BentPipe2D", 17),
             ("Stretched2D", 20), ("Stretched2D", 32)]
    if big:
        cases += [("Laplace3D", 40), ("BentPipe2D", 1500), ("UniFlow2D", 2500), ("Laplace3D", 200)]
    out = {}
    for preset, nx in cases:
        A = mk.generate_stencil(mk.ProblemSpec(preset, nx))
        out["%s_%d" % (preset, nx)] = {
            "n": A.n, "nnz": A.nnz, "row_ptr": sha(A.row_ptr), "col_idx": sha(A.col_idx),
            "values": sha(A.values), "values_f32": sha(A.values.astype(np.float32)),
        }
        print("stencil", preset, nx, A.n, A.nnz, flush=True)
    return out


def random_csr(rng, n, density=0.3, dtype=np.float64):
    """Same recipe as the reference tests' conftest.random_csr."""
    mask = rng.random((n, n)) < density
    np.fill_diagonal(mask, True)
    dense = np.where(mask, rng.standard_normal((n, n)), 0.0)
    dense[np.arange(n), np.arange(n)] += float(n)
    dense = dense.astype(dtype)
    rows, cols = np.nonzero(dense)
    return mk.csr_from_coo(rows, cols, dense[rows, cols], n, dtype=dtype)


def spmv_fixture():
    rng = np.random.default_rng(7)
    arrs = {}
    mats = {
        "bentpipe64": mk.generate_stencil(mk.ProblemSpec("BentPipe2D", 64)),
        "laplace3d12": mk.generate_stencil(mk.ProblemSpec("Laplace3D", 12)),
        "stretched20": mk.generate_stencil(mk.ProblemSpec("Stretched2D", 20)),
        "uniflow30": mk.generate_stencil(mk.ProblemSpec("UniFlow2D", 30)),
        "random150": random_csr(rng, 150),
    }
    # ragged rows, an empty row and an irregular pattern
    rows = np.array([0, 0, 0, 2, 2, 3, 3, 3, 3, 4])
    cols = np.array([0, 3, 4, 1, 2, 0, 1, 3, 4, 4])
    mats["ragged5"] = mk.csr_from_coo(rows, cols, rng.standard_normal(10), 5)
    for name, A in mats.items():
        x = rng.standard_normal(A.n)
        A32 = mk.convert_matrix(A, mk.Precision.binary32)
        arrs[name + "/row_ptr"] = A.row_ptr
        arrs[name + "/col_idx"] = A.col_idx
        arrs[name + "/values"] = A.values
        arrs[name + "/x"] = x
        arrs[name + "/y64"] = mk.spmv(A, x)
        arrs[name + "/y32"] = mk.spmv(A32, x.astype(np.float32))
    np.savez_compressed(os.path.join(OUT, "spmv.npz"), **arrs)


def _report(rep, wall):
    return {
        "converged": bool(rep.converged), "iters": int(rep.total_iters),
        "restarts": int(rep.restarts), "relres": float(rep.final_explicit_relres),
        "loss": bool(rep.loss_of_accuracy), "stalled": bool(getattr(rep, "stalled", False)),
        "baseline": float(rep.baseline), "phases": dict(rep.phase_iters),
        "history": [[e.iteration, e.phase, e.implicit_relres, e.explicit_relres]
                    for e in rep.history],
        "wall": wall,
    }


def with_rule_u(fn):
    """Run fn with the non-reference breakdown rule beta <= u*||w||."""
    orig = _k.cgs2_append

    def cgs2_u(basis, w):
        # reference body (kernels.py:114-126) with threshold u*||w||
        w_norm = _k.norm2(w)
        V = basis.columns()
        c1 = V.T @ w
        w = w - V @ c1
        c2 = V.T @ w
        w = w - V @ c2
        beta = _k.norm2(w)
        appended = float(beta) > basis.precision.unit_roundoff * float(w_norm)
        if appended:
            basis.append(w / beta)
        return c1 + c2, beta, appended

    for mod in (_g, _p):
        mod.cgs2_append = cgs2_u
    try:
        return fn()
    finally:
        for mod in (_g, _p):
            mod.cgs2_append = orig


def runs_fixture(big):
    L = lambda preset, nx: mk.generate_stencil(mk.ProblemSpec(preset, nx))  # noqa: E731
    P = mk.Precision
    runs, xs = {}, {}

    def record(name, fn, keep_x=True):
        t0 = time.perf_counter()
        rep = fn()
        runs[name] = _report(rep, time.perf_counter() - t0)
        if keep_x:
            xs[name] = rep.x
        print("run", name, runs[name]["iters"], runs[name]["restarts"],
              runs[name]["converged"], "%.2fs" % runs[name]["wall"], flush=True)

    def gm(A, b, **kw):
        cfg = mk.SolverConfig(**kw)
        return lambda: mk.gmres_restarted(A, None, b.astype(cfg.precision.dtype),
                                          np.zeros(A.n, cfg.precision.dtype), cfg)

    def ir(A, b, m=50, rtol=1e-10, M=None, **kw):
        inner = mk.SolverConfig(m=m, rtol=1e-4, precision=P.binary32, max_iters=kw.pop("max_iters", 20000))
        cfg = mk.IrConfig(inner=inner, rtol=rtol, **kw)
        return lambda: mk.gmres_ir(A, b, np.zeros(A.n), cfg, M=M)

    def fd(A, b, switch, m=50):
        cfg = mk.FdConfig(switch_iter=switch,
                          low=mk.SolverConfig(m=m, rtol=1e-10, precision=P.binary32),
                          high=mk.SolverConfig(m=m, rtol=1e-10))
        return lambda: mk.gmres_fd(A, b, np.zeros(A.n), cfg)

    l16, l32 = L("Laplace2D", 16), L("Laplace2D", 32)
    record("gmres_l2d16_m50", gm(l16, np.ones(l16.n), m=50, rtol=1e-10))
    record("gmres_l2d16_m10", gm(l16, np.ones(l16.n), m=10, rtol=1e-10))
    record("gmres_l2d16_m5_cap8", gm(l16, np.ones(l16.n), m=5, rtol=1e-10, max_iters=8))
    record("gmres_l2d16_m5_r2", gm(l16, np.ones(l16.n), m=5, rtol=1e-10, max_restarts=2))
    l8_32 = mk.convert_matrix(L("Laplace2D", 8), P.binary32)
    record("gmres32_l2d8_m20", gm(l8_32, np.ones(64), m=20, rtol=1e-4, precision=P.binary32))
    for m in (25, 50, 100):
        record("gmres_l2d32_m%d" % m, gm(l32, np.ones(l32.n), m=m, rtol=1e-10))
        record("ir_l2d32_m%d" % m, ir(l32, np.ones(l32.n), m=m))
    record("ir_l2d16_m50", ir(l16, np.ones(l16.n)))
    record("ir_l2d16_cap60", ir(l16, np.ones(l16.n), max_iters=60))
    l4 = L("Laplace2D", 4)
    record("ir_stall_l2d4", ir(l4, 1e-15 * np.ones(l4.n), m=10, rtol=1e-14))
    for s in (0, 50, 100, 150, 200):
        record("fd_l2d32_s%d" % s, fd(l32, np.ones(l32.n), s))
    record("fd_l2d16_s50", fd(l16, np.ones(l16.n), 50))
    bp = L("BentPipe2D", 64)
    record("gmres_bp64", gm(bp, np.ones(bp.n), m=50, rtol=1e-10))
    record("ir_bp64", ir(bp, np.ones(bp.n)))
    uf = L("UniFlow2D", 48)
    record("gmres_uf48", gm(uf, np.ones(uf.n), m=50, rtol=1e-10))
    record("ir_uf48", ir(uf, np.ones(uf.n)))
    l3 = L("Laplace3D", 40)
    record("gmres_l3d40", gm(l3, np.ones(l3.n), m=50, rtol=1e-10), keep_x=False)
    record("ir_l3d40", ir(l3, np.ones(l3.n)), keep_x=False)
    record("ir_l3d40_rule_u", lambda: with_rule_u(ir(l3, np.ones(l3.n))), keep_x=False)

    # preconditioned runs
    st = L("Stretched2D", 32)
    b = np.ones(st.n)
    M32 = mk.build_gmres_poly(mk.convert_matrix(st, P.binary32), 20, b.astype(np.float32))
    Mw = mk.wrap_low_precision_preconditioner(M32, P.binary64)
    cfg = mk.SolverConfig(m=50, rtol=1e-10, max_iters=2000)
    record("loss_recover_st32", lambda: mk.gmres_restarted(st, Mw, b, np.zeros(st.n), cfg))
    record("loss_giveup_st32", lambda: mk.gmres_restarted(st, Mw, b, np.zeros(st.n), cfg,
                                                          explicit_restart_on_loss=False))
    runs["poly_st32_roots"] = {"roots_re": M32.data.roots.real.tolist(),
                               "roots_im": M32.data.roots.imag.tolist(),
                               "degree": M32.data.degree, "truncated": M32.data.truncated}
    rng = np.random.default_rng(7)
    b7 = rng.standard_normal(l16.n)
    Mp = mk.build_gmres_poly(l16, 10, b7)
    record("poly10_l2d16_seed7", lambda: mk.gmres_restarted(
        l16, Mp, b7, np.zeros(l16.n), mk.SolverConfig(m=50, rtol=1e-10)))
    runs["poly10_l2d16_roots"] = {"roots_re": Mp.data.roots.real.tolist(),
                                  "roots_im": Mp.data.roots.imag.tolist(),
                                  "degree": Mp.data.degree, "truncated": Mp.data.truncated}
    Mj = mk.build_block_jacobi(l16, 16)
    record("jacobi16_l2d16", lambda: mk.gmres_restarted(
        l16, Mj, np.ones(l16.n), np.zeros(l16.n), mk.SolverConfig(m=50, rtol=1e-10)))
    bp24 = L("BentPipe2D", 24)
    Mj1 = mk.build_block_jacobi(bp24, 1)
    record("jacobi1_bp24", lambda: mk.gmres_restarted(
        bp24, Mj1, np.ones(bp24.n), np.zeros(bp24.n), mk.SolverConfig(m=50, rtol=1e-10)))
    Mj32 = mk.build_block_jacobi(bp24, 1, P.binary32)
    record("ir_jacobi1_bp24", ir(bp24, np.ones(bp24.n), M=Mj32))
    Mj8 = mk.build_block_jacobi(bp24, 8, P.binary32)
    record("ir_jacobi8_bp24", ir(bp24, np.ones(bp24.n), M=Mj8))
    record("ir_poly20_st32", ir(st, b, M=M32))
    if big:
        c2 = L("BentPipe2D", 1500)
        record("ir_bp1500", ir(c2, np.ones(c2.n), max_iters=100000), keep_x=False)
    with open(os.path.join(OUT, "runs.json"), "w") as f:
        json.dump(runs, f, indent=1)
    np.savez_compressed(os.path.join(OUT, "runs_x.npz"), **xs)


def main():
    big = "--big" in sys.argv
    with open(os.path.join(OUT, "stencils.json"), "w") as f:
        json.dump(stencil_fixture(big), f, indent=1)
    spmv_fixture()
    runs_fixture(big)


if __name__ == "__main__":
    main()
