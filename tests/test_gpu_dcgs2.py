"""The lagged one-reduction CGS2 cycle (SolverConfig.orthogonalization =
"dcgs2") is the reference's CGS2 Arnoldi reordered (fused_dcgs2.cuh): same
Hessenberg in exact arithmetic.  Bars: implicit-residual histories of one
cycle agree with the CGS2 kernel to rounding, restarted / IR solves converge
to 1e-10 with iteration counts within one restart cycle of CGS2's (equal on
the reference goldens that have margin)."""

import numpy as np
import pytest

import paper_2105_07544_b200 as mk

pytestmark = pytest.mark.gpu
P = mk.Precision


def L(preset, nx):
    return mk.generate_stencil(mk.ProblemSpec(preset, nx))


@pytest.mark.parametrize("preset,nx,prec,tol", [("BentPipe2D", 64, P.binary64, 1e-8),
                                                 ("Laplace3D", 16, P.binary64, 1e-8),
                                                 ("UniFlow2D", 48, P.binary64, 1e-8),
                                                 ("BentPipe2D", 64, P.binary32, 2e-3)])
def test_one_cycle_history_matches_cgs2(cuda, preset, nx, prec, tol):
    A = mk.convert_matrix(L(preset, nx), prec)
    b = np.ones(A.n, prec.dtype)
    # fp32: exit at 1e-5, above the cycle's attainable accuracy
    cfg = dict(m=40, rtol=1e-300 if prec is P.binary64 else 1e-5, precision=prec, breakdown_rule="u")
    x1, s1 = mk.gmres_cycle(A, None, b, np.zeros(A.n, prec.dtype), mk.SolverConfig(**cfg))
    x2, s2 = mk.gmres_cycle(A, None, b, np.zeros(A.n, prec.dtype), mk.SolverConfig(orthogonalization="dcgs2", **cfg))
    assert s1.steps == s2.steps
    h1, h2 = np.array(s1.implicit_relres), np.array(s2.implicit_relres)
    keep = h1 > (1e-12 if prec is P.binary64 else 1e-4)
    assert np.all(np.abs(h1 - h2)[keep] <= tol * h1[keep]), np.max(np.abs(h1 - h2)[keep] / h1[keep])
    assert np.abs(x1 - x2).max() <= (1e-9 if prec is P.binary64 else 1e-3) * np.abs(x1).max()


def test_restarted_counts(cuda, runs):
    for name, (preset, nx) in {"gmres_l2d32_m50": ("Laplace2D", 32), "gmres_bp64": ("BentPipe2D", 64),
                               "gmres_uf48": ("UniFlow2D", 48)}.items():
        A = L(preset, nx)
        rep = mk.gmres_restarted(A, None, np.ones(A.n), np.zeros(A.n),
                                 mk.SolverConfig(m=50, rtol=1e-10, orthogonalization="dcgs2"))
        g = runs[name]
        assert rep.converged and rep.final_explicit_relres <= 1e-10
        assert abs(rep.total_iters - g["iters"]) <= 50, (name, rep.total_iters, g["iters"])


def test_ir_converges_like_cgs2(cuda):
    for preset, nx in (("BentPipe2D", 96), ("Laplace3D", 24)):
        A = L(preset, nx)
        reps = []
        for orth in ("cgs2", "dcgs2"):
            inner = mk.SolverConfig(m=50, rtol=1e-4, precision=P.binary32, orthogonalization=orth, max_iters=20000)
            reps.append(mk.gmres_ir(A, np.ones(A.n), np.zeros(A.n), mk.IrConfig(inner=inner, rtol=1e-10)))
        assert all(r.converged and r.final_explicit_relres <= 1e-10 for r in reps)
        assert abs(reps[0].total_iters - reps[1].total_iters) <= 50, (reps[0].total_iters, reps[1].total_iters)


def test_lucky_breakdown_detected(cuda):
    # b = ones on a 4x4 Laplacian spans a 3-dimensional Krylov space
    A = L("Laplace2D", 4)
    cfg = mk.SolverConfig(m=10, rtol=1e-300, orthogonalization="dcgs2")
    _, st = mk.gmres_cycle(A, None, np.ones(16), np.zeros(16), cfg)
    _, st2 = mk.gmres_cycle(A, None, np.ones(16), np.zeros(16), mk.SolverConfig(m=10, rtol=1e-300))
    assert st.breakdown and st2.breakdown and st.steps == st2.steps


def test_jacobi1_lagged_matches_cgs2(cuda):
    """Block Jacobi k=1 inside the lagged cycle (SpMV input M u, correction
    x0 + M V d): same convergence as the CGS2 kernel."""
    A = mk.synthetic_irregular(12000, band=300, signs="negative", dominance=1.01, shift=1e-3)
    b = np.ones(A.n)
    J = mk.build_block_jacobi(A, 1)
    r1 = mk.gmres_restarted(A, J, b, np.zeros(A.n), mk.SolverConfig(m=50, rtol=1e-10, max_iters=5000))
    r2 = mk.gmres_restarted(A, J, b, np.zeros(A.n), mk.SolverConfig(m=50, rtol=1e-10, max_iters=5000,
                                                                    orthogonalization="dcgs2"))
    assert r1.converged and r2.converged and abs(r1.total_iters - r2.total_iters) <= 50
    assert np.abs(r1.x - r2.x).max() <= 1e-7 * np.abs(r1.x).max()
    Al = mk.convert_matrix(A, P.binary32)
    J32 = mk.build_block_jacobi(Al, 1)
    inner = mk.SolverConfig(m=50, rtol=1e-4, precision=P.binary32, max_iters=5000, orthogonalization="dcgs2")
    ir = mk.gmres_ir(A, b, np.zeros(A.n), mk.IrConfig(inner=inner, rtol=1e-10), M=J32, A_low=Al)
    assert ir.converged and ir.final_explicit_relres <= 1e-10
