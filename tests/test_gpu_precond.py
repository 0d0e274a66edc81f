"""Preconditioner application on the GPU vs the oracle / dense solves, and
preconditioned solves vs the reference goldens."""

import numpy as np
import pytest

import paper_2105_07544_b200 as mk
from oracle import mpk_oracle as O

pytestmark = pytest.mark.gpu
P = mk.Precision


def L(preset, nx):
    return mk.generate_stencil(mk.ProblemSpec(preset, nx))


def test_identity_returns_input(cuda, rng):
    M = mk.identity(6, P.binary64)
    v = rng.standard_normal(6)
    assert M.apply(v) is v and M.kind == "identity"


def test_block_jacobi_apply(cuda, rng):
    from conftest import random_csr

    A, dense = random_csr(mk, rng, 24)
    M = mk.build_block_jacobi(A, 5)
    assert M.data.num_blocks == 5 and M.data.starts[-1] == 24
    v = rng.standard_normal(24)
    out = M.apply(v)
    for s in range(0, 24, 5):
        e = min(s + 5, 24)
        assert np.allclose(out[s:e], np.linalg.solve(dense[s:e, s:e], v[s:e]), rtol=1e-11, atol=1e-13)
    M1 = mk.build_block_jacobi(A, 1)
    assert np.array_equal(M1.apply(v), v / np.diagonal(dense))
    M32 = mk.build_block_jacobi(A, 4, precision=P.binary32)
    assert M32.apply(v.astype(np.float32)).dtype == np.float32
    with pytest.raises(mk.PrecisionMismatchError):
        M32.apply(v)


def test_singular_block_reported(cuda):
    A = mk.csr_from_coo(np.array([0, 1, 2, 2, 3, 3]), np.array([0, 1, 2, 3, 2, 3]),
                        np.array([1.0, 1.0, 1.0, 2.0, 2.0, 4.0]), 4)
    with pytest.raises(mk.SingularBlockError) as info:
        mk.build_block_jacobi(A, 2)
    assert info.value.block_index == 1


def test_poly_apply_bit_exact_given_roots(cuda, runs):
    st = L("Stretched2D", 32)
    A32 = mk.convert_matrix(st, P.binary32)
    b = np.ones(st.n, np.float32)
    M = mk.build_gmres_poly(A32, 20, b)
    g = runs["poly_st32_roots"]
    assert M.data.degree == g["degree"]
    want_roots = np.array(g["roots_re"]) + 1j * np.array(g["roots_im"])
    assert np.abs(M.data.roots - want_roots).max() <= 1e-3 * np.abs(want_roots).max()
    # apply with the reference's exact roots: bit-identical to the oracle's product form
    M.data.roots = want_roots
    M._desc = None
    v = np.random.default_rng(5).standard_normal(st.n).astype(np.float32)
    ref = O.Poly(want_roots, g["degree"], 20, False, st.row_ptr, st.col_idx,
                 st.values.astype(np.float32))
    assert np.array_equal(M.apply(v), ref(v))


def test_poly_on_identity_truncates(cuda, rng):
    n = 12
    idx = np.arange(n)
    A = mk.csr_from_coo(idx, idx, np.ones(n), n)
    M = mk.build_gmres_poly(A, 5, np.ones(n))
    assert M.data.truncated and M.data.degree == 1 and M.data.requested_degree == 5
    v = rng.standard_normal(n)
    assert np.allclose(M.apply(v), v, rtol=1e-14)


def test_loss_of_accuracy_goldens(cuda, runs):
    st = L("Stretched2D", 32)
    b = np.ones(st.n)
    M32 = mk.build_gmres_poly(mk.convert_matrix(st, P.binary32), 20, b.astype(np.float32))
    W = mk.wrap_low_precision_preconditioner(M32, P.binary64)
    assert W.kind == "cast[poly]"
    cfg = mk.SolverConfig(m=50, rtol=1e-10, max_iters=2000)
    rep = mk.gmres_restarted(st, W, b, np.zeros(st.n), cfg)
    g = runs["loss_recover_st32"]
    assert rep.loss_of_accuracy and rep.converged
    assert abs(rep.total_iters - g["iters"]) <= 50
    rep = mk.gmres_restarted(st, W, b, np.zeros(st.n), cfg, explicit_restart_on_loss=False)
    assert rep.loss_of_accuracy and not rep.converged
    assert abs(rep.total_iters - runs["loss_giveup_st32"]["iters"]) <= 50


def test_preconditioned_goldens(cuda, runs):
    l16 = L("Laplace2D", 16)
    Mj = mk.build_block_jacobi(l16, 16)
    rep = mk.gmres_restarted(l16, Mj, np.ones(256), np.zeros(256), mk.SolverConfig(m=50, rtol=1e-10))
    assert rep.converged and rep.total_iters == runs["jacobi16_l2d16"]["iters"]
    bp24 = L("BentPipe2D", 24)
    Mj1 = mk.build_block_jacobi(bp24, 1)
    rep = mk.gmres_restarted(bp24, Mj1, np.ones(576), np.zeros(576), mk.SolverConfig(m=50, rtol=1e-10))
    assert rep.converged and rep.total_iters == runs["jacobi1_bp24"]["iters"]
    inner = mk.SolverConfig(m=50, rtol=1e-4, precision=P.binary32, max_iters=20000)
    for k, name in ((1, "ir_jacobi1_bp24"), (8, "ir_jacobi8_bp24")):
        Mk = mk.build_block_jacobi(bp24, k, P.binary32)
        rep = mk.gmres_ir(bp24, np.ones(576), np.zeros(576), mk.IrConfig(inner=inner, rtol=1e-10), M=Mk)
        assert rep.converged and abs(rep.total_iters - runs[name]["iters"]) <= 50
    rng = np.random.default_rng(7)
    b7 = rng.standard_normal(256)
    Mp = mk.build_gmres_poly(l16, 10, b7)
    rep = mk.gmres_restarted(l16, Mp, b7, np.zeros(256), mk.SolverConfig(m=50, rtol=1e-10))
    assert rep.converged and abs(rep.total_iters - runs["poly10_l2d16_seed7"]["iters"]) <= 1
    st = L("Stretched2D", 32)
    M32 = mk.build_gmres_poly(mk.convert_matrix(st, P.binary32), 20, np.ones(st.n, np.float32))
    rep = mk.gmres_ir(st, np.ones(st.n), np.zeros(st.n), mk.IrConfig(inner=inner, rtol=1e-10), M=M32)
    assert rep.converged and abs(rep.total_iters - runs["ir_poly20_st32"]["iters"]) <= 50


def test_jacobi1_fused_cycle_matches_multikernel_and_oracle(cuda):
    """Block Jacobi k=1 runs inside the persistent cycle kernel (diagonal
    scaling of the SpMV input and of the correction); same iteration counts
    as the multi-kernel path and within one cycle of the oracle."""
    from oracle import mpk_oracle as O
    from paper_2105_07544_b200.engine import CycleWorkspace

    A = mk.synthetic_irregular(12000, band=300, signs="negative", dominance=1.01, shift=1e-3)
    b = np.ones(A.n)
    J = mk.build_block_jacobi(A, 1)
    cfg = mk.SolverConfig(m=50, rtol=1e-10, max_iters=5000)
    fused = mk.gmres_restarted(A, J, b, np.zeros(A.n), cfg)
    ws = CycleWorkspace.get(A.n, 50, P.binary64)
    ws.flags = 4
    try:
        multi = mk.gmres_restarted(A, J, b, np.zeros(A.n), cfg)
    finally:
        ws.flags = 0
    assert fused.converged and multi.converged
    assert abs(fused.total_iters - multi.total_iters) <= 2
    ref = O.restarted((A.row_ptr, A.col_idx, A.values), O.jacobi_build(A.row_ptr, A.col_idx, A.values, 1,
                                                                         np.float64),
                      b, np.zeros(A.n), 50, 1e-10, 5000)
    assert ref.converged and abs(fused.total_iters - ref.iters) <= 50
    assert np.abs(fused.x - ref.x).max() <= 1e-7 * np.abs(ref.x).max()
    # GMRES-IR with the fp32 diagonal
    Al = mk.convert_matrix(A, P.binary32)
    J32 = mk.build_block_jacobi(Al, 1)
    inner = mk.SolverConfig(m=50, rtol=1e-4, precision=P.binary32, max_iters=5000)
    ir = mk.gmres_ir(A, b, np.zeros(A.n), mk.IrConfig(inner=inner, rtol=1e-10), M=J32, A_low=Al)
    assert ir.converged and ir.final_explicit_relres <= 1e-10


@pytest.mark.parametrize("k,prec", [(1, P.binary64), (5, P.binary64), (16, P.binary32), (42, P.binary64),
                                    (64, P.binary32)])
def test_device_block_lu_matches_lapack(cuda, rng, k, prec):
    """mpk_block_lu (device setup) vs the oracle's scipy.linalg.lu_factor
    (preconditioners.py:96-130): same pivot rows, factors equal to rounding,
    P L U reconstructing each block, thresholds equal."""
    from conftest import random_csr

    n = 3 * k + (k // 2 if k > 1 else 0) + 1
    A, dense = random_csr(mk, rng, n, diag_shift=0.0)   # real pivoting
    M = mk.build_block_jacobi(A, k, precision=prec)
    ref = O.jacobi_build(A.row_ptr, A.col_idx, A.values, k, prec.dtype)
    tol = 1e-12 if prec is P.binary64 else 2e-5
    assert M.data.num_blocks == len(ref.factors)
    for bi, ((lu, piv), (rlu, rpiv)) in enumerate(zip(M.data.factors, ref.factors)):
        assert lu.shape == rlu.shape and lu.dtype == prec.dtype
        assert np.array_equal(piv, rpiv), bi
        scale = np.abs(rlu).max()
        assert np.abs(lu.astype(np.float64) - rlu).max() <= tol * 10 * scale * lu.shape[0], bi
    # the apply: equal to the oracle's lu_solve with the reference factors to rounding
    v = rng.standard_normal(n).astype(prec.dtype)
    got = M.apply(v)
    want = ref(v)
    assert np.allclose(got, want, rtol=tol * 100, atol=tol * 100 * np.abs(want).max())


def test_device_block_lu_singular_matches_reference_rule(cuda):
    """The pivot test pivot <= kb*u*max row sum names the same block as the
    reference (SingularBlockError(block, pivot, threshold))."""
    # block 2 (rows 4-5) exactly singular, block 1 nearly singular but above the threshold
    rows = np.array([0, 1, 2, 2, 3, 3, 4, 4, 5, 5])
    cols = np.array([0, 1, 2, 3, 2, 3, 4, 5, 4, 5])
    vals = np.array([1.0, 2.0, 1.0, 1.0, 1.0, 1.0 + 1e-9, 1.0, 2.0, 2.0, 4.0])
    A = mk.csr_from_coo(rows, cols, vals, 6)
    with pytest.raises(mk.SingularBlockError) as info:
        mk.build_block_jacobi(A, 2)
    try:
        O.jacobi_build(A.row_ptr, A.col_idx, A.values, 2, np.float64)
    except ValueError as e:
        _, bi, pv, lim = e.args
    assert info.value.block_index == bi == 2
    assert info.value.threshold == lim
    assert info.value.pivot == pv == 0.0


def test_device_block_lu_large_batch(cuda):
    """C5-shaped setup (jacobi:42 over a banded irregular CSR): every block's
    apply equals the dense solve to rounding."""
    A = mk.synthetic_irregular(20000, signs="negative", dominance=1.001, shift=1e-3, far_frac=0.01, band=200)
    M = mk.build_block_jacobi(A, 42)
    v = np.random.default_rng(5).standard_normal(A.n)
    got = M.apply(v)
    ref = O.jacobi_build(A.row_ptr, A.col_idx, A.values, 42, np.float64)
    want = ref(v)
    assert np.abs(got - want).max() <= 1e-10 * np.abs(want).max()


@pytest.mark.parametrize("preset,nx,deg", [("UniFlow2D", 64, 25), ("Laplace2D", 32, 10), ("Stretched2D", 32, 20)])
def test_poly_fused_cycle_matches_multikernel(cuda, preset, nx, deg):
    """The GMRES polynomial runs inside the persistent cycle kernel (z = p(A) v_k
    and the correction's p(A)(V_k d) with one grid barrier per SpMV, same
    per-row roundings as k_poly_*): same counts and histories to rounding as
    the multi-kernel path (desc flag 4), and within a cycle of the oracle."""
    from oracle import mpk_oracle as O
    from paper_2105_07544_b200 import _lib
    from paper_2105_07544_b200.engine import CycleWorkspace

    A = L(preset, nx)
    A32 = mk.convert_matrix(A, P.binary32)
    M32 = mk.build_gmres_poly(A32, deg, np.ones(A.n, np.float32))
    inner = mk.SolverConfig(m=50, rtol=1e-4, precision=P.binary32, max_iters=3000)
    cfg = mk.IrConfig(inner=inner, rtol=1e-10)
    fused = mk.gmres_ir(A, np.ones(A.n), np.zeros(A.n), cfg, M=M32, A_low=A32)
    assert _lib.last_cycle_kernel() == "k_cycle_reg/poly"
    ws = CycleWorkspace.get(A.n, 50, P.binary32)
    ws.flags = 4
    try:
        multi = mk.gmres_ir(A, np.ones(A.n), np.zeros(A.n), cfg, M=M32, A_low=A32)
        assert _lib.last_cycle_kernel() == "multi-kernel"
    finally:
        ws.flags = 0
    assert fused.converged == multi.converged
    assert abs(fused.total_iters - multi.total_iters) <= 50
    # the first cycle's implicit residuals agree to rounding (the two paths
    # reduce the dot products in different orders)
    def first_cycle(rep):
        out = []
        for e in rep.history[1:]:
            if e.phase != "inner":
                break
            out.append(e.implicit_relres)
        return np.array(out)
    hf, hm = first_cycle(fused), first_cycle(multi)
    # fp32 with a degree-10..25 polynomial: the two reduction orders agree
    # to ~1e-7 over the first steps, then drift apart (observed up to 6%
    # late in the cycle, both within a cycle of the oracle's count below)
    assert np.abs(hf[:5] / hm[:5] - 1).max() <= 1e-5
    rp, ci, v = O.stencil_csr(preset, nx)
    d = M32.data
    ref = O.refine((rp, ci, v), np.ones(A.n), np.zeros(A.n), 50, 1e-10, 3000,
                   M=O.Poly(d.roots, d.degree, d.requested_degree, d.truncated, rp, ci, v.astype(np.float32)))
    assert fused.converged == ref.converged
    if ref.converged:
        assert abs(fused.total_iters - ref.iters) <= 50
