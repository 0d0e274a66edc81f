"""Ragged and tiny systems through the persistent cycle kernels: n = 1, n < m
(lucky breakdown at step n), and n not a multiple of the 16-byte pack width
(4 fp32 / 2 fp64 rows), so every kernel's tail rows are exercised.  The
oracle (reference gmres.py:134-308 restated) is the checker: one-cycle
implicit histories to rounding, equal step counts, same solution."""

import numpy as np
import pytest

import paper_2105_07544_b200 as mk

pytestmark = pytest.mark.gpu
P = mk.Precision

SIZES = (1, 2, 3, 5, 7, 63, 65, 130, 1001)


def _system(n, seed=7, diag_shift=None):
    rng = np.random.default_rng(seed + n)
    from conftest import random_csr

    return random_csr(mk, rng, n, density=min(1.0, 8.0 / n + 0.02), diag_shift=diag_shift)


@pytest.mark.parametrize("orth", ["cgs2", "dcgs2"])
@pytest.mark.parametrize("n", SIZES)
def test_one_cycle_fp64_vs_oracle(cuda, n, orth):
    from oracle import mpk_oracle as O

    A, dense = _system(n)
    b = np.random.default_rng(n).standard_normal(n)
    m = 20
    x, st = mk.gmres_cycle(A, None, b, np.zeros(n), mk.SolverConfig(m=m, rtol=1e-300, orthogonalization=orth))
    xo, so = O.one_cycle((A.row_ptr, A.col_idx, A.values), None, b, np.zeros(n), m, 1e-300)
    assert st.steps == so.steps, (st.steps, so.steps)
    assert st.breakdown == so.breakdown
    h, ho = np.array(st.implicit_relres), np.array(so.implicit)
    keep = ho > 1e-12
    assert np.all(np.abs(h - ho)[keep] <= 1e-8 * ho[keep])
    want = np.linalg.solve(dense, b)
    if n <= m:   # the Krylov space is exhausted inside the cycle: exact solve
        assert np.abs(x - want).max() <= 1e-9 * np.abs(want).max()
    assert np.abs(x - xo).max() <= 1e-9 * np.abs(xo).max()


@pytest.mark.parametrize("orth", ["cgs2", "dcgs2"])
@pytest.mark.parametrize("n", SIZES)
def test_restarted_and_ir_ragged(cuda, n, orth):
    from oracle import mpk_oracle as O

    A, dense = _system(n)
    b = np.ones(n)
    want = np.linalg.solve(dense, b)
    rep = mk.gmres_restarted(A, None, b, np.zeros(n), mk.SolverConfig(m=10, rtol=1e-12, orthogonalization=orth))
    ref = O.restarted((A.row_ptr, A.col_idx, A.values), None, b, np.zeros(n), 10, 1e-12)
    assert rep.converged and ref.converged
    assert abs(rep.total_iters - ref.iters) <= 10, (rep.total_iters, ref.iters)
    assert np.abs(rep.x - want).max() <= 1e-10 * np.abs(want).max()
    inner = mk.SolverConfig(m=10, rtol=1e-4, precision=P.binary32, orthogonalization=orth)
    ir = mk.gmres_ir(A, b, np.zeros(n), mk.IrConfig(inner=inner, rtol=1e-12))
    assert ir.converged and ir.final_explicit_relres <= 1e-12
    assert np.abs(ir.x - want).max() <= 1e-10 * np.abs(want).max()


@pytest.mark.parametrize("orth", ["cgs2", "dcgs2"])
@pytest.mark.parametrize("n", (63, 65, 130, 1001))
def test_one_cycle_fp32_vs_oracle(cuda, n, orth):
    """fp32 cycle (the GMRES-IR inner solver) on odd sizes: the oracle in
    float32 (same roundings, sequential sums) is the checker; the device's
    fixed-order tree sums differ in the last bits only."""
    from oracle import mpk_oracle as O

    A64, _ = _system(n, diag_shift=3.0)   # slow convergence: all 20 steps above 1e-5
    A = mk.convert_matrix(A64, P.binary32)
    b = np.random.default_rng(n).standard_normal(n).astype(np.float32)
    cfg = mk.SolverConfig(m=20, rtol=1e-300, precision=P.binary32, orthogonalization=orth)
    x, st = mk.gmres_cycle(A, None, b, np.zeros(n, np.float32), cfg)
    xo, so = O.one_cycle((A.row_ptr, A.col_idx, A.values), None, b, np.zeros(n, np.float32), 20, 1e-300)
    h, ho = np.array(st.implicit_relres), np.array(so.implicit)
    k = min(len(h), len(ho))
    keep = ho[:k] > 1e-5
    assert keep.sum() >= 8
    assert np.all(np.abs(h[:k] - ho[:k])[keep] <= 2e-3 * ho[:k][keep])
    assert np.abs(x.astype(np.float64) - xo).max() <= 1e-3 * np.abs(xo).max()
