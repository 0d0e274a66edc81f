"""Matrix Market input -> RCM reordering -> GPU solve (the
paper's real-matrix workflow; cli.py:137-151).  The
reader and RCM are bit-exact against reference fixtures on CPU
(tests/test_mmio_reorder.py); here the permuted systems are solved on the
GPU and checked against the oracle on the same permuted system."""

import os

import numpy as np
import pytest

import paper_2105_07544_b200 as mk
from oracle import mpk_oracle as O

pytestmark = pytest.mark.gpu
P = mk.Precision
MM = os.path.join(os.path.dirname(__file__), "golden", "mm")


def csr_of(A):
    return (np.asarray(A.row_ptr), np.asarray(A.col_idx), np.asarray(A.values))


@pytest.mark.parametrize("name", ["laplace2d20_scrambled", "bentpipe16", "stretched12"])
def test_mm_rcm_solve_matches_oracle(cuda, name):
    A = mk.read_matrix_market(os.path.join(MM, name + ".mtx"))
    b = np.ones(A.n)
    Ap, bp = mk.permute_system(A, b, mk.rcm_ordering(A))
    assert Ap.stencil is None   # CSR operator path
    rep = mk.gmres_restarted(Ap, None, bp, np.zeros(A.n), mk.SolverConfig(m=50, rtol=1e-10))
    ref = O.restarted(csr_of(Ap), None, bp, np.zeros(A.n), 50, 1e-10)
    assert rep.converged == ref.converged
    assert abs(rep.total_iters - ref.iters) <= 50
    inner = mk.SolverConfig(m=50, rtol=1e-4, precision=P.binary32)
    ir = mk.gmres_ir(Ap, bp, np.zeros(A.n), mk.IrConfig(inner=inner, rtol=1e-10))
    ref_ir = O.refine(csr_of(Ap), bp, np.zeros(A.n), 50, 1e-10, 100000)
    assert ir.converged and ref_ir.converged
    assert abs(ir.total_iters - ref_ir.iters) <= 50
    # the solution of the permuted system, un-permuted, solves the original
    x = np.empty(A.n)
    x[mk.rcm_ordering(A)] = ir.x
    r = b - mk.spmv(A, x)
    assert np.linalg.norm(r) <= 1e-9 * np.linalg.norm(b)


def test_scrambled_large_system_rcm_banded_window(cuda, tmp_path):
    """A BentPipe2D(300) system written to Matrix Market with its unknowns
    scrambled, read back, RCM-reordered: RCM restores a banded profile (the
    x-window SpMV applies) and the GPU solve matches the original system's."""
    A0 = mk.generate_stencil(mk.ProblemSpec("BentPipe2D", 300))
    perm = np.random.default_rng(11).permutation(A0.n)
    As, _ = mk.permute_system(A0, np.ones(A0.n), perm)
    path = tmp_path / "scr.mtx"
    mk.write_matrix_market(As, str(path))
    A = mk.read_matrix_market(str(path))
    assert A.band_width() > 10000            # scrambled: no band
    q = mk.rcm_ordering(A)
    Ar, br = mk.permute_system(A, np.ones(A.n), q)
    assert Ar.band_width() <= 2 * 300 + 64   # RCM: bandwidth of order nx
    # exact SpMV against the oracle (bit-exact, CSR path)
    x = np.random.default_rng(2).standard_normal(A.n)
    assert np.array_equal(mk.spmv(Ar, x), O.spmv_seq(*csr_of(Ar), x))
    inner = mk.SolverConfig(m=50, rtol=1e-4, precision=P.binary32)
    ir = mk.gmres_ir(Ar, br, np.zeros(A.n), mk.IrConfig(inner=inner, rtol=1e-10))
    base = mk.gmres_ir(A0, np.ones(A0.n), np.zeros(A0.n), mk.IrConfig(inner=inner, rtol=1e-10))
    assert ir.converged and ir.final_explicit_relres <= 1e-10
    assert abs(ir.total_iters - base.total_iters) <= 0.25 * base.total_iters + 50
