"""Parity at BASELINE sizes through size-independent properties (the oracle
is too slow for whole solves there):

* SpMV at C2 (2.25M rows) and C4 (8M rows): matrix-free stencil == CSR ==
  the sequential CPU restatement, bit for bit, fp64 and fp32;
* one fp32 and one fp64 Arnoldi cycle at C2: the basis V (kept on the
  device) is orthonormal, V^T V = I to the precision's CGS2 level, and the
  Arnoldi relation A V_k = V_{k+1} Hbar holds;
* a partial GMRES-IR solve at C2 decreases the explicit residual monotonically
  per refinement and equals the residual recomputed from the returned x.
"""

import numpy as np
import pytest

import paper_2105_07544_b200 as mk

pytestmark = pytest.mark.gpu
P = mk.Precision


@pytest.mark.parametrize("preset,nx", [("BentPipe2D", 1500), ("Laplace3D", 200)])
def test_spmv_bit_exact_at_baseline_size(cuda, preset, nx):
    from oracle import mpk_oracle as O

    A = mk.generate_stencil(mk.ProblemSpec(preset, nx))
    x = np.random.default_rng(1).standard_normal(A.n)
    ref = O.spmv_seq(A.row_ptr, A.col_idx, A.values, x)
    for prec in (P.binary64, P.binary32):
        B = mk.convert_matrix(A, prec)
        xs = x.astype(prec.dtype)
        want = ref if prec is P.binary64 else O.spmv_seq(B.row_ptr, B.col_idx, B.values, xs)
        B.use_stencil = True
        ys = mk.spmv(B, xs)
        B.use_stencil = False
        yc = mk.spmv(B, xs)
        assert ys.tobytes() == want.tobytes() and yc.tobytes() == want.tobytes(), prec


@pytest.mark.parametrize("prec,tol", [(P.binary32, 5e-6), (P.binary64, 1e-12)])   # reference bars: test_gmres.py:135-151
def test_arnoldi_cycle_properties_at_c2(cuda, prec, tol):
    import torch

    from paper_2105_07544_b200.engine import CycleWorkspace

    A = mk.generate_stencil(mk.ProblemSpec("BentPipe2D", 1500))
    B = mk.convert_matrix(A, prec)
    n, m = A.n, 50
    b = torch.ones(n, dtype=prec.torch_dtype, device=cuda)
    x, st = mk.gmres_cycle(B, None, b, torch.zeros_like(b),
                           mk.SolverConfig(m=m, rtol=1e-30 if prec is P.binary64 else 1e-12, precision=prec,
                                           breakdown_rule="u"))
    assert st.steps == m and not st.breakdown
    ws = CycleWorkspace.get(n, m, prec)
    V = ws.V.view(m + 1, ws.ld)[:m, :n].double()          # columns v_0..v_{m-1}
    G = V @ V.t()
    assert (G - torch.eye(m, device=cuda, dtype=torch.float64)).abs().max().item() <= tol
    H = torch.as_tensor(ws.raw_hessenberg(m - 1), device=cuda)   # (m) x (m-1) unrotated columns
    Vk = ws.V.view(m + 1, ws.ld)[: m - 1, :n]
    AV = torch.stack([torch.as_tensor(mk.spmv(B, Vk[j].clone()), device=cuda) for j in range(m - 1)]).double()
    res = AV - (H.t() @ V)                                   # rows: A v_j - sum_i H[i, j] v_i
    assert res.norm().item() <= 20 * tol * AV.norm().item()


def test_partial_ir_residuals_consistent_at_c2(cuda):
    import torch

    A = mk.generate_stencil(mk.ProblemSpec("BentPipe2D", 1500))
    b = torch.ones(A.n, dtype=torch.float64, device=cuda)
    inner = mk.SolverConfig(m=50, rtol=1e-4, precision=P.binary32, max_iters=500)
    rep = mk.gmres_ir(A, b, torch.zeros_like(b), mk.IrConfig(inner=inner, rtol=1e-10))
    outer = [h.explicit_relres for h in rep.history if h.phase == "outer"]
    assert rep.total_iters == 500 and len(outer) == 11
    assert all(b2 < a2 for a2, b2 in zip(outer, outer[1:]))
    r = b - torch.as_tensor(mk.spmv(A, rep.x), device=cuda)
    assert abs(r.norm().item() / rep.baseline - rep.final_explicit_relres) <= 1e-12
