"""Pin the CPU oracle (oracle/mpk_oracle.py) to the golden vectors produced
by the unmodified reference (tests/golden/make_golden.py)."""

import hashlib

import numpy as np
import pytest

from oracle import mpk_oracle as O


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


BIG = {"Laplace3D_40", "BentPipe2D_1500", "UniFlow2D_2500", "Laplace3D_200"}


def test_oracle_stencils_bit_exact(stencil_golden):
    for key, g in stencil_golden.items():
        if key in BIG:
            continue
        preset, nx = key.rsplit("_", 1)
        rp, ci, v = O.stencil_csr(preset, int(nx))
        assert (rp.size - 1, v.size) == (g["n"], g["nnz"]), key
        assert sha(rp) == g["row_ptr"] and sha(ci) == g["col_idx"], key
        assert sha(v) == g["values"], key
        assert sha(v.astype(np.float32)) == g["values_f32"], key


@pytest.mark.slow
def test_oracle_stencils_benchmark_sizes(stencil_golden):
    for key in sorted(BIG & set(stencil_golden)):
        preset, nx = key.rsplit("_", 1)
        rp, ci, v = O.stencil_csr(preset, int(nx))
        g = stencil_golden[key]
        assert sha(rp) == g["row_ptr"] and sha(ci) == g["col_idx"] and sha(v) == g["values"], key


def test_oracle_spmv_bit_exact(spmv_golden):
    names = sorted({k.split("/")[0] for k in spmv_golden.files})
    for name in names:
        g = lambda f: spmv_golden[name + "/" + f]  # noqa: E731
        rp, ci, v, x = g("row_ptr"), g("col_idx"), g("values"), g("x")
        assert np.array_equal(O.spmv_seq(rp, ci, v, x), g("y64")), name
        assert np.array_equal(O.spmv_seq_numpy(rp, ci, v, x), g("y64")), name
        v32, x32 = v.astype(np.float32), x.astype(np.float32)
        assert np.array_equal(O.spmv_seq(rp, ci, v32, x32), g("y32")), name
        assert np.array_equal(O.spmv_seq_numpy(rp, ci, v32, x32), g("y32")), name


def _same_history(got, want):
    assert len(got) == len(want)
    for a, b in zip(got, want):
        assert a[0] == b[0] and a[1] == b[1]
        assert a[2] == b[2] and a[3] == b[3]


def _check(runs, name, out, x=None, runs_x=None):
    g = runs[name]
    assert (out.iters, out.restarts, out.converged) == (g["iters"], g["restarts"], g["converged"]), name
    assert out.stalled == g["stalled"] and out.loss == g["loss"], name
    _same_history([list(h) for h in out.history], g["history"])
    if runs_x is not None and name in runs_x.files:
        assert np.array_equal(out.x, runs_x[name]), name


def test_oracle_reproduces_reference_runs(runs, runs_x):
    S = O.stencil_csr
    l16, l32, l4 = S("Laplace2D", 16), S("Laplace2D", 32), S("Laplace2D", 4)
    one = lambda A: np.ones(A[0].size - 1)  # noqa: E731
    zero = lambda A: np.zeros(A[0].size - 1)  # noqa: E731
    _check(runs, "gmres_l2d16_m50", O.restarted(l16, None, one(l16), zero(l16), 50, 1e-10), runs_x=runs_x)
    _check(runs, "gmres_l2d16_m10", O.restarted(l16, None, one(l16), zero(l16), 10, 1e-10), runs_x=runs_x)
    _check(runs, "gmres_l2d16_m5_cap8", O.restarted(l16, None, one(l16), zero(l16), 5, 1e-10, max_iters=8))
    _check(runs, "gmres_l2d16_m5_r2", O.restarted(l16, None, one(l16), zero(l16), 5, 1e-10, max_restarts=2))
    for m in (25, 50, 100):
        _check(runs, "gmres_l2d32_m%d" % m, O.restarted(l32, None, one(l32), zero(l32), m, 1e-10))
        _check(runs, "ir_l2d32_m%d" % m, O.refine(l32, one(l32), zero(l32), m, 1e-10, 20000), runs_x=runs_x)
    _check(runs, "ir_l2d16_cap60", O.refine(l16, one(l16), zero(l16), 50, 1e-10, 60))
    _check(runs, "ir_stall_l2d4", O.refine(l4, 1e-15 * one(l4), zero(l4), 10, 1e-14, 20000))
    for s in (0, 50, 100, 150, 200):
        _check(runs, "fd_l2d32_s%d" % s, O.switch(l32, one(l32), zero(l32), s), runs_x=runs_x)
    bp = S("BentPipe2D", 64)
    _check(runs, "gmres_bp64", O.restarted(bp, None, one(bp), zero(bp), 50, 1e-10), runs_x=runs_x)
    _check(runs, "ir_bp64", O.refine(bp, one(bp), zero(bp), 50, 1e-10, 20000), runs_x=runs_x)


def test_oracle_reproduces_preconditioned_runs(runs, runs_x):
    S = O.stencil_csr
    st = S("Stretched2D", 32)
    rp, ci, v = st
    b = np.ones(rp.size - 1)
    P = O.poly_build(rp, ci, v.astype(np.float32), 20, b.astype(np.float32))
    g = runs["poly_st32_roots"]
    assert P.degree == g["degree"] and P.truncated == g["truncated"]
    assert np.array_equal(P.roots.real, g["roots_re"]) and np.array_equal(P.roots.imag, g["roots_im"])
    W = O.cast_wrap(P, np.float32, np.float64)
    _check(runs, "loss_recover_st32", O.restarted(st, W, b, np.zeros_like(b), 50, 1e-10, 2000))
    _check(runs, "loss_giveup_st32", O.restarted(st, W, b, np.zeros_like(b), 50, 1e-10, 2000,
                                                 restart_on_loss=False))
    _check(runs, "ir_poly20_st32", O.refine(st, b, np.zeros_like(b), 50, 1e-10, 20000, M=P))
    bp24 = S("BentPipe2D", 24)
    b24 = np.ones(576)
    _check(runs, "ir_jacobi8_bp24", O.refine(bp24, b24, np.zeros(576), 50, 1e-10, 20000,
                                             M=O.jacobi_build(*bp24, 8, np.float32)))
    l16 = S("Laplace2D", 16)
    _check(runs, "jacobi16_l2d16", O.restarted(l16, O.jacobi_build(*l16, 16, np.float64),
                                               np.ones(256), np.zeros(256), 50, 1e-10))


def test_oracle_breakdown_rule_u_matches_reference_patch(runs):
    l3 = O.stencil_csr("Laplace3D", 40)
    out = O.refine(l3, np.ones(64000), np.zeros(64000), 50, 1e-10, 20000, rule="u")
    _check(runs, "ir_l3d40_rule_u", out)


def test_oracle_dcgs2_cycle_is_cgs2_reordered():
    """The oracle's lagged one-reduction CGS2 (dcgs2_cycle, this repo's
    option) is the reference's CGS2 Arnoldi reordered: fp64 cycle residual
    histories agree to rounding, and fp32-inner IR takes the same count."""
    rp, ci, v = O.stencil_csr("Laplace2D", 24)
    n = len(rp) - 1
    b = np.ones(n)
    _, a = O.one_cycle((rp, ci, v), None, b, np.zeros(n), 40, 1e-12)
    _, d = O.dcgs2_cycle((rp, ci, v), None, b, np.zeros(n), 40, 1e-12)
    assert a.steps == d.steps
    assert np.allclose(np.log10(a.implicit), np.log10(d.implicit), atol=1e-6)
    A = O.stencil_csr("Laplace3D", 16)
    n = len(A[0]) - 1
    c = O.refine(A, np.ones(n), np.zeros(n), 50, 1e-10, 20000, rule="u")
    d = O.refine(A, np.ones(n), np.zeros(n), 50, 1e-10, 20000, rule="u", orth="dcgs2")
    assert c.converged and d.converged and abs(c.iters - d.iters) <= 50
