"""Solver-level parity on the GPU against the reference's golden runs
(tests/golden/runs.json, produced by the unmodified mpkrylov).

Contract (BASELINE north star): convergence to the same tolerance, iteration
counts within one restart cycle, residual histories within a stated
tolerance.  Dot products are tree-reduced on the device instead of
OpenBLAS's order, so only rounding differs:

* fp64 GMRES: iteration and restart counts identical; every history value
  within 5% relative (observed <= 2.6e-2, drift under m=10 restarts;
  <= 2e-4 for m >= 25) plus 1e-13 absolute.
* fp32 / GMRES-IR / GMRES-FD: the fp32 cycle is accurate only to about
  u32*kappa(A) (~2e-5 on Laplace2D 32), so below that level the values are
  rounding noise.  Counts within one restart cycle (m); history values
  compared while they are above 1e-4 (15% relative: observed <= 9% on the
  convection-dominated BentPipe2D 64, where the fp32 Arnoldi vectors carry
  u32*kappa(A) errors that grow over 550 inner steps).
"""

import numpy as np
import pytest

import paper_2105_07544_b200 as mk

pytestmark = pytest.mark.gpu

P = mk.Precision
# history tolerances: (relative, absolute, floor below which values are noise)
HIST_TOL = {"fp64": (5e-2, 1e-13, 0.0), "fp32": (1.5e-1, 0.0, 1e-4)}


def L(preset, nx):
    return mk.generate_stencil(mk.ProblemSpec(preset, nx))


def compare(rep, g, slack=0, hist="fp64", exact_iters=True):
    assert rep.converged == g["converged"]
    if exact_iters:
        assert rep.total_iters == g["iters"], (rep.total_iters, g["iters"])
        assert rep.restarts == g["restarts"]
    else:
        assert abs(rep.total_iters - g["iters"]) <= slack, (rep.total_iters, g["iters"])
    assert rep.stalled == g["stalled"]
    assert rep.loss_of_accuracy == g["loss"]
    got = [(e.iteration, e.phase, e.implicit_relres, e.explicit_relres) for e in rep.history]
    want = g["history"]
    rtol, atol, floor = HIST_TOL[hist]
    worst = 0.0
    for a, b in zip(got, want):
        if a[0] != b[0] or a[1] != b[1]:
            break   # trajectories may separate once counts differ
        for i in (2, 3):
            if a[i] is not None and b[i] is not None and abs(b[i]) >= floor:
                d = abs(a[i] - b[i]) - atol
                worst = max(worst, d / abs(b[i]))
        if hist == "fp32" and min(v for v in (a[2], a[3], b[2], b[3]) if v is not None) < floor:
            break   # past the fp32 attainable accuracy: noise
    assert worst <= rtol, worst
    if g["converged"]:
        assert rep.final_explicit_relres <= 1e-10 or g["relres"] > 1e-10
    return worst


def gm(A, b, **kw):
    cfg = mk.SolverConfig(**kw)
    return mk.gmres_restarted(A, None, b.astype(cfg.precision.dtype),
                              np.zeros(A.n, cfg.precision.dtype), cfg)


def ir(A, b, m=50, rtol=1e-10, M=None, max_iters=20000, **kw):
    inner = mk.SolverConfig(m=m, rtol=1e-4, precision=P.binary32, max_iters=max_iters)
    return mk.gmres_ir(A, b, np.zeros(A.n), mk.IrConfig(inner=inner, rtol=rtol, **kw), M=M)


def fd(A, b, s, m=50):
    cfg = mk.FdConfig(switch_iter=s, low=mk.SolverConfig(m=m, rtol=1e-10, precision=P.binary32),
                      high=mk.SolverConfig(m=m, rtol=1e-10))
    return mk.gmres_fd(A, b, np.zeros(A.n), cfg)


def test_fp64_restarted_goldens(cuda, runs, runs_x):
    l16, l32 = L("Laplace2D", 16), L("Laplace2D", 32)
    compare(gm(l16, np.ones(256), m=50, rtol=1e-10), runs["gmres_l2d16_m50"])
    compare(gm(l16, np.ones(256), m=10, rtol=1e-10), runs["gmres_l2d16_m10"])
    compare(gm(l16, np.ones(256), m=5, rtol=1e-10, max_iters=8), runs["gmres_l2d16_m5_cap8"])
    compare(gm(l16, np.ones(256), m=5, rtol=1e-10, max_restarts=2), runs["gmres_l2d16_m5_r2"])
    for m in (25, 50, 100):
        compare(gm(l32, np.ones(1024), m=m, rtol=1e-10), runs["gmres_l2d32_m%d" % m])
    rep = gm(l16, np.ones(256), m=50, rtol=1e-10)
    assert np.abs(rep.x - runs_x["gmres_l2d16_m50"]).max() <= 1e-9 * np.abs(rep.x).max()
    compare(gm(L("BentPipe2D", 64), np.ones(4096), m=50, rtol=1e-10), runs["gmres_bp64"])
    compare(gm(L("UniFlow2D", 48), np.ones(48 * 48), m=50, rtol=1e-10), runs["gmres_uf48"])


def test_fp32_restarted(cuda, runs):
    A = mk.convert_matrix(L("Laplace2D", 8), P.binary32)
    rep = gm(A, np.ones(64), m=20, rtol=1e-4, precision=P.binary32)
    compare(rep, runs["gmres32_l2d8_m20"], hist="fp32", exact_iters=False, slack=20)
    assert rep.x.dtype == np.float32 and rep.history[0].phase == "single"


def test_ir_goldens(cuda, runs):
    l16, l32 = L("Laplace2D", 16), L("Laplace2D", 32)
    compare(ir(l32, np.ones(1024)), runs["ir_l2d32_m50"], hist="fp32", exact_iters=False, slack=50)
    compare(ir(l32, np.ones(1024), m=25), runs["ir_l2d32_m25"], hist="fp32", exact_iters=False, slack=25)
    compare(ir(l32, np.ones(1024), m=100), runs["ir_l2d32_m100"], hist="fp32", exact_iters=False, slack=100)
    compare(ir(l16, np.ones(256)), runs["ir_l2d16_m50"], hist="fp32", exact_iters=False, slack=50)
    rep = ir(l16, np.ones(256), max_iters=60)
    assert rep.total_iters <= 60
    compare(ir(L("BentPipe2D", 64), np.ones(4096)), runs["ir_bp64"], hist="fp32", exact_iters=False,
            slack=50)


def test_ir_stall_on_fp32_invisible_residual(cuda, runs):
    A = L("Laplace2D", 4)
    rep = ir(A, 1e-15 * np.ones(16), m=10, rtol=1e-14)
    g = runs["ir_stall_l2d4"]
    assert rep.stalled and not rep.converged
    assert rep.restarts == g["restarts"]
    # b = const on the 4x4 grid has a 3-dimensional Krylov space (the square's
    # symmetry orbits); how fast refinement 2 exhausts the fp32-visible part
    # of the residual depends on the last bits of x after refinement 1, i.e.
    # on dot-product rounding (OpenBLAS vs device tree): within one cycle
    assert abs(rep.total_iters - g["iters"]) <= 10, (rep.total_iters, g["iters"])
    assert rep.history[0].explicit_relres == 1.0
    assert [h.phase for h in rep.history[:4]] == ["outer", "inner", "inner", "inner"]


def test_ir_history_layout(cuda):
    A = L("Laplace2D", 16)
    rep = ir(A, np.ones(256))
    assert {e.phase for e in rep.history} == {"inner", "outer"}
    inner = [e for e in rep.history if e.phase == "inner"]
    assert [e.iteration for e in inner] == list(range(1, rep.total_iters + 1))
    outer = [e for e in rep.history if e.phase == "outer"]
    assert outer[-1].explicit_relres == rep.final_explicit_relres
    assert rep.phase_iters == {"inner": rep.total_iters, "outer": rep.restarts}


def test_fd_goldens(cuda, runs):
    l32 = L("Laplace2D", 32)
    rep0 = fd(l32, np.ones(1024), 0)
    pure = gm(l32, np.ones(1024), m=50, rtol=1e-10)
    assert np.array_equal(rep0.x, pure.x) and rep0.total_iters == pure.total_iters
    assert rep0.phase_iters == {"single": 0, "double": 71}
    for s in (50, 100, 150, 200):
        g = runs["fd_l2d32_s%d" % s]
        rep = fd(l32, np.ones(1024), s)
        compare(rep, g, hist="fp32", exact_iters=False, slack=50)
        assert rep.phase_iters["single"] == s


def test_lucky_breakdown_and_zero_rhs(cuda):
    nx = 16
    A = L("Laplace2D", nx)
    grid = (np.arange(nx) + 1) / (nx + 1) * np.pi
    b = np.outer(np.sin(grid), np.sin(grid)).ravel()
    rep = gm(A, b, m=50, rtol=1e-10)
    assert rep.converged and rep.total_iters == 1 and rep.final_explicit_relres <= 1e-12
    with pytest.raises(mk.ZeroRightHandSideError):
        gm(A, np.zeros(A.n), m=5)
    with pytest.raises(mk.ZeroRightHandSideError):
        ir(A, np.zeros(A.n))


def test_exact_initial_guess_and_identity(cuda, rng):
    n = 30
    idx = np.arange(n)
    A = mk.csr_from_coo(idx, idx, np.ones(n), n)
    b = rng.standard_normal(n)
    rep = mk.gmres_restarted(A, None, b, b.copy(), mk.SolverConfig(m=10, rtol=1e-8))
    assert rep.converged and rep.total_iters == 0 and rep.final_explicit_relres == 0.0
    rep = mk.gmres_restarted(A, None, b, np.zeros(n), mk.SolverConfig(m=10, rtol=1e-12))
    assert rep.total_iters == 1 and np.allclose(rep.x, b, atol=1e-14)


def test_random_nonsymmetric_vs_dense_solve(cuda, rng):
    from conftest import random_csr

    for n in (24, 80, 128):
        A, dense = random_csr(mk, rng, n)
        b = rng.standard_normal(n)
        rep = mk.gmres_restarted(A, None, b, np.zeros(n), mk.SolverConfig(m=30, rtol=1e-12))
        want = np.linalg.solve(dense, b)
        assert rep.converged
        assert np.abs(rep.x - want).max() <= 1e-7 * np.abs(want).max()


def test_collected_basis_orthonormal_and_arnoldi(cuda):
    A = L("Laplace2D", 16)
    n = A.n
    x, st = mk.gmres_cycle(A, None, np.ones(n), np.zeros(n), mk.SolverConfig(m=30, rtol=1e-300),
                           collect_basis=True)
    k = st.steps
    V, H = st.basis, st.hessenberg
    assert V.shape == (n, k + 1) and H.shape == (k + 1, k)
    assert np.abs(V.T @ V - np.eye(k + 1)).max() <= 1e-12
    AV = np.column_stack([mk.spmv(A, V[:, j].copy()) for j in range(k)])
    assert np.linalg.norm(AV - V @ H) <= 1e-10 * np.linalg.norm(A.values) * np.sqrt(k)


def test_device_tensors_through_the_solver(cuda):
    import torch

    A = L("BentPipe2D", 32)
    b = torch.ones(A.n, dtype=torch.float64, device=cuda)
    inner = mk.SolverConfig(m=50, rtol=1e-4, precision=P.binary32)
    rep = mk.gmres_ir(A, b, torch.zeros_like(b), mk.IrConfig(inner=inner, rtol=1e-10))
    assert isinstance(rep.x, torch.Tensor) and rep.x.is_cuda and rep.converged


def test_c1_laplace3d40_counts(cuda, runs):
    A = L("Laplace3D", 40)
    b = np.ones(A.n)
    # the reference stops at 206 with relres 9.57e-11; one step earlier it sits
    # within 0.1% of 1e-10, so the count is decided by last-bit rounding of the
    # dot products: hold it to the contract (one restart cycle) instead
    compare(gm(A, b, m=50, rtol=1e-10), runs["gmres_l3d40"], exact_iters=False, slack=50)
    compare(ir(A, b), runs["ir_l3d40"], hist="fp32", exact_iters=False, slack=50)
    inner = mk.SolverConfig(m=50, rtol=1e-4, precision=P.binary32, max_iters=20000, breakdown_rule="u")
    rep = mk.gmres_ir(A, b, np.zeros(A.n), mk.IrConfig(inner=inner, rtol=1e-10))
    compare(rep, runs["ir_l3d40_rule_u"], hist="fp32", exact_iters=False, slack=50)


def test_run_to_run_bit_identical(cuda):
    """SPEC determinism: fixed-order reductions everywhere, so two solves of
    the same system give bit-identical histories and solutions."""
    A = L("BentPipe2D", 96)
    b = np.ones(A.n)
    r1, r2 = ir(A, b), ir(A, b)
    assert [(h.implicit_relres, h.explicit_relres) for h in r1.history] == \
        [(h.implicit_relres, h.explicit_relres) for h in r2.history]
    assert r1.x.tobytes() == r2.x.tobytes()
    g1 = gm(A, b, m=50, rtol=1e-10)
    g2 = gm(A, b, m=50, rtol=1e-10)
    assert g1.x.tobytes() == g2.x.tobytes() and g1.total_iters == g2.total_iters


def test_l2_window_release_and_env_off(cuda):
    """The cycle kernels launch with an L2 access-policy window over their
    work vectors; mpk_l2_release returns the persisting lines to normal after
    a solve.  With MPK_L2_PERSIST=0 (a fresh process) the solve is the same
    bit for bit: the window changes cache residency, not arithmetic."""
    import json
    import os
    import subprocess
    import sys

    from paper_2105_07544_b200 import _lib

    assert _lib.load().mpk_l2_release() == 0
    code = ("import sys, json, numpy as np; sys.path.insert(0, %r); import paper_2105_07544_b200 as mk; "
            "A = mk.generate_stencil(mk.ProblemSpec('Laplace3D', 24)); "
            "inner = mk.SolverConfig(m=50, rtol=1e-4, precision=mk.Precision.binary32); "
            "r = mk.gmres_ir(A, np.ones(A.n), np.zeros(A.n), mk.IrConfig(inner=inner, rtol=1e-10)); "
            "print(json.dumps([r.total_iters, r.x.tobytes().hex()[:4096], r.final_explicit_relres]))"
            % os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    outs = []
    for flag in ("1", "0"):
        env = dict(os.environ, MPK_L2_PERSIST=flag)
        p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
        assert p.returncode == 0, p.stderr
        outs.append(json.loads(p.stdout.strip().splitlines()[-1]))
    assert outs[0] == outs[1]
