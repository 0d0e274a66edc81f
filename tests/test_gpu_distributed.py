"""Row-partitioned solver on P virtual ranks sharing the one GPU (threads,
one stream each, concurrent persistent kernels meeting at the cross-rank
barrier through the same peer-pointer code path a multi-GPU run uses).

Parity bar: every rank returns the identical report; iteration counts equal
the single-GPU solve's within one restart cycle; converged to 1e-10; the
assembled x agrees with the single-GPU x to the solve tolerance."""

import numpy as np
import pytest

import paper_2105_07544_b200 as mk
from paper_2105_07544_b200 import _lib
from paper_2105_07544_b200 import distributed as dd

from conftest import random_csr

pytestmark = pytest.mark.gpu
P32, P64 = mk.Precision.binary32, mk.Precision.binary64


def L(preset, nx):
    return mk.generate_stencil(mk.ProblemSpec(preset, nx))


def solve_dist(A, P, solver, b, m=50, rule="n_u"):
    A_low = mk.convert_matrix(A, P32) if solver == "ir" else None

    def fn(comm):
        sysm = dd.LocalSystem(comm, A, A_low)
        try:
            if solver == "ir":
                inner = mk.SolverConfig(m=m, rtol=1e-4, precision=P32, max_iters=20000, breakdown_rule=rule)
                rep = dd.dist_gmres_ir(sysm, b, np.zeros(A.n), mk.IrConfig(inner=inner, rtol=1e-10))
            else:
                rep = dd.dist_gmres_restarted(sysm, b, np.zeros(A.n),
                                              mk.SolverConfig(m=m, rtol=1e-10, max_iters=20000))
            return rep, rep.x.cpu().numpy(), (sysm.r0, sysm.r1)
        finally:
            sysm.close()

    res = dd.run_virtual_ranks(P, fn)
    x = np.zeros(A.n)
    for rep, xl, (r0, r1) in res:
        x[r0:r1] = xl
    reps = [r[0] for r in res]
    for r in reps[1:]:   # replicated bookkeeping: identical on every rank
        assert (r.total_iters, r.restarts, r.converged) == (reps[0].total_iters, reps[0].restarts,
                                                            reps[0].converged)
        assert [(h.iteration, h.implicit_relres, h.explicit_relres) for h in r.history] == \
            [(h.iteration, h.implicit_relres, h.explicit_relres) for h in reps[0].history]
    return reps[0], x


def solve_single(A, solver, b, m=50, rule="n_u"):
    if solver == "ir":
        inner = mk.SolverConfig(m=m, rtol=1e-4, precision=P32, max_iters=20000, breakdown_rule=rule)
        return mk.gmres_ir(A, b, np.zeros(A.n), mk.IrConfig(inner=inner, rtol=1e-10))
    return mk.gmres_restarted(A, None, b, np.zeros(A.n), mk.SolverConfig(m=m, rtol=1e-10, max_iters=20000))


def check(A, P, solver, b=None, m=50, rule="n_u"):
    b = np.ones(A.n) if b is None else b
    ref = solve_single(A, solver, b, m, rule)
    rep, x = solve_dist(A, P, solver, b, m, rule)
    assert rep.converged and ref.converged
    assert rep.final_explicit_relres <= 1e-10
    assert abs(rep.total_iters - ref.total_iters) <= m, (rep.total_iters, ref.total_iters)
    # early history (before rounding differences accumulate) agrees closely
    for a, c in list(zip(rep.history, ref.history))[:10]:
        if a.implicit_relres is not None and c.implicit_relres is not None:
            assert abs(a.implicit_relres - c.implicit_relres) <= 1e-3 * abs(c.implicit_relres) + 1e-12
    scale = np.abs(ref.x).max()
    assert np.abs(x - ref.x).max() <= 1e-6 * scale
    return rep, ref


@pytest.mark.parametrize("P", [2, 3])
def test_fp64_laplace2d_matches_single_gpu(cuda, P):
    rep, ref = check(L("Laplace2D", 32), P, "fp64")
    assert rep.total_iters == 71   # the reference's golden count


@pytest.mark.parametrize("P", [2, 4])
def test_ir_laplace3d(cuda, P):
    check(L("Laplace3D", 24), P, "ir")


def test_ir_bentpipe_four_ranks(cuda):
    check(L("BentPipe2D", 64), 4, "ir")


def test_csr_operator_three_ranks(cuda):
    A = L("Laplace3D", 16)
    A.use_stencil = False
    check(A, 3, "fp64")


def test_random_nonsymmetric_far_columns(cuda, rng):
    A, dense = random_csr(mk, rng, 320, density=0.05)
    b = rng.standard_normal(320)
    rep, x = solve_dist(A, 2, "fp64", b)
    assert rep.converged
    xs = np.linalg.solve(dense, b)
    assert np.abs(x - xs).max() <= 1e-8 * np.abs(xs).max()


def test_two_processes_share_the_gpu_through_ipc(cuda, tmp_path):
    """torchrun, 2 processes on GPU 0: CUDA-IPC peer pointers, system-scope
    atomics across processes (time-sliced, hence a small problem)."""
    import json
    import os
    import socket
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ, MPK_SHARE_GPU="1")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port),
                          os.path.join(root, "tools", "dist_check.py"), "Laplace2D", "32"],
                         capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-3000:]
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1]
    r = json.loads(line)
    assert r["ir_converged"] and r["fp64_converged"] and r["ir_relres"] <= 1e-10
    assert r["fp64_iters"] == r["single_fp64_iters"] == 71
    assert abs(r["ir_iters"] - 150) <= 50
    assert r["x_maxdiff"] <= 1e-8


@pytest.mark.parametrize("P", [2, 3])
def test_lagged_cgs2_row_partitioned(cuda, P):
    """The one-reduction cycle across ranks (2 cross-rank barriers per step):
    same counts as the single-GPU lagged cycle within a restart cycle."""
    A = L("Laplace3D", 24)
    A_low = mk.convert_matrix(A, P32)
    b = np.ones(A.n)

    def fn(comm):
        sysm = dd.LocalSystem(comm, A, A_low)
        try:
            inner = mk.SolverConfig(m=50, rtol=1e-4, precision=P32, max_iters=20000, orthogonalization="dcgs2")
            ir_rep = dd.dist_gmres_ir(sysm, b, np.zeros(A.n), mk.IrConfig(inner=inner, rtol=1e-10))
            kern_ir = _lib.last_cycle_kernel()
            g64 = dd.dist_gmres_restarted(sysm, b, np.zeros(A.n),
                                          mk.SolverConfig(m=50, rtol=1e-10, orthogonalization="dcgs2"))
            kern64 = _lib.last_cycle_kernel()
            return (ir_rep.total_iters, ir_rep.converged, g64.total_iters, g64.converged,
                    g64.final_explicit_relres, kern_ir, kern64)
        finally:
            sysm.close()

    res = dd.run_virtual_ranks(P, fn)
    assert all(r == res[0] for r in res)
    it_ir, c_ir, it64, c64, rel64, kern_ir, kern64 = res[0]
    # the row-partitioned lagged kernel really ran (it used to fall back to CGS2)
    assert kern_ir == "k_cycle_dcgs2/multi" and kern64 == "k_cycle_dcgs2/multi", (kern_ir, kern64)
    inner = mk.SolverConfig(m=50, rtol=1e-4, precision=P32, max_iters=20000, orthogonalization="dcgs2")
    ref_ir = mk.gmres_ir(A, b, np.zeros(A.n), mk.IrConfig(inner=inner, rtol=1e-10))
    ref64 = mk.gmres_restarted(A, None, b, np.zeros(A.n), mk.SolverConfig(m=50, rtol=1e-10, orthogonalization="dcgs2"))
    assert c_ir and c64 and rel64 <= 1e-10
    assert abs(it_ir - ref_ir.total_iters) <= 50 and abs(it64 - ref64.total_iters) <= 50


@pytest.mark.parametrize("P", [2, 3])
def test_fp32_restarted_matches_single_gpu(cuda, P):
    """fp32 row-partitioned GMRES(m) (e.g. GMRES-FD's low phase): the halo of
    x comes from the fp32 peer set (it used to be read from an
    fp64 buffer), with a nonzero x0 so the very first residual needs it."""
    A = mk.convert_matrix(L("Laplace2D", 32), P32)
    b = np.ones(A.n, np.float32)
    x0 = (0.01 * np.sin(np.arange(A.n))).astype(np.float32)
    cfg = mk.SolverConfig(m=30, rtol=1e-5, precision=P32, max_iters=3000)
    ref = mk.gmres_restarted(A, None, b, x0, cfg)

    def fn(comm):
        sysm = dd.LocalSystem(comm, A)
        try:
            rep = dd.dist_gmres_restarted(sysm, b, x0, cfg)
            return rep, rep.x.cpu().numpy(), (sysm.r0, sysm.r1)
        finally:
            sysm.close()

    res = dd.run_virtual_ranks(P, fn)
    rep = res[0][0]
    assert rep.converged and ref.converged
    assert abs(rep.total_iters - ref.total_iters) <= cfg.m
    # the first explicit residual (x0's halo) is the single-GPU one to fp32 rounding
    assert abs(rep.baseline - ref.baseline) <= 1e-5 * ref.baseline
    x = np.zeros(A.n, np.float32)
    for _, xl, (r0, r1) in res:
        x[r0:r1] = xl
    assert np.abs(x - ref.x).max() <= 1e-3 * np.abs(ref.x).max()


@pytest.mark.parametrize("P", [2, 3])
def test_jacobi1_row_partitioned(cuda, P):
    """Block-Jacobi(1) right preconditioning inside the row-partitioned cycle
    (diagonal of the GLOBAL matrix; halo rows scaled by their own a_ii):
    same report on every rank, counts within a cycle of the one-GPU solve."""
    A = mk.synthetic_irregular(6000, signs="negative", dominance=1.001, shift=1e-3, far_frac=0.01, band=300)
    A_low = mk.convert_matrix(A, P32)
    M64 = mk.build_block_jacobi(A, 1)
    M32 = mk.build_block_jacobi(A_low, 1)
    b = np.ones(A.n)
    inner = mk.SolverConfig(m=50, rtol=1e-4, precision=P32, max_iters=20000, breakdown_rule="u")

    def fn(comm):
        sysm = dd.LocalSystem(comm, A, A_low)
        try:
            r64 = dd.dist_gmres_restarted(sysm, b, np.zeros(A.n), mk.SolverConfig(m=50, rtol=1e-10, max_iters=20000),
                                          M=M64)
            rir = dd.dist_gmres_ir(sysm, b, np.zeros(A.n), mk.IrConfig(inner=inner, rtol=1e-10), M=M32)
            return r64.total_iters, rir.total_iters, rir.converged, rir.final_explicit_relres
        finally:
            sysm.close()

    res = dd.run_virtual_ranks(P, fn)
    assert all(r == res[0] for r in res)
    it64, itir, conv, rel = res[0]
    one64 = mk.gmres_restarted(A, M64, b, np.zeros(A.n), mk.SolverConfig(m=50, rtol=1e-10, max_iters=20000))
    oneir = mk.gmres_ir(A, b, np.zeros(A.n), mk.IrConfig(inner=inner, rtol=1e-10), M=M32, A_low=A_low)
    assert conv and rel <= 1e-10
    assert abs(it64 - one64.total_iters) <= 50 and abs(itir - oneir.total_iters) <= 50
