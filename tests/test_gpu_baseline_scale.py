"""Parity at BASELINE scale (VERDICT r1 "Next round" 1): full C2 / C4 solves
on the GPU against runs of the UNMODIFIED reference at the same size
(tests/golden/runs.json["ir_bp1500"], tests/golden/big/*.npz, made by
tests/golden/make_golden.py --big and tests/golden/make_big_golden.py).

What the reference itself pins, and what these tests hold:

* Restarted GMRES over hundreds of cycles is chaotic in the last bit: the
  reference's own C2 fp64 count moves with the OpenBLAS thread count
  (10504 at 4 threads, 10833 at 8), and this solver's moves
  with the reduction order (10438-10913 for 148/144/128/100/74 CTAs,
  profiles/r02_C2_fp64_spread.json).  Every pair of runs -- reference vs
  GPU, or GPU vs GPU with another CTA count -- agrees to ~1e-13 for the
  first ~37 cycles and then diverges exponentially.  So the tests pin
  (a) the histories to rounding over the pre-chaotic window, (b) the
  trajectories to a bounded band over the whole solve, and (c) the counts
  to the reference's spread widened by one restart cycle.
"""

import glob
import json
import os

import numpy as np
import pytest

import paper_2105_07544_b200 as mk

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
P = mk.Precision


def explicit(rep, phase):
    return np.array([e.explicit_relres for e in rep.history if e.phase == phase and e.explicit_relres is not None])


def big(case):
    """Reference runs of `case` at every recorded BLAS thread count."""
    return [np.load(f) for f in sorted(glob.glob(os.path.join(GOLD, "big", case + "_t*.npz")))]


@pytest.fixture(scope="module")
def bentpipe():
    return mk.generate_stencil(mk.ProblemSpec("BentPipe2D", 1500))


def test_c2_gmres_ir_matches_reference_run(bentpipe):
    """C2 GMRES-IR(50) vs the reference's full run (710 s of CPU)."""
    ref = json.load(open(os.path.join(GOLD, "runs.json")))["ir_bp1500"]
    A = bentpipe
    inner = mk.SolverConfig(m=50, rtol=1e-4, precision=P.binary32, max_iters=100000)
    rep = mk.gmres_ir(A, np.ones(A.n), np.zeros(A.n), mk.IrConfig(inner=inner, rtol=1e-10))
    assert rep.converged and rep.final_explicit_relres <= 1e-10
    # fp32 inner cycles make the count chaotic in the last bit: the
    # reference itself gives 10250 (1 OpenBLAS thread, big/c2_ir_t1.npz) and
    # 10650 (8 threads, runs.json); this solver 10400-10800 for
    # 148/144/128/100/74 CTAs (profiles/r02_C2_ir_spread.json).  Hold the
    # count to the reference's spread widened by one restart cycle.
    counts = [int(ref["iters"])] + [int(g["iters"]) for g in big("c2_ir")]
    assert min(counts) - 50 <= rep.total_iters <= max(counts) + 50, (rep.total_iters, counts)
    ours = explicit(rep, "outer")
    theirs = np.array([r[3] for r in ref["history"] if r[1] == "outer"])
    k = min(len(ours), len(theirs))
    rel = np.abs(ours[:k] / theirs[:k] - 1)
    # fp32 inner cycles: the first 30 refinements agree to 1e-5 (observed
    # 2.3e-7 .. 1.1e-6 across stream shapes)
    assert rel[:30].max() <= 1e-5, rel[:30].max()
    # then the fp32 trajectories drift apart but stay within a factor 10^0.5
    # of each other (observed max 0.34 decades)
    assert np.abs(np.log10(ours[:k] / theirs[:k])).max() <= 0.5


def test_c2_fp64_gmres_matches_reference_runs(bentpipe):
    """C2 fp64 GMRES(50) vs the reference's full runs (20 min of CPU each)."""
    runs = big("c2_fp64")
    assert runs, "missing tests/golden/big/c2_fp64_t*.npz"
    A = bentpipe
    rep = mk.gmres_restarted(A, None, np.ones(A.n), np.zeros(A.n), mk.SolverConfig(m=50, rtol=1e-10,
                                                                                   max_iters=100000))
    assert rep.converged and rep.final_explicit_relres <= 1e-10
    ours = np.array([e.explicit_relres for e in rep.history if e.explicit_relres is not None])
    impl = np.array([np.nan if e.implicit_relres is None else e.implicit_relres for e in rep.history])
    for g in runs:
        theirs = g["h_expl"][~np.isnan(g["h_expl"])]
        # pre-chaotic window: 36 restart cycles (1800 iterations) to 1e-11
        # relative (observed 3.4e-13); implicit residuals of the first 30
        # cycles to 1e-12 (observed 7e-14; 1.2e-12 by iteration 1800)
        assert np.abs(ours[:37] / theirs[:37] - 1).max() <= 1e-11
        gi = g["h_impl"][:1500]
        m = ~np.isnan(gi) & ~np.isnan(impl[:1500])
        assert np.abs(impl[:1500][m] / gi[m] - 1).max() <= 1e-12
        k = min(len(ours), len(theirs))
        assert np.abs(np.log10(ours[:k] / theirs[:k])).max() <= 0.5   # observed 0.29 decades
    # the reference's own counts: 10300 (1 OpenBLAS thread), 10504 (4),
    # 10833 (8); within one restart cycle of that spread
    counts = [int(g["iters"]) for g in runs] + [10833]
    assert min(counts) - 50 <= rep.total_iters <= max(counts) + 50, (rep.total_iters, counts)


@pytest.fixture(scope="module")
def laplace200():
    return mk.generate_stencil(mk.ProblemSpec("Laplace3D", 200))


def test_c4_fp64_gmres_matches_reference_run(laplace200):
    """C4 (north_star's config) fp64 GMRES(50) vs the reference's full run
    (36 min of CPU): same iteration count (4053 = the paper's), histories
    equal to rounding (Laplace3D is not chaotic like BentPipe2D)."""
    runs = big("c4_fp64")
    assert runs, "missing tests/golden/big/c4_fp64_t*.npz"
    A = laplace200
    rep = mk.gmres_restarted(A, None, np.ones(A.n), np.zeros(A.n), mk.SolverConfig(m=50, rtol=1e-10,
                                                                                   max_iters=100000))
    assert rep.converged and rep.final_explicit_relres <= 1e-10
    ours = np.array([e.explicit_relres for e in rep.history if e.explicit_relres is not None])
    impl = np.array([np.nan if e.implicit_relres is None else e.implicit_relres for e in rep.history])
    for g in runs:
        assert rep.total_iters == int(g["iters"]) and rep.restarts == int(g["restarts"])
        theirs = g["h_expl"][~np.isnan(g["h_expl"])]
        assert len(ours) == len(theirs)
        rel = np.abs(ours / theirs - 1)
        assert rel[:25].max() <= 1e-12 and rel.max() <= 1e-4, (rel[:25].max(), rel.max())   # observed 2.4e-5
        gi = g["h_impl"]
        m = ~np.isnan(gi) & ~np.isnan(impl)
        assert np.abs(impl[m] / gi[m] - 1).max() <= 1e-4


def test_c4_gmres_ir_matches_reference_runs(laplace200):
    """C4 GMRES-IR(50), breakdown rule "u", vs the reference's
    own runs with that rule (make_big_golden.py c4_ir_u, 1 and 4 OpenBLAS
    threads): identical counts (4100 iterations, 82 refinements = the paper's
    Trilinos count), per-refinement explicit residuals within 1e-2 relative
    (fp32 inner cycles; observed 1.5e-3, reference t1 vs t4 9e-5)."""
    runs = big("c4_ir_u")
    assert runs, "missing tests/golden/big/c4_ir_u_t*.npz"
    A = laplace200
    inner = mk.SolverConfig(m=50, rtol=1e-4, precision=P.binary32, max_iters=100000, breakdown_rule="u")
    rep = mk.gmres_ir(A, np.ones(A.n), np.zeros(A.n), mk.IrConfig(inner=inner, rtol=1e-10))
    assert rep.converged and rep.final_explicit_relres <= 1e-10
    ours = explicit(rep, "outer")
    for g in runs:
        assert rep.total_iters == int(g["iters"]) and rep.restarts == int(g["restarts"])
        theirs = g["h_expl"][g["h_phase"] == 2]
        assert len(ours) == len(theirs)
        rel = np.abs(ours / theirs - 1)
        assert rel[:7].max() <= 1e-4 and rel.max() <= 1e-2, (rel[:7].max(), rel.max())


def test_c4_gmres_fd_matches_reference_run(laplace200):
    """C4 GMRES-FD(50), fp32 for 2000 iterations then fp64 (rule "u" in both
    phases), vs the reference's full run (make_big_golden.py c4_fd_u, 4
    OpenBLAS threads: 3707 iterations, 75 restarts)."""
    runs = big("c4_fd_u")
    assert runs, "missing tests/golden/big/c4_fd_u_t*.npz"
    A = laplace200
    low = mk.SolverConfig(m=50, rtol=1e-10, precision=P.binary32, max_iters=100000, breakdown_rule="u")
    high = mk.SolverConfig(m=50, rtol=1e-10, max_iters=100000, breakdown_rule="u")
    rep = mk.gmres_fd(A, np.ones(A.n), np.zeros(A.n), mk.FdConfig(switch_iter=2000, low=low, high=high))
    assert rep.converged and rep.final_explicit_relres <= 1e-10
    ours = np.array([e.explicit_relres for e in rep.history if e.explicit_relres is not None])
    for g in runs:
        assert abs(rep.total_iters - int(g["iters"])) <= 50, (rep.total_iters, int(g["iters"]))
        theirs = g["h_expl"][~np.isnan(g["h_expl"])]
        k = min(len(ours), len(theirs))
        rel = np.abs(ours[:k] / theirs[:k] - 1)
        # fp32 phase: the first 20 restart residuals to 1e-3 (fp32 Arnoldi;
        # it then stagnates near 3e-4 at a rounding-determined level), the
        # whole run within 0.3 decades
        assert rel[:20].max() <= 1e-3, rel[:20].max()
        assert np.abs(np.log10(ours[:k] / theirs[:k])).max() <= 0.3
