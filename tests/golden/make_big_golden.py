"""BASELINE-scale golden runs of the UNMODIFIED reference (mpkrylov from
/root/reference/pkg/src), generated in the survey container and committed
because /root/reference does not exist on the GPU box.

    PYTHONPATH=/root/reference/pkg/src OPENBLAS_NUM_THREADS=T \
        python tests/golden/make_big_golden.py CASE

CASE is one of
  c2_fp64      BentPipe2D 1500^2, fp64 GMRES(50), rtol 1e-10   (gmres.py:221-308)
  c4_fp64      Laplace3D 200^3,   fp64 GMRES(50), rtol 1e-10
  c4_ir_u      Laplace3D 200^3,   GMRES-IR(50) fp32 inner, breakdown rule "u"
                                  (reference cgs2_append body with u*||w||)
  c4_fd_u      Laplace3D 200^3,   GMRES-FD(50), fp32 for 2000 iterations then fp64,
                                  breakdown rule "u" in both phases
  c1_fp64 / c1_ir   Laplace3D 40^3 (quick; used to check the thread spread)

Writes tests/golden/big/<CASE>_t<T>.npz with the counts, flags and the history
as arrays (iteration, phase code 0=cycle/1=inner/2=outer/3=low/4=high,
implicit, explicit; NaN where the reference stores None).  T is the OpenBLAS
thread count the reference ran with, recorded so the spread of the
reference's own count across BLAS thread counts is on file
(VERDICT r1 "the fp64 miss").
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)
import mpkrylov as mk  # noqa: E402
from mpkrylov import gmres as _g, kernels as _k, preconditioners as _p  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "big")
PHASES = {"cycle": 0, "inner": 1, "outer": 2, "low": 3, "high": 4}


def with_rule_u(fn):
    """Reference cgs2_append (kernels.py:114-126) with threshold u*||w||."""
    orig = _k.cgs2_append

    def cgs2_u(basis, w):
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


def main():
    case = sys.argv[1]
    threads = os.environ.get("OPENBLAS_NUM_THREADS", "default")
    P = mk.Precision
    if case.startswith("c2"):
        A = mk.generate_stencil(mk.ProblemSpec("BentPipe2D", 1500))
    elif case.startswith("c4"):
        A = mk.generate_stencil(mk.ProblemSpec("Laplace3D", 200))
    else:
        A = mk.generate_stencil(mk.ProblemSpec("Laplace3D", 40))
    b = np.ones(A.n)
    if "_fd" in case:
        low = mk.SolverConfig(m=50, rtol=1e-10, precision=P.binary32, max_iters=100000)
        high = mk.SolverConfig(m=50, rtol=1e-10, max_iters=100000)
        cfg = mk.FdConfig(switch_iter=2000, low=low, high=high)
        run = lambda: mk.gmres_fd(A, b, np.zeros(A.n), cfg)  # noqa: E731
        if case.endswith("_u"):
            run0 = run
            run = lambda: with_rule_u(run0)  # noqa: E731
    elif case.endswith("fp64"):
        cfg = mk.SolverConfig(m=50, rtol=1e-10, max_iters=100000)
        run = lambda: mk.gmres_restarted(A, None, b, np.zeros(A.n), cfg)  # noqa: E731
    else:
        inner = mk.SolverConfig(m=50, rtol=1e-4, precision=P.binary32, max_iters=100000)
        cfg = mk.IrConfig(inner=inner, rtol=1e-10)
        run = lambda: mk.gmres_ir(A, b, np.zeros(A.n), cfg)  # noqa: E731
        if case.endswith("_u"):
            run0 = run
            run = lambda: with_rule_u(run0)  # noqa: E731
    t0 = time.perf_counter()
    rep = run()
    wall = time.perf_counter() - t0
    h = rep.history
    nan = float("nan")
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(
        os.path.join(OUT, "%s_t%s.npz" % (case, threads)),
        converged=bool(rep.converged), iters=int(rep.total_iters), restarts=int(rep.restarts),
        relres=float(rep.final_explicit_relres), loss=bool(rep.loss_of_accuracy),
        stalled=bool(getattr(rep, "stalled", False)), baseline=float(rep.baseline),
        wall=wall, threads=str(threads),
        h_iter=np.array([e.iteration for e in h], np.int32),
        h_phase=np.array([PHASES.get(e.phase, 9) for e in h], np.int8),
        h_impl=np.array([nan if e.implicit_relres is None else e.implicit_relres for e in h]),
        h_expl=np.array([nan if e.explicit_relres is None else e.explicit_relres for e in h]),
    )
    print(case, "threads", threads, "iters", rep.total_iters, "restarts", rep.restarts,
          "relres", rep.final_explicit_relres, "converged", rep.converged, "%.1fs" % wall,
          flush=True)


if __name__ == "__main__":
    main()
