"""Run BASELINE-scale solves on the GPU and dump their histories in the
format of tests/golden/make_big_golden.py (for comparison with the
reference's own runs on the CPU box).

    python tools/dump_big.py c2_fp64 c2_ir c4_fp64 c4_ir_u [--out gpurun_out]
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2105_07544_b200 as mk  # noqa: E402

PHASES = {"cycle": 0, "inner": 1, "outer": 2, "low": 3, "high": 4}


def run(case):
    P = mk.Precision
    if case.startswith("c2"):
        A = mk.generate_stencil(mk.ProblemSpec("BentPipe2D", 1500))
    elif case.startswith("c4"):
        A = mk.generate_stencil(mk.ProblemSpec("Laplace3D", 200))
    else:
        A = mk.generate_stencil(mk.ProblemSpec("Laplace3D", 40))
    b = np.ones(A.n)
    rule = "u" if case.endswith("_u") else "n_u"
    orth = "dcgs2" if "dcgs2" in case else "cgs2"
    if "fp64" in case:
        cfg = mk.SolverConfig(m=50, rtol=1e-10, max_iters=100000, breakdown_rule=rule, orthogonalization=orth)
        fn = lambda: mk.gmres_restarted(A, None, b, np.zeros(A.n), cfg)  # noqa: E731
    else:
        inner = mk.SolverConfig(m=50, rtol=1e-4, precision=P.binary32, max_iters=100000, breakdown_rule=rule,
                                orthogonalization=orth)
        fn = lambda: mk.gmres_ir(A, b, np.zeros(A.n), mk.IrConfig(inner=inner, rtol=1e-10))  # noqa: E731
    t0 = time.perf_counter()
    rep = fn()
    wall = time.perf_counter() - t0
    h = rep.history
    nan = float("nan")
    return rep, wall, dict(
        converged=bool(rep.converged), iters=int(rep.total_iters), restarts=int(rep.restarts),
        relres=float(rep.final_explicit_relres), loss=bool(rep.loss_of_accuracy), wall=wall,
        h_iter=np.array([e.iteration for e in h], np.int32),
        h_phase=np.array([PHASES.get(e.phase, 9) for e in h], np.int8),
        h_impl=np.array([nan if e.implicit_relres is None else e.implicit_relres for e in h]),
        h_expl=np.array([nan if e.explicit_relres is None else e.explicit_relres for e in h]))


def main():
    out = "gpurun_out"
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    if "--out" in sys.argv:
        out = sys.argv[sys.argv.index("--out") + 1]
        args.remove(out)
    os.makedirs(out, exist_ok=True)
    for case in args:
        rep, wall, d = run(case)
        np.savez_compressed(os.path.join(out, "ours_%s.npz" % case), **d)
        print(case, "iters", rep.total_iters, "restarts", rep.restarts, "relres", rep.final_explicit_relres,
              "converged", rep.converged, "%.2fs" % wall, flush=True)


if __name__ == "__main__":
    main()
