"""Histories of the reference-suite cases whose exact counts differ
(tools/run_ref_suite.sh), through the `mpkrylov` API: run with
PYTHONPATH=/root/reference/pkg/src (the reference, CPU) or
PYTHONPATH=tools/ref_suite (this package on cuda:0); writes JSON."""
import json
import sys

import numpy as np

import mpkrylov as mk


def lap(nx, preset="Laplace2D"):
    return mk.generate_stencil(mk.ProblemSpec(preset, nx))


def inner(m=50):
    return mk.SolverConfig(m=m, rtol=1e-4, precision=mk.Precision.binary32, max_iters=20000)


def fd(switch):
    return mk.FdConfig(switch_iter=switch, low=mk.SolverConfig(m=50, rtol=1e-10, precision=mk.Precision.binary32),
                       high=mk.SolverConfig(m=50, rtol=1e-10))


def rep(r):
    return {"iters": int(r.total_iters), "restarts": int(r.restarts), "converged": bool(r.converged),
            "relres": float(r.final_explicit_relres),
            "stalled": bool(getattr(r, "stalled", False)), "loss": bool(getattr(r, "loss_of_accuracy", False)),
            "hist": [[int(h.iteration), h.phase, None if h.implicit_relres is None else float(h.implicit_relres),
                      None if h.explicit_relres is None else float(h.explicit_relres)] for h in r.history]}


out = {}
A = lap(4)
out["stall"] = rep(mk.gmres_ir(A, 1e-15 * np.ones(A.n), np.zeros(A.n), mk.IrConfig(inner=inner(10), rtol=1e-14)))
A = lap(32)
out["noise_m100"] = rep(mk.gmres_ir(A, np.ones(A.n), np.zeros(A.n), mk.IrConfig(inner=inner(100), rtol=1e-10)))
out["ir_m50"] = rep(mk.gmres_ir(A, np.ones(A.n), np.zeros(A.n), mk.IrConfig(inner=inner(50), rtol=1e-10)))
out["fd50"] = rep(mk.gmres_fd(A, np.ones(A.n), np.zeros(A.n), fd(50)))
As = mk.generate_stencil(mk.ProblemSpec("Stretched2D", 32))
b = np.ones(As.n)
M = mk.wrap_low_precision_preconditioner(
    mk.build_gmres_poly(mk.convert_matrix(As, mk.Precision.binary32), 20, b.astype(np.float32)), mk.Precision.binary64)
out["loss"] = rep(mk.gmres_restarted(As, M, b, np.zeros(As.n), mk.SolverConfig(m=50, rtol=1e-10, max_iters=2000)))
json.dump(out, open(sys.argv[1], "w"), indent=0)
for k, v in out.items():
    print(k, v["iters"], v["restarts"], v["converged"], v["stalled"], v["loss"], "%.3e" % v["relres"])
