"""Profiling driver: one GMRES-IR (or fp64 GMRES) solve of a BASELINE config,
for ncu launch lists / full captures.  Not a benchmark (numbers under a
profiler are not bench values)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2105_07544_b200 as mk
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--solver", default="ir")
ap.add_argument("--max-iters", type=int, default=100000)
ap.add_argument("--orth", default="cgs2")
ap.add_argument("--basis", default="working")
a = ap.parse_args()
spec = {"C1": ("Laplace3D", 40), "C2": ("BentPipe2D", 1500), "C4": ("Laplace3D", 200)}[a.config]
A = mk.generate_stencil(mk.ProblemSpec(*spec))
b = torch.ones(A.n, dtype=torch.float64, device="cuda"); x0 = torch.zeros_like(b)
if a.solver == "ir":
    inner = mk.SolverConfig(m=50, rtol=1e-4, precision=mk.Precision.binary32, max_iters=a.max_iters,
                            orthogonalization=a.orth, basis_precision=a.basis, breakdown_rule="u" if a.config == "C4" else "n_u")
    rep = mk.gmres_ir(A, b, x0, mk.IrConfig(inner=inner, rtol=1e-10), A_low=mk.convert_matrix(A, mk.Precision.binary32))
else:
    rep = mk.gmres_restarted(A, None, b, x0, mk.SolverConfig(m=50, rtol=1e-10, max_iters=a.max_iters))
torch.cuda.synchronize()
print("iters", rep.total_iters, "relres", rep.final_explicit_relres)
