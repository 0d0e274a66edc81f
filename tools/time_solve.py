"""Time a capped solve of a BASELINE config (CUDA events; for A/B experiments,
not the bench).  python tools/time_solve.py --config C2 --solver ir --max-iters 1000"""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2105_07544_b200 as mk
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--solver", default="ir")
ap.add_argument("--max-iters", type=int, default=1000)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--m", type=int, default=50)
ap.add_argument("--orth", default="cgs2")
ap.add_argument("--rule", default="n_u")
ap.add_argument("--basis", default="working")
a = ap.parse_args()
spec = {"C1": ("Laplace3D", 40), "C2": ("BentPipe2D", 1500), "C4": ("Laplace3D", 200),
        "C3": ("UniFlow2D", 2500)}[a.config]
A = mk.generate_stencil(mk.ProblemSpec(*spec))
b = torch.ones(A.n, dtype=torch.float64, device="cuda"); x0 = torch.zeros_like(b)
P = mk.Precision
if a.solver == "ir":
    Al = mk.convert_matrix(A, P.binary32)
    inner = mk.SolverConfig(m=a.m, rtol=1e-4, precision=P.binary32, max_iters=a.max_iters, orthogonalization=a.orth,
                           breakdown_rule=a.rule, basis_precision=a.basis)
    run = lambda: mk.gmres_ir(A, b, x0, mk.IrConfig(inner=inner, rtol=1e-10), A_low=Al)
else:
    run = lambda: mk.gmres_restarted(A, None, b, x0, mk.SolverConfig(m=a.m, rtol=1e-10, max_iters=a.max_iters,
                                                                                orthogonalization=a.orth))
run()
best = 1e30
for _ in range(a.reps):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); rep = run(); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print("%s %s %s %s m=%d TR=%s iters %d relres %.3e  %.2f ms  %.1f us/iter" % (a.config, a.solver, a.orth, a.basis, a.m, os.environ.get("MPK_FUSED_TR", "default"),
      rep.total_iters, rep.final_explicit_relres, best, best * 1e3 / rep.total_iters))
