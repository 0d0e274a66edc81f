"""Polynomial-preconditioner probe (default C3: UniFlow2D 2500^2 + GMRES poly(25)): setup time, capped IR and
fp64 runs (per-iteration time, residual reached)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2105_07544_b200 as mk
P = mk.Precision
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2500
cap = int(sys.argv[2]) if len(sys.argv) > 2 else 100
deg = int(sys.argv[3]) if len(sys.argv) > 3 else 25
preset = sys.argv[4] if len(sys.argv) > 4 else "UniFlow2D"
A = mk.generate_stencil(mk.ProblemSpec(preset, nx))
Al = mk.convert_matrix(A, P.binary32)
t0 = time.time()
if deg:
    M32 = mk.build_gmres_poly(Al, deg, np.ones(A.n, np.float32), rule="u")
    M64 = mk.build_gmres_poly(A, deg, np.ones(A.n))
else:
    class _D: degree = 0
    class _M: data = _D()
    M32 = M64 = None
torch.cuda.synchronize()
print("%s %d: setup %.2f s, degrees %s / %s" % (preset, nx, time.time() - t0, M32.data.degree if M32 else 0,
      M64.data.degree if M64 else 0), flush=True)
b = torch.ones(A.n, dtype=torch.float64, device="cuda"); x0 = torch.zeros_like(b)
for name, run in (("ir", lambda mi: mk.gmres_ir(A, b, x0, mk.IrConfig(inner=mk.SolverConfig(m=50, rtol=1e-4, precision=P.binary32, max_iters=mi, breakdown_rule="u"), rtol=1e-10), M=M32, A_low=Al)),
                  ("fp64", lambda mi: mk.gmres_restarted(A, M64, b, x0, mk.SolverConfig(m=50, rtol=1e-10, max_iters=mi)))):
    run(10)
    torch.cuda.synchronize(); t = time.time()
    rep = run(cap)
    torch.cuda.synchronize(); dt = time.time() - t
    print("%s: %d iters, relres %.3e, converged %s, %.3f s, %.1f us/iter" % (name, rep.total_iters, rep.final_explicit_relres, rep.converged, dt, dt * 1e6 / max(rep.total_iters, 1)), flush=True)
