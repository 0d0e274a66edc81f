"""cProfile of the host side of GMRES-IR / fp64 GMRES solves (C1 Laplace3D
40^3: short cycles, so host bookkeeping is visible)."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2105_07544_b200 as mk
P = mk.Precision
A = mk.generate_stencil(mk.ProblemSpec("Laplace3D", 40))
A32 = mk.convert_matrix(A, P.binary32)
b = torch.ones(A.n, dtype=torch.float64, device="cuda"); x0 = torch.zeros_like(b)
inner = mk.SolverConfig(m=50, rtol=1e-4, precision=P.binary32)
cfg = mk.IrConfig(inner=inner, rtol=1e-10)
cfg64 = mk.SolverConfig(m=50, rtol=1e-10)
for _ in range(3):
    mk.gmres_ir(A, b, x0, cfg, A_low=A32); mk.gmres_restarted(A, None, b, x0, cfg64)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    r = mk.gmres_ir(A, b, x0, cfg, A_low=A32)
torch.cuda.synchronize()
print("IR solve wall %.3f ms (%d iters, %d refinements)" % ((time.perf_counter() - t0) / 20 * 1e3, r.total_iters, r.restarts))
t0 = time.perf_counter()
for _ in range(20):
    r = mk.gmres_restarted(A, None, b, x0, cfg64)
torch.cuda.synchronize()
print("fp64 solve wall %.3f ms (%d iters, %d restarts)" % ((time.perf_counter() - t0) / 20 * 1e3, r.total_iters, r.restarts))
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    mk.gmres_ir(A, b, x0, cfg, A_low=A32)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
