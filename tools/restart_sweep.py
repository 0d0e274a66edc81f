"""Restart-length sweep of the paper (BentPipe2D 1500^2,
m = 25..400, fp64 GMRES vs GMRES-IR to 1e-10), timed with CUDA events.
Prints one JSON object; python tools/restart_sweep.py [m ...]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2105_07544_b200 as mk
P = mk.Precision
ms = [int(v) for v in sys.argv[1:]] or [25, 50, 100, 150, 200, 300, 400]
A = mk.generate_stencil(mk.ProblemSpec("BentPipe2D", 1500))
Al = mk.convert_matrix(A, P.binary32)
b = torch.ones(A.n, dtype=torch.float64, device="cuda"); x0 = torch.zeros_like(b)
def timed(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); rep = fn(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3, rep
out = []
for m in ms:
    inner = mk.SolverConfig(m=m, rtol=1e-4, precision=P.binary32, max_iters=100000)
    t_ir, r_ir = timed(lambda: mk.gmres_ir(A, b, x0, mk.IrConfig(inner=inner, rtol=1e-10), A_low=Al))
    t_64, r_64 = timed(lambda: mk.gmres_restarted(A, None, b, x0, mk.SolverConfig(m=m, rtol=1e-10, max_iters=100000)))
    row = {"m": m, "fp64_s": t_64, "fp64_iters": r_64.total_iters, "ir_s": t_ir, "ir_iters": r_ir.total_iters,
           "speedup": t_64 / t_ir, "converged": bool(r_ir.converged and r_64.converged)}
    if m <= 51:   # third precision: binary16 Krylov basis in the inner cycles
        inner16 = mk.SolverConfig(m=m, rtol=1e-4, precision=P.binary32, max_iters=100000,
                                  basis_precision="binary16")
        t_h, r_h = timed(lambda: mk.gmres_ir(A, b, x0, mk.IrConfig(inner=inner16, rtol=1e-10), A_low=Al))
        row.update(ir16_s=t_h, ir16_iters=r_h.total_iters, ir16_speedup=t_64 / t_h,
                   ir16_converged=bool(r_h.converged))
    out.append(row)
    print(json.dumps(row), flush=True)
print(json.dumps({"sweep": "BentPipe2D 1500^2, b = ones, rtol 1e-10, one B200", "rows": out}))
