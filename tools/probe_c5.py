"""C5 calibration probe: generate the synthetic irregular CSR, build Jacobi(1),
run capped fp64 GMRES(50)+J1, GMRES-IR+J1 and GMRES-FD; print iterations and
us/iteration.  python tools/probe_c5.py N signs dominance shift far_frac [cap]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2105_07544_b200 as mk
P = mk.Precision
n = int(sys.argv[1]); signs = sys.argv[2]; dom = float(sys.argv[3]); shift = float(sys.argv[4])
far = float(sys.argv[5]); cap = int(sys.argv[6]) if len(sys.argv) > 6 else 2000
t0 = time.time()
A = mk.synthetic_irregular(n, signs=signs, dominance=dom, shift=shift, far_frac=far)
t1 = time.time()
lens = np.diff(A.row_ptr)
print("n %d nnz %d mean %.1f std %.1f max %d; gen %.1f s" % (n, A.nnz, lens.mean(), lens.std(), lens.max(), t1 - t0), flush=True)
Al = mk.convert_matrix(A, P.binary32)
J64 = mk.build_block_jacobi(A, 1)
J32 = mk.build_block_jacobi(Al, 1)
print("setup %.1f s" % (time.time() - t1), flush=True)
b = torch.ones(n, dtype=torch.float64, device="cuda"); x0 = torch.zeros_like(b)
runs = [("fp64+J1", lambda mi: mk.gmres_restarted(A, J64, b, x0, mk.SolverConfig(m=50, rtol=1e-10, max_iters=mi))),
        ("IR+J1", lambda mi: mk.gmres_ir(A, b, x0, mk.IrConfig(inner=mk.SolverConfig(m=50, rtol=1e-4, precision=P.binary32, max_iters=mi, breakdown_rule="u"), rtol=1e-10), M=J32, A_low=Al)),
        ("fp64", lambda mi: mk.gmres_restarted(A, None, b, x0, mk.SolverConfig(m=50, rtol=1e-10, max_iters=mi)))]
for name, run in runs:
    run(5)
    torch.cuda.synchronize(); t = time.time()
    rep = run(cap)
    torch.cuda.synchronize(); dt = time.time() - t
    print("%-8s %5d iters relres %.3e conv %s  %.3f s  %.1f us/iter" % (name, rep.total_iters, rep.final_explicit_relres, rep.converged, dt, dt * 1e6 / max(rep.total_iters, 1)), flush=True)
