"""C5 GMRES-IR(50)+J1 with the banded-CSR x window on and off (band forced
to 0), CUDA events, same build."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2105_07544_b200 as mk
P = mk.Precision
A = mk.synthetic_irregular(4000000, signs="negative", dominance=1.001, shift=1e-3, far_frac=0.01, band=2000)
for band0 in (False, True, False, True):
    B = mk.CsrMatrix(A.n, A.row_ptr, A.col_idx, A.values, validate=False)
    if band0:
        B._band = 0
    Bl = mk.convert_matrix(B, P.binary32)
    M32 = mk.build_block_jacobi(Bl, 1)
    inner = mk.SolverConfig(m=50, rtol=1e-4, precision=P.binary32, max_iters=100000, breakdown_rule="u")
    b = torch.ones(A.n, dtype=torch.float64, device="cuda"); x0 = torch.zeros_like(b)
    cfg = mk.IrConfig(inner=inner, rtol=1e-10)
    mk.gmres_ir(B, b, x0, cfg, M=M32, A_low=Bl)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rep = mk.gmres_ir(B, b, x0, cfg, M=M32, A_low=Bl)
    e1.record(); torch.cuda.synchronize()
    print("window %s band %d: IR %d iters %.3f s" % ("off" if band0 else "on", Bl.band_width(), rep.total_iters,
                                                   e0.elapsed_time(e1) / 1e3), flush=True)
