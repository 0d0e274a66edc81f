"""Standalone SpMV timing (CUDA events): C5 synthetic CSR and stencil configs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2105_07544_b200 as mk
from paper_2105_07544_b200.sparse import spmv_into
P = mk.Precision
peak = 6539.5
def bench(name, A, reps=20):
    for prec in (P.binary64, P.binary32):
        B = mk.convert_matrix(A, prec)
        sv0 = 4 if prec is P.binary32 else 8
        npair = max(1, min(20, -(-384 * 2**20 // (2 * sv0 * A.n))))   # vectors never L2-resident across launches
        pairs = [(torch.randn(A.n, dtype=prec.torch_dtype, device="cuda"),
                  torch.empty(A.n, dtype=prec.torch_dtype, device="cuda")) for _ in range(npair)]
        x, y = pairs[0]
        spmv_into(B, x, y); torch.cuda.synchronize()
        # captured in a CUDA graph: a Python launch loop is host-bound for short kernels
        side = torch.cuda.Stream(); side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side): spmv_into(B, x, y)
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(reps): spmv_into(B, *pairs[i % npair])
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        sv = 4 if prec is P.binary32 else 8
        if B.stencil is not None and B.use_stencil:
            byt = 2.0 * sv * A.n
        else:
            byt = sv * (A.nnz + 2.0 * A.n) + 4.0 * (A.nnz + A.n + 1)
        print("%-28s %s %.3f ms  %.0f GB/s alg (%.0f%% of %.0f)" % (name, prec.value, ms, byt / ms / 1e6, 100 * byt / ms / 1e6 / peak, peak), flush=True)
A = mk.synthetic_irregular(4000000, signs="negative", dominance=1.001, shift=1e-3)
bench("C5 synthetic CSR", A)
S = mk.generate_stencil(mk.ProblemSpec("BentPipe2D", 1500))
bench("C2 BentPipe stencil", S)
S.use_stencil = False
bench("C2 BentPipe CSR", S)
L = mk.generate_stencil(mk.ProblemSpec("Laplace3D", 200))
bench("C4 Laplace3D stencil", L)
L.use_stencil = False
bench("C4 Laplace3D CSR", L)
