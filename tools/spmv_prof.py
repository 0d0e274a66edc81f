"""One standalone SpMV launch per (matrix, form, precision), for ncu captures:
    ncu --set full -k regex:k_spmv python tools/spmv_prof.py
Order: C4 stencil f32, C4 stencil f64, C2 CSR f32, C2 CSR f64, C5 CSR f32, C5 CSR f64."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2105_07544_b200 as mk
from paper_2105_07544_b200.sparse import spmv_into
P = mk.Precision


def once(A, prec):
    B = mk.convert_matrix(A, prec)
    x = torch.randn(A.n, dtype=prec.torch_dtype, device="cuda")
    y = torch.empty_like(x)
    spmv_into(B, x, y)
    torch.cuda.synchronize()


L = mk.generate_stencil(mk.ProblemSpec("Laplace3D", 200))
once(L, P.binary32)
once(L, P.binary64)
S = mk.generate_stencil(mk.ProblemSpec("BentPipe2D", 1500))
S.use_stencil = False
once(S, P.binary32)
once(S, P.binary64)
C = mk.synthetic_irregular(4000000, signs="negative", dominance=1.001, shift=1e-3, far_frac=0.01, band=2000)
once(C, P.binary32)
once(C, P.binary64)
