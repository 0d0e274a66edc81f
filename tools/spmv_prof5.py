"""C5 standalone CSR SpMV launches for ncu: fp32/fp64, x-window on (row
statistics) and off (band forced to 0)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2105_07544_b200 as mk
from paper_2105_07544_b200.sparse import spmv_into
P = mk.Precision
C = mk.synthetic_irregular(4000000, signs="negative", dominance=1.001, shift=1e-3, far_frac=0.01, band=2000)
for band0 in (False, True):
    for prec in (P.binary32, P.binary64):
        B = mk.convert_matrix(C, prec)
        B._desc = None
        if band0:
            B._band = 0
        x = torch.randn(C.n, dtype=prec.torch_dtype, device="cuda")
        y = torch.empty_like(x)
        spmv_into(B, x, y)
        torch.cuda.synchronize()
        print(prec.value, "band", B.band_width(), flush=True)
