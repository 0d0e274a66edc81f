"""Phase breakdown of the persistent cycle kernel (clock64 per section, CTA
0 and the max over CTAs) on one cycle of a BASELINE config."""
import argparse, ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2105_07544_b200 as mk
from paper_2105_07544_b200 import _lib
from paper_2105_07544_b200.engine import CycleWorkspace
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--prec", default="fp32")
a = ap.parse_args()
spec = {"C1": ("Laplace3D", 40), "C2": ("BentPipe2D", 1500), "C4": ("Laplace3D", 200)}[a.config]
A = mk.generate_stencil(mk.ProblemSpec(*spec))
P = mk.Precision
prec = P.binary32 if a.prec == "fp32" else P.binary64
Al = mk.convert_matrix(A, prec)
b = torch.ones(A.n, dtype=prec.torch_dtype, device="cuda")
cfg = mk.SolverConfig(m=50, rtol=1e-30 if prec is P.binary64 else 1e-7, precision=prec,
                      breakdown_rule="u" if a.config == "C4" else "n_u")
mk.gmres_cycle(Al, None, b, torch.zeros_like(b), cfg)
ws = CycleWorkspace.get(A.n, 50, prec)
ws.flags = 8
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
x, st = mk.gmres_cycle(Al, None, b, torch.zeros_like(b), cfg)
e1.record(); torch.cuda.synchronize()
ws.flags = 0
nct = 148
buf = (ctypes.c_uint64 * (nct * 16))()
_lib.check(_lib.load().mpk_fused_prof_read(buf, nct))
p = np.array(buf[:], dtype=np.float64).reshape(nct, 16)
names = ["v_k", "SpMV", "stream A", "barrier A", "reduce A", "stream B", "barrier B", "reduce B",
         "stream C", "barrier C", "reduce C", "Givens(last)", "Givens", "epilogue"]
tot0 = p[0, :14].sum()
print("%s %s: cycle %.3f ms, %d steps, event %.3f ms" % (a.config, a.prec, tot0 / 1.965e6, st.steps, e0.elapsed_time(e1)))
for i, nm in enumerate(names):
    print("  %-12s cta0 %8.1f us (%4.1f%%)   mean %8.1f us  max %8.1f us" % (nm, p[0, i] / 1965, 100 * p[0, i] / tot0,
          p[:, i].mean() / 1965, p[:, i].max() / 1965))
