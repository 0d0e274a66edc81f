"""Per-CTA stream time of the persistent cycle (phase profiler, desc flag
bit 3), twice, to tell systematic imbalance (the same CTAs slow in both
runs) from jitter."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2105_07544_b200 as mk
from paper_2105_07544_b200 import _lib
from paper_2105_07544_b200.engine import CycleWorkspace
cfgname = sys.argv[1] if len(sys.argv) > 1 else "C2"
spec = {"C1": ("Laplace3D", 40), "C2": ("BentPipe2D", 1500), "C4": ("Laplace3D", 200)}[cfgname]
A = mk.generate_stencil(mk.ProblemSpec(*spec))
P = mk.Precision
Al = mk.convert_matrix(A, P.binary32)
b = torch.ones(A.n, dtype=torch.float32, device="cuda")
cfg = mk.SolverConfig(m=50, rtol=1e-7, precision=P.binary32, breakdown_rule="u")
mk.gmres_cycle(Al, None, b, torch.zeros_like(b), cfg)
ws = CycleWorkspace.get(A.n, 50, P.binary32)
runs = []
for rep in range(3):
    ws.flags = 8
    mk.gmres_cycle(Al, None, b, torch.zeros_like(b), cfg)
    torch.cuda.synchronize()
    ws.flags = 0
    nct = 148
    buf = (ctypes.c_uint64 * (nct * 16))()
    _lib.check(_lib.load().mpk_fused_prof_read(buf, nct))
    raw = np.array(buf[:], dtype=np.float64).reshape(nct, 16)
    p = raw / 1965.0
    p[:, 15] = raw[:, 15]   # smid
    runs.append(p)
for p in runs:
    streams = p[:, 2] + p[:, 5] + p[:, 8] + p[:, 1]
    waits = p[:, 3] + p[:, 6] + p[:, 9]
    print("streams+spmv us: mean %.0f min %.0f max %.0f | waits mean %.0f" % (streams.mean(), streams.min(),
                                                                             streams.max(), waits.mean()))
s = [p[:, 2] + p[:, 5] + p[:, 8] + p[:, 1] for p in runs]
print("corr run0-run1 %.3f run1-run2 %.3f" % (np.corrcoef(s[0], s[1])[0, 1], np.corrcoef(s[1], s[2])[0, 1]))
order = np.argsort(-s[0])
print("slowest CTAs run0:", order[:12].tolist(), "their run1 rank:", [int((s[1] > s[1][i]).sum()) for i in order[:12]])
print("smid of the slowest CTAs (run0, run1):", [int(runs[0][i, 15]) for i in order[:12]],
      [int(runs[1][i, 15]) for i in order[:12]])
print("per-CTA stream us (run0):", np.round(s[0]).astype(int).tolist())
print("per-CTA smid (run0):", runs[0][:, 15].astype(int).tolist())
