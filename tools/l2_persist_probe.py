"""Probe: does an L2 persisting access-policy window over the cycle's work
vectors (w, w', w'': 3 x 32 MB fp32 at C4) speed up the persistent cycle?
Sets cudaLimitPersistingL2CacheSize and the stream's access-policy window
with cuda-python, then times the capped C4 / C2 IR solve (CUDA events)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from cuda.bindings import runtime as rt
import paper_2105_07544_b200 as mk
from paper_2105_07544_b200.engine import CycleWorkspace
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--mb", type=int, default=64)      # persisting set-aside
ap.add_argument("--vecs", type=int, default=3)     # work vectors in the window
ap.add_argument("--ratio", type=float, default=-1)
a = ap.parse_args()
spec = {"C2": ("BentPipe2D", 1500), "C4": ("Laplace3D", 200)}[a.config]
P = mk.Precision
A = mk.generate_stencil(mk.ProblemSpec(*spec))
Al = mk.convert_matrix(A, P.binary32)
b = torch.ones(A.n, dtype=torch.float64, device="cuda"); x0 = torch.zeros_like(b)
inner = mk.SolverConfig(m=50, rtol=1e-4, precision=P.binary32, max_iters=1000,
                        breakdown_rule="u" if a.config == "C4" else "n_u")
run = lambda: mk.gmres_ir(A, b, x0, mk.IrConfig(inner=inner, rtol=1e-10), A_low=Al)
run()
ws = CycleWorkspace.get(A.n, 50, P.binary32)
def timed():
    best = 1e30
    for _ in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); rep = run(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best, rep.total_iters
t0, it = timed()
err, = rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize, a.mb << 20)[:1]
_, maxwin = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxAccessPolicyWindowSize, 0)
_, got = rt.cudaDeviceGetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize)
nbytes = min(a.vecs * ws.ld * 4, maxwin)
val = rt.cudaStreamAttrValue()
w = val.accessPolicyWindow
w.base_ptr = ws.work.data_ptr()
w.num_bytes = nbytes
w.hitRatio = a.ratio if a.ratio > 0 else min(1.0, got / nbytes)
w.hitProp = rt.cudaAccessProperty.cudaAccessPropertyPersisting
w.missProp = rt.cudaAccessProperty.cudaAccessPropertyStreaming
stream = torch.cuda.current_stream().cuda_stream
e2, = rt.cudaStreamSetAttribute(stream, rt.cudaStreamAttrID.cudaLaunchAttributeAccessPolicyWindow, val)[:1]
t1, it1 = timed()
print("%s setlimit=%s got=%d MB maxwin=%d MB window=%d MB ratio=%.2f attr=%s | off %.2f ms (%d it) | on %.2f ms (%d it) | %.3fx"
      % (a.config, err, got >> 20, maxwin >> 20, nbytes >> 20, w.hitRatio, e2, t0, it, t1, it1, t0 / t1))
