"""Diagnostics: GPU solver histories vs the reference goldens (prints worst diffs)."""
import json, sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2105_07544_b200 as mk
P = mk.Precision
runs = json.load(open("tests/golden/runs.json"))
L = lambda p, nx: mk.generate_stencil(mk.ProblemSpec(p, nx))

def show(name, rep):
    g = runs[name]
    got = [(e.iteration, e.phase, e.implicit_relres, e.explicit_relres) for e in rep.history]
    want = g["history"]
    print("==", name, "iters", rep.total_iters, g["iters"], "restarts", rep.restarts, g["restarts"],
          "conv", rep.converged, g["converged"], "relres %.3e %.3e" % (rep.final_explicit_relres, g["relres"]))
    rows = []
    for a, b in zip(got, want):
        for i in (2, 3):
            if a[i] is not None and b[i] is not None:
                rows.append((abs(a[i] - b[i]) / max(abs(b[i]), 1e-300), a[0], a[1], i, a[i], b[i]))
    rows.sort(reverse=True)
    for r in rows[:4]:
        print("   rel %.3e it %d %s col %d got %.6e want %.6e" % r)
    # first divergence > 1e-3
    for a, b in zip(got, want):
        for i in (2, 3):
            if a[i] is not None and b[i] is not None and abs(a[i] - b[i]) > 1e-3 * abs(b[i]):
                print("   first >1e-3: it", a[0], a[1], i, a[i], b[i]); break
        else:
            continue
        break

def gm(A, b, **kw):
    cfg = mk.SolverConfig(**kw)
    return mk.gmres_restarted(A, None, b.astype(cfg.precision.dtype), np.zeros(A.n, cfg.precision.dtype), cfg)
def ir(A, b, m=50, **kw):
    inner = mk.SolverConfig(m=m, rtol=1e-4, precision=P.binary32, max_iters=kw.pop("max_iters", 20000))
    return mk.gmres_ir(A, b, np.zeros(A.n), mk.IrConfig(inner=inner, rtol=1e-10))
def fd(A, b, s, m=50):
    cfg = mk.FdConfig(switch_iter=s, low=mk.SolverConfig(m=m, rtol=1e-10, precision=P.binary32), high=mk.SolverConfig(m=m, rtol=1e-10))
    return mk.gmres_fd(A, b, np.zeros(A.n), cfg)

l16, l32 = L("Laplace2D", 16), L("Laplace2D", 32)
show("gmres_l2d16_m50", gm(l16, np.ones(256), m=50, rtol=1e-10))
show("gmres_l2d16_m10", gm(l16, np.ones(256), m=10, rtol=1e-10))
show("gmres_l2d16_m5_cap8", gm(l16, np.ones(256), m=5, rtol=1e-10, max_iters=8))
for m in (25, 50, 100):
    show("gmres_l2d32_m%d" % m, gm(l32, np.ones(1024), m=m, rtol=1e-10))
show("gmres_bp64", gm(L("BentPipe2D", 64), np.ones(4096), m=50, rtol=1e-10))
show("gmres_uf48", gm(L("UniFlow2D", 48), np.ones(48*48), m=50, rtol=1e-10))
show("gmres32_l2d8_m20", gm(mk.convert_matrix(L("Laplace2D", 8), P.binary32), np.ones(64), m=20, rtol=1e-4, precision=P.binary32))
for m in (25, 50, 100):
    show("ir_l2d32_m%d" % m, ir(l32, np.ones(1024), m=m))
show("ir_l2d16_m50", ir(l16, np.ones(256)))
show("ir_bp64", ir(L("BentPipe2D", 64), np.ones(4096)))
for s in (50, 100, 150, 200):
    show("fd_l2d32_s%d" % s, fd(l32, np.ones(1024), s))
show("fd_l2d16_s50", fd(l16, np.ones(256), 50))
