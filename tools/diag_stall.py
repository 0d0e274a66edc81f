import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2105_07544_b200 as mk
P = mk.Precision
g = json.load(open("tests/golden/runs.json"))["ir_stall_l2d4"]
A = mk.generate_stencil(mk.ProblemSpec("Laplace2D", 4))
inner = mk.SolverConfig(m=10, rtol=1e-4, precision=P.binary32, max_iters=20000)
rep = mk.gmres_ir(A, 1e-15 * np.ones(16), np.zeros(16), mk.IrConfig(inner=inner, rtol=1e-14))
print("ours", rep.total_iters, rep.restarts, rep.stalled)
for h, w in zip(rep.history, g["history"] + [None] * 20):
    print((h.iteration, h.phase, h.implicit_relres, h.explicit_relres), w)
for flag in (4,):
    from paper_2105_07544_b200.engine import CycleWorkspace
    ws = CycleWorkspace.get(16, 10, P.binary32); ws.flags = flag
    rep = mk.gmres_ir(A, 1e-15 * np.ones(16), np.zeros(16), mk.IrConfig(inner=inner, rtol=1e-14))
    print("multi-kernel path", rep.total_iters, rep.restarts, [(h.iteration, h.implicit_relres) for h in rep.history if h.phase == "inner"][-3:])
    ws.flags = 0
