"""Multi-process check of the row-partitioned solver (torchrun; one process
per rank).  With MPK_SHARE_GPU=1 every rank uses GPU 0 and gloo, which
exercises the CUDA-IPC peer mapping and the system-scope barrier on a
one-GPU box (time-sliced, so slow).  Prints one JSON line from rank 0."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

share = os.environ.get("MPK_SHARE_GPU") == "1"
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(0 if share else local)
dist.init_process_group("gloo" if share else "nccl")
import paper_2105_07544_b200 as mk
from paper_2105_07544_b200 import distributed as dd

P = mk.Precision
comm = dd.TorchComm()
if share:
    comm.ctas = max(1, int(mk._lib.load().mpk_sm_count()) // comm.size)
A = mk.generate_stencil(mk.ProblemSpec(sys.argv[1] if len(sys.argv) > 1 else "Laplace2D",
                                       int(sys.argv[2]) if len(sys.argv) > 2 else 32))
sysm = dd.LocalSystem(comm, A, mk.convert_matrix(A, P.binary32))
inner = mk.SolverConfig(m=50, rtol=1e-4, precision=P.binary32, max_iters=20000,
                        breakdown_rule="u" if len(sys.argv) > 3 and sys.argv[3] == "u" else "n_u")
import time
from paper_2105_07544_b200.engine import HOST_STATS
dd.dist_gmres_ir(sysm, np.ones(A.n), np.zeros(A.n), mk.IrConfig(inner=inner, rtol=1e-10))   # warm-up
HOST_STATS.update(on=True, sync_s=0.0, reads=0, host_collectives=0)
t0 = time.perf_counter()
ir = dd.dist_gmres_ir(sysm, np.ones(A.n), np.zeros(A.n), mk.IrConfig(inner=inner, rtol=1e-10))
wall = time.perf_counter() - t0
stats = dict(HOST_STATS)
HOST_STATS["on"] = False
g64 = dd.dist_gmres_restarted(sysm, np.ones(A.n), np.zeros(A.n), mk.SolverConfig(m=50, rtol=1e-10))
xs = [None] * comm.size
dist.all_gather_object(xs, (sysm.r0, g64.x.cpu().numpy()))
if comm.rank == 0:
    x = np.zeros(A.n)
    for r0, xl in xs:
        x[r0:r0 + xl.size] = xl
    ref = mk.gmres_restarted(A, None, np.ones(A.n), np.zeros(A.n), mk.SolverConfig(m=50, rtol=1e-10))
    print(json.dumps({"ir_wall_s": wall, "ir_refinements": ir.restarts,
                      "host_s_per_refinement_excl_sync": (wall - stats["sync_s"]) / max(stats["reads"], 1),
                      "host_collectives_during_solve": stats["host_collectives"], "reads": stats["reads"],
                      "ir_iters": ir.total_iters, "ir_converged": ir.converged, "ir_relres": ir.final_explicit_relres,
                      "fp64_iters": g64.total_iters, "fp64_converged": g64.converged,
                      "single_fp64_iters": ref.total_iters,
                      "x_maxdiff": float(np.abs(x - ref.x).max() / np.abs(ref.x).max())}), flush=True)
sysm.close()
dist.destroy_process_group()
