"""compute-sanitizer workload for the kernels changed or added in round 2
(memcheck / racecheck / synccheck):
  * lagged CGS2 (k_cycle_dcgs2) with cycles of 50 steps (> 32: the R-column
    race of ADVICE r1), fp32 and fp64, stencil and CSR;
  * k_cycle_reg BIG instantiation (m = 60), every register stream shape
    (m = 50 walks basis widths 1..51);
  * row-partitioned cycles on 2 virtual ranks (k_cycle_reg MULTI and
    k_cycle_dcgs2 MULTI) + the per-restart collectives (comm push / reduce);
  * the banded-CSR x-window SpMV (standalone and in the cycle) and the
    device block-LU setup (k = 1, 8, 42);
  * the lagged CGS2 over a 16-bit basis and the preset-specialised stencil
    SpMV (k_spmv_pre)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2105_07544_b200 as mk
from paper_2105_07544_b200 import distributed as dd
P = mk.Precision
A = mk.generate_stencil(mk.ProblemSpec("BentPipe2D", 40))
b = np.ones(A.n)
for orth in ("cgs2", "dcgs2"):
    cfg = mk.SolverConfig(m=50, rtol=1e-10, max_iters=100, orthogonalization=orth)
    print(orth, "fp64", mk.gmres_restarted(A, None, b, np.zeros(A.n), cfg).total_iters)
    inner = mk.SolverConfig(m=50, rtol=1e-4, precision=P.binary32, max_iters=100, orthogonalization=orth)
    print(orth, "ir", mk.gmres_ir(A, b, np.zeros(A.n), mk.IrConfig(inner=inner, rtol=1e-10)).total_iters)
inner16 = mk.SolverConfig(m=50, rtol=1e-4, precision=P.binary32, max_iters=100, basis_precision="binary16")
print("binary16 basis ir", mk.gmres_ir(A, b, np.zeros(A.n), mk.IrConfig(inner=inner16, rtol=1e-10)).total_iters)
print("big", mk.gmres_restarted(A, None, b, np.zeros(A.n), mk.SolverConfig(m=60, rtol=1e-10, max_iters=120)).total_iters)
C = mk.synthetic_irregular(6000, signs="negative", dominance=1.001, shift=1e-3, far_frac=0.01, band=300)
print("band", C.band_width())
J1 = mk.build_block_jacobi(C, 1)
for orth in ("cgs2", "dcgs2"):
    cfg = mk.SolverConfig(m=50, rtol=1e-10, max_iters=100, orthogonalization=orth)
    print("csr+J1", orth, mk.gmres_restarted(C, J1, np.ones(C.n), np.zeros(C.n), cfg).total_iters)
print("spmv", float(mk.spmv(C, np.ones(C.n)).sum()), float(mk.spmv(mk.convert_matrix(C, P.binary32),
                                                                   np.ones(C.n, np.float32)).sum()))
for k in (8, 42):
    Mk = mk.build_block_jacobi(C, k)
    print("lu", k, float(Mk.apply(np.ones(C.n)).sum()))
print("lu32", float(mk.build_block_jacobi(C, 16, precision=P.binary32).apply(np.ones(C.n, np.float32)).sum()))


def dist(orth, solver):
    A_low = mk.convert_matrix(A, P.binary32)

    def fn(comm):
        sysm = dd.LocalSystem(comm, A, A_low)
        try:
            if solver == "ir":
                inner = mk.SolverConfig(m=50, rtol=1e-4, precision=P.binary32, max_iters=100,
                                        orthogonalization=orth)
                return dd.dist_gmres_ir(sysm, b, np.zeros(A.n), mk.IrConfig(inner=inner, rtol=1e-10)).total_iters
            return dd.dist_gmres_restarted(sysm, b, np.zeros(A.n), mk.SolverConfig(
                m=50, rtol=1e-10, max_iters=100, orthogonalization=orth)).total_iters
        finally:
            sysm.close()
    return dd.run_virtual_ranks(2, fn)


# concurrent virtual ranks need both persistent kernels resident at once;
# compute-sanitizer serialises kernels, so this part runs only with --dist
# (the cross-rank barrier times out under the tools)
if "--dist" in sys.argv:
    for orth in ("cgs2", "dcgs2"):
        print("dist", orth, dist(orth, "fp64"), dist(orth, "ir"))
inner_b = mk.SolverConfig(m=50, rtol=1e-4, precision=P.binary32, max_iters=100, basis_precision="bfloat16")
print("bfloat16 basis ir", mk.gmres_ir(A, b, np.zeros(A.n), mk.IrConfig(inner=inner_b, rtol=1e-10)).total_iters)
Ad = mk.generate_stencil(mk.ProblemSpec("Laplace3D", 12), on_device=True)
Ad.use_stencil = False
print("assembly + short-row CSR spmv", float(mk.spmv(Ad, np.ones(Ad.n)).sum()))
L2 = mk.generate_stencil(mk.ProblemSpec("Laplace2D", 40))
Mp = mk.build_gmres_poly(mk.convert_matrix(L2, P.binary32), 6, np.ones(L2.n, np.float32))
inner_p = mk.SolverConfig(m=30, rtol=1e-4, precision=P.binary32, max_iters=60)
print("fused poly ir", mk.gmres_ir(L2, np.ones(L2.n), np.zeros(L2.n), mk.IrConfig(inner=inner_p, rtol=1e-10),
                                   M=Mp).total_iters)
# round 2 (session 3): lagged CGS2 over the 16-bit basis, stencil SpMV with
# the preset fixed at compile time (every preset, both precisions)
for bp in ("binary16", "bfloat16"):
    inner_dh = mk.SolverConfig(m=50, rtol=1e-4, precision=P.binary32, max_iters=100, orthogonalization="dcgs2",
                               basis_precision=bp)
    print("dcgs2", bp, "ir", mk.gmres_ir(A, b, np.zeros(A.n), mk.IrConfig(inner=inner_dh, rtol=1e-10)).total_iters)
for pre, nx in (("Laplace3D", 12), ("Laplace2D", 36), ("UniFlow2D", 36), ("BentPipe2D", 36)):
    S = mk.generate_stencil(mk.ProblemSpec(pre, nx))
    print("spmv_pre", pre, float(mk.spmv(S, np.ones(S.n)).sum()),
          float(mk.spmv(mk.convert_matrix(S, P.binary32), np.ones(S.n, np.float32)).sum()))
print("sanitize ok")
