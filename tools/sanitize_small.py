"""Small solves for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel family once -- persistent cycle (stencil + CSR, fp32 + fp64,
Jacobi-1), multi-kernel cycle (block Jacobi 4, polynomial), residual, SpMV."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2105_07544_b200 as mk
P = mk.Precision
A = mk.generate_stencil(mk.ProblemSpec("BentPipe2D", 24))
b = np.ones(A.n)
print(mk.gmres_restarted(A, None, b, np.zeros(A.n), mk.SolverConfig(m=20, rtol=1e-10, max_iters=60)).total_iters)
inner = mk.SolverConfig(m=20, rtol=1e-4, precision=P.binary32, max_iters=60)
print(mk.gmres_ir(A, b, np.zeros(A.n), mk.IrConfig(inner=inner, rtol=1e-10)).total_iters)
L3 = mk.generate_stencil(mk.ProblemSpec("Laplace3D", 10))
print(mk.gmres_restarted(L3, None, np.ones(L3.n), np.zeros(L3.n), mk.SolverConfig(m=10, rtol=1e-10, max_iters=30)).total_iters)
C = mk.synthetic_irregular(3000, band=100)
J1 = mk.build_block_jacobi(C, 1)
print(mk.gmres_restarted(C, J1, np.ones(C.n), np.zeros(C.n), mk.SolverConfig(m=20, rtol=1e-10, max_iters=60)).total_iters)
J4 = mk.build_block_jacobi(A, 4)
print(mk.gmres_restarted(A, J4, b, np.zeros(A.n), mk.SolverConfig(m=20, rtol=1e-10, max_iters=40)).total_iters)
Al = mk.convert_matrix(A, P.binary32)
Mp = mk.build_gmres_poly(Al, 5, np.ones(A.n, np.float32))
print(mk.gmres_ir(A, b, np.zeros(A.n), mk.IrConfig(inner=inner, rtol=1e-10), M=Mp, A_low=Al).total_iters)
print(float(mk.spmv(C, np.ones(C.n)).sum()))
print("sanitize ok")
