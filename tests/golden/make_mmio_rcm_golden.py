"""Golden fixtures for Matrix Market I/O and RCM, produced by the UNMODIFIED
reference (PYTHONPATH=/root/reference/pkg/src) in the build container:

  python tests/golden/make_mmio_rcm_golden.py

tests/golden/rcm.npz       reference rcm_ordering permutations + bandwidths
tests/golden/mm/*.mtx      files written by the reference writer / edge cases
tests/golden/mm_read.npz   the reference reader's CSR arrays for each file
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import mpkrylov as ref  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def matrices():
    rng = np.random.default_rng(11)
    out = {}
    L = ref.generate_stencil(ref.ProblemSpec("Laplace2D", 20))
    p = rng.permutation(L.n)
    Ls, _ = ref.permute_system(L, np.zeros(L.n), p)
    out["laplace2d20_scrambled"] = Ls
    out["bentpipe16"] = ref.generate_stencil(ref.ProblemSpec("BentPipe2D", 16))
    n = 300
    dense = np.where(rng.random((n, n)) < 0.02, rng.standard_normal((n, n)), 0.0)
    np.fill_diagonal(dense, 5.0)
    r, c = np.nonzero(dense)
    out["random300"] = ref.csr_from_coo(r, c, dense[r, c], n)
    # three components + isolated vertices
    ent = [(i, i, 2.0) for i in range(40)]
    for a, b in [(0, 5), (5, 9), (9, 17), (20, 21), (21, 30), (30, 22), (33, 38)]:
        ent += [(a, b, -1.0), (b, a, -1.0)]
    out["components40"] = ref.csr_from_triplets(ent, 40)
    out["stretched12"] = ref.generate_stencil(ref.ProblemSpec("Stretched2D", 12))
    return out


def main():
    mats = matrices()
    rcm = {}
    mm = {}
    for name, A in mats.items():
        perm = ref.rcm_ordering(A)
        rcm[name + "_perm"] = perm
        rcm[name + "_bw"] = np.array([ref.bandwidth(A)])
        B, _ = ref.permute_system(A, np.zeros(A.n), perm)
        rcm[name + "_bw_rcm"] = np.array([ref.bandwidth(B)])
        rcm[name + "_rp"], rcm[name + "_ci"], rcm[name + "_v"] = A.row_ptr, A.col_idx, A.values
        path = os.path.join(HERE, "mm", name + ".mtx")
        ref.write_matrix_market(A, path)
    edge = {
        "crlf_comments": "%%MatrixMarket matrix coordinate real general\r\n% c\r\n\r\n3 3 4\r\n1 1 1.5\r\n"
                         "% mid\r\n2 1 -2.0\r\n3 3 4e-3\r\n2 2 7\r\n",
        "symmetric": "%%MatrixMarket matrix coordinate real symmetric\n4 4 5\n1 1 2.0\n2 1 -1.0\n3 2 -1.5\n"
                     "4 4 3.0\n4 1 0.25\n",
        "integer_dups": "%%MatrixMarket matrix coordinate integer general\n3 3 5\n1 1 2\n1 1 3\n2 3 -4\n3 3 1\n"
                        "3 1 7\n",
    }
    for name, text in edge.items():
        with open(os.path.join(HERE, "mm", name + ".mtx"), "w", newline="") as f:
            f.write(text)
    for fn in sorted(os.listdir(os.path.join(HERE, "mm"))):
        A = ref.read_matrix_market(os.path.join(HERE, "mm", fn))
        k = fn[:-4]
        mm[k + "_rp"], mm[k + "_ci"], mm[k + "_v"] = A.row_ptr, A.col_idx, A.values
        mm[k + "_hdr"] = np.array(ref.read_matrix_market_header(os.path.join(HERE, "mm", fn))[:2])
    np.savez_compressed(os.path.join(HERE, "rcm.npz"), **rcm)
    np.savez_compressed(os.path.join(HERE, "mm_read.npz"), **mm)
    print("wrote", len(rcm), "rcm arrays,", len(mm), "mm arrays")


if __name__ == "__main__":
    main()
