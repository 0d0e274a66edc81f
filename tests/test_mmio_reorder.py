"""Matrix Market I/O and RCM (the data formats feeding the solve path for the
paper's SuiteSparse set) against fixtures produced by the unmodified
reference (tests/golden/make_mmio_rcm_golden.py): identical CSR arrays,
identical permutations, and the reference's error behaviour."""

import os

import numpy as np
import pytest

import paper_2105_07544_b200 as mk

from conftest import GOLDEN, random_csr

MM = os.path.join(GOLDEN, "mm")


@pytest.fixture(scope="module")
def mm_gold():
    return np.load(os.path.join(GOLDEN, "mm_read.npz"))


@pytest.fixture(scope="module")
def rcm_gold():
    return np.load(os.path.join(GOLDEN, "rcm.npz"))


def test_reader_matches_reference_on_every_fixture(mm_gold):
    names = sorted(f[:-4] for f in os.listdir(MM))
    assert len(names) == 8
    for k in names:
        A = mk.read_matrix_market(os.path.join(MM, k + ".mtx"))
        assert np.array_equal(A.row_ptr, mm_gold[k + "_rp"]), k
        assert np.array_equal(A.col_idx, mm_gold[k + "_ci"]), k
        assert A.values.tobytes() == mm_gold[k + "_v"].tobytes(), k
        n, nnz, _ = mk.read_matrix_market_header(os.path.join(MM, k + ".mtx"))
        assert [n, nnz] == list(mm_gold[k + "_hdr"])


def test_write_read_roundtrip_bit_exact(tmp_path, rng):
    for _ in range(4):
        A, _ = random_csr(mk, rng, int(rng.integers(2, 30)))
        p = str(tmp_path / "m.mtx")
        mk.write_matrix_market(A, p)
        B = mk.read_matrix_market(p)
        assert np.array_equal(B.row_ptr, A.row_ptr) and np.array_equal(B.col_idx, A.col_idx)
        assert B.values.tobytes() == A.values.tobytes()
    # the writer's text equals the reference writer's
    A = mk.read_matrix_market(os.path.join(MM, "random300.mtx"))
    p = str(tmp_path / "r.mtx")
    mk.write_matrix_market(A, p)
    assert open(p).read() == open(os.path.join(MM, "random300.mtx")).read()


@pytest.mark.parametrize("text,needle", [
    ("%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n", "coordinate"),
    ("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n", "real-valued"),
    ("%%MatrixMarket matrix coordinate pattern general\n1 1 1\n1 1\n", "real-valued"),
    ("%%MatrixMarket matrix coordinate real general\n2 3 1\n1 1 1.0\n", "square"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n2 2 1.0\n", "declares 3"),
    ("%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1.0\n", "symmetry"),
    ("%%MatrixMarket vector coordinate real general\n1 1 1\n1 1 1.0\n", "object"),
    ("not a header\n1 1 1\n1 1 1.0\n", "header"),
    ("%%MatrixMarket matrix coordinate real general\n% only comments\n", "size line"),
])
def test_reader_rejections(tmp_path, text, needle):
    p = tmp_path / "bad.mtx"
    p.write_text(text)
    with pytest.raises(mk.MatrixMarketError) as e:
        mk.read_matrix_market(str(p))
    assert needle in str(e.value) and str(p) in str(e.value)


def test_out_of_range_index_is_entry_error(tmp_path):
    p = tmp_path / "oob.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n")
    with pytest.raises(mk.EntryOutOfRangeError):
        mk.read_matrix_market(str(p))


@pytest.mark.parametrize("name", ["laplace2d20_scrambled", "bentpipe16", "random300", "components40",
                                  "stretched12"])
def test_rcm_permutation_matches_reference(rcm_gold, name):
    A = mk.CsrMatrix(int(rcm_gold[name + "_rp"].size - 1), rcm_gold[name + "_rp"], rcm_gold[name + "_ci"],
                     rcm_gold[name + "_v"])
    perm = mk.rcm_ordering(A)
    assert np.array_equal(perm, rcm_gold[name + "_perm"])
    assert mk.bandwidth(A) == int(rcm_gold[name + "_bw"][0])
    B, _ = mk.permute_system(A, np.zeros(A.n), perm)
    assert mk.bandwidth(B) == int(rcm_gold[name + "_bw_rcm"][0])


def test_rcm_identity_and_large(rng):
    A = mk.csr_from_triplets([(i, i, 1.0) for i in range(9)], 9)
    assert np.array_equal(mk.rcm_ordering(A), np.arange(9))
    # a scrambled 2-D grid of 250k vertices: native sweep, bandwidth restored to ~nx
    L = mk.generate_stencil(mk.ProblemSpec("Laplace2D", 500))
    p = rng.permutation(L.n)
    Ls, _ = mk.permute_system(L, np.zeros(L.n), p)
    perm = mk.rcm_ordering(Ls)
    assert np.array_equal(np.sort(perm), np.arange(L.n))
    B, _ = mk.permute_system(Ls, np.zeros(L.n), perm)
    assert mk.bandwidth(B) <= 2 * 500 + 2
