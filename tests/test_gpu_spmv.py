"""Bit-exact parity of the device SpMV (CSR and matrix-free stencil paths)
and the casts against the reference's golden vectors and the oracle."""

import numpy as np
import pytest

import paper_2105_07544_b200 as mk
from oracle import mpk_oracle as O

pytestmark = pytest.mark.gpu


def test_spmv_matches_reference_golden(cuda, spmv_golden):
    names = sorted({k.split("/")[0] for k in spmv_golden.files})
    for name in names:
        g = lambda f: spmv_golden[name + "/" + f]  # noqa: E731
        A = mk.CsrMatrix(g("row_ptr").size - 1, g("row_ptr"), g("col_idx"), g("values"))
        assert np.array_equal(mk.spmv(A, g("x")), g("y64")), name
        A32 = mk.convert_matrix(A, mk.Precision.binary32)
        assert np.array_equal(mk.spmv(A32, g("x").astype(np.float32)), g("y32")), name


# nx % 4 == 0 rows take the preset-specialised row-group kernel (k_spmv_pre)
# in both precisions, the others the generic k_spmv's scalar rows
@pytest.mark.parametrize("preset,nx", [("Laplace2D", 33), ("Laplace3D", 17), ("UniFlow2D", 40),
                                       ("BentPipe2D", 70), ("Stretched2D", 31), ("Laplace2D", 2),
                                       ("Laplace3D", 16), ("Laplace2D", 64), ("BentPipe2D", 64),
                                       ("Laplace3D", 36)])
def test_stencil_and_csr_paths_bit_identical(cuda, preset, nx):
    A = mk.generate_stencil(mk.ProblemSpec(preset, nx))
    x = np.random.default_rng(nx).standard_normal(A.n)
    want = O.spmv_seq(A.row_ptr, A.col_idx, A.values, x)
    A.use_stencil = True
    assert np.array_equal(mk.spmv(A, x), want)
    A.use_stencil = False
    assert np.array_equal(mk.spmv(A, x), want)
    A32 = mk.convert_matrix(A, mk.Precision.binary32)
    x32 = x.astype(np.float32)
    want32 = O.spmv_seq(A.row_ptr, A.col_idx, A.values.astype(np.float32), x32)
    for flag in (True, False):
        A32.use_stencil = flag
        assert np.array_equal(mk.spmv(A32, x32), want32)


def test_spmv_large_bentpipe_stencil_vs_csr(cuda):
    A = mk.generate_stencil(mk.ProblemSpec("BentPipe2D", 1500))
    x = np.random.default_rng(1).standard_normal(A.n)
    A.use_stencil = True
    y1 = mk.spmv(A, x)
    A.use_stencil = False
    y2 = mk.spmv(A, x)
    assert np.array_equal(y1, y2)
    assert np.array_equal(y1, O.spmv_seq(A.row_ptr, A.col_idx, A.values, x))


def test_device_tensors_in_device_tensors_out(cuda):
    import torch

    A = mk.generate_stencil(mk.ProblemSpec("Laplace2D", 8))
    x = torch.randn(A.n, dtype=torch.float64, device=cuda)
    y = mk.spmv(A, x)
    assert isinstance(y, torch.Tensor) and y.is_cuda
    assert np.array_equal(y.cpu().numpy(), O.spmv_seq(A.row_ptr, A.col_idx, A.values, x.cpu().numpy()))


def test_spmv_guards(cuda):
    A = mk.generate_stencil(mk.ProblemSpec("Laplace2D", 4))
    with pytest.raises(mk.DimensionMismatchError):
        mk.spmv(A, np.ones(5))
    with pytest.raises(mk.PrecisionMismatchError):
        mk.spmv(A, np.ones(16, dtype=np.float32))


def test_convert_vector_rounds_to_nearest_keeps_subnormals(cuda):
    v = np.array([1.0 + 2.0 ** -30, 3e-40, -1e-45, 1e300, np.pi, -0.0])
    with np.errstate(over="ignore"):
        want = v.astype(np.float32)
    got = mk.convert_vector(v, mk.Precision.binary32)
    assert got.dtype == np.float32
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    back = mk.convert_vector(got, mk.Precision.binary64)
    assert np.array_equal(back, want.astype(np.float64))


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_irregular_csr_warp_rows_bit_exact(cuda, dtype):
    """Config-5 family (row lengths 2..1000): the warp-cooperative CSR path
    (coalesced entry loads, staged products, row-sequential sums) equals the
    sequential csr_matvec order bit for bit, including rows spanning several
    256-entry chunks."""
    from oracle import mpk_oracle as O

    A = mk.synthetic_irregular(20000, band=500, max_len=1000)
    A = mk.convert_matrix(A, mk.Precision.from_dtype(np.dtype(dtype)))
    x = np.random.default_rng(5).standard_normal(A.n).astype(dtype)
    y = mk.spmv(A, x)
    ref = O.spmv_seq(A.row_ptr, A.col_idx, A.values, x)
    assert y.tobytes() == ref.tobytes()
    # a row far longer than one chunk
    n = 3000
    rows = np.concatenate([np.zeros(2500, np.int64), np.arange(n)])
    cols = np.concatenate([np.arange(2500), np.arange(n)])
    vals = np.random.default_rng(6).standard_normal(rows.size).astype(dtype)
    B = mk.csr_from_coo(rows, cols, vals, n)
    xb = np.random.default_rng(7).standard_normal(n).astype(dtype)
    assert mk.spmv(B, xb).tobytes() == O.spmv_seq(B.row_ptr, B.col_idx, B.values, xb).tobytes()
