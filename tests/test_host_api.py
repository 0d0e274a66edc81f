"""Host-side contract of the drop-in API (no GPU): configuration validation,
CSR validation/COO compression, stencil assembly (bit-exact vs the reference
golden hashes), preconditioner spec parsing, error types."""

import hashlib

import numpy as np
import pytest

import paper_2105_07544_b200 as mk


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


BIG = {"Laplace3D_200", "UniFlow2D_2500"}


def test_stencils_bit_exact_vs_reference(stencil_golden):
    for key, g in stencil_golden.items():
        if key in BIG:
            continue
        preset, nx = key.rsplit("_", 1)
        A = mk.generate_stencil(mk.ProblemSpec(preset, int(nx)))
        assert (A.n, A.nnz) == (g["n"], g["nnz"]), key
        assert sha(A.row_ptr) == g["row_ptr"] and sha(A.col_idx) == g["col_idx"], key
        assert sha(A.values) == g["values"], key
        assert sha(mk.convert_matrix(A, mk.Precision.binary32).values) == g["values_f32"], key
        assert mk.stencil_dimensions(mk.ProblemSpec(preset, int(nx))) == (g["n"], g["nnz"])


@pytest.mark.slow
def test_stencils_bit_exact_benchmark_sizes(stencil_golden):
    for key in sorted(BIG & set(stencil_golden)):
        preset, nx = key.rsplit("_", 1)
        A = mk.generate_stencil(mk.ProblemSpec(preset, int(nx)))
        g = stencil_golden[key]
        assert sha(A.row_ptr) == g["row_ptr"] and sha(A.col_idx) == g["col_idx"], key
        assert sha(A.values) == g["values"], key


def test_closed_form_counts():
    for nx in (2, 5, 40):
        assert mk.stencil_dimensions(mk.ProblemSpec("Laplace2D", nx)) == (nx * nx, 5 * nx * nx - 4 * nx)
        assert mk.stencil_dimensions(mk.ProblemSpec("Laplace3D", nx)) == (nx ** 3, 7 * nx ** 3 - 6 * nx * nx)


def test_solver_config_validation():
    for bad in (dict(m=0), dict(rtol=0.0), dict(rtol=1.5), dict(max_iters=0), dict(max_restarts=0),
                dict(breakdown_rule="x")):
        with pytest.raises(ValueError):
            mk.SolverConfig(**bad)
    inner = mk.SolverConfig(m=50, rtol=1e-4, precision=mk.Precision.binary32)
    with pytest.raises(ValueError):
        mk.IrConfig(inner=mk.SolverConfig(m=50))
    with pytest.raises(ValueError):
        mk.IrConfig(inner=inner, rtol=0.0)
    with pytest.raises(ValueError):
        mk.IrConfig(inner=inner, max_refinements=0)
    hi = mk.SolverConfig(m=50, rtol=1e-10)
    lo = mk.SolverConfig(m=50, rtol=1e-10, precision=mk.Precision.binary32)
    with pytest.raises(ValueError, match="switch_iter 30 is not a multiple of the restart length 50"):
        mk.FdConfig(switch_iter=30, low=lo, high=hi)
    with pytest.raises(ValueError):
        mk.FdConfig(switch_iter=-50, low=lo, high=hi)
    with pytest.raises(ValueError):
        mk.FdConfig(switch_iter=50, low=hi, high=hi)


def test_csr_validation_errors():
    with pytest.raises(mk.DimensionMismatchError):
        mk.CsrMatrix(3, np.array([0, 2, 4, 4]), np.array([0, 1, 1, 2, 2]), np.ones(5))
    with pytest.raises(mk.DimensionMismatchError):
        mk.CsrMatrix(3, np.array([0, 3, 2, 5]), np.array([0, 1, 1, 2, 2]), np.ones(5))
    with pytest.raises(mk.EntryOutOfRangeError):
        mk.CsrMatrix(2, np.array([0, 1, 2]), np.array([0, 2]), np.ones(2))
    with pytest.raises(mk.ColumnOrderError):
        mk.CsrMatrix(2, np.array([0, 2, 3]), np.array([1, 0, 1]), np.ones(3))
    with pytest.raises(mk.ColumnOrderError):
        mk.CsrMatrix(2, np.array([0, 2, 3]), np.array([0, 0, 1]), np.ones(3))
    with pytest.raises(mk.PrecisionMismatchError):
        mk.CsrMatrix(1, np.array([0, 1]), np.array([0]), np.ones(1, dtype=np.int64))
    A = mk.CsrMatrix(3, np.array([0, 0, 1, 1]), np.array([1]), np.array([5.0]))
    assert A.to_dense()[1, 1] == 5.0


def test_coo_sorts_and_sums_duplicates():
    A = mk.csr_from_coo(np.array([1, 0, 1, 0, 1]), np.array([1, 0, 0, 0, 1]),
                        np.array([2.0, 1.0, 4.0, 3.0, 5.0]), 2)
    assert np.array_equal(A.to_dense(), np.array([[4.0, 0.0], [4.0, 7.0]]))
    with pytest.raises(mk.EntryOutOfRangeError):
        mk.csr_from_coo(np.array([0]), np.array([3]), np.array([1.0]), 2)


def test_convert_matrix_shares_structure():
    A = mk.generate_stencil(mk.ProblemSpec("Laplace2D", 4))
    B = mk.convert_matrix(A, mk.Precision.binary32)
    assert B.row_ptr is A.row_ptr and B.col_idx is A.col_idx
    assert np.array_equal(B.values, A.values.astype(np.float32))
    assert mk.convert_matrix(A, mk.Precision.binary64) is A


def test_permutation_helpers(rng):
    p = rng.permutation(20)
    q = mk.invert_permutation(p)
    assert np.array_equal(p[q], np.arange(20))
    with pytest.raises(mk.InvalidPermutationError):
        mk.invert_permutation(np.array([0, 0, 2]))


def test_parse_precond_spec():
    assert mk.parse_precond_spec("none") == ("none", 0)
    assert mk.parse_precond_spec("Jacobi:16") == ("jacobi", 16)
    assert mk.parse_precond_spec("poly:25") == ("poly", 25)
    for bad in ("poly", "ilu:3", "poly:x", "poly:0"):
        with pytest.raises(ValueError):
            mk.parse_precond_spec(bad)


def test_precision_parsing():
    assert mk.Precision.parse("single") is mk.Precision.binary32
    assert mk.Precision.parse("FP64") is mk.Precision.binary64
    assert mk.Precision.binary32.unit_roundoff == 2.0 ** -24
    with pytest.raises(ValueError):
        mk.Precision.parse("half")
    with pytest.raises(mk.PrecisionMismatchError):
        mk.Precision.from_dtype(np.int32)


def test_binary16_basis_validation():
    with pytest.raises(ValueError):
        mk.SolverConfig(precision=mk.Precision.binary64, basis_precision="binary16")
    with pytest.raises(ValueError):
        mk.SolverConfig(precision=mk.Precision.binary32, m=60, basis_precision="binary16")
    # the lagged CGS2 runs over a 16-bit basis too (k_cycle_dcgs2<float, Op, false, __half>)
    mk.SolverConfig(precision=mk.Precision.binary32, orthogonalization="dcgs2", basis_precision="binary16")
    with pytest.raises(ValueError):
        mk.SolverConfig(basis_precision="float8")
    with pytest.raises(ValueError):
        mk.SolverConfig(precision=mk.Precision.binary64, basis_precision="bfloat16")
