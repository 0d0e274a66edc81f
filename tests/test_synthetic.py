"""Config-5 generator: product restatement == oracle restatement, bit for bit
(there is no reference generator: parity of this matrix is
pinned between the two restatements of the SURVEY 8(d) specification)."""

import numpy as np
import pytest

import paper_2105_07544_b200 as mk
from oracle import mpk_oracle as O


@pytest.mark.parametrize("kw", [dict(), dict(signs="negative", dominance=1.001, shift=0.0),
                                dict(far_frac=0.1, band=50), dict(mean_len=5, max_len=20, seed=7)])
def test_generator_matches_oracle_bit_exact(kw):
    n = 6000
    kw = dict(dict(band=300), **kw)
    A = mk.synthetic_irregular(n, **kw)
    rp, ci, v = O.synthetic_irregular(n, **kw)
    assert np.array_equal(A.row_ptr, rp)
    assert np.array_equal(A.col_idx, ci)
    assert A.values.tobytes() == v.tobytes()
    A.validate()   # strictly increasing columns, in range


def test_generator_statistics():
    A = mk.synthetic_irregular(20000, band=500)
    lens = np.diff(A.row_ptr)
    assert 45 < lens.mean() < 53 and lens.max() <= 1000
    d = A.to_dense() if A.n <= 2000 else None
    rows = np.repeat(np.arange(A.n), lens)
    diag = A.values[A.col_idx == rows]
    off = np.bincount(rows[A.col_idx != rows], weights=np.abs(A.values[A.col_idx != rows]), minlength=A.n)
    assert np.all(diag > 1.1 * off)   # strictly diagonally dominant (default family)
