"""BASELINE config 5: a SuiteSparse-like irregular nonsymmetric CSR matrix.

The reference has no generator for it; this is the SURVEY
§8(d) specification (restated identically by the test-side CPU checker,
bit-exact, tests/test_synthetic.py):

  row length 1 + Geometric(1/mean_len), clipped to max_len; off-diagonal
  columns clip(i + U[-band, band]) or, with probability far_frac, U[0, n);
  values N(0,1) (signs="random") or -|N(0,1)| (signs="negative", an
  M-matrix pattern); diagonal entries drawn there are dropped; duplicates
  summed as csr_from_coo does (sparse.py:155-170); diagonal =
  dominance * sum|offdiag| + shift.

Host numpy draws the random numbers; the (row, col) ordering of the ~200M
entries at n = 4M is one stable device sort (torch), the rest is the
reference's compression arithmetic.  Setup, not on the timed path.
"""

from __future__ import annotations

import numpy as np

from . import device as D
from .sparse import CsrMatrix

__all__ = ["synthetic_irregular"]


def _stable_order(keys: np.ndarray) -> np.ndarray:
    """Stable argsort of int64 keys (== np.lexsort((cols, rows)) for key = row*n + col)."""
    try:
        t = D.torch()
        if t.cuda.is_available():
            kd = t.from_numpy(keys).to(D.device())
            _, idx = t.sort(kd, stable=True)
            return idx.cpu().numpy()
    except Exception:  # noqa: BLE001 - no device: host sort below
        pass
    return np.argsort(keys, kind="stable")


def synthetic_irregular(n, seed=20240817, mean_len=49, max_len=1000, band=2000, far_frac=0.01,
                        dominance=1.1, shift=1.0, signs="random") -> CsrMatrix:
    if signs not in ("random", "negative"):
        raise ValueError("signs must be 'random' or 'negative'")
    n = int(n)
    rng = np.random.default_rng(seed)
    lens = np.minimum(1 + rng.geometric(1.0 / mean_len, size=n), max_len).astype(np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), lens - 1)
    tot = rows.size
    near = np.clip(rows + rng.integers(-band, band + 1, size=tot), 0, n - 1)
    far = rng.integers(0, n, size=tot)
    cols = np.where(rng.random(tot) < far_frac, far, near)
    vals = rng.standard_normal(tot)
    if signs == "negative":
        vals = -np.abs(vals)
    keep = cols != rows
    rows, cols, vals = rows[keep], cols[keep], vals[keep]
    # coo compression (sparse.py:155-170): stable (row, col) order, duplicates summed
    order = _stable_order(rows * n + cols)
    r, c, v = rows[order], cols[order], vals[order]
    head = np.ones(r.size, dtype=bool)
    head[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
    starts = np.flatnonzero(head)
    vv = np.add.reduceat(v, starts) if starts.size else v[:0]
    r, c = r[starts], c[starts]
    rowsum = np.bincount(r, weights=np.abs(vv), minlength=n)
    diag = dominance * rowsum + shift
    # the diagonal joins each row at its sorted position (no (i, i) entry is
    # left, so this equals compressing the concatenated triplets again)
    below = np.bincount(r[c < r], minlength=n)
    rp_off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=rp_off[1:])
    at = rp_off[:-1] + below
    ci = np.insert(c, at, np.arange(n, dtype=np.int64))
    va = np.insert(vv, at, diag)
    rp = rp_off + np.arange(n + 1, dtype=np.int64)
    return CsrMatrix(n, rp, ci, va.astype(np.float64, copy=False), validate=False)
