"""Bandwidth-reducing reordering (reference: pkg/src/mpkrylov/reorder.py).

``rcm_ordering`` returns the same permutation as the reference's reverse
Cuthill-McKee (reorder.py:22-63); the breadth-first sweep runs in native
host code (``mpk_rcm_host``), the symmetrized pattern is built with numpy.
Apply it with :func:`permute_system` (sparse.py), as the reference does.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .sparse import CsrMatrix

__all__ = ["rcm_ordering", "bandwidth"]


def _symmetrized_pattern(A: CsrMatrix):
    """Row-sorted CSR (indptr, indices) of pattern(A + A^T) minus the diagonal."""
    n = A.n
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(A.row_ptr))
    cols = A.col_idx
    off = rows != cols
    r = np.concatenate([rows[off], cols[off]])
    c = np.concatenate([cols[off], rows[off]])
    key = np.unique(r * n + c)            # sorted, duplicates (i,j)+(j,i) merged
    r, c = key // n, key % n
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=indptr[1:])
    return indptr, np.ascontiguousarray(c, dtype=np.int64)


def rcm_ordering(A: CsrMatrix) -> np.ndarray:
    """Reverse Cuthill-McKee permutation of A's symmetrized pattern: row i of
    the reordered matrix is row perm[i] of A (reference reorder.py:22-63)."""
    n = A.n
    indptr, indices = _symmetrized_pattern(A)
    perm = np.empty(n, dtype=np.int64)
    if n:
        lib = _lib.load(require_device=False)
        rc = lib.mpk_rcm_host(n, indptr.ctypes.data_as(ctypes.c_void_p),
                              indices.ctypes.data_as(ctypes.c_void_p), perm.ctypes.data_as(ctypes.c_void_p))
        if rc != 0:
            raise RuntimeError("mpk_rcm_host failed (%d)" % rc)
    return perm


def bandwidth(A: CsrMatrix) -> int:
    """max |i - j| over the stored entries (reference reorder.py:66-71)."""
    if A.nnz == 0:
        return 0
    rows = np.repeat(np.arange(A.n, dtype=np.int64), np.diff(A.row_ptr))
    return int(np.abs(rows - A.col_idx).max())
