"""Dense Krylov primitives on the device vs numpy / dense oracles
(mirrors the reference's tests/test_kernels.py)."""

import numpy as np
import pytest

import paper_2105_07544_b200 as mk

pytestmark = pytest.mark.gpu


def test_vector_primitives(cuda, rng):
    for dtype in (np.float64, np.float32):
        x = rng.standard_normal(10000).astype(dtype)
        y = rng.standard_normal(10000).astype(dtype)
        assert np.isclose(mk.dot(x, y), float(x.astype(np.float64) @ y.astype(np.float64)), rtol=1e-4)
        assert np.isclose(mk.norm2(x), np.linalg.norm(x.astype(np.float64)), rtol=1e-6)
        z = mk.axpy(2.5, x, y)
        assert z.dtype == dtype and np.array_equal(z, y + dtype(2.5) * x)
        w = mk.scale(0.5, x)
        assert np.array_equal(w, dtype(0.5) * x)
    with pytest.raises(mk.PrecisionMismatchError):
        mk.dot(np.ones(3), np.ones(3, dtype=np.float32))


def test_dot_is_deterministic(cuda, rng):
    x = rng.standard_normal(3_000_001)
    vals = {float(mk.dot(x, x)) for _ in range(5)}
    assert len(vals) == 1


@pytest.mark.parametrize("prec,tol", [(mk.Precision.binary64, 1e-14), (mk.Precision.binary32, 1e-6)])
@pytest.mark.parametrize("n,k", [(50, 12), (20000, 40), (3000, 70)])
def test_cgs2_orthonormal(cuda, rng, prec, tol, n, k):
    dt = prec.dtype
    basis = mk.KrylovBasis(n, k, prec)
    v = rng.standard_normal(n).astype(dt)
    basis.append((v / np.linalg.norm(v)).astype(dt))
    for _ in range(k - 1):
        coeffs, beta, appended = mk.cgs2_append(basis, rng.standard_normal(n).astype(dt))
        assert appended and coeffs.shape == (basis.count - 1,) and beta > 0
    V = basis.columns().astype(np.float64)
    assert np.abs(V.T @ V - np.eye(basis.count)).max() <= tol * max(1, n / 1000)


def test_cgs2_reconstructs_and_detects_breakdown(cuda, rng):
    n, k = 30, 6
    basis = mk.KrylovBasis(n, k + 1, mk.Precision.binary64)
    v = rng.standard_normal(n)
    basis.append(v / np.linalg.norm(v))
    for _ in range(k - 1):
        mk.cgs2_append(basis, rng.standard_normal(n))
    w = rng.standard_normal(n)
    cnt = basis.count
    coeffs, beta, appended = mk.cgs2_append(basis, w)
    rebuilt = basis.columns(cnt) @ coeffs + beta * basis.column(cnt)
    assert appended and np.abs(rebuilt - w).max() <= 1e-12 * np.abs(w).max()
    b2 = mk.KrylovBasis(20, 4, mk.Precision.binary64)
    v = rng.standard_normal(20)
    b2.append(v / np.linalg.norm(v))
    _, beta, appended = mk.cgs2_append(b2, 3.0 * v)
    assert not appended and b2.count == 1


def random_hessenberg(rng, m):
    h = np.zeros((m + 1, m))
    for j in range(m):
        h[: j + 1, j] = rng.standard_normal(j + 1)
        h[j + 1, j] = abs(rng.standard_normal()) + 0.5
    return h


def lstsq(gamma, h, k):
    rhs = np.zeros(k + 1)
    rhs[0] = gamma
    y, *_ = np.linalg.lstsq(h[: k + 1, :k], rhs, rcond=None)
    return y, np.linalg.norm(rhs - h[: k + 1, :k] @ y)


def test_hessenberg_tracks_lstsq(cuda, rng):
    m, gamma = 10, 2.0
    h = random_hessenberg(rng, m)
    sys_ = mk.HessenbergSystem(m, gamma)
    for j in range(1, m + 1):
        rel = sys_.update(j, h[:j, j - 1].copy(), h[j, j - 1])
        _, res = lstsq(gamma, h, j)
        assert np.isclose(rel * gamma, res, rtol=1e-10, atol=1e-12)
    y = sys_.solve()
    want, _ = lstsq(gamma, h, m)
    assert np.abs(y - want).max() <= 1e-9 * (np.abs(want).max() + 1)
    y3 = sys_.solve(3)
    want3, _ = lstsq(gamma, h, 3)
    assert np.abs(y3 - want3).max() <= 1e-9


def test_hessenberg_errors(cuda):
    s = mk.HessenbergSystem(4, 1.0)
    with pytest.raises(mk.ColumnOrderError):
        s.update(2, np.zeros(2), 1.0)
    with pytest.raises(mk.ColumnOrderError):
        s.solve()
    s = mk.HessenbergSystem(2, 1.0)
    s.update(1, np.array([0.0]), 1.0)
    s.update(2, np.array([0.0, 5.0]), 0.0)
    with pytest.raises(mk.TriangularBreakdownError) as info:
        s.solve()
    assert info.value.threshold >= 0.0
