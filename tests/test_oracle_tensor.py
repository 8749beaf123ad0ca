"""Pins for oracle/tensor.py (unfolding order, mode products, norms)."""
import math

import numpy as np

import oracle as O

from oracle.tensor import unfold, fold, mode_product, multi_mode_product, frob, unfold_columns
from workloads import from_first_mode_fastest, to_first_mode_fastest


def _x222():
    return from_first_mode_fastest(np.arange(1, 9, dtype=np.float64), (2, 2, 2))


def test_unfold_2x2x2_examples():
    x = _x222()
    np.testing.assert_array_equal(unfold(x, 0), [[1, 3, 5, 7], [2, 4, 6, 8]])
    np.testing.assert_array_equal(unfold(x, 1), [[1, 2, 5, 6], [3, 4, 7, 8]])
    np.testing.assert_array_equal(unfold(x, 2), [[1, 2, 3, 4], [5, 6, 7, 8]])


def test_mode_product_example_and_norm():
    x = _x222()
    y = mode_product(x, np.array([[1.0, 1.0]]), 2)
    assert y.shape == (2, 2, 1)
    np.testing.assert_array_equal(to_first_mode_fastest(y), [6, 8, 10, 12])
    assert abs(frob(x) ** 2 - 204.0) < 1e-12


def test_fold_inverts_unfold():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((3, 4, 5, 2))
    for j in range(4):
        np.testing.assert_array_equal(fold(unfold(x, j), j, x.shape), x)


def test_kronecker_identity():
    """eq. (kron): Y_(j) = A_j X_(j) (A_d (x) .. (x) A_{j+1} (x) A_{j-1} (x) .. A_1)^T,
    with np.kron as the independent route; fixes the column order of X_(j)."""
    rng = np.random.default_rng(1)
    dims, out = (3, 4, 5, 2), (2, 3, 4, 3)
    x = rng.standard_normal(dims)
    a = [rng.standard_normal((o, i)) for o, i in zip(out, dims)]
    y = multi_mode_product(x, a)
    for j in range(4):
        k = np.ones((1, 1))
        for m in reversed(range(4)):
            if m != j:
                k = np.kron(k, a[m])
        np.testing.assert_allclose(unfold(y, j), a[j] @ unfold(x, j) @ k.T, rtol=1e-12, atol=1e-12)


def test_unfold_columns_matches_dense_unfolding():
    rng = np.random.default_rng(2)
    dims = (3, 4, 5, 2)
    x = rng.standard_normal(dims)
    idx = np.array(np.unravel_index(np.arange(x.size), dims, order="F"))
    for j in range(4):
        c = unfold_columns(dims, j, idx)
        m = unfold(x, j)
        np.testing.assert_array_equal(m[idx[j], c], to_first_mode_fastest(x))


def test_mode_product_definition_bruteforce():
    """Entry formula of the mode product by explicit loops."""
    rng = np.random.default_rng(3)
    x = rng.standard_normal((2, 3, 4))
    a = rng.standard_normal((5, 3))
    y = mode_product(x, a, 1)
    for i1 in range(2):
        for k in range(5):
            for i3 in range(4):
                s = sum(x[i1, i2, i3] * a[k, i2] for i2 in range(3))
                assert abs(y[i1, k, i3] - s) < 1e-12


def test_approx_distance_closed_form():
    """delta between two DIFFERENT Tuckers has a closed form (the metric was only
    ever checked at 0).  Superdiagonal (3,2,1) of S:105: its rank-(2,2,2) truncation is
    diag(3,2,0) and its rank-(1,1,1) truncation diag(3,0,0), so
    ||X_hat2 - X_hat1||_F / ||X||_F = 2 / sqrt(14)."""
    from workloads import superdiagonal
    x = superdiagonal([3.0, 2.0, 1.0])
    e = np.eye(3)
    g2 = np.zeros((2, 2, 2))
    g2[0, 0, 0], g2[1, 1, 1] = 3.0, 2.0
    t2 = (g2, [e[:, :2]] * 3)
    t1 = (np.full((1, 1, 1), 3.0), [e[:, :1]] * 3)
    assert abs(O.approx_distance(x, t2, t1) - 2 / math.sqrt(14)) < 1e-15
    assert abs(O.approx_distance(x, t1, t2) - 2 / math.sqrt(14)) < 1e-15
    # the full tensor against its rank-1 truncation: sqrt(2^2 + 1^2) / sqrt(14)
    t3 = (x, [e] * 3)
    assert abs(O.approx_distance(x, t3, t1) - math.sqrt(5 / 14)) < 1e-15
    # sign/basis invariance: flipping a factor column and the matching core slice is the
    # same approximation (distance 0), flipping only the factor is not (distance 2*2/sqrt(14))
    f = [e[:, :2].copy() for _ in range(3)]
    f[1][:, 1] *= -1
    g = g2.copy()
    g[:, 1, :] *= -1
    assert O.approx_distance(x, t2, (g, f)) < 1e-15
    assert abs(O.approx_distance(x, t2, (g2, f)) - 4 / math.sqrt(14)) < 1e-15


def test_projector_distance_closed_form():
    """||A A^T - B B^T||_2 = sin(theta) for two planes in R^4 sharing one direction and
    rotated by theta in the other (largest principal angle theta); 0 for a rotated basis of
    the same subspace; 1 for orthogonal complements."""
    for th in (1e-9, 1e-5, 0.3, 1.2):
        a = np.zeros((4, 2))
        a[0, 0] = a[1, 1] = 1.0
        b = np.zeros((4, 2))
        b[0, 0] = 1.0
        b[1, 1], b[2, 1] = math.cos(th), math.sin(th)
        assert abs(O.projector_distance(a, b) - math.sin(th)) <= 1e-15 + 1e-13 * math.sin(th)
    rng = np.random.default_rng(0)
    q = np.linalg.qr(rng.standard_normal((9, 3)))[0]
    rot = np.linalg.qr(rng.standard_normal((3, 3)))[0]
    assert O.projector_distance(q, q @ rot) < 1e-15
    full = np.linalg.qr(rng.standard_normal((6, 6)))[0]
    assert abs(O.projector_distance(full[:, :3], full[:, 3:]) - 1.0) < 1e-14


def test_spectral_gap_kappa():
    """kappa = u s_1 / (s_r - s_{r+1}) (SURVEY c.4 gate)."""
    s = np.array([4.0, 2.0, 1.5, 1.0])
    assert abs(O.spectral_gap_kappa(s, 2, 1e-16) - 1e-16 * 4.0 / 0.5) < 1e-30
    assert O.spectral_gap_kappa(s, 4, 1e-16) == 0.0
    assert O.spectral_gap_kappa(np.array([1.0, 1.0]), 1, 1e-16) == float("inf")
