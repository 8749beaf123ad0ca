"""Pins for oracle/tensor.py (unfolding order, mode products, norms)."""
import numpy as np

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
