"""Oracle tensor algebra (test infrastructure only; see oracle/__init__.py).

PAPER.md §2.1: mode-j unfolding X_(j) in R^{I_j x prod_{k!=j} I_k} whose
columns are the mode-j fibers; mode product Y = X x_j A <=> Y_(j) = A X_(j)
(P:29-31); multi-mode product and its Kronecker form eq. (kron).

Column order of X_(j) (DESIGN reading R2): c = sum_{k!=j} i_k prod_{m<k, m!=j} I_m
(0-based, lower modes fastest), which is the order for which eq. (kron) reads
Y_(j) = A_j X_(j) (A_d (x) ... (x) A_{j+1} (x) A_{j-1} (x) ... (x) A_1)^T.
Pinned by the 2x2x2 example and the Kronecker identity (tests/test_oracle_tensor.py).
Modes are 0-based in code (mode j here is the paper's j+1).
"""
from __future__ import annotations

import numpy as np


def unfold(x: np.ndarray, j: int) -> np.ndarray:
    """X_(j): move mode j to the front, then lay the remaining modes out with the
    lowest mode fastest (Fortran order)."""
    return np.reshape(np.moveaxis(x, j, 0), (x.shape[j], -1), order="F")


def fold(m: np.ndarray, j: int, dims) -> np.ndarray:
    """Inverse of `unfold` for a tensor whose mode-j size is m.shape[0]."""
    dims = list(dims)
    dims[j] = m.shape[0]
    rest = [dims[k] for k in range(len(dims)) if k != j]
    t = np.reshape(m, [m.shape[0]] + rest, order="F")
    return np.moveaxis(t, 0, j)


def unfold_columns(dims, j: int, idx) -> np.ndarray:
    """Unfolding column c of X_(j) for 0-based multi-indices idx (d x nnz):
    c = sum_{k!=j} i_k prod_{m<k, m!=j} I_m (DESIGN reading R2)."""
    c = np.zeros(np.asarray(idx[0]).shape, dtype=np.int64)
    stride = 1
    for k in range(len(dims)):
        if k == j:
            continue
        c = c + np.asarray(idx[k], dtype=np.int64) * stride
        stride *= int(dims[k])
    return c


def mode_product(x: np.ndarray, a: np.ndarray, j: int) -> np.ndarray:
    """Y = X x_j A, i.e. Y_(j) = A X_(j)."""
    return fold(a @ unfold(x, j), j, x.shape)


def multi_mode_product(x: np.ndarray, mats, transpose: bool = False) -> np.ndarray:
    """X x_1 M_1 x_2 ... x_d M_d (entries of `mats` may be None = identity)."""
    y = x
    for j, m in enumerate(mats):
        if m is None:
            continue
        y = mode_product(y, m.T if transpose else m, j)
    return y


def frob(x) -> float:
    return float(np.sqrt(np.sum(np.asarray(x, dtype=np.float64) ** 2)))


def reconstruct(core: np.ndarray, factors) -> np.ndarray:
    """X_hat = [G; A_1, ..., A_d] = G x_1 A_1 ... x_d A_d."""
    return multi_mode_product(np.asarray(core, dtype=np.float64), factors)


def rel_error(x: np.ndarray, core: np.ndarray, factors) -> float:
    """||X - X_hat||_F / ||X||_F by direct reconstruction."""
    xh = reconstruct(core, factors)
    x64 = np.asarray(x, dtype=np.float64)
    return frob(x64 - xh) / frob(x64)


def approx_distance(x: np.ndarray, t1, t2) -> float:
    """delta = ||X_hat1 - X_hat2||_F / ||X||_F (DESIGN §5 parity metric; SURVEY c.4: a
    direct elementwise difference of the two reconstructions, not core algebra).
    Pinned by closed forms in tests/test_oracle_tensor.py (2/sqrt(14) between the rank-2
    and rank-1 truncations of the S:105 superdiagonal tensor)."""
    a = reconstruct(t1[0], t1[1])
    b = reconstruct(t2[0], t2[1])
    return frob(a - b) / frob(np.asarray(x, dtype=np.float64))


def projector_distance(a: np.ndarray, b: np.ndarray) -> float:
    """||A A^T - B B^T||_2 for two orthonormal bases of equal width (north_star parity
    criterion, SURVEY c.4).  For equal dimensions this is the sine of the largest principal
    angle, evaluated as ||(I - B B^T) A||_2 (no cancellation for small angles).  Pinned by
    the closed form sin(theta) for planes rotated by theta (tests/test_oracle_tensor.py)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError("projector_distance: bases of different shapes")
    return float(np.linalg.norm(a - b @ (b.T @ a), 2))


def spectral_gap_kappa(s, r: int, u: float) -> float:
    """Gate of the projector criterion (SURVEY c.4): kappa = u * s_1 / (s_r - s_{r+1}) for the
    singular values s of B (descending) and the working unit roundoff u; the criterion
    applies when kappa <= 1e-5.  r = len(s) (no s_{r+1}) gives kappa = 0."""
    s = np.asarray(s, dtype=np.float64)
    if r >= s.size:
        return 0.0
    gap = s[r - 1] - s[r]
    return float("inf") if gap <= 0 else float(u * s[0] / gap)
