"""Oracle error-bound formulas (test infrastructure only; see oracle/__init__.py).

Delta_j (eq. delta), Thm 3.1/3.2 expected-error bound,
Thm 5.1 SP bound with g(I,r) = sqrt(1+4r(I-r)) and f_p(r) = sqrt(1+r/(p-1)).
"""
from __future__ import annotations

import math
import numpy as np

from .tensor import unfold


def delta_tail(x: np.ndarray, j: int, r: int) -> float:
    """Delta_j = sqrt(sum_{i>r_j} sigma_i^2(X_(j))) (eq. delta)."""
    s = np.linalg.svd(unfold(np.asarray(x, dtype=np.float64), j), compute_uv=False)
    return float(math.sqrt(float(np.sum(s[r:] ** 2))))


def bound_expected_error(deltas, ranks, p: int) -> float:
    """(sum_j (1 + r_j/(p-1)) Delta_j^2)^{1/2}, Thm 3.1 / Thm 3.2 (needs p >= 2)."""
    if p < 2:
        raise ValueError("bound needs p >= 2")
    return math.sqrt(sum((1.0 + r / (p - 1.0)) * dl * dl for dl, r in zip(deltas, ranks)))


def g_cond(I: int, ell: int) -> float:
    """g(I, r) = sqrt(1 + 4 r (I - r)) (Thm 5.1)."""
    return math.sqrt(1.0 + 4.0 * ell * (I - ell))


def f_p(r: int, p: int) -> float:
    """f_p(r) = sqrt(1 + r/(p-1)) (Thm 5.1)."""
    if p < 2:
        raise ValueError("f_p needs p >= 2")
    return math.sqrt(1.0 + r / (p - 1.0))


def bound_sp(dims, ranks, p: int, deltas, order=None) -> float:
    """sum_j (prod_{k<=j} g(I_k, l_k)) f_p(r_j) Delta_j (Thm 5.1), evaluated in the
    processing order (the theorem is stated for rho = [1..d])."""
    order = list(range(len(dims))) if order is None else list(order)
    tot, prod_g = 0.0, 1.0
    for j in order:
        prod_g *= g_cond(dims[j], ranks[j] + p)
        tot += prod_g * f_p(ranks[j], p) * deltas[j]
    return tot
