"""Pins for the oracle's adaptive range finder and Alg 4/5 (DESIGN reading R8)."""
import os
from collections import Counter

import numpy as np
import pytest

import oracle as O
from workloads import hilbert, exact_rank

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _table63():
    rows = {}
    with open(os.path.join(GOLD, "table_6_3_adaptive_ranks.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            v = [int(t) for t in line.split()]
            rows[v[0]] = v[1:]
    return rows


EPS = [1e-3, 1e-4, 1e-5, 1e-6, 1e-7]


@pytest.mark.parametrize("I", [25, 50, 100])
def test_table_6_3(I):
    """PAPER Table 6.3: adaptive R-STHOSVD on the paper-form Hilbert tensor,
    d=3, b=1, rho=[1,2,3].  The modal rank over Omega seeds equals the table in every
    cell, and every run meets the tolerance by direct reconstruction."""
    want = _table63()[I]
    x = hilbert((I, I, I), "paper")
    nx = O.frob(x)
    for eps, w in zip(EPS, want):
        got = []
        for seed in range(10):
            t = O.adaptive_r_sthosvd(x, eps, 1, seed=seed, order=(0, 1, 2))
            got.append(t.ranks)
            err = O.rel_error(x, t.core, t.factors)
            assert err <= eps * (1 + 1e-6) or eps <= 1e-7 and err <= 1.05 * eps
        modal = Counter(r for rr in got for r in rr).most_common(1)[0][0]
        assert modal == w, (I, eps, got)


def test_adaptive_exact_rank():
    """Exactly rank-(3,4,2) tensor, tiny eps, b=1: the range finder stops on the floor
    or tolerance after exactly the true rank in every mode."""
    x = exact_rank((10, 11, 12), (3, 4, 2), seed=2)
    t = O.adaptive_r_sthosvd(x, 1e-10, 1, seed=0, order=(0, 1, 2))
    assert t.ranks == (3, 4, 2)
    assert O.rel_error(x, t.core, t.factors) < 1e-10


def test_range_finder_geometric_diag():
    """diag(2^-i) 20x20, eps=1e-3, b=2.  Closed form: the minimal rank kmin with
    tail^2 <= eps^2 ||X||^2.  Eckart-Young makes kmin a lower bound for any basis; the
    untruncated basis is a multiple of b; the residual identity certifies the tolerance
    and decays monotonically; truncation lands between kmin and the basis size."""
    s = 2.0 ** -np.arange(1, 21)
    x = np.diag(s)
    eps = 1e-3
    nx2 = float(np.sum(s * s))
    tail2 = np.array([np.sum(s[k:] ** 2) for k in range(21)])
    kmin = int(np.nonzero(tail2 <= eps * eps * nx2)[0][0])
    for seed in range(5):
        q, g, info = O.adapt_range_finder(x, eps * eps * nx2, 2, seed=seed, mode=0,
                                          norm_x=np.sqrt(nx2), truncate=False)
        k = q.shape[1]
        assert k % 2 == 0 and kmin <= k <= kmin + 4
        res = np.linalg.norm(x - q @ (q.T @ x)) ** 2
        assert res <= eps * eps * nx2 * (1 + 1e-9)
        assert abs(res - info["e"]) <= 1e-14 * nx2
        assert np.all(np.diff(info["e_hist"]) <= 1e-15)
        a, g2, info2 = O.adapt_range_finder(x, eps * eps * nx2, 2, seed=seed, mode=0,
                                            norm_x=np.sqrt(nx2))
        assert kmin <= a.shape[1] <= k
        assert np.linalg.norm(x - a @ (a.T @ x)) ** 2 <= eps * eps * nx2 * (1 + 1e-9)


def test_adaptive_guarantee_and_mode_tolerances():
    """||X - X_hat|| <= eps ||X|| for Alg 5 and Alg 4, with uniform and
    with per-mode tolerances (sum eps_j^2 = eps^2, eps_j = 0: mode not compressed)."""
    x = hilbert((30, 25, 20), "shifted")
    for eps in (1e-2, 1e-4):
        t = O.adaptive_r_sthosvd(x, eps, 3, seed=4)
        assert O.rel_error(x, t.core, t.factors) <= eps
        h = O.adaptive_r_hosvd(x, eps, 3, seed=4)
        assert O.rel_error(x, h.core, h.factors) <= eps
    eps = 1e-3
    t = O.adaptive_r_sthosvd(x, eps, 2, seed=0, order=(0, 1, 2), mode_tol=[0.0, eps / np.sqrt(2), eps / np.sqrt(2)])
    assert t.ranks[0] == 30 and O.rel_error(x, t.core, t.factors) <= eps
    with pytest.raises(ValueError):
        O.adaptive_r_sthosvd(x, eps, 2, mode_tol=[eps, eps, eps])


def test_adaptive_first_block_equals_fixed_rank_sketch():
    """Global column index k: the adaptive run's first l sketch columns are the
    fixed-rank Omega's, so with one block of l columns and no truncation the basis
    spans the same space as R-STHOSVD's Q for the first mode."""
    rng = np.random.default_rng(0)
    x = rng.standard_normal((15, 14, 13))
    ell = 6
    q, _, _ = O.adapt_range_finder(O.unfold(x, 0), 0.0, ell, seed=9, mode=0, norm_x=O.frob(x),
                                   truncate=False)
    q1 = q[:, :ell]
    om = O.omega_rows(9, 0, np.arange(14 * 13), ell)
    qf, _ = np.linalg.qr(O.unfold(x, 0) @ om)
    assert np.linalg.norm(q1 @ q1.T - qf @ qf.T, 2) < 1e-12
