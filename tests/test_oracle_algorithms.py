"""Pins for the oracle's fixed-rank algorithms (Algs 1-3) and bounds."""
import math

import numpy as np
import pytest
import scipy.linalg

import oracle as O
from workloads import hilbert, exact_rank, superdiagonal


def test_qr_example():
    q, r = np.linalg.qr(np.array([[3.0], [4.0]]))
    assert np.allclose(np.abs(q[:, 0]), [0.6, 0.8]) and abs(abs(r[0, 0]) - 5) < 1e-15


def test_superdiagonal_deterministic():
    """diag(3,2,1) superdiagonal, rank (2,2,2): abs error 1, rel 1/sqrt(14)."""
    x = superdiagonal([3.0, 2.0, 1.0])
    for t in (O.hosvd(x, (2, 2, 2)), O.sthosvd(x, (2, 2, 2))):
        e = O.rel_error(x, t.core, t.factors)
        assert abs(e - 1 / math.sqrt(14)) < 1e-14
    assert abs(O.delta_tail(x, 0, 2) - 1.0) < 1e-14


def test_randsvd_full_sketch_equals_hosvd():
    """l = I_n: Q spans R^{I_n}, so RandSVD = SVD and R-HOSVD = HOSVD (special case)."""
    rng = np.random.default_rng(0)
    x = rng.standard_normal((6, 7, 5))
    ranks = (3, 4, 2)
    rh = O.r_hosvd(x, ranks, p=10, seed=3)                    # l clamped to I_n
    assert rh.ell == (6, 7, 5)
    h = O.hosvd(x, ranks)
    assert O.approx_distance(x, (rh.core, rh.factors), (h.core, h.factors)) < 1e-12
    rs = O.r_sthosvd(x, ranks, p=10, seed=3, order=(0, 1, 2))
    s = O.sthosvd(x, ranks, order=(0, 1, 2))
    assert O.approx_distance(x, (rs.core, rs.factors), (s.core, s.factors)) < 1e-12


@pytest.mark.parametrize("dims,ranks", [((8, 9, 10), (2, 3, 2)), ((50, 50, 50), (5, 5, 5)),
                                        ((16, 12, 40), (4, 5, 6)), ((6, 7, 5, 4), (2, 3, 2, 2))])
@pytest.mark.parametrize("p", [0, 2, 5])
def test_exact_recovery(dims, ranks, p):
    """Exact multilinear rank r and p >= 0: relative error <= 1e-12 (BASELINE north_star)."""
    x = exact_rank(dims, ranks, seed=11)
    for t in (O.r_hosvd(x, ranks, p, seed=5), O.r_sthosvd(x, ranks, p, seed=5)):
        assert O.rel_error(x, t.core, t.factors) <= 1e-12
        for a in t.factors:
            assert np.allclose(a.T @ a, np.eye(a.shape[1]), atol=1e-12)


def test_sthosvd_identity():
    """||X - X_hat||^2 = ||X||^2 - ||G||^2 for (R-)STHOSVD (orthonormal factors,
    Thm 2.3 first equality), within 1e-12 ||X||^2."""
    rng = np.random.default_rng(4)
    for x in (hilbert((20, 22, 24)), rng.standard_normal((10, 12, 9, 5))):
        ranks = tuple(max(1, s // 4) for s in x.shape)
        for t in (O.r_sthosvd(x, ranks, 3, seed=1), O.sthosvd(x, ranks)):
            nx2 = float(np.sum(x * x))
            lhs = (O.rel_error(x, t.core, t.factors) ** 2) * nx2
            rhs = nx2 - float(np.sum(t.core ** 2))
            assert abs(lhs - rhs) <= 1e-12 * nx2
            assert abs(sum(t.mode_residual_sq.values()) - rhs) <= 1e-12 * nx2 if t.mode_residual_sq else True


def _hosvd_err_independent(x, ranks):
    """Deterministic HOSVD error by an independent library route (scipy eigh of the
    Gram X_(j) X_(j)^T instead of numpy's gesdd SVD), for cross-checking."""
    facs = []
    for j in range(x.ndim):
        m = O.unfold(x, j)
        w, v = scipy.linalg.eigh(m @ m.T)
        facs.append(v[:, ::-1][:, :ranks[j]])
    g = O.multi_mode_product(x, facs, transpose=True)
    return O.rel_error(x, g, facs)


def test_hilbert_c1_deterministic_and_randomized():
    """BASELINE configs[0] (shifted Hilbert 50^3, r=5, p=5).  Deterministic values are
    checked against an independent eigh route; the randomized errors equal the
    deterministic ones to ~1e-9 for any seed and lie below the
    Thm 3.1/3.2 bound."""
    x = hilbert((50, 50, 50), "shifted")
    r = (5, 5, 5)
    h = O.hosvd(x, r)
    eh = O.rel_error(x, h.core, h.factors)
    assert abs(eh - _hosvd_err_independent(x, r)) < 1e-10
    es = O.rel_error(x, *(lambda t: (t.core, t.factors))(O.sthosvd(x, r)))
    assert abs(eh - 7.008974e-4) < 5e-10 and abs(es - 7.007534e-4) < 5e-10
    nx = O.frob(x)
    assert abs(nx - 6.719862729) < 1e-8
    deltas = [O.delta_tail(x, j, 5) for j in range(3)]
    bound = O.bound_expected_error(deltas, r, 5) / nx
    assert abs(bound - 1.118213e-3) < 1e-9
    for seed in (0, 1, 2):
        rh = O.r_hosvd(x, r, 5, seed)
        rs = O.r_sthosvd(x, r, 5, seed, order=(0, 1, 2))
        erh = O.rel_error(x, rh.core, rh.factors)
        ers = O.rel_error(x, rs.core, rs.factors)
        assert abs(erh - eh) < 1e-8 and abs(ers - es) < 1e-8
        assert erh < bound and ers < bound


def test_bound_formulas():
    assert abs(O.bound_expected_error([1, 1, 1], [2, 2, 2], 3) - math.sqrt(6)) < 1e-15
    assert abs(O.g_cond(25, 10) - math.sqrt(601)) < 1e-12
    assert abs(O.f_p(4, 5) - math.sqrt(2)) < 1e-15
    # p = r + 1 => (1 + r/(p-1)) = 2: the sqrt(2) factor of P:216-217
    d = [0.3, 0.1, 0.2, 0.05, 0.4]
    assert abs(O.bound_expected_error(d, [4] * 5, 5) - math.sqrt(2) * math.sqrt(sum(v * v for v in d))) < 1e-14
    # p = ceil(r/eps) + 1 => factor <= sqrt(1+eps)
    r, eps = 5, 0.1
    p = math.ceil(r / eps) + 1
    assert O.bound_expected_error([1.0], [r], p) <= math.sqrt(1 + eps) + 1e-15
    assert abs(O.bound_sp((10,), (3,), 2, [0.5]) - O.g_cond(10, 5) * O.f_p(3, 2) * 0.5) < 1e-14


@pytest.mark.parametrize("algo", ["rhosvd", "rsthosvd"])
def test_expected_error_bound_seed_average(algo):
    """Thm 3.1 / 3.2: mean over 20 Omega seeds <= the bound (1.5x slack per S:248)."""
    rng = np.random.default_rng(7)
    core = rng.standard_normal((12, 12, 12)) * np.exp(-0.6 * np.add.outer(
        np.add.outer(np.arange(12), np.arange(12)), np.arange(12)))
    x = O.multi_mode_product(core, [np.linalg.qr(rng.standard_normal((n, 12)))[0] for n in (20, 18, 16)])
    r, p = (3, 3, 3), 3
    deltas = [O.delta_tail(x, j, r[j]) for j in range(3)]
    bound = O.bound_expected_error(deltas, r, p)
    errs = []
    for s in range(20):
        t = O.r_hosvd(x, r, p, s) if algo == "rhosvd" else O.r_sthosvd(x, r, p, s)
        errs.append(O.rel_error(x, t.core, t.factors) * O.frob(x))
    assert np.mean(errs) <= 1.5 * bound
    # deterministic counterpart obeys the deterministic bound (Thm 2.2/2.3)
    h = O.hosvd(x, r)
    assert O.rel_error(x, h.core, h.factors) * O.frob(x) <= math.sqrt(sum(d * d for d in deltas)) * (1 + 1e-12)


def test_auto_order():
    assert O.auto_order((40, 4096, 10)) == (1, 0, 2)        # S:409 (paper rho=[2,1,*])
    assert O.auto_order((807, 613, 1922)) == (2, 0, 1)      # S:410 (Table 6.5 rho=[3,1,2])
    assert O.auto_order((7, 7, 7)) == (0, 1, 2)
    assert O.auto_order((8000, 8000, 200000, 1200)) == (2, 0, 1, 3)


def test_rank_caps_clamp():
    assert O.rank_caps((25, 25, 25, 25, 25), 0, 25, 5) == (25, 25)   # Fig 6.1 sweep to r=25
    assert O.rank_caps((4, 3, 2), 2, 2, 3) == (2, 2)


def test_ordering_invariance_of_bound_and_rsthosvd_orders():
    """Every processing order gives a valid approximation under the same bound (Thm 3.2)."""
    import itertools
    x = hilbert((12, 10, 8), "paper")
    r, p = (3, 3, 3), 3
    deltas = [O.delta_tail(x, j, r[j]) for j in range(3)]
    bound = O.bound_expected_error(deltas, r, p)
    for order in itertools.permutations(range(3)):
        t = O.r_sthosvd(x, r, p, 0, order)
        assert O.rel_error(x, t.core, t.factors) * O.frob(x) <= 1.5 * bound


def test_canonical_signs_rule():
    """Reading R4b: the entry of largest magnitude of each column becomes positive; on a tie
    of magnitudes the FIRST such row decides; a zero column keeps sign +1."""
    u = np.array([[0.1, -3.0, 0.0, 2.0],
                  [-0.5, 2.0, 0.0, -2.0],
                  [0.5, 1.0, 0.0, 1.0]])
    s = O.canonical_signs(u)
    np.testing.assert_array_equal(s, [-1.0, -1.0, 1.0, 1.0])
    # applied by randsvd: every returned column has a positive largest-magnitude entry
    rng = np.random.default_rng(5)
    xm = rng.standard_normal((30, 40))
    omega = rng.standard_normal((40, 8))
    uu, _, vt, _ = O.randsvd(xm, 5, 3, omega)
    idx = np.argmax(np.abs(uu), axis=0)
    assert np.all(uu[idx, np.arange(5)] > 0)
    # the sign is applied to (U, V) together, so U S V^T is unchanged
    u0, s0, vt0 = np.linalg.svd(np.linalg.qr(xm @ omega)[0].T @ xm, full_matrices=False)
    q = np.linalg.qr(xm @ omega)[0]
    np.testing.assert_allclose((uu * s0[:5]) @ vt, (q @ u0[:, :5] * s0[:5]) @ vt0[:5], atol=1e-12)


def test_subspace_iteration_pins():
    """Randomized subspace iteration (NEXT-3; SPEC S:254-262 examples):
    q = 0 is the plain range finder; range(Q_q) = range((X X^T)^q X Omega) computed directly
    (no intermediate orthonormalisation, a different route); exact low rank is still recovered;
    on a slowly decaying spectrum one step does not increase the error (20 paired seeds)."""
    rng = np.random.default_rng(2)
    xm = rng.standard_normal((40, 60)) * (0.8 ** np.arange(60))[None, :]
    om = rng.standard_normal((60, 8))
    u0, _, _, i0 = O.randsvd(xm, 5, 3, om, 0)
    u1, _, _, i1 = O.randsvd(xm, 5, 3, om, 1)
    ua, _, _, _ = O.randsvd(xm, 5, 3, om)
    np.testing.assert_array_equal(u0, ua)
    direct = np.linalg.qr(xm @ (xm.T @ (xm @ om)))[0]
    assert O.projector_distance(i1["q"], direct) <= 1e-10
    x = exact_rank((9, 10, 11), (2, 3, 2), seed=4)
    for t in (O.r_hosvd(x, (2, 3, 2), 2, 1, power=1), O.r_sthosvd(x, (2, 3, 2), 2, 1, power=2)):
        assert O.rel_error(x, t.core, t.factors) <= 1e-12
    s = 1.0 / np.arange(1, 31) ** 0.3                        # slow decay
    u, _ = np.linalg.qr(rng.standard_normal((30, 30)))
    v, _ = np.linalg.qr(rng.standard_normal((50, 30)))
    a = (u * s) @ v.T
    e0 = e1 = 0.0
    for seed in range(20):
        om = np.random.default_rng(100 + seed).standard_normal((50, 6))
        for q, acc in ((0, 0), (1, 1)):
            uu, _, _, inf = O.randsvd(a, 4, 2, om, q)
            err = np.linalg.norm(a - inf["q"] @ (inf["q"].T @ a))
            if q == 0:
                e0 += err
            else:
                e1 += err
    assert e1 <= e0
