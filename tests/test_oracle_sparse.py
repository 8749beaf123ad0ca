"""Pins for the oracle's SP-STHOSVD (Alg 6) and the sRRQR reading R9."""
import itertools

import numpy as np
import pytest

import oracle as O
from workloads import superdiagonal, sparse_zipf, from_first_mode_fastest


def _coo(x):
    idx = np.array(np.nonzero(x))
    return idx, x[tuple(idx)]


def test_srrqr_small_examples():
    q = np.eye(5)[:, :3]                                      # S:180 identity columns
    sel, _ = O.srrqr_select(q)
    assert sel == [0, 1, 2]
    q = np.array([[1.0], [1.0]]) / np.sqrt(2)                 # S:180 2x1 case
    sel, _ = O.srrqr_select(q)
    a = O.oblique_factor(q, sel)
    assert sel == [0] and np.allclose(a, [[1.0], [1.0]])      # S:189, tie -> smallest index
    assert np.linalg.norm(np.linalg.inv(q[sel]), 2) <= O.g_cond(2, 1)


@pytest.mark.parametrize("I,ell", [(30, 6), (20, 4), (200, 15), (9, 3)])
def test_srrqr_properties(I, ell):
    """Thm 5.1: A contains I_l at S, |A_ik| <= eta, 1 <= ||A||_2 <= g(I,l)."""
    rng = np.random.default_rng(I + ell)
    q, _ = np.linalg.qr(rng.standard_normal((I, ell)) * np.exp(-0.2 * np.arange(I))[:, None])
    sel, swaps = O.srrqr_select(q, 2.0)
    a = O.oblique_factor(q, sel)
    np.testing.assert_allclose(a[sel], np.eye(ell), atol=1e-12)
    assert np.max(np.abs(a)) <= 2.0 + 1e-12
    n2 = np.linalg.norm(a, 2)
    assert 1 - 1e-12 <= n2 <= O.g_cond(I, ell)
    assert sel == sorted(sel) and len(set(sel)) == ell


def test_srrqr_bruteforce_local_optimality():
    """Brute force on tiny inputs: the selected rows' |det| is within eta^l of the best
    subset's (maxvol guarantee) and no single swap improves it by more than eta."""
    rng = np.random.default_rng(3)
    for trial in range(20):
        I, ell = 7, 3
        q, _ = np.linalg.qr(rng.standard_normal((I, ell)))
        sel, _ = O.srrqr_select(q, 2.0)
        best = max(abs(np.linalg.det(q[list(c)])) for c in itertools.combinations(range(I), ell))
        got = abs(np.linalg.det(q[sel]))
        assert got * 2.0 ** ell >= best
        for k in range(ell):
            for i in range(I):
                if i in sel:
                    continue
                s2 = list(sel)
                s2[k] = i
                assert abs(np.linalg.det(q[s2])) <= 2.0 * got * (1 + 1e-12)


def test_sp_superdiagonal_example():
    """5^3 superdiagonal (5,4,3,2,1), r=(2,2,2), p=2: core is a 4x4x4 sub-tensor
    of x with entries copied bit-exactly."""
    x = superdiagonal([5.0, 4.0, 3.0, 2.0, 1.0])
    idx, vals = _coo(x)
    t = O.sp_sthosvd(idx, vals, x.shape, (2, 2, 2), 2, seed=0, order=(0, 1, 2))
    assert t.core_dims == (4, 4, 4)
    g = t.dense_core()
    sub = x[np.ix_(*t.selections)]
    np.testing.assert_array_equal(g, sub)


def _dense_sp_sthosvd(x, ranks, p, seed, order, eta=2.0):
    """Independent dense route for Alg 6: dense unfoldings, full Omega, np.take."""
    g = np.asarray(x, dtype=np.float64)
    sels, facs = [None] * x.ndim, [None] * x.ndim
    for j in order:
        gj = O.unfold(g, j)
        om = O.omega_rows(seed, j, np.arange(gj.shape[1]), ranks[j] + p)
        q, _ = np.linalg.qr(gj @ om)
        s, _ = O.srrqr_select(q, eta)
        facs[j] = O.oblique_factor(q, s)
        sels[j] = s
        g = np.take(g, s, axis=j)
    return g, facs, sels


def test_sp_sparse_matches_dense_route():
    """COO path (occupied-column Omega rows, unfold_columns, compaction) equals the
    dense-unfolding route on a random sparse 12x10x9 tensor."""
    rng = np.random.default_rng(5)
    x = rng.standard_normal((12, 10, 9)) * (rng.random((12, 10, 9)) < 0.3)
    idx, vals = _coo(x)
    for order in [(0, 1, 2), (2, 0, 1)]:
        t = O.sp_sthosvd(idx, vals, x.shape, (2, 3, 2), 2, seed=4, order=order)
        g, facs, sels = _dense_sp_sthosvd(x, (2, 3, 2), 2, 4, order)
        assert [list(s) for s in t.selections] == [list(s) for s in sels]
        np.testing.assert_array_equal(t.dense_core(), g)
        for a, b in zip(t.factors, facs):
            np.testing.assert_allclose(a, b, atol=1e-12)


def test_sp_sketch_equals_dense_unfolding_product():
    """Alg 6 line 4: the COO sketch (Omega rows drawn only for occupied columns, summed per
    row) equals X_(j) Omega_j with the full dense unfolding and every Omega row; a tensor with
    an empty slice and a single heavy row covers the degenerate rows."""
    rng = np.random.default_rng(8)
    x = rng.standard_normal((7, 6, 5)) * (rng.random((7, 6, 5)) < 0.25)
    x[3] = 0.0                                               # empty mode-0 row
    x[5] = rng.standard_normal((6, 5))                       # dense (heavy) mode-0 row
    idx, vals = _coo(x)
    for j in range(3):
        y = O.sp_sketch(idx, vals, x.shape, j, 4, seed=2)
        xj = O.unfold(x, j)
        om = O.omega_rows(2, j, np.arange(xj.shape[1]), 4)
        np.testing.assert_allclose(y, xj @ om, rtol=0, atol=1e-12)
        if j == 0:
            assert np.all(y[3] == 0.0)


def test_sp_structure_on_zipf_counts():
    """Scaled-down C5 (BASELINE configs[4] recipe): every core entry is an entry of X
    bit-exactly, nnz never increases, A_j[S_j] = I, 1 <= ||A_j||_2 <= g(I_j, l_j)."""
    dims = (80, 80, 2000, 12)
    idx, vals = sparse_zipf(dims, 20000, seed=5)
    t = O.sp_sthosvd(idx, vals, dims, (3, 3, 3, 3), 2, seed=0)
    assert t.order == (2, 0, 1, 3)
    assert all(a >= b for a, b in zip(t.nnz_history, t.nnz_history[1:]))
    lookup = {tuple(c): v for c, v in zip(idx.T.tolist(), vals.tolist())}
    for c, v in zip(t.core_idx.T.tolist(), t.core_vals.tolist()):
        orig = tuple(int(t.selections[j][c[j]]) for j in range(4))
        assert lookup[orig] == v
    for j in range(4):
        a = t.factors[j]
        np.testing.assert_allclose(a[t.selections[j]], np.eye(a.shape[1]), atol=1e-12)
        n2 = np.linalg.norm(a, 2)
        assert 1 - 1e-12 <= n2 <= O.g_cond(dims[j], 5)


def test_sp_bound_seed_average():
    """Thm 5.1 expected-error bound holds on a small dense-as-sparse tensor."""
    rng = np.random.default_rng(9)
    core = rng.standard_normal((8, 8, 8)) * np.exp(-0.5 * np.add.outer(np.add.outer(np.arange(8), np.arange(8)), np.arange(8)))
    x = O.multi_mode_product(core, [np.linalg.qr(rng.standard_normal((n, 8)))[0] for n in (14, 13, 12)])
    idx, vals = _coo(x)
    r, p = (3, 3, 3), 2
    deltas = [O.delta_tail(x, j, r[j]) for j in range(3)]
    bound = O.bound_sp(x.shape, r, p, deltas, (0, 1, 2))
    errs = []
    for s in range(10):
        t = O.sp_sthosvd(idx, vals, x.shape, r, p, seed=s, order=(0, 1, 2))
        errs.append(O.rel_error(x, t.dense_core(), t.factors) * O.frob(x))
    assert np.mean(errs) <= bound


def test_sp_rank_cap_strict():
    x = superdiagonal([3.0, 2.0, 1.0])
    idx, vals = _coo(x)
    with pytest.raises(ValueError):
        O.sp_sthosvd(idx, vals, x.shape, (1, 1, 1), 2)   # l = 3 is not < 3


def test_sp_hosvd_core_is_cartesian_selection():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((10, 10, 10))
    idx, vals = _coo(x)
    t = O.sp_hosvd(idx, vals, x.shape, (3, 3, 3), 2, seed=2)
    np.testing.assert_array_equal(t.dense_core(), x[np.ix_(*t.selections)])
