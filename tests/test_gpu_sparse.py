"""GPU parity of SP-STHOSVD (Alg 6; sRRQR per DESIGN reading R9) through the C ABI
against the CPU oracle on the same COO inputs: selections S_j equal, core
entries bit-exact copies of the input values, oblique factors A_j = Q (P^T Q)^-1 close
(they do not depend on the QR basis), and Thm 5.1's structure (A_j[S_j,:] = I, |A| <= eta)."""
import numpy as np
import pytest

import oracle as O
from workloads import superdiagonal, sparse_zipf

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1905_07311_b200.rtucker import Context
    c = Context(0)
    yield c
    c.close()


def _run(ctx, idx, vals, dims, ranks, p, seed=0, order=None, eta=2.0, device=True, flags=0):
    import torch
    from paper_1905_07311_b200.rtucker import RESULT_HOST
    if device:
        it = torch.as_tensor(np.ascontiguousarray(idx, dtype=np.int32), device="cuda")
        vt = torch.as_tensor(np.ascontiguousarray(vals), device="cuda")
        return ctx.sparse_sthosvd(it, vt, dims, ranks, p, seed, order, eta, flags | RESULT_HOST).numpy()
    return ctx.sparse_sthosvd(np.ascontiguousarray(idx, dtype=np.int32), np.ascontiguousarray(vals), dims, ranks, p,
                              seed, order, eta, flags | RESULT_HOST).numpy()


def _check(g, o, eta, a_tol):
    d = len(o.selections)
    for j in range(d):
        assert list(g.selections[j]) == list(o.selections[j]), (j, g.selections[j], o.selections[j])
        a = g.factors[j]
        np.testing.assert_allclose(a[np.asarray(o.selections[j])], np.eye(a.shape[1]), atol=1e-10)
        assert np.max(np.abs(a)) <= eta * (1 + 1e-9)
        err = np.linalg.norm(a - o.factors[j]) / np.linalg.norm(o.factors[j])
        assert err <= a_tol, (j, err)
    assert tuple(g.nnz_history) == tuple(o.nnz_history)
    # core: same entries (bit-exact values), compare as sorted coordinate lists
    gk = np.lexsort(g.core_idx[::-1])
    ok = np.lexsort(o.core_idx[::-1])
    np.testing.assert_array_equal(g.core_idx[:, gk], o.core_idx[:, ok])
    np.testing.assert_array_equal(g.core_vals[gk], np.asarray(o.core_vals)[ok])


def _col_err(y, yo):
    return np.max(np.linalg.norm(y - yo, axis=0) / np.maximum(np.linalg.norm(yo, axis=0), 1e-300))


@pytest.mark.parametrize("dtype,flags", [(np.float64, 0), (np.float32, "fp64"), (np.float32, 0)])
def test_coo_sketch_elementwise(ctx, dtype, flags):
    """Alg 6 line 4 element by element against the oracle: the row-sorted, lane-segmented
    fixed-point sketch (sparse.cu) on C5-shaped Zipf counts at 1/100 of the draws (heavy rows
    spanning many lanes and warps, ragged tails), every mode.  fp64 normals: the fixed-point sum
    is the exact sum rounded once (R20), so ~1e-13 per column; fp32 normals (R3, RMS 3e-7)."""
    from paper_1905_07311_b200.rtucker import ACCUM_FP64
    idx, vals = sparse_zipf(ndraws=500_000, seed=4)
    vals = vals.astype(dtype)
    dims = (8000, 8000, 200000, 1200)
    f = ACCUM_FP64 if flags == "fp64" else 0
    tol = 1e-6 if (dtype == np.float32 and not f) else 1e-12
    for j in range(4):
        y = ctx.debug_coo_sketch(idx, vals, dims, j, 15, seed=5, flags=f)
        yo = O.sp_sketch(idx, vals, dims, j, 15, seed=5)
        assert _col_err(y, yo) <= tol, (j, _col_err(y, yo))
        assert np.all(y[np.abs(yo).sum(axis=1) == 0] == 0.0)      # empty rows stay exactly zero


def test_coo_sketch_degenerate(ctx):
    """Edge cases of the sorted sketch: one row holding every nonzero (one segment across all
    lanes and warps), a single nonzero, a ragged nnz, ell = 1, 16, 17 and 29 (column passes)."""
    rng = np.random.default_rng(12)
    dims = (50, 40, 30)
    n = 40 * 30
    heavy = np.array([np.full(n, 7), np.repeat(np.arange(40), 30), np.tile(np.arange(30), 40)])
    hv = rng.standard_normal(n)
    cases = [(heavy, hv), (np.array([[3], [2], [1]]), np.array([2.5])),
             (np.array([rng.integers(0, d_, 1037) for d_ in dims]), rng.standard_normal(1037))]
    for idx, vals in cases:
        key = np.ravel_multi_index(idx, dims)
        _, first = np.unique(key, return_index=True)
        idx, vals = idx[:, np.sort(first)], vals[np.sort(first)]
        for ell in (1, 16, 17, 29):
            for j in range(3):
                y = ctx.debug_coo_sketch(idx, vals, dims, j, ell, seed=1)
                yo = O.sp_sketch(idx, vals, dims, j, ell, seed=1)
                assert _col_err(y, yo) <= 1e-12, (idx.shape, ell, j)
    y = ctx.debug_coo_sketch(np.zeros((3, 0), np.int32), np.zeros(0), dims, 1, 5, seed=1)
    assert y.shape == (40, 5) and np.all(y == 0.0)


def test_superdiagonal_spec_example(ctx):
    """Superdiagonal 5^3 with (5,4,3,2,1), r=(2,2,2), p=2 -> the 4x4x4 leading sub-tensor."""
    x = superdiagonal([5, 4, 3, 2, 1])
    idx = np.array(np.nonzero(x))
    vals = x[tuple(idx)]
    g = _run(ctx, idx, vals, x.shape, (2, 2, 2), 2, seed=0)
    o = O.sp_sthosvd(idx, vals, x.shape, (2, 2, 2), 2, seed=0)
    _check(g, o, 2.0, 1e-10)
    assert g.ranks == (4, 4, 4)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_zipf_small_scale(ctx, dtype):
    """BASELINE configs[4] at 1/100 of the draws (Zipf(1.1) indices, 1+Poisson(2) counts)."""
    idx, vals = sparse_zipf(ndraws=500_000)
    vals = vals.astype(dtype)
    dims = (8000, 8000, 200000, 1200)
    g = _run(ctx, idx, vals, dims, (10, 10, 10, 10), 5, seed=0)
    o = O.sp_sthosvd(idx, vals, dims, (10, 10, 10, 10), 5, seed=0)
    # fp32 values -> fp32 normals on the GPU (fp64 products/sums), the oracle draws fp64
    # normals: Y agrees to ~1e-7 relative, so A to ~1e-5
    _check(g, o, 2.0, 1e-9 if dtype == np.float64 else 1e-4)
    assert g.order == (2, 0, 1, 3)


def test_host_input_order_and_eta(ctx):
    rng = np.random.default_rng(3)
    dims = (40, 30, 25)
    n = 3000
    idx = np.array([rng.integers(0, d_, n) for d_ in dims])
    key = np.ravel_multi_index(idx, dims)
    _, first = np.unique(key, return_index=True)
    idx = idx[:, np.sort(first)]
    vals = rng.random(idx.shape[1])
    for order, eta in [((1, 2, 0), 2.0), ((0, 1, 2), 1.1)]:
        g = _run(ctx, idx, vals, dims, (4, 3, 5), 3, seed=7, order=order, eta=eta, device=False)
        o = O.sp_sthosvd(idx, vals, dims, (4, 3, 5), 3, seed=7, order=order, eta=eta)
        _check(g, o, eta, 1e-9)
        assert g.swaps == tuple(o.swaps)


def test_srrqr_on_oracle_q(ctx):
    """N9 fed the oracle's Q reproduces the oracle's selection exactly (SURVEY c.4)."""
    rng = np.random.default_rng(11)
    for I, ell in [(200, 15), (5000, 15), (64, 8)]:
        q, _ = np.linalg.qr(rng.standard_normal((I, ell)) * np.exp(-0.02 * np.arange(I))[:, None])
        sel, a, swaps = ctx.debug_srrqr(q, 2.0)
        osel, oswaps = O.srrqr_select(q, 2.0)
        assert list(sel) == list(osel) and swaps == oswaps
        np.testing.assert_allclose(a, O.oblique_factor(q, osel), rtol=0, atol=1e-10)


def test_sparse_bit_reproducible_and_debug_checks(ctx):
    """The sparse sketch sums in fixed point (int64 words, sparse.cu): reruns are bit-identical
    (RTUCKER_DETERMINISTIC) although the reduction order of the CTAs, warps and
    atomics varies between runs; RTUCKER_DEBUG_CHECKS rejects an out-of-range index."""
    from paper_1905_07311_b200.rtucker import DEBUG_CHECKS, RTuckerError
    idx, vals = sparse_zipf(ndraws=300_000, seed=9)
    dims = (8000, 8000, 200000, 1200)
    a = _run(ctx, idx, vals, dims, (10, 10, 10, 10), 5, seed=3)
    b = _run(ctx, idx, vals, dims, (10, 10, 10, 10), 5, seed=3, flags=DEBUG_CHECKS)
    for fa, fb in zip(a.factors, b.factors):
        np.testing.assert_array_equal(fa, fb)
    np.testing.assert_array_equal(a.core_idx, b.core_idx)
    bad = idx.copy()
    bad[1, 7] = dims[1]
    with pytest.raises(RTuckerError) as e:
        _run(ctx, bad, vals, dims, (10, 10, 10, 10), 5, seed=3, flags=DEBUG_CHECKS)
    assert e.value.name == "EINVAL"


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_sp_hosvd(ctx, dtype):
    """SP-HOSVD (NEXT-2): every mode selected on X, core = X x_j P_j^T (one filter by all
    selections), against the oracle's sp_hosvd: selections, factors, core entries bit-exact."""
    from paper_1905_07311_b200.rtucker import SP_HOSVD
    idx, vals = sparse_zipf(dims=(800, 700, 20000, 120), ndraws=200_000, seed=6)
    vals = vals.astype(dtype)
    dims = (800, 700, 20000, 120)
    g = _run(ctx, idx, vals, dims, (6, 6, 6, 6), 4, seed=2, flags=SP_HOSVD)
    o = O.sp_hosvd(idx, vals, dims, (6, 6, 6, 6), 4, seed=2)
    for j in range(4):
        assert list(g.selections[j]) == list(o.selections[j]), j
        err = np.linalg.norm(g.factors[j] - o.factors[j]) / np.linalg.norm(o.factors[j])
        assert err <= (1e-9 if dtype == np.float64 else 1e-4), (j, err)
    assert g.nnz_history[:2] == tuple(o.nnz_history)
    gk, ok = np.lexsort(g.core_idx[::-1]), np.lexsort(o.core_idx[::-1])
    np.testing.assert_array_equal(g.core_idx[:, gk], o.core_idx[:, ok])
    np.testing.assert_array_equal(g.core_vals[gk], np.asarray(o.core_vals)[ok])


def test_sparse_invalid(ctx):
    from paper_1905_07311_b200.rtucker import RTuckerError
    idx = np.array([[0, 1, 2], [0, 1, 2], [0, 1, 2]])
    vals = np.array([1.0, 2.0, 3.0])
    for kw in (dict(ranks=(2, 1, 1), p=1), dict(eta=0.5)):   # r + p >= min(I, prod others)
        a = dict(ranks=(1, 1, 1), p=0, eta=2.0)
        a.update(kw)
        with pytest.raises(RTuckerError) as e:
            _run(ctx, idx, vals, (3, 3, 3), a["ranks"], a["p"], eta=a["eta"], device=False)
        assert e.value.name == "EINVAL", kw


@pytest.mark.slow
def test_zipf_full_scale_c5(ctx):
    """BASELINE configs[4] at full scale (50M draws -> ~40.7M nnz), against the oracle."""
    import time
    idx, vals = sparse_zipf()
    dims = (8000, 8000, 200000, 1200)
    t0 = time.perf_counter()
    g = _run(ctx, idx, vals, dims, (10, 10, 10, 10), 5, seed=0)
    t1 = time.perf_counter()
    o = O.sp_sthosvd(idx, vals, dims, (10, 10, 10, 10), 5, seed=0)
    t2 = time.perf_counter()
    print(f"C5 nnz={idx.shape[1]} gpu {t1 - t0:.3f}s (incl. H2D) oracle {t2 - t1:.1f}s nnz chain {g.nnz_history}")
    _check(g, o, 2.0, 1e-4)


def test_gamma_tensor_error_ordering(ctx):
    """NEXT-4 (Fig 6.4): on the synthetic sparse gamma-tensor (gamma = 10, 200^3,
    ~185k nonzeros) SP-STHOSVD at target rank r (rank r + p) is no better than R-STHOSVD and
    STHOSVD at rank r + p, and stays within a small factor of them ("slightly higher")."""
    import torch
    from paper_1905_07311_b200.rtucker import EXACT_SVD, RESULT_HOST
    from workloads import synthetic_sparse_gamma, to_first_mode_fastest
    x = synthetic_sparse_gamma(10.0, seed=1)
    idx = np.array(np.nonzero(x), dtype=np.int32)
    vals = x[tuple(idx)]
    r, ell = 10, 15
    sp = _run(ctx, idx, vals, x.shape, (r, r, r), 5, seed=0, order=(0, 1, 2))
    o = O.sp_sthosvd(idx, vals, x.shape, (r, r, r), 5, seed=0, order=(0, 1, 2))
    _check(sp, o, 2.0, 1e-9)
    core = np.zeros((ell,) * 3)
    core[tuple(sp.core_idx)] = sp.core_vals
    e_sp = np.linalg.norm(x - O.reconstruct(core, sp.factors)) / np.linalg.norm(x)
    xd = torch.as_tensor(to_first_mode_fastest(x), device="cuda")
    rs = ctx.sthosvd(xd, x.shape, (ell,) * 3, 5, 0, (0, 1, 2), RESULT_HOST).numpy()
    st = ctx.sthosvd(xd, x.shape, (ell,) * 3, 0, 0, (0, 1, 2), EXACT_SVD | RESULT_HOST).numpy()
    e_rs, e_st = O.rel_error(x, rs.core, rs.factors), O.rel_error(x, st.core, st.factors)
    assert e_st <= e_rs * (1 + 1e-9) and e_rs <= e_sp * (1 + 1e-9) and e_sp <= 10 * e_rs, (e_st, e_rs, e_sp)
