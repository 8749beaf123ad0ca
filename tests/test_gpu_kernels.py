"""GPU parity of the individual kernels through the C ABI against the CPU oracle
(or, for the QR / eig / srrqr steps, against LAPACK on the same fp64 inputs)."""
import numpy as np
import pytest

import oracle as O
from oracle.philox import philox4x32_10
from workloads import hilbert, tucker_c2, to_first_mode_fastest

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


def test_philox_words_bit_exact(ctx):
    rng = np.random.default_rng(0)
    n = 100000
    ctr = rng.integers(0, 2 ** 32, size=(n, 4), dtype=np.uint64).astype(np.uint32)
    for key in [(0, 0), (0xFFFFFFFF, 0xFFFFFFFF), (0xA4093822, 0x299F31D0)]:
        got = ctx.debug_philox(ctr, *key)
        ref = np.stack(philox4x32_10([ctr[:, i].astype(np.uint64) for i in range(4)],
                                     [np.uint64(key[0]), np.uint64(key[1])]), axis=1)
        np.testing.assert_array_equal(got, ref)


@pytest.mark.parametrize("k0,ell", [(0, 64), (5, 7), (3, 1), (60, 10)])
def test_omega_fp64(ctx, k0, ell):
    cols = np.concatenate([np.arange(20000), np.array([2 ** 32 + 5, 2 ** 40 + 123])]).astype(np.int64)
    got = ctx.debug_omega(cols, ell, seed=0x1234567890ABCDEF, mode=3, k0=k0, dtype="f64")
    ref = O.omega_rows(0x1234567890ABCDEF, 3, cols, ell, k0=k0)
    np.testing.assert_allclose(got, ref, rtol=1e-13, atol=1e-13)


def test_omega_fp32(ctx):
    cols = np.arange(1_000_000, dtype=np.int64)
    got = ctx.debug_omega(cols, 4, seed=7, mode=1, dtype="f32").astype(np.float64)
    ref = O.omega_rows(7, 1, cols, 4)
    d = got - ref
    assert np.sqrt(np.mean(d * d)) <= 3e-7
    assert np.max(np.abs(d)) <= 2e-5


def _sketch_ref(x, mode, ell, seed, k0=0):
    xm = O.unfold(np.asarray(x, dtype=np.float64), mode)
    return xm @ O.omega_rows(seed, mode, np.arange(xm.shape[1]), ell, k0=k0)


def _check_elementwise(got, x, mode, ell, seed, k0, rel):
    """Element-by-element check of a sketch against the oracle product: every entry within
    rel * (|X_(n)| |Omega|)_ik, the scale of the rounding-error bound of that entry's dot
    product (a wrong or missing element cannot hide in a Frobenius norm)."""
    xm = O.unfold(np.asarray(x, dtype=np.float64), mode)
    om = O.omega_rows(seed, mode, np.arange(xm.shape[1]), ell, k0=k0)
    ref = xm @ om
    scale = np.abs(xm) @ np.abs(om)
    bad = np.abs(got - ref) > rel * scale + 1e-300
    assert not bad.any(), (int(bad.sum()), np.argwhere(bad)[:5])


CASES = [
    ("hilbert50", lambda: hilbert((50, 50, 50), "shifted"), [10, 64, 70]),
    ("ragged", lambda: np.asfortranarray(np.random.default_rng(1).standard_normal((37, 41, 29))), [13, 33]),
    ("hilbert25^5", lambda: hilbert((25,) * 5, "shifted"), [10]),
    ("c2_f32", lambda: tucker_c2(), [30, 50]),
    ("hilbert25^5_f32", lambda: hilbert((25,) * 5, "shifted", dtype=np.float32), [10]),
]


@pytest.mark.parametrize("name,make,ells", CASES, ids=[c[0] for c in CASES])
def test_sketch_all_modes(ctx, name, make, ells):
    x = make()
    tol = 1e-13 if x.dtype == np.float64 else 2e-6
    for mode in range(x.ndim):
        for ell in ells:
            ell = min(ell, x.shape[mode] * 4)
            got = ctx.debug_sketch(x, x.shape, mode, ell, seed=11)
            ref = _sketch_ref(x, mode, ell, 11)
            err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
            assert err <= tol, (name, mode, ell, err)
            _check_elementwise(got, x, mode, ell, 11, 0, 1e-14 if x.dtype == np.float64 else 1e-6)


@pytest.mark.parametrize("shape", [(1, 5, 1), (2, 7, 3), (3, 130, 5), (16, 129, 2), (17, 257, 33), (5, 4, 1500),
                                   (260, 3, 2), (1, 1, 40)])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_sketch_fp64_edge_shapes(ctx, shape, dtype):
    """The double-buffered fp64 tensor-core sketch at its corner cases: fewer columns than one
    16-column chunk, exactly one / two chunks per split, a contiguous lower extent L below the
    chunk (the incremental (l, r) split wraps several times per chunk), ragged 128-row tiles,
    and both input types (fp32 data under the FP64 policy takes the same kernel).  Tolerance
    2e-13 (|X||Omega|)_ik: with one or a few terms per entry nothing averages the generator's
    own accuracy (fp64 normals within 1e-13 of the oracle's, test_omega_*; seen: 7e-14 on the
    single-column case)."""
    from paper_1905_07311_b200.rtucker import ACCUM_FP64
    rng = np.random.default_rng(sum(shape))
    x = np.asfortranarray(rng.standard_normal(shape).astype(dtype))
    for mode in range(3):
        for ell in (1, 9, 64):
            got = ctx.debug_sketch(x, x.shape, mode, ell, seed=21, flags=ACCUM_FP64)
            _check_elementwise(got, x, mode, ell, 21, 0, 2e-13)


def test_sketch_fp32_with_fp64_policy(ctx):
    from paper_1905_07311_b200.rtucker import ACCUM_FP64
    x = hilbert((25,) * 5, "shifted", dtype=np.float32)
    got = ctx.debug_sketch(x, x.shape, 2, 10, seed=3, flags=ACCUM_FP64)
    ref = _sketch_ref(x, 2, 10, 3)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-13


def test_sketch_block_offset(ctx):
    """Adaptive blocks continue the global column index k (reading R3)."""
    x = np.asfortranarray(np.random.default_rng(2).standard_normal((30, 20, 10)))
    got = ctx.debug_sketch(x, x.shape, 1, 6, seed=9, k0=13)
    ref = _sketch_ref(x, 1, 6, 9, k0=13)
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)
    _check_elementwise(got, x, 1, 6, 9, 13, 1e-14)


@pytest.mark.parametrize("m,n", [(800, 60), (50, 10), (25, 10), (1000, 1), (64, 64), (4096, 15), (20003, 15),
                                 (5001, 40), (3000, 30)])
def test_householder_qr(ctx, m, n):
    rng = np.random.default_rng(m + n)
    y = rng.standard_normal((m, n)) * np.logspace(0, -9, n)[None, :]
    q = ctx.debug_qr(y)
    assert np.linalg.norm(q.T @ q - np.eye(n)) <= 1e-13 * n
    qr, _ = np.linalg.qr(y)
    assert np.linalg.norm(qr - q @ (q.T @ qr), 2) <= 1e-10  # ||(I - Q Q^T) Q_ref||_2 = sin of the largest angle
    # rank-deficient sketch: exact rank 3 with 10 columns
    if m >= 10 and n >= 10:
        y = rng.standard_normal((m, 3)) @ rng.standard_normal((3, 10))
        q = ctx.debug_qr(y)
        assert np.linalg.norm(q.T @ q - np.eye(10)) <= 1e-12
        assert np.linalg.norm(y - q @ (q.T @ y)) <= 1e-12 * np.linalg.norm(y)


@pytest.mark.parametrize("n", [1, 2, 7, 10, 30, 60, 64, 65, 150])
def test_sym_eig(ctx, n):
    """Unpreconditioned one-sided Jacobi on the Gram against LAPACK eigh.  n <= ~110: one CTA
    with the matrices in shared memory; n = 150: the grid-synchronised variant
    (jacobi_grid_kernel, one warp per pair) used by the adaptive variant's large ranks."""
    rng = np.random.default_rng(n)
    u, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.sort(np.logspace(0, -12, n) * (1 + 0.1 * rng.random(n)))[::-1]
    a = (u * lam) @ u.T
    a = (a + a.T) / 2
    w, v = ctx.debug_eig(a)
    print(f"n={n} jacobi sweeps={ctx.last_sweeps}")
    assert ctx.last_sweeps < 40
    wr = np.sort(np.linalg.eigvalsh(a))[::-1]
    np.testing.assert_allclose(w, wr, rtol=0, atol=1e-15 * n)
    assert np.all(np.diff(w) <= 0)
    assert np.linalg.norm(v.T @ v - np.eye(n)) <= 1e-13 * n
    assert np.linalg.norm(a @ v - v * w[None, :]) <= 1e-14 * n


@pytest.mark.parametrize("shape,ell,k0", [((800, 800, 40), 60, 0), ((800, 300, 7), 10, 0), ((96, 1001, 3), 64, 0),
                                          ((800, 200, 11), 5, 10), ((128, 64, 8), 33, 4), ((100, 300, 5), 20, 0),
                                          ((36, 500, 2), 7, 3), ((900, 64, 3), 60, 0)])
def test_sketch_tc_mode1(ctx, shape, ell, k0):
    """Mode-1 fp32 sketch (the tcgen05 3xTF32 path: L == 1, I % 4 == 0) against the fp64
    oracle product on the same fp32 bits, incl. ragged column counts and block offsets k0.
    Routes: MN-major A with one 3-D TMA per stage (I % 32 == 0: 800, 96, 128), MN-major A
    with 32-row 2-D boxes (100, 36: the last box ragged), the transposing K-major kernel
    (I = 900: more than 7 M-tiles).
    Tolerance: fp32 accumulation in TMEM over a CTA's column range (a few hundred to a few
    thousand terms, relative error ~ sqrt(K) u32) -> 1e-5 relative."""
    rng = np.random.default_rng(sum(shape) + ell)
    x = np.asfortranarray(rng.standard_normal(shape).astype(np.float32))
    got = ctx.debug_sketch(x, x.shape, 0, ell, seed=5, k0=k0)
    ref = _sketch_ref(x, 0, ell, 5, k0=k0)
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    colerr = np.max(np.linalg.norm(got - ref, axis=0) / np.linalg.norm(ref, axis=0))
    assert err <= 1e-5 and colerr <= 2e-5, (err, colerr)
    _check_elementwise(got, x, 0, ell, 5, k0, 1e-6)


@pytest.mark.parametrize("shape,mode,ell,k0", [((80, 800, 30), 1, 60, 0), ((16, 96, 9), 1, 33, 4), ((40, 24, 200), 2, 20, 0),
                                               ((8, 8, 8, 296), 3, 64, 0), ((24, 56, 17), 1, 17, 10)])
def test_sketch_tc_kmajor(ctx, shape, mode, ell, k0):
    """fp32 sketch of a mode with L > 1 (tcgen05 3xTF32, K-major 5-D TMA tiles: L % 8 == 0,
    I % 8 == 0) against the fp64 oracle product on the same fp32 bits; same tolerance as the
    mode-1 kernel (fp32 accumulation over a CTA's column range)."""
    rng = np.random.default_rng(sum(shape) + ell + mode)
    x = np.asfortranarray(rng.standard_normal(shape).astype(np.float32))
    got = ctx.debug_sketch(x, x.shape, mode, ell, seed=7, k0=k0)
    ref = _sketch_ref(x, mode, ell, 7, k0=k0)
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    colerr = np.max(np.linalg.norm(got - ref, axis=0) / np.linalg.norm(ref, axis=0))
    assert err <= 1e-5 and colerr <= 2e-5, (err, colerr)
    _check_elementwise(got, x, mode, ell, 7, k0, 1e-6)


@pytest.mark.parametrize("shape,J,graded", [((800, 300, 5), 60, False), ((96, 1001, 3), 17, True), ((64, 50, 7), 64, True),
                                          ((800, 129, 1), 60, False), ((4, 300, 2), 1, False)])
def test_ozaki_bpass(ctx, shape, J, graded):
    """Mode-1 HYBRID B-pass on the int8 tensor cores (Ozaki-style exact slice products, DESIGN
    R18) against the fp64 product on the same fp32 bits: B and its Gram to 2e-9 relative
    (slices keep 35 bits of every column-scaled operand).  `graded` scales the columns of X
    over 12 decades and zeroes one, exercising the per-column exponents."""
    rng = np.random.default_rng(sum(shape) + J)
    x = rng.standard_normal(shape)
    if graded:
        x *= np.logspace(0, -12, shape[1])[None, :, None]
        x[:, 1, 0] = 0.0
    x = np.asfortranarray(x.astype(np.float32))
    q, _ = np.linalg.qr(rng.standard_normal((shape[0], J)))
    b, g = ctx.debug_ttm(x, x.shape, 0, q)
    x1 = O.unfold(np.asarray(x, dtype=np.float64), 0)
    bref = q.T @ x1
    bgot = b.cpu().numpy().reshape((J, -1), order="F")
    assert np.linalg.norm(bgot - bref) <= 2e-9 * np.linalg.norm(bref)
    # per column, against the column's natural scale ||q_j|| ||x_p|| (the slices are scaled per column)
    scale = np.linalg.norm(q, axis=0)[:, None] * np.linalg.norm(x1, axis=0)[None, :]
    assert np.all(np.abs(bgot - bref) <= 2e-9 * scale + 1e-300)
    gref = bref @ bref.T
    assert np.linalg.norm(g - gref) <= 2e-9 * np.linalg.norm(gref)


@pytest.mark.gpu
@pytest.mark.parametrize("shape,mode,J,graded", [((96, 64, 30), 1, 60, False), ((200, 24, 8), 1, 13, True),
                                                 ((20, 64, 36), 2, 36, True), ((8, 16, 12), 2, 5, False)])
def test_ozaki_bpass_strided(ctx, shape, mode, J, graded):
    """Gram-only HYBRID B-pass of a strided mode (L > 1: the Ozaki kernel's 3-D-box variant,
    R-HOSVD modes n > 1) against the fp64 Gram of Q^T X_(n) on the same fp32 bits, 2e-9
    relative (DESIGN R18).  Ragged 128-column tiles (L = 200, 96, 1280, 128) and, with `graded`,
    per-column scales over 12 decades with one zero column."""
    rng = np.random.default_rng(sum(shape) + J + mode)
    x = rng.standard_normal(shape)
    if graded:  # scale the unfolding columns (indices other than `mode`)
        other = [k for k in range(3) if k != mode]
        x *= np.logspace(0, -12, shape[other[0]]).reshape([-1 if k == other[0] else 1 for k in range(3)])
        idx = [0, 0, 0]
        idx[mode] = slice(None)
        x[tuple(idx)] = 0.0
    x = np.asfortranarray(x.astype(np.float32))
    q, _ = np.linalg.qr(rng.standard_normal((shape[mode], J)))
    _, g = ctx.debug_ttm(x, x.shape, mode, q, want_out=False)
    bref = q.T @ O.unfold(np.asarray(x, dtype=np.float64), mode)
    gref = bref @ bref.T
    g = g.cpu().numpy().reshape(J, J) if hasattr(g, "cpu") else np.asarray(g).reshape(J, J)
    assert np.linalg.norm(g - gref) <= 2e-9 * np.linalg.norm(gref)


@pytest.mark.parametrize("kind,n,k", [("c4like", 60, 50), ("hilbert", 60, 5), ("rankdef", 40, 7), ("small", 10, 5),
                                      ("odd", 33, 20), ("one", 1, 1), ("two", 2, 1), ("c4like", 65, 50),
                                      ("hilbert", 65, 5), ("rankdef", 150, 9), ("c4like", 300, 250),
                                      ("c4like", 760, 730)])
def test_gram_eig(ctx, kind, n, k):
    """Hot-path eigensolvers against LAPACK eigh: n <= 64 the register-resident preconditioned
    Jacobi (gram_eig_kernel), n > 64 - the adaptive truncation sizes - the grid tridiagonal
    solver (trideig.cu: Householder tridiagonalisation, multisection, twisted eigenvectors,
    orthonormal completion of degenerate clusters, Newton-Schulz polish): eigenvalues to
    ~eps lambda_1, the leading-k projector to the accuracy the gap allows, and the WHOLE basis
    orthonormal, including the numerically degenerate clusters of rank-deficient / Hilbert
    Grams."""
    rng = np.random.default_rng(n + k)
    if kind == "c4like" or kind in ("small", "odd", "one", "two"):
        u, _ = np.linalg.qr(rng.standard_normal((n, n)))
        lam = np.arange(1, n + 1) ** -3.0
        a = (u * lam) @ u.T
    elif kind == "hilbert":
        a = 1.0 / (np.arange(n)[:, None] + np.arange(n)[None, :] + 1.0)
    else:
        b = rng.standard_normal((n, k)) @ rng.standard_normal((k, 300))
        a = b @ b.T
    a = (a + a.T) / 2
    w, v = ctx.debug_gram_eig(a)
    # fp64 Jacobi sweeps, or (32 < n <= 64, the fp32-data selection) fp32 sweeps + 1000 x steps
    assert ctx.last_sweeps % 1000 <= 20 and ctx.last_sweeps // 1000 <= 4
    we, ve = np.linalg.eigh(a)
    o = np.argsort(-we)
    we, ve = we[o], ve[:, o]
    np.testing.assert_allclose(w[:k], we[:k], rtol=1e-11, atol=1e-14 * we[0])
    gap = we[k - 1] - (we[k] if k < n else 0.0)
    p1, p2 = v[:, :k] @ v[:, :k].T, ve[:, :k] @ ve[:, :k].T
    assert np.linalg.norm(p1 - p2, 2) <= 1e-13 * we[0] / gap + 1e-12
    if n > 64:  # tridiagonal solver: the whole basis (degenerate clusters completed)
        assert np.linalg.norm(v.T @ v - np.eye(n)) <= 1e-13 * n
        assert np.linalg.norm(a @ v - v * w[None, :]) <= 1e-14 * n * we[0]
    else:       # Jacobi on the pivoted Cholesky factor: the leading k (zero columns past the rank)
        assert np.linalg.norm(v[:, :k].T @ v[:, :k] - np.eye(k)) <= 1e-12


def _mixed_case(kind, n, rng):
    u, _ = np.linalg.qr(rng.standard_normal((n, n)))
    if kind == "c4like":      # C4's mode Grams: lambda_i ~ i^-3 (odeco sigma_i = i^-1.5)
        lam = np.arange(1, n + 1) ** -3.0
    elif kind == "graded":    # ten decades
        lam = np.logspace(0, -10, n)
    elif kind == "pairs":     # exactly repeated eigenvalues (any basis of a pair is correct)
        lam = np.repeat(np.arange(1, n // 2 + 1) ** -2.0, 2)[:n]
        lam = np.concatenate([lam, np.full(n - len(lam), lam[-1])])
    elif kind == "tie_at_r":  # eigenvalues r-1 and r (0-based, r = n - 10) 1e-9 apart: the split
        lam = np.arange(1, n + 1) ** -1.0  # is unresolved after refinement -> fp64 Jacobi fallback
        lam[n - 10] = lam[n - 11] * (1 - 1e-9)
    elif kind == "tie_in":    # eigenvalues 4 and 5 1e-9 apart, both kept: any basis of the pair
        lam = np.arange(1, n + 1) ** -1.0
        lam[5] = lam[4] * (1 - 1e-9)
    else:                     # rank-deficient: the fp64 Jacobi fallback
        lam = np.concatenate([np.arange(1, n - 4) ** -1.0, np.zeros(5)])
    return (u * lam) @ u.T


@pytest.mark.parametrize("kind", ["c4like", "graded", "pairs", "tie_at_r", "tie_in", "rankdef"])
@pytest.mark.parametrize("n", [33, 48, 60, 64])
def test_gram_eig_mixed(ctx, kind, n):
    """The fp32-data eigensolver (fp32 one-sided Jacobi on the pivoted Cholesky factor
    + fp64 Ogita-Aishima refinement on the tensor cores, 32 < n <= 64) against LAPACK eigh:
    eigenvalues to ~eps lambda_1, the whole basis orthonormal to 1e-13, residual
    ||A V - V diag(w)|| <= 1e-13 n lambda_1, and the leading-r projector (r = n - 10, the
    truncation rank it is called with) to the absolute-accuracy class eps lambda_1 / gap; a
    rank-deficient Gram takes the fp64 Jacobi fallback."""
    rng = np.random.default_rng(1000 + n)
    a = _mixed_case(kind, n, rng)
    a = (a + a.T) / 2
    r = n - 10
    w, v = ctx.debug_gram_eig_ex(a, rel_acc=False, r_need=r)
    we, ve = np.linalg.eigh(a)
    o = np.argsort(-we)
    we, ve = we[o], ve[:, o]
    # (a numerically degenerate pair inside the kept set is mixed: its Rayleigh quotients and
    # residual at the pair's gap)
    np.testing.assert_allclose(w, we, rtol=0, atol=1e-9 * we[0] if kind == "tie_in" else 1e-13 * n * we[0])
    gap = we[r - 1] - we[r]
    p1, p2 = v[:, :r] @ v[:, :r].T, ve[:, :r] @ ve[:, :r].T
    assert np.linalg.norm(p1 - p2, 2) <= 1e-14 * n * we[0] / gap + 1e-12
    if kind in ("rankdef", "tie_at_r"):  # the fp64 Jacobi fallback ran (fp64 sweep count)
        assert ctx.last_sweeps < 1000, ctx.last_sweeps
        assert np.linalg.norm(v[:, :r].T @ v[:, :r] - np.eye(r)) <= 1e-12
    else:  # the mixed path: fp32 sweeps + 1000 x refinement steps (<= 4)
        assert 1000 <= ctx.last_sweeps < 5000, ctx.last_sweeps
        assert np.linalg.norm(v.T @ v - np.eye(n)) <= 1e-12
        res_tol = 1e-9 * we[0] if kind == "tie_in" else 1e-13 * n * we[0]
        assert np.linalg.norm(a @ v - v * w[None, :]) <= res_tol


@pytest.mark.parametrize("m,n,k,ta,tb", [(730, 900, 760, True, False), (70, 40, 65, False, False),
                                         (300, 257, 1000, False, True), (129, 300, 77, True, True),
                                         (760, 760, 4000, False, True)])
def test_gemm_f64(ctx, m, n, k, ta, tb):
    """The library's fp64 tensor-core GEMM (both the simple and the pipelined cp.async kernel,
    every transposition, ragged edges) against numpy: fp64 accuracy (1e-14 relative)."""
    rng = np.random.default_rng(m + n + k)
    a = rng.standard_normal((k, m) if ta else (m, k))
    b = rng.standard_normal((n, k) if tb else (k, n))
    c = ctx.debug_gemm(a, b, ta, tb)
    ref = (a.T if ta else a) @ (b.T if tb else b)
    assert np.max(np.abs(c - ref)) <= 1e-14 * np.sqrt(k) * np.max(np.abs(a)) * np.max(np.abs(b)) * 10


@pytest.mark.parametrize("L,K,R", [(1, 760, 20000), (730, 120, 30), (7, 65, 50), (1, 30, 1000), (50, 700, 40)])
def test_gram_f64(ctx, L, K, R):
    """Gram B_(n) B_(n)^T of a (L, K, R) fp64 tensor (adaptive truncation), gather layout for
    L > 1, split K with a fixed-order reduction: fp64 accuracy and exact symmetry."""
    rng = np.random.default_rng(L + K + R)
    b = rng.standard_normal(L * K * R)
    c = ctx.debug_gram(b, L, K, R)
    x = O.unfold(b.reshape((L, K, R), order="F"), 1)
    ref = x @ x.T
    assert np.max(np.abs(c - ref)) <= 1e-13 * np.max(np.abs(ref))
    np.testing.assert_array_equal(c, c.T)
