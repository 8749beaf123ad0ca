"""Oracle Tucker algorithms (test infrastructure only; see oracle/__init__.py).

Each function follows one algorithm of PAPER.md step by step, in the paper's order:
  randsvd              Alg 1
  r_hosvd              Alg 2
  r_sthosvd            Alg 3
  adapt_range_finder   AdaptRangeFinder, DESIGN reading R8
  adaptive_r_hosvd     Alg 4
  adaptive_r_sthosvd   Alg 5
  sp_sthosvd           Alg 6
  sp_hosvd             §5.3 variant 1
  hosvd / sthosvd      deterministic comparators
  auto_order           processing-order heuristic
All arithmetic is fp64 (fp32 inputs are promoted exactly).  Modes are 0-based.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from .philox import omega_rows
from .tensor import unfold, fold, multi_mode_product, unfold_columns
from .srrqr import srrqr_select, oblique_factor


@dataclass
class TuckerResult:
    core: np.ndarray                 # logical shape (r_1..r_d)
    factors: list                    # A_j : I_j x r_j
    ranks: tuple
    ell: tuple
    order: tuple
    seed: int
    mode_residual_sq: dict = field(default_factory=dict)
    extra: dict = field(default_factory=dict)


@dataclass
class SpTuckerResult:
    core_idx: np.ndarray             # (d, nnz) 0-based in the core dims
    core_vals: np.ndarray
    core_dims: tuple
    factors: list                    # A_j : I_j x l_j (oblique)
    selections: list                 # S_j : sorted original mode-j indices (length l_j)
    order: tuple
    seed: int
    nnz_history: list = field(default_factory=list)
    swaps: list = field(default_factory=list)

    def dense_core(self) -> np.ndarray:
        g = np.zeros(self.core_dims, dtype=np.float64)
        g[tuple(self.core_idx)] = self.core_vals
        return g


def auto_order(dims) -> tuple:
    """Process the largest modes first; ties by ascending mode index."""
    return tuple(sorted(range(len(dims)), key=lambda j: (-int(dims[j]), j)))


def rank_caps(dims, j: int, r: int, p: int):
    """l_j = min(r_j + p, I_j, prod_{i!=j} I_i) evaluated on the given (current) dims
    (Alg 2/3 requirement P:160, clamped per DESIGN reading R5); r <= l."""
    others = int(np.prod([dims[i] for i in range(len(dims)) if i != j], dtype=np.int64))
    cap = min(int(dims[j]), others)
    ell = min(int(r) + int(p), cap)
    return ell, min(int(r), ell)


def canonical_signs(u: np.ndarray) -> np.ndarray:
    """DESIGN reading R4b: the thin SVD fixes singular vectors only up to sign; we
    fix it so that the entry of largest magnitude of each column of U_hat = Q U_B(:,1:r)
    is positive (first such row on ties).  Needed because in Alg 3 the next sketch
    G_(rho_j) Omega depends on the basis of the shrunk core.  Returns the +-1 vector."""
    idx = np.argmax(np.abs(u), axis=0)
    s = np.sign(u[idx, np.arange(u.shape[1])])
    s[s == 0] = 1.0
    return s


def randsvd(xm: np.ndarray, r: int, p: int, omega: np.ndarray, power: int = 0):
    """Alg 1 RandSVD(X, r, p, Omega).  Returns (U_hat, Sigma_hat, V_hat^T)
    plus the diagnostics (Q, B, U_B, all singular values of B).  Signs per reading R4b.
    power = q >= 1 adds q steps of randomized subspace iteration after line 2 (the paper's
    remedy for slow spectral decay, "see Halko et al."): Z = X^T Q,
    re-orthonormalised, then Y = X Z and Q = qr(Y) again, so range(Q) = range((X X^T)^q X Omega)."""
    y = xm @ omega                                        # line 1: Y = X Omega
    q, _ = np.linalg.qr(y, mode="reduced")                # line 2: Y = QR (Householder, LAPACK)
    for _ in range(power):                                # subspace iteration
        z, _ = np.linalg.qr(xm.T @ q, mode="reduced")     #   Z = orth(X^T Q)
        q, _ = np.linalg.qr(xm @ z, mode="reduced")       #   Q = orth(X Z)
    b = q.T @ xm                                          # line 3: B = Q^T X
    ub, s, vt = np.linalg.svd(b, full_matrices=False)     # line 4: thin SVD of B
    u = q @ ub[:, :r]                                     # line 5: U_hat = Q U_B(:, 1:r)
    sg = canonical_signs(u)
    u, vt = u * sg[None, :], vt[:r, :] * sg[:, None]      # (U, V) -> (U D, V D), D = diag(+-1)
    return u, s[:r], vt, dict(q=q, b=b, ub=ub, s_all=s)   # line 6


def _omega_for(seed, j, ncols, ell, k0=0):
    return omega_rows(seed, j, np.arange(ncols, dtype=np.int64), ell, k0=k0)


def r_hosvd(x: np.ndarray, ranks, p: int, seed: int = 0, power: int = 0) -> TuckerResult:
    """Alg 2: A_j from RandSVD of every X_(j) with independent Omega_j,
    then G = X x_1 A_1^T ... x_d A_d^T."""
    x = np.asarray(x, dtype=np.float64)
    d = x.ndim
    factors, rr, ells, svals = [None] * d, [0] * d, [0] * d, [None] * d
    for j in range(d):                                    # for j = 1:d
        ell, r = rank_caps(x.shape, j, ranks[j], p)
        xj = unfold(x, j)
        om = _omega_for(seed, j, xj.shape[1], ell)        # draw Omega_j
        u, _, _, info = randsvd(xj, r, ell - r, om, power) # RandSVD(X_(j), r_j, p, Omega_j)
        factors[j], rr[j], ells[j] = u, r, ell            # A_j <- U_hat
        svals[j] = info["s_all"]                          # (diagnostic: projector-test gate)
    core = multi_mode_product(x, factors, transpose=True) # G = X x_j A_j^T
    return TuckerResult(core, factors, tuple(rr), tuple(ells), tuple(range(d)), seed,
                        extra=dict(s_all=svals))


def r_sthosvd(x: np.ndarray, ranks, p: int, seed: int = 0, order=None, power: int = 0) -> TuckerResult:
    """Alg 3: sequential over rho; RandSVD of the current core unfolding,
    then G_(rho_j) <- Sigma_hat V_hat^T (line 6)."""
    x = np.asarray(x, dtype=np.float64)
    d = x.ndim
    order = auto_order(x.shape) if order is None else tuple(order)
    g = x                                                 # G = X
    factors, rr, ells, res, svals = [None] * d, [0] * d, [0] * d, {}, [None] * d
    for j in order:
        ell, r = rank_caps(g.shape, j, ranks[j], p)
        gj = unfold(g, j)
        om = _omega_for(seed, j, gj.shape[1], ell)        # Omega_{rho_j}, current dims
        u, s, vt, info = randsvd(gj, r, ell - r, om, power)
        svals[j] = info["s_all"]                          # (diagnostic: projector-test gate)
        factors[j], rr[j], ells[j] = u, r, ell            # A_{rho_j} <- U_hat
        g_new = fold(s[:, None] * vt, j, g.shape)         # G_(rho_j) <- Sigma_hat V_hat^T
        res[j] = float(np.sum(g * g) - np.sum(g_new * g_new))
        g = g_new
    return TuckerResult(g, factors, tuple(rr), tuple(ells), order, seed, res, dict(s_all=svals))


def adapt_range_finder(xm: np.ndarray, tau_sq: float, b: int, seed: int, mode: int,
                       norm_x: float, floor_rel: float = 1e-13, truncate: bool = True):
    """AdaptRangeFinder(X, eps, b) per DESIGN reading R8:
    blocks of b Gaussian columns (global column index k continues across blocks);
    W = X Omega_blk; W <- (I - QQ^T) W twice; Q_i = qr(W); B_i = Q_i^T X;
    E = ||X||^2 - sum ||B_i||^2 (exact identity); stop when E <= tau^2, when the
    column count reaches min(m, n), or when an appended block's projected norm is
    <= floor_rel*||X||_F (range exhausted; the block is discarded).
    truncate=True: SVD of B = [B_1; ...] and r = min{r : ||X||^2 - sum_{i<=r} s_i^2 <= tau^2},
    A = Q U_B(:,1:r), G_new = U_B(:,1:r)^T B.  truncate=False: A = Q, G_new = B.
    Returns (A, G_new_matrix, info)."""
    m, n = xm.shape
    cap = min(m, n)
    norm2 = float(np.sum(xm * xm))
    e = norm2
    qs, bs = [], []
    k = 0
    q = np.zeros((m, 0))
    e_hist, stop = [], "tol"
    while True:
        if e <= tau_sq:
            stop = "tol"
            break
        if k >= cap:
            stop = "cap"
            break
        bb = min(b, cap - k)
        om = omega_rows(seed, mode, np.arange(n, dtype=np.int64), bb, k0=k)
        w = xm @ om                                       # W = X Omega(:, k:k+b)
        w = w - q @ (q.T @ w)                             # project out current basis
        w = w - q @ (q.T @ w)                             # ... twice (re-orthogonalisation)
        if np.linalg.norm(w) <= floor_rel * norm_x:
            stop = "floor"
            break
        qi, _ = np.linalg.qr(w, mode="reduced")           # Q_i
        bi = qi.T @ xm                                    # B_i = Q_i^T X
        q = np.hstack([q, qi])
        bs.append(bi)
        e -= float(np.sum(bi * bi))                       # E -= ||B_i||^2
        e_hist.append(e)
        k += bb
    bmat = np.vstack(bs) if bs else np.zeros((0, n))
    info = dict(k=k, e=e, e_hist=e_hist, stop=stop, norm2=norm2)
    if not truncate or k == 0:
        return q, bmat, info
    ub, s, vt = np.linalg.svd(bmat, full_matrices=False)
    cums = np.cumsum(s ** 2)
    ok = np.nonzero(norm2 - cums <= tau_sq)[0]
    r = int(ok[0]) + 1 if ok.size else k
    info.update(r=r, s=s)
    a = q @ ub[:, :r]
    sg = canonical_signs(a)                               # reading R4b
    return a * sg[None, :], (s[:r, None] * vt[:r, :]) * sg[:, None], info


def _mode_tols(eps, d, mode_tol):
    if mode_tol is None:
        return [eps / math.sqrt(d)] * d                   # eps/sqrt(d) per mode
    mt = [float(t) for t in mode_tol]
    if abs(sum(t * t for t in mt) - eps * eps) > 1e-12 * max(1.0, eps * eps):
        raise ValueError("sum eps_j^2 must equal eps^2 (P:317)")
    return mt


def adaptive_r_sthosvd(x: np.ndarray, eps: float, b: int, seed: int = 0, order=None,
                       mode_tol=None, truncate: bool = True, floor_rel: float = 1e-13) -> TuckerResult:
    """Alg 5: A_{rho_j} = AdaptRangeFinder(G_(rho_j), eps_j, b),
    G_(rho_j) <- A^T G_(rho_j); threshold tau_j = eps_j ||X||_F (reading R8)."""
    x = np.asarray(x, dtype=np.float64)
    d = x.ndim
    order = auto_order(x.shape) if order is None else tuple(order)
    tols = _mode_tols(eps, d, mode_tol)
    nx = math.sqrt(float(np.sum(x * x)))
    g = x
    factors, rr, res, infos = [None] * d, [0] * d, {}, {}
    for j in order:
        gj = unfold(g, j)
        if tols[j] == 0.0:                                # eps_j = 0: mode not compressed
            factors[j], rr[j], res[j] = np.eye(gj.shape[0]), gj.shape[0], 0.0   # (R8)
            infos[j] = dict(k=gj.shape[0], stop="uncompressed")
            continue
        a, gnew, info = adapt_range_finder(gj, (tols[j] * nx) ** 2, b, seed, j, nx, floor_rel, truncate)
        factors[j], rr[j] = a, a.shape[1]
        g_new = fold(gnew, j, g.shape)
        res[j] = float(np.sum(g * g) - np.sum(g_new * g_new))
        infos[j] = info
        g = g_new
    return TuckerResult(g, factors, tuple(rr), tuple(i["k"] for i in (infos[j] for j in range(d))),
                        order, seed, res, dict(infos=infos))


def adaptive_r_hosvd(x: np.ndarray, eps: float, b: int, seed: int = 0, mode_tol=None,
                     truncate: bool = True, floor_rel: float = 1e-13) -> TuckerResult:
    """Alg 4: A_j = AdaptRangeFinder(X_(j), eps/sqrt(d), b) for each j,
    then G = X x_j A_j^T."""
    x = np.asarray(x, dtype=np.float64)
    d = x.ndim
    tols = _mode_tols(eps, d, mode_tol)
    nx = math.sqrt(float(np.sum(x * x)))
    factors, infos = [None] * d, {}
    for j in range(d):
        if tols[j] == 0.0:                                # eps_j = 0: mode not compressed
            factors[j], infos[j] = np.eye(x.shape[j]), dict(k=x.shape[j], stop="uncompressed")
            continue
        a, _, info = adapt_range_finder(unfold(x, j), (tols[j] * nx) ** 2, b, seed, j, nx,
                                        floor_rel, truncate)
        factors[j], infos[j] = a, info
    core = multi_mode_product(x, factors, transpose=True)
    return TuckerResult(core, factors, tuple(a.shape[1] for a in factors),
                        tuple(infos[j]["k"] for j in range(d)), tuple(range(d)), seed, {},
                        dict(infos=infos))


def hosvd(x: np.ndarray, ranks) -> TuckerResult:
    """Deterministic HOSVD: leading r_j left singular vectors of each X_(j)."""
    x = np.asarray(x, dtype=np.float64)
    factors = []
    for j in range(x.ndim):
        u, _, _ = np.linalg.svd(unfold(x, j), full_matrices=False)
        factors.append(u[:, :ranks[j]])
    core = multi_mode_product(x, factors, transpose=True)
    return TuckerResult(core, factors, tuple(ranks), tuple(ranks), tuple(range(x.ndim)), -1)


def sthosvd(x: np.ndarray, ranks, order=None) -> TuckerResult:
    """Deterministic STHOSVD: SVD of the current core unfolding, shrink."""
    x = np.asarray(x, dtype=np.float64)
    order = tuple(range(x.ndim)) if order is None else tuple(order)
    g, factors = x, [None] * x.ndim
    for j in order:
        u, s, vt = np.linalg.svd(unfold(g, j), full_matrices=False)
        r = ranks[j]
        sg = canonical_signs(u[:, :r])
        factors[j] = u[:, :r] * sg[None, :]
        g = fold((s[:r, None] * vt[:r, :]) * sg[:, None], j, g.shape)
    return TuckerResult(g, factors, tuple(ranks), tuple(ranks), order, -1)


def sp_sketch(idx, vals, cur_dims, j, ell, seed):
    """Alg 6 line 4: Y = G_(j) Omega_j for a COO tensor, with only the Omega rows of
    the occupied columns of the unfolding drawn."""
    cols = unfold_columns(cur_dims, j, idx)
    ucols, inv = np.unique(cols, return_inverse=True)
    om = omega_rows(seed, j, ucols, ell)                  # Omega rows of occupied columns
    gj = sp.coo_matrix((np.asarray(vals).astype(np.float64), (np.asarray(idx[j]).astype(np.int64), inv)),
                       shape=(int(cur_dims[j]), ucols.size)).tocsr()
    return np.asarray(gj @ om)


def _sp_mode(idx, vals, cur_dims, j, ell, seed, eta):
    """One pass of Alg 6 lines 3-7 on the current sparse core (COO)."""
    y = sp_sketch(idx, vals, cur_dims, j, ell, seed)      # line 4: Y = G_(j) Omega
    q, _ = np.linalg.qr(y, mode="reduced")                # line 5: thin QR
    sel, swaps = srrqr_select(q, eta)                     # line 6: strong RRQR on Q^T
    a = oblique_factor(q, sel)                            # line 7: A = Q (P^T Q)^{-1}
    return q, sel, swaps, a


def _check_sp_caps(dims, j, r, p):
    others = int(np.prod([dims[i] for i in range(len(dims)) if i != j], dtype=np.int64))
    ell = int(r) + int(p)
    if not ell < min(int(dims[j]), others):              # strict inequality
        raise ValueError("SP-STHOSVD needs r_j + p < min(I_j, prod_{i!=j} I_i)")
    return ell


def sp_sthosvd(idx, vals, dims, ranks, p: int, seed: int = 0, order=None, eta: float = 2.0) -> SpTuckerResult:
    """Alg 6 SP-STHOSVD on a COO tensor (idx: d x nnz 0-based, vals).
    Line 8, G_(rho_j) <- P^T G_(rho_j): keep the nonzeros whose mode-j index is
    selected and renumber it to its position in the sorted selection."""
    idx = np.array(idx, dtype=np.int64, copy=True)
    vals = np.asarray(vals).copy()
    dims = tuple(int(x) for x in dims)
    d = len(dims)
    order = auto_order(dims) if order is None else tuple(order)
    cur = list(dims)
    factors, sels, hist, swaps = [None] * d, [None] * d, [idx.shape[1]], [0] * d
    for j in order:
        ell = _check_sp_caps(cur, j, ranks[j], p)
        _, sel, sw, a = _sp_mode(idx, vals, cur, j, ell, seed, eta)
        sel = np.asarray(sel, dtype=np.int64)
        keep = np.isin(idx[j], sel)                       # P^T G: rows in the selection
        idx = idx[:, keep]
        vals = vals[keep]
        idx[j] = np.searchsorted(sel, idx[j])             # renumber to 0..l-1
        cur[j] = ell
        factors[j], sels[j], swaps[j] = a, sel, sw
        hist.append(idx.shape[1])
    return SpTuckerResult(idx, vals, tuple(cur), factors, sels, order, seed, hist, swaps)


def sp_hosvd(idx, vals, dims, ranks, p: int, seed: int = 0, eta: float = 2.0) -> SpTuckerResult:
    """SP-HOSVD (§5.3 variant 1): every mode handled independently on X;
    core = X x_j P_j^T for all j.  (DESIGN: NEXT-2 item; oracle side only.)"""
    idx = np.array(idx, dtype=np.int64, copy=True)
    vals = np.asarray(vals).copy()
    dims = tuple(int(x) for x in dims)
    d = len(dims)
    factors, sels, swaps = [None] * d, [None] * d, [0] * d
    for j in range(d):
        ell = _check_sp_caps(dims, j, ranks[j], p)
        _, sel, sw, a = _sp_mode(idx, vals, dims, j, ell, seed, eta)
        factors[j], sels[j], swaps[j] = a, np.asarray(sel, dtype=np.int64), sw
    keep = np.ones(idx.shape[1], dtype=bool)
    for j in range(d):
        keep &= np.isin(idx[j], sels[j])
    cidx = idx[:, keep]
    for j in range(d):
        cidx[j] = np.searchsorted(sels[j], cidx[j])
    return SpTuckerResult(cidx, vals[keep], tuple(len(s) for s in sels), factors, sels,
                          tuple(range(d)), seed, [idx.shape[1], int(keep.sum())], swaps)
