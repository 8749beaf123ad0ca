"""Seeded input generators (no method arithmetic; see workloads/__init__.py).

Tensor convention shared by every part of the repo:
a d-mode tensor X in R^{I_1 x ... x I_d} is stored *first-mode-fastest*:
element (i_1..i_d) (0-based) sits at i_1 + I_1*(i_2 + I_2*(i_3 + ...)).
In numpy we keep the logical shape (I_1, ..., I_d) and use Fortran order for the
memory image; `to_first_mode_fastest` / `from_first_mode_fastest` convert.

Recipes:
  hilbert        P:484-486 eq. (hilbert); `form="paper"` is 1/(i_1+..+i_d),
                 `form="shifted"` is BASELINE.json's 1/(i_1+..+i_d-(d-1)) (1-based i).
  tucker_c2      BASELINE.json configs[1]: core 40^3 with N(0,1)/(ijk), Haar factors,
                 additive Gaussian noise of std 1e-3*||X0||_F/sqrt(N) (DESIGN reading R10).
  odeco          BASELINE.json configs[3]: superdiagonal core sigma_i=i^-1.5 with Haar
                 factors plus relative noise (std = rel*||X0||_F/sqrt(N)).
  sparse_zipf    BASELINE.json configs[4]: i.i.d. bounded Zipf(s) indices per mode,
                 values 1+Poisson(2), duplicates merged by summation.
  synthetic_sparse_gamma  P:490-495 eq. (sparse): sum of sparse outer products.
"""
from __future__ import annotations

import math
import numpy as np

__all__ = [
    "hilbert", "tucker_c2", "odeco", "exact_rank", "superdiagonal", "sparse_zipf",
    "synthetic_sparse_gamma", "haar", "to_first_mode_fastest", "from_first_mode_fastest",
    "CONFIGS",
]


def to_first_mode_fastest(x: np.ndarray) -> np.ndarray:
    """1-D memory image of a logical-shape tensor, first mode fastest."""
    return np.ravel(x, order="F")


def from_first_mode_fastest(flat, dims) -> np.ndarray:
    """Logical-shape view of a first-mode-fastest memory image."""
    return np.reshape(np.asarray(flat), tuple(int(d) for d in dims), order="F")


def haar(rng: np.random.Generator, m: int, n: int) -> np.ndarray:
    """m x n matrix with orthonormal columns: Q of a Gaussian QR with sign(diag R)=+1
    (DESIGN reading R12: "Haar-random orthonormal")."""
    g = rng.standard_normal((m, n))
    q, r = np.linalg.qr(g)
    s = np.sign(np.diag(r))
    s[s == 0] = 1.0
    return q * s[None, :]


def hilbert(dims, form: str = "shifted", dtype=np.float64) -> np.ndarray:
    """Hilbert tensor.  form='paper': 1/(sum i_j); form='shifted':
    1/(sum i_j - (d-1)) as in BASELINE.json configs[0] and configs[2] (1-based i_j)."""
    dims = tuple(int(d) for d in dims)
    d = len(dims)
    off = 0 if form == "paper" else (d - 1)
    if form not in ("paper", "shifted"):
        raise ValueError(form)
    s = np.zeros(dims, dtype=np.float64)
    for j, n in enumerate(dims):
        shape = [1] * d
        shape[j] = n
        s = s + np.arange(1, n + 1, dtype=np.float64).reshape(shape)
    x = 1.0 / (s - off)
    return np.asfortranarray(x.astype(dtype))


def _mode_mult(x: np.ndarray, a: np.ndarray, n: int) -> np.ndarray:
    """Input-construction helper only (core x_n factor), via tensordot."""
    y = np.tensordot(a, x, axes=([1], [n]))  # new axis first
    return np.moveaxis(y, 0, n)


def tucker_c2(seed: int = 2, dims=(64, 64, 400), core=(40, 40, 40), noise: float = 1e-3,
              dtype=np.float32) -> np.ndarray:
    """BASELINE configs[1]: image-stack-shaped Tucker tensor + noise (DESIGN §3 C2)."""
    rng = np.random.default_rng(seed)
    c = core
    z = rng.standard_normal(int(np.prod(c))).reshape(c, order="F")
    w = np.ones(c)
    for j, n in enumerate(c):
        shape = [1] * len(c)
        shape[j] = n
        w = w * np.arange(1, n + 1, dtype=np.float64).reshape(shape)
    g = z / w
    x0 = g
    for j, (I, r) in enumerate(zip(dims, c)):
        x0 = _mode_mult(x0, haar(rng, I, r), j)
    n_el = x0.size
    std = noise * np.linalg.norm(x0.ravel()) / math.sqrt(n_el)
    e = rng.standard_normal(n_el).reshape(dims, order="F") * std
    return np.asfortranarray((x0 + e).astype(dtype))


def odeco(I: int = 800, R: int | None = None, seed: int = 4, noise: float = 1e-4,
          dtype=np.float32, device=None, third: int | None = None, slabs=None):
    """Orthogonally decomposable 3-mode tensor (BASELINE configs[3]):
    X0 = sum_{i<=R} sigma_i u_i o v_i o w_i, sigma_i = i^-1.5, Haar U, V (I x R) and W
    (third x R); X = X0 + E with E iid N(0, (noise*||X0||_F/sqrt(N))^2).

    device=None: numpy fp64 construction, returns a logical-shape numpy array.
    device='cuda'/'cpu' torch device: builds slab-wise with torch (fp32 matmuls, no TF32)
    and returns a flat first-mode-fastest torch tensor of `dtype` on that device; the
    noise of mode-3 slab c is drawn with a torch generator seeded by seed*1000003 + c (so
    bits differ from the numpy variant; parity tests feed the same bits to both
    implementations).  slabs=(lo, hi) builds only mode-3 slabs lo..hi-1 (a shard).
    """
    R = I if R is None else R
    K = I if third is None else third
    rng = np.random.default_rng(seed)
    U = haar(rng, I, R)
    V = haar(rng, I, R)
    W = haar(rng, K, R)
    sig = np.arange(1, R + 1, dtype=np.float64) ** -1.5
    if device is None:
        # X0[a,b,c] = sum_i U[a,i] sig_i V[b,i] W[c,i]
        x0 = np.einsum("ai,bi,ci->abc", U * sig[None, :], V, W, optimize=True)
        n_el = x0.size
        std = noise * math.sqrt(float(np.sum(sig ** 2))) / math.sqrt(n_el)
        e = rng.standard_normal(n_el).reshape(x0.shape, order="F") * std
        return np.asfortranarray((x0 + e).astype(dtype))
    import torch
    tdev = torch.device(device)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        Us = torch.as_tensor(U * sig[None, :], dtype=torch.float32, device=tdev)
        Vt = torch.as_tensor(V.T.copy(), dtype=torch.float32, device=tdev)
        Wt = torch.as_tensor(W, dtype=torch.float32, device=tdev)
        tdt = torch.float32 if dtype in (np.float32, "float32") else torch.float64
        lo, hi = (0, K) if slabs is None else (int(slabs[0]), int(slabs[1]))
        out = torch.empty(hi - lo, I, I, dtype=tdt, device=tdev)  # [c][b][a]: a fastest
        n_el = I * I * K
        std = noise * math.sqrt(float(np.sum(sig ** 2))) / math.sqrt(n_el)
        gen = torch.Generator(device=tdev)
        chunk = 64
        for c0 in range(lo, hi, chunk):
            c1 = min(hi, c0 + chunk)
            # slab[c] (a x b) = (U diag(sig*W[c,:])) V^T ; stored transposed so a is fastest
            scl = Wt[c0:c1]                                   # (cc, R)
            left = Us[None, :, :] * scl[:, None, :]           # (cc, I, R)
            slab = torch.matmul(left, Vt[None])               # (cc, I(a), I(b))
            slab = slab.transpose(1, 2)                       # (cc, b, a)
            for c in range(c0, c1):                           # per-slab noise stream: any slab
                gen.manual_seed(int(seed) * 1_000_003 + c)    # range reproduces the same bits
                nz = torch.randn((I, I), generator=gen, device=tdev, dtype=torch.float32)
                out[c - lo] = (slab[c - c0] + std * nz).to(tdt)
        return out.reshape(-1)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def exact_rank(dims, ranks, seed: int = 0, dtype=np.float64) -> np.ndarray:
    """Tensor of exact multilinear rank `ranks`: Gaussian core, Haar factors."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(tuple(ranks))
    for j, (I, r) in enumerate(zip(dims, ranks)):
        x = _mode_mult(x, haar(rng, I, r), j)
    return np.asfortranarray(x.astype(dtype))


def superdiagonal(values, d: int = 3, dtype=np.float64) -> np.ndarray:
    n = len(values)
    x = np.zeros((n,) * d, dtype=np.float64)
    for i, v in enumerate(values):
        x[(i,) * d] = v
    return np.asfortranarray(x.astype(dtype))


def _bounded_zipf(rng: np.random.Generator, n: int, size: int, s: float) -> np.ndarray:
    """0-based draws k-1 with P(k) proportional to k^-s on {1..n} (inverse CDF)."""
    w = np.arange(1, n + 1, dtype=np.float64) ** (-s)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    u = rng.random(size)
    return np.minimum(np.searchsorted(cdf, u, side="right"), n - 1).astype(np.int64)


def sparse_zipf(dims=(8000, 8000, 200000, 1200), ndraws: int = 50_000_000, s: float = 1.1,
                lam: float = 2.0, seed: int = 5):
    """BASELINE configs[4] (DESIGN §3 C5): returns (idx, vals) with idx an int32 array
    (d, nnz) (SoA, 0-based), vals float32; lexicographically sorted with mode 1 slowest,
    duplicate coordinates merged by summation (exact integer sums)."""
    rng = np.random.default_rng(seed)
    dims = tuple(int(x) for x in dims)
    key = np.zeros(ndraws, dtype=np.int64)
    for n in dims:
        key = key * n + _bounded_zipf(rng, n, ndraws, s)
    val = 1 + rng.poisson(lam, ndraws).astype(np.int64)
    ukey, inv = np.unique(key, return_inverse=True)
    sums = np.bincount(inv, weights=val, minlength=ukey.size)
    idx = np.empty((len(dims), ukey.size), dtype=np.int32)
    rem = ukey.copy()
    for j in range(len(dims) - 1, -1, -1):
        idx[j] = (rem % dims[j]).astype(np.int32)
        rem //= dims[j]
    return idx, sums.astype(np.float32)


def synthetic_sparse_gamma(gamma: float, n: int = 200, terms: int = 200, density: float = 0.05,
                           seed: int = 0):
    """P:490-495 eq. (sparse): X = sum_{i<=10} gamma/i^2 x_i o y_i o z_i +
    sum_{i=11}^{terms} 1/i^2 x_i o y_i o z_i with sprand-like sparse vectors (uniform
    values at `density` random positions).  Returns the dense logical tensor (fp64)."""
    rng = np.random.default_rng(seed)

    def sprand():
        v = np.zeros(n)
        k = max(1, int(round(density * n)))
        pos = rng.choice(n, size=k, replace=False)
        v[pos] = rng.random(k)
        return v

    x = np.zeros((n, n, n))
    for i in range(1, terms + 1):
        c = (gamma if i <= 10 else 1.0) / i ** 2
        a, b, z = sprand(), sprand(), sprand()
        x += c * np.einsum("a,b,c->abc", a, b, z)
    return np.asfortranarray(x)


# Named configurations (BASELINE.json configs).
CONFIGS = {
    "C1": dict(kind="hilbert", dims=(50, 50, 50), form="shifted", dtype="f64", ranks=(5, 5, 5), p=5,
               seed=0, order=(0, 1, 2)),
    "C2": dict(kind="tucker_c2", dims=(64, 64, 400), dtype="f32", ranks=(20, 20, 40), p=10, seed=0,
               data_seed=2, block=5, tol=1e-2),
    "C3": dict(kind="hilbert", dims=(25, 25, 25, 25, 25), form="shifted", dtype="f64",
               ranks=(5, 5, 5, 5, 5), p=5, seed=0, order=(0, 1, 2, 3, 4)),
    "C4": dict(kind="odeco", dims=(800, 800, 800), dtype="f32", ranks=(50, 50, 50), p=10, seed=0,
               data_seed=4, order=(0, 1, 2), block=10, tol=1e-3),
    "C5": dict(kind="sparse_zipf", dims=(8000, 8000, 200000, 1200), ndraws=50_000_000,
               ranks=(10, 10, 10, 10), p=5, seed=0, data_seed=5),
}
