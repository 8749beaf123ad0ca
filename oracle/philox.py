"""Oracle Gaussian test matrices Omega (test infrastructure only; see oracle/__init__.py).

PAPER.md fixes only the distribution: "the entries Omega_ij are independent and
identically distributed N(0,1)" (Alg 1) and that Omega "need not be stored
explicitly. Its entries may be generated on-the-fly".  The concrete generator
is DESIGN.md reading R3 (= SURVEY §8(c) item 3), binding for both implementations:

  Philox4x32-10 (Salmon et al. 2011; multipliers 0xD2511F53, 0xCD9E8D57; Weyl key
  increments 0x9E3779B9, 0xBB67AE85; 10 rounds),
  key     = (seed & 0xffffffff, seed >> 32)
  counter = (k >> 2, n | (v << 8), c & 0xffffffff, c >> 32)
     n = 0-based mode, v = draw type (0 = range finder), c = 0-based unfolding column
     (over the current dims), k = 0-based sketch column (global across adaptive blocks)
  u_i     = (w_i + 0.5) * 2^-32  in (0, 1)
  Box-Muller: k&3 = 0: sqrt(-2 ln u0) cos(2 pi u1);  1: sqrt(-2 ln u0) sin(2 pi u1)
              k&3 = 2: sqrt(-2 ln u2) cos(2 pi u3);  3: sqrt(-2 ln u2) sin(2 pi u3)

Written with numpy uint64 arithmetic, fp64 Box-Muller.  Pinned by the Random123
known-answer vectors and libcurand's host Philox generator (tests/test_oracle_philox.py).
"""
from __future__ import annotations

import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = np.uint64(0x9E3779B9)
W1 = np.uint64(0xBB67AE85)
MASK = np.uint64(0xFFFFFFFF)
S32 = np.uint64(32)


def philox4x32_10(ctr, key):
    """Philox4x32 with 10 rounds.  ctr: 4 uint arrays (broadcastable), key: 2 uint
    arrays.  Returns 4 uint32 arrays.  One round (Salmon et al.):
        (hi0, lo0) = mulhilo(M0, c0); (hi1, lo1) = mulhilo(M1, c2)
        c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
    and the key is bumped by the Weyl constants between rounds."""
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint64) & MASK for x in ctr)
    k0, k1 = (np.asarray(x, dtype=np.uint64) & MASK for x in key)
    for rnd in range(10):
        if rnd > 0:
            k0 = (k0 + W0) & MASK
            k1 = (k1 + W1) & MASK
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> S32, p0 & MASK
        hi1, lo1 = p1 >> S32, p1 & MASK
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0), lo1, (hi0 ^ c3 ^ k1), lo0
    return tuple(x.astype(np.uint32) for x in (c0, c1, c2, c3))


def philox_words(seed: int, mode: int, cols, j, v: int = 0):
    """The 4 words for counter (j, mode | v<<8, c lo, c hi) and key(seed)."""
    cols = np.asarray(cols, dtype=np.uint64)
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    key = (np.uint64(seed & 0xFFFFFFFF), np.uint64(seed >> 32))
    ctr = (np.full(cols.shape, j, dtype=np.uint64),
           np.full(cols.shape, (int(mode) | (int(v) << 8)) & 0xFFFFFFFF, dtype=np.uint64),
           cols & MASK, cols >> S32)
    return philox4x32_10(ctr, key)


def omega_rows(seed: int, mode: int, cols, ell: int, k0: int = 0, v: int = 0) -> np.ndarray:
    """Rows `cols` and columns k0 .. k0+ell-1 of Omega_mode, fp64, shape (len(cols), ell).

    Counter-based, so any subset of rows equals the corresponding rows of the full
    matrix (partition invariance) and adaptive blocks continue the global k."""
    cols = np.asarray(cols, dtype=np.int64).ravel()
    out = np.empty((cols.size, ell), dtype=np.float64)
    if ell == 0 or cols.size == 0:
        return out
    two32 = 2.0 ** -32
    for j in range(k0 >> 2, ((k0 + ell - 1) >> 2) + 1):
        w = philox_words(seed, mode, cols.astype(np.uint64), j, v)
        u = [(w_i.astype(np.float64) + 0.5) * two32 for w_i in w]
        ra = np.sqrt(-2.0 * np.log(u[0]))
        rb = np.sqrt(-2.0 * np.log(u[2]))
        z = (ra * np.cos(2.0 * np.pi * u[1]), ra * np.sin(2.0 * np.pi * u[1]),
             rb * np.cos(2.0 * np.pi * u[3]), rb * np.sin(2.0 * np.pi * u[3]))
        for q in range(4):
            k = 4 * j + q
            if k0 <= k < k0 + ell:
                out[:, k - k0] = z[q]
    return out
