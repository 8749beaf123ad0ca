"""Oracle row selection for SP-STHOSVD (test infrastructure only; see oracle/__init__.py).

Alg 6 line 6: "Use strong RRQR on Q^T with parameter eta = 2 ...
Let P = S_1 ... which contains the columns from the identity matrix", and line 7
(P:382): A = Q (P^T Q)^{-1}.  Thm 5.1: A contains an l x l identity and
1 <= ||A||_2 <= g(I, l) = sqrt(1 + 4 l (I - l)).

DESIGN reading R9 (= SURVEY §8(c) item 9): the selection takes k = l = rank(Q)
columns of Q^T, so the R22 block of Gu-Eisenstat's strong RRQR is empty and the
strong-RRQR condition reduces to |(Q Q_S^{-1})_{ik}| <= eta for all i, k ("maxvol").
Procedure: Businger-Golub column-pivoted QR of Q^T (pivot = largest remaining
column norm, ties to the smallest index) gives the initial S; then while
max_{i not in S, k} |A_ik| > eta swap S_k <- i (largest entry; ties to smallest i then
smallest k) and recompute A.  Each swap multiplies |det Q_S| by > eta, so it stops.
Finally S is sorted ascending (this fixes the renumbering of the selected indices).
"""
from __future__ import annotations

import numpy as np


class SingularSelection(ArithmeticError):
    pass


def cpqr_select(qt: np.ndarray, k: int | None = None) -> list[int]:
    """Businger-Golub CPQR pivots of qt (l x I); returns the first k pivot columns.
    Residual column norms are recomputed from the updated matrix at every step."""
    r = np.array(qt, dtype=np.float64, copy=True)
    ell, n = r.shape
    k = ell if k is None else k
    piv: list[int] = []
    chosen = np.zeros(n, dtype=bool)
    for j in range(k):
        norms = np.sum(r[j:, :] ** 2, axis=0)
        norms[chosen] = -1.0
        p = int(np.argmax(norms))          # first maximum -> smallest index on ties
        piv.append(p)
        chosen[p] = True
        v = r[j:, p].copy()
        nv = np.linalg.norm(v)
        if nv == 0.0:
            continue
        alpha = -nv if v[0] >= 0 else nv
        v[0] -= alpha
        vn = np.linalg.norm(v)
        if vn == 0.0:
            continue
        v /= vn
        r[j:, :] -= 2.0 * np.outer(v, v @ r[j:, :])
    return piv


def oblique_factor(q: np.ndarray, sel) -> np.ndarray:
    """A = Q (P^T Q)^{-1} by an LU solve on the l x l block Q[S, :]."""
    qs = q[np.asarray(sel), :]
    try:
        if not np.all(np.isfinite(qs)) or np.linalg.matrix_rank(qs) < qs.shape[0]:
            raise np.linalg.LinAlgError("rank-deficient P^T Q")
        at = np.linalg.solve(qs.T, q.T)   # (Q_S^T) A^T = Q^T  <=>  A Q_S = Q
    except np.linalg.LinAlgError as e:
        raise SingularSelection(str(e)) from e
    return at.T


def srrqr_select(q: np.ndarray, eta: float = 2.0, max_swaps: int = 10000):
    """Strong-RRQR row selection of q (I x l, orthonormal columns) per reading R9.
    Returns (sorted selection, number of swaps)."""
    q = np.asarray(q, dtype=np.float64)
    n, ell = q.shape
    sel = cpqr_select(q.T, ell)
    swaps = 0
    while swaps < max_swaps:
        a = oblique_factor(q, sel)
        m = np.abs(a)
        m[np.asarray(sel), :] = -1.0
        flat = int(np.argmax(m))           # row-major: smallest i, then smallest k
        i, kk = divmod(flat, ell)
        if m[i, kk] <= eta:
            break
        sel[kk] = i
        swaps += 1
    return sorted(sel), swaps
