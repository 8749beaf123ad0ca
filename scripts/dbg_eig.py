"""Eigensolver accuracy probe: V and w of debug_gram_eig vs LAPACK on random / graded Grams."""
import sys
import numpy as np
sys.path.insert(0, '.')
from paper_1905_07311_b200.rtucker import Context
c = Context(0, allocator='library')
rng = np.random.default_rng(0)
for n in (10, 60, 64, 65, 100, 150, 300):
    for kind in ("rand", "graded", "hilbert"):
        if kind == "rand":
            b = rng.standard_normal((n, n)); a = b @ b.T
        elif kind == "graded":
            u, _ = np.linalg.qr(rng.standard_normal((n, n))); a = (u * np.arange(1, n + 1) ** -3.0) @ u.T
        else:
            x = 1.0 / (np.arange(n)[:, None] + np.arange(3 * n)[None, :] + 1.0); a = x @ x.T
        a = (a + a.T) / 2
        w, v = c.debug_gram_eig(a)
        we, ve = np.linalg.eigh(a); o = np.argsort(-we); we, ve = we[o], ve[:, o]
        k = min(10, n - 1)
        gap = we[k - 1] - we[k]
        pd = np.linalg.norm(v[:, :k] @ v[:, :k].T - ve[:, :k] @ ve[:, :k].T, 2)
        print(f"n={n:4d} {kind:8s} werr={np.max(np.abs(w - we)) / we[0]:.1e} orth={np.linalg.norm(v.T @ v - np.eye(n)):.1e} "
              f"resid={np.linalg.norm(a @ v - v * w) / we[0]:.1e} proj{k}={pd:.1e} (eps*l1/gap={2.2e-16 * we[0] / gap:.1e}) "
              f"nan={np.isnan(v).any()}", flush=True)
