import numpy as np, sys
sys.path.insert(0, '.')
from paper_1905_07311_b200.rtucker import Context
ctx = Context(0)
for m, n in [(2000, 10), (800, 60), (400, 50), (64, 64)]:
    rng = np.random.default_rng(0)
    y = rng.standard_normal((m, n))
    q = ctx.debug_qr(y)
    qr, _ = np.linalg.qr(y)
    # compare up to column signs
    s = np.sign(np.sum(q * qr, axis=0))
    d = q - qr * s
    blocks = [np.abs(d[i:i + m // 4]).max() for i in range(0, m, max(1, m // 4))]
    print(m, n, "orth", np.linalg.norm(q.T @ q - np.eye(n)), "blockerr", ["%.1e" % b for b in blocks],
          "colerr", ["%.1e" % v for v in np.abs(d).max(axis=0)[:8]])
