import numpy as np, sys, os
sys.path.insert(0, '.')
from paper_1905_07311_b200.rtucker import Context
ctx = Context(0)
np.set_printoptions(precision=4, suppress=True, linewidth=150)
rng = np.random.default_rng(0)
for m, n in [(8, 2), (8, 3), (12, 4)]:
    y = rng.standard_normal((m, n))
    q = ctx.debug_qr(y)
    qr, _ = np.linalg.qr(y)
    s = np.sign(np.sum(q * qr, axis=0))
    print(m, n, os.environ.get("RTUCKER_QR_NCTA"), "orth", np.linalg.norm(q.T @ q - np.eye(n)))
    print(np.hstack([q, qr * s]))
