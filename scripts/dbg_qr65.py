import sys
import numpy as np
sys.path.insert(0, '.')
from paper_1905_07311_b200.rtucker import Context
c = Context(0, allocator='library')
rng = np.random.default_rng(0)
for m, n in ((70, 65), (100, 65), (70, 64), (200, 100)):
    y = rng.standard_normal((m, n))
    q = c.debug_qr(y)
    print(m, n, "orth", np.linalg.norm(q.T @ q - np.eye(n)), "span", np.linalg.norm(y - q @ (q.T @ y)) / np.linalg.norm(y))
