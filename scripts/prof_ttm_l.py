"""Run the L > 1 B-pass of the C4 step's second mode once: B = Q^T G1_(2), G1 = (50, 800, 800) fp64,
Q 800 x 60 (fp64 products, fp64 B + Gram).  usage: prof_ttm_l.py [reps] [L]"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1905_07311_b200.rtucker import Context
ctx = Context(0)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
L = int(sys.argv[2]) if len(sys.argv) > 2 else 50
x = torch.randn(L * 800 * 800, device="cuda", dtype=torch.float64)
q, _ = np.linalg.qr(np.random.default_rng(0).standard_normal((800, 60)))
for _ in range(reps):
    out, g = ctx.debug_ttm(x, (L, 800, 800), 1, q)
print("ok", float(g[0, 0]))
