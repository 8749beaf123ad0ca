"""Run the mode-1 HYBRID B-pass (fp64 products, fp64 B + Gram) on a C4-size tensor once."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1905_07311_b200.rtucker import Context
ctx = Context(0)
I = 800
x = torch.randn(I * I * I, device="cuda", dtype=torch.float32)
q, _ = np.linalg.qr(np.random.default_rng(0).standard_normal((I, 60)))
mode = int(sys.argv[1]) if len(sys.argv) > 1 else 0
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    out, g = ctx.debug_ttm(x, (I, I, I), mode, q)
print("ok", float(g[0, 0]))
