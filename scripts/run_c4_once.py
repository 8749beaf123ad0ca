"""One C4 R-STHOSVD through the library (for ncu captures of individual kernels)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1905_07311_b200.rtucker import Context
from workloads import odeco
x = odeco(800, seed=4, dtype=np.float32, device="cuda")
ctx = Context(0)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    ctx.sthosvd(x, (800, 800, 800), (50, 50, 50), 10, 0, (0, 1, 2)).free()
ctx.sync()
print("ok")
