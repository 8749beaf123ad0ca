"""One eager adaptive R-STHOSVD call on C4 (tol 1e-3, block 10): the command profiled by
`ncu --metrics gpu__time_duration.sum` for the adaptive launch list."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1905_07311_b200.rtucker import Context
from workloads import odeco
x = odeco(800, seed=4, dtype=np.float32, device="cuda:0")
torch.cuda.synchronize()
ctx = Context(0)
ctx.adaptive(x, (800, 800, 800), 1e-3, 10, order=(0, 1, 2), seed=0).free()
torch.cuda.synchronize()
print("done")
