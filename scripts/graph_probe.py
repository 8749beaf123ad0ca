"""Experiment: capture one C4 R-STHOSVD step into a CUDA graph and replay it, to measure the
launch/gap overhead of the eager step (not part of the product path)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1905_07311_b200.rtucker import Context
from workloads import odeco
I = 800
x = odeco(I, seed=4, dtype=np.float32, device="cuda:0", slabs=(0, I))
torch.cuda.synchronize()
s = torch.cuda.Stream()
ctx = Context(0, stream=s)
step = lambda: ctx.sthosvd(x, (I, I, I), (50, 50, 50), 10, 0, (0, 1, 2))
for _ in range(3):
    step().free()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
res = []
e0.record(s)
for _ in range(10):
    res.append(step())
e1.record(s)
torch.cuda.synchronize()
print("eager ms/step", e0.elapsed_time(e1) / 10)
for r in res:
    r.free()
g = torch.cuda.CUDAGraph()
try:
    with torch.cuda.graph(g, stream=s, capture_error_mode="relaxed"):
        r = step()
    torch.cuda.synchronize()
    g.replay(); torch.cuda.synchronize()
    e0.record(s)
    for _ in range(10):
        g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    print("graph ms/step", e0.elapsed_time(e1) / 10)
except Exception as ex:
    print("capture failed:", repr(ex)[:300])
