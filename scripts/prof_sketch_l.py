"""Mode-2 sketch of the C4 step's shrunk core G1 = (50, 800, 800) fp64 through the debug ABI
(fp64 products, fp32 normals as in the HYBRID policy).  usage: prof_sketch_l.py [reps]"""
import ctypes as C
import sys
import torch
sys.path.insert(0, ".")
from paper_1905_07311_b200.rtucker import Context
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
ctx = Context(0)
x = torch.randn(50 * 800 * 800, device="cuda", dtype=torch.float64)
for _ in range(reps):
    y = ctx.debug_sketch(x, (50, 800, 800), 1, 60, seed=3)
print("ok", float(y[0, 0]))
