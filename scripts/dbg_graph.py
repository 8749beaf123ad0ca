import sys, time
import numpy as np
sys.path.insert(0, '.')
import torch
from paper_1905_07311_b200.rtucker import Context, GRAPH
from workloads import odeco
x = odeco(800, seed=4, dtype=np.float32, device="cuda")
s = torch.cuda.Stream()
c = Context(0, stream=s)
for i in range(4):
    torch.cuda.synchronize(); t = time.perf_counter()
    r = c.sthosvd(x, (800, 800, 800), (50, 50, 50), 10, 0, (0, 1, 2), GRAPH)
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(i, f"enqueue {1e3*(t1-t):.3f} ms, total {1e3*(t2-t):.3f} ms", flush=True)
    r.free()
