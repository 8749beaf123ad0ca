"""One adaptive R-STHOSVD call on C4 (tol 1e-3, block 10) with per-phase CUDA events: prints
each phase's total ms and launch count per mode, and the wall time of an eager call."""
import sys, time
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
t0 = time.perf_counter()
r = ctx.adaptive(x, (800, 800, 800), 1e-3, 10, order=(0, 1, 2), seed=0)
torch.cuda.synchronize()
print(f"eager call {1e3 * (time.perf_counter() - t0):.1f} ms, ranks {list(r.numpy().core.shape)}")
r.free()
ctx.set_profiling(True)
ctx.phase_times(reset=True)
ctx.adaptive(x, (800, 800, 800), 1e-3, 10, order=(0, 1, 2), seed=0).free()
ph = ctx.phase_times(reset=True)
tot = 0.0
for k, (ms, n) in sorted(ph.items(), key=lambda t: -t[1][0]):
    tot += ms
    print(f"{k[0]:>7} m{k[1] + 1}: {ms:9.2f} ms total, {n:5d} launches-scopes, {ms / n:8.3f} ms each")
print(f"sum of phases {tot:.1f} ms")
