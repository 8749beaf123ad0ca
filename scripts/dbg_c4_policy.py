"""C4 relative error under the precision policies (identity e^2 = 1 - ||G||^2/||X||^2),
oracle value 0.02206951830024321 (test_c4_full_size_rsthosvd)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1905_07311_b200.rtucker import Context, RESULT_HOST, ACCUM_FAST, ACCUM_HYBRID, ACCUM_FP64
from workloads import odeco
x = odeco(800, seed=4, dtype=np.float32, device="cuda")
nx2 = float((x.double() ** 2).sum())
ctx = Context(0)
eo = 0.02206951830024321
for name, fl in (("HYBRID", ACCUM_HYBRID), ("FAST", ACCUM_FAST), ("FP64", ACCUM_FP64)):
    g = ctx.sthosvd(x, (800, 800, 800), (50, 50, 50), 10, 0, (0, 1, 2), fl | RESULT_HOST).numpy()
    e = np.sqrt(max(0.0, 1 - np.sum(g.core ** 2) / nx2))
    print(f"{name}: e={e:.10f} rel diff {abs(e - eo) / eo:.2e}")
