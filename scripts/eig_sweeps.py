import ctypes as C, sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1905_07311_b200.rtucker import Context
ctx = Context(0)
n = 60
rng = np.random.default_rng(0)
for name, spec in [("i^-3", np.arange(1, n + 1) ** -3.0), ("logspace12", np.logspace(0, -12, n)), ("flat+1e-4", np.r_[np.arange(1, 51) ** -3.0, np.full(10, 1e-8)])]:
    u, _ = np.linalg.qr(rng.standard_normal((n, n)))
    a = (u * spec) @ u.T
    at = torch.as_tensor(np.asfortranarray(a).ravel(order="F"), device="cuda")
    w = torch.empty(n, dtype=torch.float64, device="cuda"); v = torch.empty_like(at); sw = C.c_int32()
    for _ in range(3):
        assert ctx.lib.rtucker_debug_gram_eig(ctx.h, n, at.data_ptr(), w.data_ptr(), v.data_ptr(), C.byref(sw)) == 0
    torch.cuda.synchronize()
    import time
    t0 = time.perf_counter()
    for _ in range(20):
        ctx.lib.rtucker_debug_gram_eig(ctx.h, n, at.data_ptr(), w.data_ptr(), v.data_ptr(), C.byref(sw))
    torch.cuda.synchronize()
    print(name, "sweeps", sw.value, "us", (time.perf_counter() - t0) / 20 * 1e6)
