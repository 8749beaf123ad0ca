"""Launch the hot-path Gram eigensolvers at n = 40 / 60 / 64 (C4-like spectrum) for both
precisions (rel_acc 0: mixed fp32 Jacobi + fp64 refinement; 1: fp64 preconditioned Jacobi);
run under `ncu --metrics gpu__time_duration.sum` for per-kernel device times."""
import ctypes as C, sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1905_07311_b200.rtucker import Context
ctx = Context(0)
for n in (40, 60, 64):
    rng = np.random.default_rng(n)
    u, _ = np.linalg.qr(rng.standard_normal((n, n)))
    a = (u * np.arange(1, n + 1) ** -3.0) @ u.T
    at = torch.as_tensor(np.asfortranarray(a).ravel(order="F"), device="cuda")
    w = torch.empty(n, dtype=torch.float64, device="cuda"); v = torch.empty_like(at); sw = C.c_int32()
    for rel in (0, 1):
        for _ in range(3):
            assert ctx.lib.rtucker_debug_gram_eig_ex(ctx.h, n, at.data_ptr(), w.data_ptr(), v.data_ptr(), C.byref(sw), rel, n - 10) == 0
        print(f"n={n} rel_acc={rel} sweeps_info={sw.value}", flush=True)
