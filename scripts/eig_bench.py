"""Launch gram_eig (n x n PSD with graded spectrum) a few times, for ncu source-level captures."""
import ctypes as C, sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1905_07311_b200.rtucker import Context
ctx = Context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(0)
u, _ = np.linalg.qr(rng.standard_normal((n, n)))
a = (u * np.logspace(0, -12, n)) @ u.T
at = torch.as_tensor(np.asfortranarray(a).ravel(order="F"), device="cuda")
w = torch.empty(n, dtype=torch.float64, device="cuda"); v = torch.empty_like(at); sw = C.c_int32()
for _ in range(3):
    assert ctx.lib.rtucker_debug_gram_eig(ctx.h, n, at.data_ptr(), w.data_ptr(), v.data_ptr(), C.byref(sw)) == 0
print("sweeps", sw.value)
