"""Time individual library steps through the debug ABI (CUDA events on the library stream)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1905_07311_b200.rtucker import Context

ctx = Context(0)
lib = ctx.lib
st = ctx.stream


def timeit(fn, reps=20):
    for _ in range(3):
        assert fn() == 0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


rng = np.random.default_rng(0)
for n in (10, 60, 64):
    u, _ = np.linalg.qr(rng.standard_normal((n, n)))
    a = (u * np.arange(1, n + 1) ** -3.0) @ u.T
    at = torch.as_tensor(np.asfortranarray(a).ravel(order="F"), device="cuda")
    w = torch.empty(n, dtype=torch.float64, device="cuda")
    v = torch.empty_like(at)
    sw = C.c_int32()
    for name, f in (("gram_eig", lib.rtucker_debug_gram_eig), ("sym_eig", lib.rtucker_debug_eig)):
        us = timeit(lambda: f(ctx.h, n, at.data_ptr(), w.data_ptr(), v.data_ptr(), C.byref(sw)))
        print(f"{name} n={n}: {us:.1f} us (incl. host sync) sweeps={sw.value}")
for m, n in ((800, 60), (400, 50), (50, 10), (200000, 15)):
    y = torch.randn(m * n, dtype=torch.float64, device="cuda")
    q = torch.empty_like(y)
    us = timeit(lambda: lib.rtucker_debug_qr(ctx.h, m, n, y.data_ptr(), q.data_ptr()))
    print(f"qr {m}x{n}: {us:.1f} us (ncta env={os.environ.get('RTUCKER_QR_NCTA', 'auto')})")
