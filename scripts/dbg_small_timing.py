"""CUDA-event timing of the small solves through the C ABI (debug exports), n = 60 Gram, 800 x 60 QR."""
import sys
import numpy as np
sys.path.insert(0, '.')
import torch
from paper_1905_07311_b200.rtucker import Context
c = Context(0, allocator='library')
rng = np.random.default_rng(0)
u, _ = np.linalg.qr(rng.standard_normal((60, 60)))
a = (u * np.arange(1, 61) ** -3.0) @ u.T
y = rng.standard_normal((800, 60)) * np.arange(1, 61) ** -1.5
for name, fn in (("gram_eig60", lambda: c.debug_gram_eig(a)), ("qr800x60", lambda: c.debug_qr(y))):
    for _ in range(3):
        fn()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    import time
    t = time.perf_counter()
    for _ in range(20):
        fn()
    print(name, f"{(time.perf_counter() - t) / 20 * 1e6:.0f} us/call incl. host copies", flush=True)
