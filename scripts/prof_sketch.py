"""Time the mode-n sketch through the debug ABI on a C4-sized fp32 tensor (CUDA events)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1905_07311_b200.rtucker import Context
import ctypes as C

I = int(sys.argv[1]) if len(sys.argv) > 1 else 800
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 0
ell = int(sys.argv[3]) if len(sys.argv) > 3 else 60
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
x = torch.randn(I * I * I, device="cuda", dtype=torch.float32)
ctx = Context(0, stream=torch.cuda.current_stream())
desc, keep = ctx.dense_desc(x, (I, I, I))
y = torch.empty(I * ell, dtype=torch.float64, device="cuda")
f = lambda: ctx.lib.rtucker_debug_sketch(ctx.h, C.byref(desc), mode, ell, 0, 0, 0, y.data_ptr())
for _ in range(2):
    assert f() == 0
torch.cuda.synchronize()
import time
t0 = time.perf_counter()
for _ in range(reps):
    st = f()
    assert st == 0, st
torch.cuda.synchronize()
ms = (time.perf_counter() - t0) * 1e3 / reps  # includes host enqueue; reps >= 10 amortises
print(f"sketch I={I} mode={mode} ell={ell}: {ms * 1e3:.1f} us  {I ** 3 * 4 / ms / 1e6:.0f} GB/s")
