import ctypes as C, sys, torch
sys.path.insert(0, ".")
from paper_1905_07311_b200.rtucker import Context
ctx = Context(0)
m, n = int(sys.argv[1]), int(sys.argv[2])
y = torch.randn(m * n, dtype=torch.float64, device="cuda"); q = torch.empty_like(y)
for _ in range(3):
    assert ctx.lib.rtucker_debug_qr(ctx.h, m, n, y.data_ptr(), q.data_ptr()) == 0
ctx.sync()
