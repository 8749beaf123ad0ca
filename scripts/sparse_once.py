"""One SP-STHOSVD call on C5 (bench.py's sparse workload) for ncu captures of the sparse kernels."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1905_07311_b200.rtucker import Context
from workloads import sparse_zipf
dims = (8000, 8000, 200000, 1200)
idx, vals = sparse_zipf()
it = torch.as_tensor(np.ascontiguousarray(idx), device="cuda")
vt = torch.as_tensor(np.ascontiguousarray(vals), device="cuda")
ctx = Context(0)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    ctx.sparse_sthosvd(it, vt, dims, (10, 10, 10, 10), 5, 0, None, 2.0).free()
ctx.sync()
print("ok")
