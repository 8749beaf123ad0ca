"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
C1 and C3 (fp64 Hilbert) R-STHOSVD and R-HOSVD, C2 (fp32) R-STHOSVD with the tcgen05 / Ozaki
kernels, adaptive C2, the sparse path on 1% of C5, and the grid eigensolver at n = 120."""
import sys
import numpy as np
sys.path.insert(0, '.')
import torch
from paper_1905_07311_b200.rtucker import Context, RESULT_HOST
from workloads import hilbert, tucker_c2, sparse_zipf, to_first_mode_fastest

c = Context(0, allocator="library")
dev = lambda x: torch.as_tensor(to_first_mode_fastest(x), device="cuda")
x1 = hilbert((50, 50, 50), "shifted")
c.sthosvd(dev(x1), x1.shape, (5, 5, 5), 5, 0, (0, 1, 2), RESULT_HOST).numpy()
c.hosvd(dev(x1), x1.shape, (5, 5, 5), 5, 0, RESULT_HOST).numpy()
x3 = hilbert((25,) * 5, "shifted")
c.sthosvd(dev(x3), x3.shape, (5,) * 5, 5, 0, tuple(range(5)), RESULT_HOST).numpy()
x2 = tucker_c2()
c.sthosvd(dev(x2), x2.shape, (20, 20, 40), 10, 0, None, RESULT_HOST).numpy()
c.hosvd(dev(x2), x2.shape, (20, 20, 40), 10, 0, RESULT_HOST).numpy()
c.adaptive(dev(x2), x2.shape, 1e-2, 5, flags=RESULT_HOST).numpy()
idx, vals = sparse_zipf(ndraws=500_000)
c.sparse_sthosvd(torch.as_tensor(idx, device="cuda"), torch.as_tensor(vals, device="cuda"),
                 (8000, 8000, 200000, 1200), (10, 10, 10, 10), 5, 0, None, 2.0, RESULT_HOST).numpy()
a = np.random.default_rng(0).standard_normal((120, 120)); a = a @ a.T
c.debug_gram_eig(a)
c.sync()
print("sanitize cases done")
