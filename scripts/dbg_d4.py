import sys
import numpy as np
sys.path.insert(0, '.')
import torch
import oracle as O
from workloads import hilbert, to_first_mode_fastest
from paper_1905_07311_b200.rtucker import Context, RESULT_HOST
c = Context(0, allocator='library')
x = hilbert((70, 9, 13, 11), "paper")
for algo in ("sthosvd",):
    xd = torch.as_tensor(to_first_mode_fastest(x), device="cuda")
    g = c.sthosvd(xd, x.shape, (40, 3, 5, 4), 25, 0, None, RESULT_HOST).numpy()
    o = O.r_sthosvd(x, (40, 3, 5, 4), 25, 0, None)
    print("order", g.order, o.order, "ranks", g.ranks, o.ranks, "ell", g.ell, o.ell)
    for j in range(4):
        a, b = g.factors[j], o.factors[j]
        print(j, a.shape, "orth", np.linalg.norm(a.T @ a - np.eye(a.shape[1])), "proj", O.projector_distance(a, b),
              "nan", np.isnan(a).any())
    print("core", np.linalg.norm(g.core), np.linalg.norm(o.core), "resid", g.mode_residual_sq, o.mode_residual_sq)
    print("delta", O.approx_distance(x, (g.core, g.factors), (o.core, o.factors)))
