"""Fig 6.4 analogue (NEXT-4): the synthetic sparse gamma-tensor
X = sum_{i<=10} gamma/i^2 x_i o y_i o z_i + sum_{i=11}^{200} 1/i^2 x_i o y_i o z_i (5 % sparse
vectors, 200^3), gamma in {2, 10, 200}, p = 5, rho = [1, 2, 3].  SP-STHOSVD with target rank r
returns rank r + p, so it is compared with STHOSVD (RTUCKER_EXACT_SVD) and R-STHOSVD
at rank r + p on the densified tensor.  All three on the GPU; the figure prints no numbers, so
the check is qualitative (the paper: SP "slightly higher for the lower r").  JSON to stdout."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle as O  # noqa: E402  (reconstruction of the results for the error only)
from paper_1905_07311_b200.rtucker import Context, EXACT_SVD, RESULT_HOST  # noqa: E402
from workloads import synthetic_sparse_gamma, to_first_mode_fastest  # noqa: E402

ctx = Context(0)
out = []
for gamma in (2.0, 10.0, 200.0):
    x = synthetic_sparse_gamma(gamma, seed=1)
    idx = np.array(np.nonzero(x), dtype=np.int32)
    vals = x[tuple(idx)]
    xd = torch.as_tensor(to_first_mode_fastest(x), device="cuda")
    nx = np.linalg.norm(x)
    for r in (5, 10, 15, 20, 30, 40):
        ell = r + 5
        sp = ctx.sparse_sthosvd(torch.as_tensor(idx, device="cuda"), torch.as_tensor(vals, device="cuda"), x.shape,
                                (r, r, r), 5, 0, (0, 1, 2), 2.0, RESULT_HOST).numpy()
        core = np.zeros((ell, ell, ell))
        core[tuple(sp.core_idx)] = sp.core_vals
        e_sp = np.linalg.norm(x - O.reconstruct(core, sp.factors)) / nx
        rs = ctx.sthosvd(xd, x.shape, (ell,) * 3, 5, 0, (0, 1, 2), RESULT_HOST).numpy()
        st = ctx.sthosvd(xd, x.shape, (ell,) * 3, 0, 0, (0, 1, 2), EXACT_SVD | RESULT_HOST).numpy()
        row = {"gamma": gamma, "r": r, "rank": ell, "nnz": int(idx.shape[1]),
               "SP-STHOSVD": float(e_sp), "R-STHOSVD": float(O.rel_error(x, rs.core, rs.factors)),
               "STHOSVD": float(O.rel_error(x, st.core, st.factors)), "sp_core_nnz": int(sp.core_vals.size)}
        out.append(row)
        print(json.dumps(row), file=sys.stderr, flush=True)
print(json.dumps({"experiment": "Fig 6.4 analogue: relative error vs rank, synthetic sparse gamma-tensor 200^3",
                  "readings": "SP-STHOSVD(r) has rank r+p; STHOSVD and R-STHOSVD at rank r+p (P:606-607)",
                  "rows": out}))
