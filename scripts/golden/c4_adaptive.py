"""Writes tests/golden/c4_adaptive_oracle.json: the ORACLE's adaptive R-STHOSVD (Alg 5,
P:339-352; AdaptRangeFinder per DESIGN reading R8) on BASELINE configs[3] (C4: odeco 800^3
fp32, data seed 4, eps = 1e-3, block 10, order (1,2,3), Omega seed 0).  Calls only oracle/
and workloads/ (the input generator); nothing from the CUDA path.  Stored: realised ranks,
columns drawn, stop reasons, the last residuals E around the stop (near-tie certification,
DESIGN §5), ||X - X_hat|| / ||X|| and a SHA-256 of the input bytes.

    python scripts/golden/c4_adaptive.py [--size 800]
"""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
from workloads import odeco  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=800)
ap.add_argument("--eps", type=float, default=1e-3)
ap.add_argument("--block", type=int, default=10)
ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "c4_adaptive_oracle.json"))
a = ap.parse_args()

t0 = time.time()
x = odeco(a.size, seed=4, dtype=np.float32)
sha = hashlib.sha256(np.asfortranarray(x).tobytes(order="F")).hexdigest()
t1 = time.time()
o = O.adaptive_r_sthosvd(x, a.eps, a.block, seed=0, order=(0, 1, 2), floor_rel=1e-6)
t2 = time.time()
nx2 = float(np.sum(x.astype(np.float64) ** 2))
tau2 = (a.eps / np.sqrt(3)) ** 2 * nx2


def mode_rec(j):
    inf = o.extra["infos"][j]
    r = int(inf.get("r", o.ranks[j]))
    # truncation decision r = min{r : ||G||^2 - sum_{i<=r} s_i^2 <= tau^2}: the margins at r-1
    # and r (relative to tau^2) certify how far the rank decision is from a tie
    cums = np.cumsum(np.asarray(inf["s"], dtype=np.float64) ** 2)
    marg = [float((inf["norm2"] - cums[r - 2] - tau2) / tau2) if r >= 2 else None,
            float((inf["norm2"] - cums[r - 1] - tau2) / tau2)]
    return dict(stop=inf["stop"], k=int(inf["k"]), r=r, trunc_margin=marg,
                e_hist_tail=[float(e) for e in inf["e_hist"][-3:]])


# ||X - X_hat||^2 = ||X||^2 - ||G||^2 (orthonormal factors, Thm 2.3 identity)
err = float(np.sqrt(max(0.0, 1.0 - float(np.sum(o.core ** 2)) / nx2)))
rec = dict(config="C4 odeco %d^3 fp32 data seed 4" % a.size, eps=a.eps, block=a.block, seed=0,
           order=[0, 1, 2], sha256_fortran_bytes=sha, ranks=list(o.ranks), columns=list(o.ell),
           norm_sq=nx2, rel_err_identity=err,
           modes={str(j): mode_rec(j) for j in range(3)},
           seconds=dict(generate=t1 - t0, oracle=t2 - t1),
           source="scripts/golden/c4_adaptive.py (oracle only)")
with open(a.out, "w") as f:
    json.dump(rec, f, indent=1)
print(json.dumps(rec))
