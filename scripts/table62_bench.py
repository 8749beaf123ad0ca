"""Table 6.2 analogue on one B200 (NEXT-4): deterministic HOSVD / STHOSVD (RTUCKER_EXACT_SVD)
against R-HOSVD / R-STHOSVD on the paper's 5-mode Hilbert tensors X = 1/(i_1 + ... + i_5)
(P:484-487), I in {25, 35, 45, 50}, r = 5, p = 5, rho = [1..5], fp64, median of 3
after a warm-up (the paper averages 3 runs).  The paper's MATLAB CPU times are quoted beside
(context only).  Writes one JSON object to stdout."""
import json
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1905_07311_b200.rtucker import Context, EXACT_SVD  # noqa: E402
from workloads import hilbert, to_first_mode_fastest  # noqa: E402

PAPER_S = {25: (3.0030, 1.2609, 0.6455, 0.2875), 35: (14.5255, 5.5288, 3.1974, 1.2090),
           45: (70.0536, 17.3744, 15.0629, 3.5587), 50: (101.4981, 27.7725, 21.9745, 5.5606)}
stream = torch.cuda.Stream()
ctx = Context(0, stream=stream)
rows = []
for I in (25, 35, 45, 50):
    x = hilbert((I,) * 5, "paper")
    xd = torch.as_tensor(to_first_mode_fastest(x), device="cuda")
    del x
    dims, r = (I,) * 5, (5,) * 5
    calls = {"HOSVD": lambda: ctx.hosvd(xd, dims, r, 5, 0, EXACT_SVD),
             "R-HOSVD": lambda: ctx.hosvd(xd, dims, r, 5, 0),
             "STHOSVD": lambda: ctx.sthosvd(xd, dims, r, 5, 0, tuple(range(5)), EXACT_SVD),
             "R-STHOSVD": lambda: ctx.sthosvd(xd, dims, r, 5, 0, tuple(range(5)))}
    row = {"I": I, "elements": I ** 5}
    for name, f in calls.items():
        f().free()
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            res = f()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
            err = None
            res.free()
        row[name + "_ms"] = statistics.median(ts)
    p = PAPER_S[I]
    row["paper_cpu_s"] = {"HOSVD": p[0], "R-HOSVD": p[1], "STHOSVD": p[2], "R-STHOSVD": p[3]}
    row["speedup_randomized_over_deterministic"] = {"HOSVD": row["HOSVD_ms"] / row["R-HOSVD_ms"],
                                                    "STHOSVD": row["STHOSVD_ms"] / row["R-STHOSVD_ms"]}
    rows.append(row)
    print(json.dumps(row), file=sys.stderr, flush=True)
print(json.dumps({"experiment": "Table 6.2 analogue (P:534-546), one B200, fp64, median of 3 (ms)",
                  "paper_hardware": "MATLAB on a 3.4 GHz Intel Core i7 desktop (P:477), seconds, context only",
                  "rows": rows}))
