"""Full-size C4 component checks on the GPU (torch fp64 references on the device)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1905_07311_b200.rtucker import Context
from workloads import odeco

I = 800
ctx = Context(0)
x = odeco(I, seed=4, dtype=np.float32, device="cuda")
X1 = x.view(I * I, I).t() if False else x.view(I, I * I)  # placeholder
# X_(1): first-mode-fastest flat -> element (i, c) at i + I c  => reshape (C, I) row-major, transpose
X1 = x.view(I * I, I).t()          # (I, C) view, X1[i, c]
ell = 60
y = ctx.debug_sketch(x, (I, I, I), 0, ell, seed=0)
# reference: Omega rows from the library's own fp32 generator, fp64 product on the device
ref = torch.zeros(I, ell, dtype=torch.float64, device="cuda")
C = I * I
for c0 in range(0, C, 64000):
    cols = np.arange(c0, min(C, c0 + 64000))
    om = torch.as_tensor(ctx.debug_omega(cols, ell, seed=0, mode=0, dtype="f32"), device="cuda").double()
    ref += X1[:, c0:c0 + len(cols)].double() @ om
ref = ref.cpu().numpy()
err = np.linalg.norm(y - ref) / np.linalg.norm(ref)
colerr = np.max(np.linalg.norm(y - ref, axis=0) / np.linalg.norm(ref, axis=0))
print(f"sketch mode1 full size: rel err {err:.3e}, worst column {colerr:.3e}")
# B-pass with a random orthonormal Q
q, _ = np.linalg.qr(np.random.default_rng(0).standard_normal((I, ell)))
out, gram = ctx.debug_ttm(x, (I, I, I), 0, q)
Bref = torch.as_tensor(q, device="cuda").t() @ X1.double()      # (ell, C)
B = out.view(C, ell).t()                                         # stored (1, ell, C): B[k + ell c]
print(f"bpass mode1: rel err {float(torch.linalg.norm(B - Bref) / torch.linalg.norm(Bref)):.3e}")
gref = (Bref @ Bref.t()).cpu().numpy()
print(f"gram: rel err {np.linalg.norm(gram - gref) / np.linalg.norm(gref):.3e}")
