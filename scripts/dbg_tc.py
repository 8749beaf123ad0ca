import sys
import numpy as np
sys.path.insert(0, ".")
import oracle as O
from paper_1905_07311_b200.rtucker import Context
ctx = Context(0)
np.set_printoptions(precision=4, suppress=True, linewidth=150)


def ref(x, ell, seed=5):
    xm = O.unfold(np.asarray(x, dtype=np.float64), 0)
    return xm @ O.omega_rows(seed, 0, np.arange(xm.shape[1]), ell)


for name, x in [("e00", None), ("ones", None), ("rand", None)]:
    shape = (128, 16, 1)
    if name == "e00":
        x = np.zeros(shape, np.float32); x[0, 0, 0] = 1
    elif name == "ones":
        x = np.ones(shape, np.float32)
    else:
        x = np.random.default_rng(0).standard_normal(shape).astype(np.float32)
    x = np.asfortranarray(x)
    g = ctx.debug_sketch(x, x.shape, 0, 32, seed=5)
    r = ref(x, 32)
    print(name, "max|got|", np.abs(g).max(), "max|ref|", np.abs(r).max(), "relerr", np.linalg.norm(g - r) / np.linalg.norm(r))
    nz = np.argwhere(np.abs(g) > 1e-6)
    print(" nonzeros got (first 10):", nz[:10].tolist(), "count", len(nz))
    print(" got[:3,:8]\n", g[:3, :8], "\n ref[:3,:8]\n", r[:3, :8])
