import sys, time, subprocess
import numpy as np
sys.path.insert(0, '.')
import torch
from paper_1905_07311_b200.rtucker import Context, GRAPH
from workloads import odeco
x = odeco(800, seed=4, dtype=np.float32, device="cuda")
s = torch.cuda.Stream()
c = Context(0, stream=s)
for smi in (False, True):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv", "-lms", "100"], stdout=subprocess.DEVNULL) if smi else None
    time.sleep(1)
    for flags in (GRAPH, 0):
        for _ in range(3):
            c.sthosvd(x, (800, 800, 800), (50, 50, 50), 10, 0, (0, 1, 2), flags).free()
        torch.cuda.synchronize(); t = time.perf_counter()
        rs = [c.sthosvd(x, (800, 800, 800), (50, 50, 50), 10, 0, (0, 1, 2), flags) for _ in range(10)]
        t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
        print("smi", smi, "graph", bool(flags), f"enqueue {1e2*(t1-t):.3f} ms/step, total {1e2*(t2-t):.3f} ms/step", flush=True)
        for r in rs: r.free()
    if p: p.terminate()
