import sys
import numpy as np
sys.path.insert(0, '.')
import torch
from paper_1905_07311_b200.rtucker import Context
c = Context(0, allocator='library')
rng = np.random.default_rng(0)
y = rng.standard_normal((800, 60)) * np.arange(1, 61) ** -1.5
for _ in range(5):
    c.debug_qr(y)
