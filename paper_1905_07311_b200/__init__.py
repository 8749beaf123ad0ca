"""B200-native randomized Tucker hot path (arXiv 1905.07311): R-HOSVD, R-STHOSVD,
adaptive R-STHOSVD and SP-STHOSVD behind a C ABI (include/rtucker.h), sm_100a CUDA.

`from paper_1905_07311_b200 import rtucker` gives the ctypes binding (Context, ...).
"""
from . import rtucker  # noqa: F401
from .rtucker import Context, RTuckerError, load_library  # noqa: F401
