"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This package holds NO arithmetic of the method (no sketch, QR, SVD, TTM chain,
selection).  It only builds input tensors, following the recipes in DESIGN.md §3
(and SURVEY.md §8(d) d.2).  Both implementations consume the same bits from here.
"""
from .generators import (  # noqa: F401
    hilbert, tucker_c2, odeco, exact_rank, superdiagonal, sparse_zipf,
    synthetic_sparse_gamma, haar, to_first_mode_fastest, from_first_mode_fastest,
    CONFIGS,
)
