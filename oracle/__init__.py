"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously correct fp64 implementation of what the randomized Tucker
hot path computes (PAPER.md Algs 1-6),
written step by step in the paper's order and notation, with numpy/LAPACK primitives
(matmul, QR, SVD) as the only library steps.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / `--impl
reference` leg may import anything from here.  The product path
(`paper_1905_07311_b200/`, `include/`, the CUDA library) never imports, links or
executes this package; the two share no code.  The only shared module is `workloads/`
(seeded input generators, which hold none of the method's arithmetic).

Pins: every function is checked by `tests/test_oracle_*.py` against values the paper
prints, closed forms, library routines reached by special cases, invariants or brute
force (DESIGN.md §4 lists them).  Functions without such a pin say "parity unpinned"
in their docstring.
"""
from .philox import philox4x32_10, philox_words, omega_rows  # noqa: F401
from .tensor import (  # noqa: F401
    unfold, fold, mode_product, multi_mode_product, frob, reconstruct, rel_error,
    approx_distance, unfold_columns, projector_distance, spectral_gap_kappa,
)
from .algorithms import (  # noqa: F401
    TuckerResult, SpTuckerResult, randsvd, r_hosvd, r_sthosvd, adapt_range_finder,
    adaptive_r_sthosvd, adaptive_r_hosvd, hosvd, sthosvd, sp_sthosvd, sp_hosvd,
    auto_order, rank_caps, canonical_signs, sp_sketch,
)
from .srrqr import cpqr_select, srrqr_select, oblique_factor  # noqa: F401
from .bounds import delta_tail, bound_expected_error, bound_sp, g_cond, f_p  # noqa: F401
