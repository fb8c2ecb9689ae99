"""B200 (sm_100a) FP64 implementation of the ADMM hot path of arXiv 2406.07048.

The compute lives in the C-ABI library ``libca.so`` (include/ca.h); this package is
a thin ctypes binding with the same names.  There is no CPU fallback: importing
works anywhere, but every compute call needs the built library and a B200.
"""
from ._ca import (  # noqa: F401
    CA_OK,
    CA_W_NOT_CONVERGED,
    CA_W_PAIR_FAILURES,
    CAError,
    Problem,
    fp64_peak,
    nccl_unique_id,
    obstacle_partition,
    lib,
    library_path,
)
