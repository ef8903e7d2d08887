"""B200-native IRCUR (Iterated Robust CUR, arXiv 2010.07422) hot path.

Drop-in for the reference package's `ircur.solve` (solver.py:304-416):
same signature, result types and error behaviour, with every arithmetic step
of the iteration in hand-written sm_100a CUDA kernels behind a C-ABI
(include/ircur_b200.h, built into libircur_b200.so).
"""

from .convert import cur_to_svd, factors_to_svd
from .sampling import IndexSet, RngSeed, draw_index_sets, sample_count, sample_indices
from .solver import (
    Context,
    DeviceResult,
    clear_cache,
    materialize,
    materialize_device,
    solve,
    solve_batch,
    solve_batch_device,
    solve_device,
    threshold_at,
)
from .types import CurFactors, PinvFactor, SolverConfig, SolverTrace, SparseEstimate, SvdFactors

__all__ = [
    "Context", "CurFactors", "DeviceResult", "IndexSet", "PinvFactor", "RngSeed", "SolverConfig",
    "cur_to_svd", "factors_to_svd",
    "SolverTrace", "SparseEstimate", "SvdFactors", "clear_cache", "draw_index_sets", "materialize",
    "materialize_device", "sample_count", "sample_indices", "solve", "solve_batch", "solve_batch_device", "solve_device", "threshold_at",
]

__version__ = "0.1.0"
