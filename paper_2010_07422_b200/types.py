"""Result and configuration types of the IRCUR drop-in.

Same names, fields, defaults, validation and shape invariants as the
reference (`solver.py:49-150`, `matcore.py:115-193`), so code written
against `ircur.solve` reads the B200 results unchanged.  Host-facing arrays
are float64 numpy arrays, as in the reference.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .sampling import IndexSet, RngSeed

MODES = ("fixed", "resampled")
PINV_CUTOFF = 1e-12  # matcore.py:22


@dataclass
class SolverConfig:
    """All tunables of the solver (solver.py:49-86)."""

    rank: int
    eps: float = 1e-5
    zeta0: float | None = None
    gamma: float = 0.65
    c_rows: float = 4.0
    c_cols: float = 4.0
    mode: str = "fixed"
    max_iter: int = 200
    seed: RngSeed = field(default_factory=lambda: RngSeed(0))

    def __post_init__(self) -> None:
        if self.rank < 1:
            raise ValueError(f"rank must be >= 1, got {self.rank}")
        if not self.eps > 0:
            raise ValueError(f"eps must be > 0, got {self.eps}")
        if self.zeta0 is not None and not self.zeta0 > 0:
            raise ValueError(f"zeta0 must be > 0 (or None), got {self.zeta0}")
        if not 0.0 < self.gamma < 1.0:
            raise ValueError(f"gamma must lie in (0, 1), got {self.gamma}")
        if self.c_rows <= 0 or self.c_cols <= 0:
            raise ValueError("sampling constants must be > 0")
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}, got {self.mode!r}")
        if self.max_iter < 1:
            raise ValueError(f"max_iter must be >= 1, got {self.max_iter}")


@dataclass
class SvdFactors:
    """Compact SVD triple (matcore.py:115-125)."""

    W: np.ndarray
    sigma: np.ndarray
    V: np.ndarray

    def dense(self) -> np.ndarray:
        return (self.W * self.sigma) @ self.V.T


@dataclass
class PinvFactor:
    """Factored pseudo-inverse of the core (matcore.py:142-193)."""

    W: np.ndarray
    sigma: np.ndarray
    V: np.ndarray
    inv_sigma: np.ndarray

    @property
    def rows(self) -> int:
        return self.W.shape[0]

    @property
    def cols(self) -> int:
        return self.V.shape[0]

    @property
    def effective_rank(self) -> int:
        return int(np.count_nonzero(self.inv_sigma))

    def apply_left(self, X: np.ndarray) -> np.ndarray:
        """U^+ X for X with rows(U) rows."""
        return self.V @ ((self.W.T @ X) * self.inv_sigma[:, None])

    def apply_right(self, X: np.ndarray) -> np.ndarray:
        """X U^+ for X with cols(U) columns."""
        return ((X @ self.V) * self.inv_sigma) @ self.W.T

    def dense_core(self) -> np.ndarray:
        return (self.W * self.sigma) @ self.V.T


@dataclass
class CurFactors:
    """L = C U_r^+ R held in factored form (solver.py:89-114).

    `device` (not part of the reference type) keeps the B200 context that
    produced the factors so `materialize` can stream L on the GPU.
    """

    C: np.ndarray
    core_pinv: PinvFactor
    R: np.ndarray
    rows: IndexSet
    cols: IndexSet
    device: object = field(default=None, repr=False, compare=False)

    def __post_init__(self) -> None:
        if self.C.shape != (self.rows.bound, self.cols.size):
            raise ValueError("C shape inconsistent with index sets")
        if self.R.shape != (self.rows.size, self.cols.bound):
            raise ValueError("R shape inconsistent with index sets")
        if (self.core_pinv.rows, self.core_pinv.cols) != (self.rows.size, self.cols.size):
            raise ValueError("core factor shape inconsistent with index sets")

    @property
    def shape(self) -> tuple[int, int]:
        return (self.rows.bound, self.cols.bound)


@dataclass
class SparseEstimate:
    """S on the sampled slabs only (solver.py:117-129)."""

    row_values: np.ndarray
    col_values: np.ndarray
    rows: IndexSet
    cols: IndexSet


@dataclass
class SolverTrace:
    """Per-iteration history (solver.py:132-150).  `seconds` come from CUDA
    events around each device iteration; `allocated` is the transient device
    allocation per iteration in 8-byte units (0: the workspace is allocated
    once per context, before the loop)."""

    errors: list = field(default_factory=list)
    thresholds: list = field(default_factory=list)
    iterations: int = 0
    converged: bool = False
    seconds: list = field(default_factory=list)
    allocated: list = field(default_factory=list)
    sampled_rows: list = field(default_factory=list)
    sampled_cols: list = field(default_factory=list)
