"""Solver configuration / report records (solver.py:25-95).

`RobustLoss`, `SolverOptions` and `SolverReport` keep the reference's fields
and defaults; `DeviceOptions` holds the B200-only knobs (how the reduced
camera system is solved).  The LM loop itself runs in csrc/ba.cu.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class RobustLoss:
    """rho applied to the squared residual norm s = ||r||^2 (solver.py:25-51)."""

    kind: str = "trivial"        # trivial | huber | cauchy
    param: float = 1.0

    def __post_init__(self):
        if self.kind not in ("trivial", "huber", "cauchy"):
            raise ValueError(f"unknown loss kind {self.kind!r}")


TRIVIAL_LOSS = RobustLoss()


@dataclass
class SolverOptions:
    max_iters: int = 50
    grad_tol: float = 1e-10
    param_tol: float = 1e-12
    initial_lambda: float = 1e-4
    max_lambda: float = 1e32


@dataclass
class SolverReport:
    initial_cost: float
    final_cost: float
    iterations: int
    termination: str


@dataclass
class DeviceOptions:
    """How the reduced camera system S dc = b is solved on the B200.

    linear_solver: "auto" (dense Cholesky when 6*free_frames <= dense_max_dim,
    two-level PCG otherwise), "dense" or "pcg".  pcg_rtol is the relative
    residual |r|/|b| at which PCG stops; the PCG preconditioner is block-Jacobi
    plus a rigid-motion coarse space over clusters of `coarse_cluster`
    consecutive free frames.
    """

    linear_solver: str = "auto"
    pcg_rtol: float = 1e-8       # tested to LM termination at configs[2] (tests/test_gpu_configs.py)
    pcg_max_iters: int = 2000
    dense_max_dim: int = 210
    coarse_cluster: int = 8      # frames per coarse cluster; < 0 = block-Jacobi only
    coarse_refresh: int = 8      # rebuild the coarse operator every N linearisations
    coarse_max_lambda: float = 1e-2  # above this damping: block-Jacobi only (S is diagonally dominant)
    coarse_drift: float = 4.0    # re-assemble A_c = P^T S(lambda) P when lambda moved by more than this
    # point-sharded ranks: 1 = row-partitioned PCG (one launch when the ranks
    # share a device, one launch per device meeting at a cross-launch barrier
    # in a multi-device context), 2 = per-rank launches on a shared device
    # too, 0 = the replicated PCG on the all-reduced S (separate processes)
    pcg_partition: int = 1


DEFAULT_DEVICE_OPTIONS = DeviceOptions()
