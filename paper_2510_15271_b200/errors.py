"""Exception classes of the hot path (mirror of sfmkit/errors.py:4-153).

The drop-in raises the same exception classes as the reference.  When the
reference package itself is importable (a user migrating from `sfmkit`),
its classes are used, so `except sfmkit.errors.NonPositiveDepth` keeps
working; otherwise the same-named classes defined here are used.
"""

from __future__ import annotations

import importlib


class SfmError(Exception):
    """Base class (errors.py:4)."""


class NonPositiveDepth(SfmError):
    """Point does not project: depth in the camera frame is <= 0 (errors.py:10)."""


class OutOfModelDomain(SfmError):
    """Point/pixel outside the camera model's domain (errors.py:14)."""


class UndistortDiverged(SfmError):
    """Iterative undistortion failed to converge (errors.py:18)."""


class SolverDiverged(SfmError):
    """Damping overflow (errors.py:78)."""


class SingularSystem(SfmError):
    """Normal equations could not be factored (errors.py:82)."""


class InsufficientParallax(SfmError):
    """Triangulation angle below the configured minimum (errors.py:98)."""


class CheiralityViolation(SfmError):
    """Triangulated point behind an observing camera (errors.py:102)."""


class ParallelRays(SfmError):
    """Midpoint triangulation: rays (numerically) parallel (errors.py:106)."""


class NoGauge(SfmError):
    """BA has neither a fixed pose nor absolute priors (errors.py:110)."""


_NAMES = ("SfmError", "NonPositiveDepth", "OutOfModelDomain", "UndistortDiverged",
          "SolverDiverged", "SingularSystem", "InsufficientParallax",
          "CheiralityViolation", "ParallelRays", "NoGauge")

try:  # migrate transparently: raise the reference's own classes when present
    _ref = importlib.import_module("sfmkit.errors")
    for _n in _NAMES:
        if hasattr(_ref, _n):
            globals()[_n] = getattr(_ref, _n)
except ImportError:
    _ref = None


def raise_for_code(code: int, message: str):
    """Maps a C-ABI return code onto the reference exception class."""
    from . import _native as n
    if code == n.SFM_E_NON_POSITIVE_DEPTH:
        raise NonPositiveDepth(message)
    if code == n.SFM_E_OUT_OF_MODEL_DOMAIN:
        raise OutOfModelDomain(message)
    if code == n.SFM_E_UNDISTORT_DIVERGED:
        raise UndistortDiverged(message)
    if code == n.SFM_E_SOLVER_DIVERGED:
        raise SolverDiverged(message)
    if code == n.SFM_E_NO_GAUGE:
        raise NoGauge(message)
    if code == n.SFM_E_INVALID:
        raise ValueError(message)
    if code == n.SFM_E_OOM:
        raise MemoryError(message)
    raise RuntimeError(f"libsfm_b200 error {code}: {message}")


def raise_for_tri_status(status: int):
    """Per-track status of sfm_triangulate -> the reference exception."""
    from . import _native as n
    if status == n.TRI_OK:
        return
    if status == n.TRI_INSUFFICIENT_PARALLAX:
        raise InsufficientParallax("max triangulation angle below threshold or point at infinity")
    if status == n.TRI_CHEIRALITY:
        raise CheiralityViolation("point behind camera")
    if status == n.TRI_PARALLEL_RAYS:
        raise ParallelRays("ray system ill-conditioned")
    if status == n.TRI_TOO_FEW_OBS:
        raise ValueError("need at least two observations")
    if status == n.TRI_CAMERA_ERROR:
        raise UndistortDiverged("unprojection failed")
    if status == n.TRI_CAMERA_DOMAIN:
        raise OutOfModelDomain("distorted radius beyond 90 deg")
    raise RuntimeError(f"triangulation status {status}")
