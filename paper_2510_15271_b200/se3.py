"""Host-side rigid transforms for the drop-in data model.

Same conventions as the reference (se3.py:1-8): a Pose maps source-frame
points into its target frame (x' = R x + t), tangent vectors are (phi, rho),
perturbations act on the left, quaternions are unit (w, x, y, z) with the
canonical sign w >= 0.  The device restatement of these formulas lives in
csrc/sfm_math.cuh; this module only serves the Python object model
(keyframe poses, scene generation, write-back).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def canonical_quat(q) -> np.ndarray:
    """Unit quaternion with canonical sign (se3.py:20-29)."""
    q = np.asarray(q, dtype=float).reshape(4)
    n = np.linalg.norm(q)
    if n < 1e-12:
        raise ValueError("zero quaternion")
    q = q / n
    lead = q[0] if q[0] != 0 else next((c for c in q[1:] if c != 0), 0.0)
    return -q if lead < 0 else q


def quat_product(a, b) -> np.ndarray:
    aw, av = a[0], np.asarray(a[1:])
    bw, bv = b[0], np.asarray(b[1:])
    return np.concatenate(([aw * bw - av @ bv], aw * bv + bw * av + np.cross(av, bv)))


def rotation_matrix(q) -> np.ndarray:
    w, x, y, z = q
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
        [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
        [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
    ])


def hat(v) -> np.ndarray:
    return np.array([[0.0, -v[2], v[1]], [v[2], 0.0, -v[0]], [-v[1], v[0], 0.0]])


@dataclass(frozen=True)
class Pose:
    """Unit quaternion (w, x, y, z) + translation."""

    quat: np.ndarray = field(default_factory=lambda: np.array([1.0, 0.0, 0.0, 0.0]))
    t: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def __post_init__(self):
        object.__setattr__(self, "quat", canonical_quat(self.quat))
        object.__setattr__(self, "t", np.asarray(self.t, dtype=float).reshape(3))

    @staticmethod
    def identity():
        return Pose()

    @property
    def R(self) -> np.ndarray:
        return rotation_matrix(self.quat)

    def apply(self, x):
        return np.asarray(x, dtype=float) @ self.R.T + self.t

    def inverse(self) -> "Pose":
        qc = self.quat * np.array([1.0, -1.0, -1.0, -1.0])
        return Pose(qc, -(rotation_matrix(qc) @ self.t))

    def __matmul__(self, other: "Pose") -> "Pose":
        return Pose(quat_product(self.quat, other.quat), self.R @ other.t + self.t)

    def matrix(self) -> np.ndarray:
        T = np.eye(4)
        T[:3, :3], T[:3, 3] = self.R, self.t
        return T

    def almost_equal(self, other, tol=1e-9) -> bool:
        return float(np.linalg.norm(log_map(self.inverse() @ other))) < tol


def _so3_left_jacobian(phi, inverse=False):
    theta = np.linalg.norm(phi)
    P = hat(phi)
    if inverse:
        c = 1.0 / 12.0 if theta < 1e-6 else \
            1.0 / theta ** 2 - (1.0 + np.cos(theta)) / (2.0 * theta * np.sin(theta))
        return np.eye(3) - 0.5 * P + c * (P @ P)
    if theta < 1e-6:
        a, b = 0.5, 1.0 / 6.0
    else:
        a = (1.0 - np.cos(theta)) / theta ** 2
        b = (theta - np.sin(theta)) / theta ** 3
    return np.eye(3) + a * P + b * (P @ P)


def exp_map(xi) -> Pose:
    """SE(3) exponential of (phi, rho) (se3.py:190-194)."""
    xi = np.asarray(xi, dtype=float)
    phi, rho = xi[:3], xi[3:]
    theta = np.linalg.norm(phi)
    half = 0.5 * theta
    if theta < 1e-8:
        w, s = 1.0 - half * half / 2.0, 0.5 - half * half / 12.0
    else:
        w, s = np.cos(half), np.sin(half) / theta
    return Pose(np.concatenate(([w], s * phi)), _so3_left_jacobian(phi) @ rho)


def log_map(p: Pose) -> np.ndarray:
    """Inverse of exp_map (se3.py:157-168, :197-201)."""
    w, v = p.quat[0], p.quat[1:]
    n = np.linalg.norm(v)
    phi = 2.0 * v if n < 1e-10 else (2.0 * np.arctan2(n, w) / n) * v
    return np.concatenate([phi, _so3_left_jacobian(phi, inverse=True) @ p.t])


def compose(a: Pose, b: Pose) -> Pose:
    return a @ b
