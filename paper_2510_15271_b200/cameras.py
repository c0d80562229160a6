"""Camera model record of the drop-in data model (cameras.py:35-54).

Only the parameters cross to the device; the projection / unprojection
arithmetic runs in csrc/sfm_math.cuh.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .se3 import Pose

PINHOLE = "pinhole"
PINHOLE_RADIAL = "pinhole_radial"
EQUIDISTANT_FISHEYE = "equidistant_fisheye"
KINDS = (PINHOLE, PINHOLE_RADIAL, EQUIDISTANT_FISHEYE)


@dataclass(frozen=True)
class CameraModel:
    kind: str
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    distortion: tuple = ()

    def __post_init__(self):
        if self.kind not in KINDS:
            raise ValueError(f"unknown camera kind {self.kind!r}")
        if self.fx <= 0 or self.fy <= 0:
            raise ValueError("focal lengths must be positive")
        object.__setattr__(self, "distortion", tuple(float(d) for d in self.distortion))
        if self.kind == PINHOLE_RADIAL and len(self.distortion) != 2:
            raise ValueError("pinhole_radial expects (k1, k2)")


@dataclass(frozen=True)
class RigCalibration:
    """Rigid multi-camera assembly (cameras.py:182-208)."""

    camera_ids: tuple
    cam_from_rig: dict = field(default_factory=dict)

    def __post_init__(self):
        object.__setattr__(self, "camera_ids", tuple(self.camera_ids))

    def extrinsic(self, camera_id) -> Pose:
        return self.cam_from_rig[camera_id]

    @property
    def reference_id(self):
        """The camera whose extrinsic is the identity (cameras.py:197-202)."""
        for cid in self.camera_ids:
            if self.cam_from_rig[cid].almost_equal(Pose.identity()):
                return cid
        raise ValueError("no reference camera")
