"""B200-native LM bundle adjustment + iterative triangulation (cuSfM mapping
core) behind the reference `sfmkit.mapping` entry points.

    from paper_2510_15271_b200 import bundle_adjust, iterative_map, ...

The compute path is libsfm_b200.so (hand-written sm_100a CUDA, C-ABI in
include/sfm_b200.h) called through ctypes; see DESIGN.md.
"""

from .cameras import CameraModel, RigCalibration
from .errors import (CheiralityViolation, InsufficientParallax, NoGauge, NonPositiveDepth,
                     OutOfModelDomain, ParallelRays, SfmError, SolverDiverged)
from .keyframes import Keyframe
from .mapping import (FAILED, LOCALIZATION_ADJUST, LOCALIZATION_FIXED, PENDING, PURE,
                      RIG_EXTRINSIC, TRIANGULATED, BAArrays, Landmark, MappingConfig,
                      Observation, SparseMap, StageConfig, Track, bundle_adjust, flatten_ba,
                      iterative_map, mean_reprojection_error, ransac_triangulate,
                      ransac_triangulate_batch, remove_outliers, reprojection_error,
                      shard_ranges, solve_arrays, triangulate_dlt, triangulate_midpoint)
from .se3 import Pose, exp_map, log_map
from .solver import DeviceOptions, RobustLoss, SolverOptions, SolverReport

__version__ = "0.1.0"
