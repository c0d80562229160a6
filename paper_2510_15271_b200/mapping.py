"""Drop-in for sfmkit.mapping's hot path, executed on the B200.

Same names, signatures, defaults, in-place mutations, reports and exception
classes as the reference module (/root/reference/pkg/src/sfmkit/mapping.py):

    bundle_adjust          mapping.py:390-527   -> sfm_ba_solve
    ransac_triangulate     mapping.py:255-305   -> sfm_ransac_triangulate
    triangulate_dlt        mapping.py:194-221   -> sfm_triangulate (DLT)
    triangulate_midpoint   mapping.py:224-240   -> sfm_triangulate (midpoint)
    reprojection_error     mapping.py:243-252   -> sfm_reprojection_errors
    remove_outliers        mapping.py:544-566   -> sfm_gate
    iterative_map          mapping.py:569-624   (host loop, batched device calls)
    mean_reprojection_error mapping.py:627-636  -> sfm_reprojection_errors

This module only flattens the object model into the C-ABI's arrays and maps
results and error codes back; every floating-point operation of the path
runs in libsfm_b200.so.  Objects from the reference package are accepted
(duck typing) and written back with their own types.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from itertools import chain
from operator import attrgetter

import numpy as np

from . import _native as nat
from .cameras import CameraModel
from .errors import NoGauge, raise_for_tri_status
from .keyframes import ROLLING_SHUTTER, Keyframe
from .se3 import Pose
from .solver import (DEFAULT_DEVICE_OPTIONS, RobustLoss, SolverOptions, SolverReport,
                     TRIVIAL_LOSS, DeviceOptions)

PENDING = "pending"
TRIANGULATED = "triangulated"
FAILED = "failed"

PURE = "pure"
LOCALIZATION_FIXED = "localization_fixed"
LOCALIZATION_ADJUST = "localization_adjust"
RIG_EXTRINSIC = "rig_extrinsic"


# --- object model (mapping.py:30-108) ---------------------------------------

@dataclass
class Observation:
    frame_id: int
    feature_index: int
    pixel: np.ndarray

    def __post_init__(self):
        self.pixel = np.asarray(self.pixel, dtype=float).reshape(2)


@dataclass
class Track:
    observations: list
    status: str = PENDING

    def __post_init__(self):
        if len(self.observations) < 2:
            raise ValueError("tracks need at least two observations")
        frames = [o.frame_id for o in self.observations]
        if len(set(frames)) != len(frames):
            raise ValueError("duplicate frame in track")


@dataclass
class Landmark:
    position: np.ndarray
    track: Track
    inlier_mask: np.ndarray

    def __post_init__(self):
        self.position = np.asarray(self.position, dtype=float).reshape(3)
        self.inlier_mask = np.asarray(self.inlier_mask, dtype=bool)

    def inlier_observations(self):
        return [o for o, ok in zip(self.track.observations, self.inlier_mask) if ok]


@dataclass
class SparseMap:
    keyframes: dict
    cameras: dict
    landmarks: list = field(default_factory=list)
    rig: object = None
    provenance: dict = field(default_factory=dict)
    fixed_frames: set = field(default_factory=set)

    def camera_of(self, frame_id):
        return self.cameras[self.keyframes[frame_id].camera_id]

    def pose_of(self, frame_id) -> Pose:
        return self.keyframes[frame_id].cam_from_world


@dataclass
class StageConfig:
    outlier_px: float
    loss: RobustLoss = TRIVIAL_LOSS


@dataclass
class MappingConfig:
    stage1: StageConfig = field(
        default_factory=lambda: StageConfig(4.0, RobustLoss("huber", 2.0)))
    stage2: StageConfig = field(default_factory=lambda: StageConfig(2.0))
    lambda_c: float = 1.0
    lambda_a: float = 1.0
    extrinsic_prior_weight: float = 1.0
    max_outer_iters: int = 10
    min_triangulation_angle: float = float(np.radians(0.5))
    triangulation: str = "dlt"
    seed: int = 42
    max_solver_iters: int = 50

    def __post_init__(self):
        if self.stage2.outlier_px > self.stage1.outlier_px:
            raise ValueError("stage 2 threshold must not exceed stage 1")
        if min(self.lambda_c, self.lambda_a) < 0:
            raise ValueError("weights must be non-negative")


# --- flattened arrays --------------------------------------------------------

def camera_struct(cam) -> nat.CameraModelC:
    k1, k2 = (tuple(cam.distortion) + (0.0, 0.0))[:2]
    return nat.CameraModelC(nat.CAM_KINDS[cam.kind], int(cam.width), int(cam.height), 0,
                            float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy),
                            float(k1), float(k2))


def model_table(cams_per_frame):
    """Unique camera models -> (ctypes array, per-frame model index)."""
    models, index, fm = [], {}, []
    for cam in cams_per_frame:
        key = id(cam)
        if key not in index:
            index[key] = len(models)
            models.append(cam)
        fm.append(index[key])
    arr = (nat.CameraModelC * max(len(models), 1))(*[camera_struct(c) for c in models])
    return arr, len(models), np.asarray(fm, dtype=np.int32)


@dataclass
class BAArrays:
    """The C-ABI's sfm_ba_problem as numpy arrays (include/sfm_b200.h)."""

    cam_q: np.ndarray          # [F,4]
    cam_t: np.ndarray          # [F,3]
    frame_model: np.ndarray    # [F] i32
    frame_fixed: np.ndarray    # [F] u8
    models: object             # ctypes array of CameraModelC
    n_models: int
    points: np.ndarray         # [P,3]
    obs_frame: np.ndarray      # [N] i32
    obs_point: np.ndarray      # [N] i32, non-decreasing
    obs_uv: np.ndarray         # [N,2]
    edge_ab: np.ndarray        # [E,2] i32
    prior_frame: np.ndarray    # [A] i32
    edge_weight: float = 0.0
    prior_weight: float = 0.0
    obs_offset: int = 0
    n_params_global: int = 0

    def struct(self) -> nat.BAProblemC:
        self._keep = [self.cam_q, self.cam_t, self.frame_model, self.frame_fixed, self.points,
                      self.obs_frame, self.obs_point, self.obs_uv, self.edge_ab, self.prior_frame]
        return nat.BAProblemC(
            len(self.frame_model), self.n_models, nat.ptr(self.cam_q), nat.ptr(self.cam_t),
            nat.ptr(self.frame_model), nat.ptr(self.frame_fixed), ctypes.addressof(self.models),
            len(self.points), nat.ptr(self.points), len(self.obs_frame), nat.ptr(self.obs_frame),
            nat.ptr(self.obs_point), nat.ptr(self.obs_uv), len(self.edge_ab), len(self.prior_frame),
            nat.ptr(self.edge_ab), nat.ptr(self.prior_frame), float(self.edge_weight),
            float(self.prior_weight), int(self.obs_offset), int(self.n_params_global))

    def shard(self, rank: int, world: int) -> "BAArrays":
        """Point-sharded slice for `rank` (contiguous points balanced by
        observation count); pose terms stay on rank 0 only."""
        p0, p1 = shard_ranges(self.obs_point, len(self.points), world)[rank]
        o0, o1 = np.searchsorted(self.obs_point, [p0, p1])
        n_free = int((self.frame_fixed == 0).sum())
        return BAArrays(
            self.cam_q, self.cam_t, self.frame_model, self.frame_fixed, self.models, self.n_models,
            np.ascontiguousarray(self.points[p0:p1]), np.ascontiguousarray(self.obs_frame[o0:o1]),
            np.ascontiguousarray(self.obs_point[o0:o1] - p0, dtype=np.int32),
            np.ascontiguousarray(self.obs_uv[o0:o1]),
            self.edge_ab if rank == 0 else np.zeros((0, 2), np.int32),
            self.prior_frame if rank == 0 else np.zeros(0, np.int32),
            self.edge_weight, self.prior_weight, int(o0),
            6 * n_free + 3 * len(self.points))


def shard_ranges(obs_point, n_points: int, world: int):
    """Contiguous point ranges with (near) equal observation counts
    (SURVEY.md §8e): boundaries at the points where the running observation
    count crosses r*N/world."""
    obs_point = np.asarray(obs_point)
    n = len(obs_point)
    ptr = np.searchsorted(obs_point, np.arange(n_points + 1))
    bounds = [0]
    for r in range(1, world):
        target = (r * n) // world
        p = int(np.searchsorted(ptr, target, side="left"))
        bounds.append(min(max(p, bounds[-1]), n_points))
    bounds.append(n_points)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def _options(loss: RobustLoss, sopt: SolverOptions, dopt: DeviceOptions) -> nat.BAOptionsC:
    return nat.BAOptionsC(nat.LOSS_KINDS[loss.kind], int(sopt.max_iters), float(loss.param),
                          float(sopt.grad_tol), float(sopt.param_tol), float(sopt.initial_lambda),
                          float(sopt.max_lambda), nat.LINSOLVE[dopt.linear_solver],
                          int(dopt.pcg_max_iters), float(dopt.pcg_rtol), int(dopt.dense_max_dim),
                          int(dopt.coarse_cluster), int(dopt.coarse_refresh),
                          float(dopt.coarse_max_lambda), float(dopt.coarse_drift),
                          int(dopt.pcg_partition), 0)


def solve_arrays(arrays: BAArrays, loss: RobustLoss = TRIVIAL_LOSS,
                 options: SolverOptions = None, device: DeviceOptions = None, ctx=None,
                 out=None):
    """sfm_ba_solve on flattened arrays -> (cam_q, cam_t, points, report, raw).
    `out` = (cam_q, cam_t, points) C-contiguous fp64 arrays to write the
    result into (e.g. pinned host memory); fresh arrays otherwise.  The
    library writes every entry (fixed frames copied bit-identically)."""
    ctx = ctx or nat.default_context()
    options = options or SolverOptions()
    device = device or DEFAULT_DEVICE_OPTIONS
    prob = arrays.struct()
    opt = _options(loss, options, device)
    if out is not None:
        q, t, X = out
        assert q.shape == arrays.cam_q.shape and t.shape == arrays.cam_t.shape
        assert X.shape == arrays.points.shape
    else:
        q = np.empty(arrays.cam_q.shape, dtype=np.float64)
        t = np.empty(arrays.cam_t.shape, dtype=np.float64)
        X = np.empty(arrays.points.shape, dtype=np.float64)
    rep = nat.BAReportC()
    ctx.check(ctx.lib.sfm_ba_solve(ctx.handle, ctypes.byref(prob), ctypes.byref(opt),
                                   nat.ptr(q), nat.ptr(t), nat.ptr(X), ctypes.byref(rep)))
    report = SolverReport(rep.initial_cost, rep.final_cost, rep.iterations,
                          nat.TERMINATIONS[rep.termination])
    return q, t, X, report, rep


def _next_same_camera(sparse_map):
    """frame_id -> next keyframe of the same camera by timestamp
    (mapping.py:530-541)."""
    by_cam = {}
    for f in sorted(sparse_map.keyframes):
        kf = sparse_map.keyframes[f]
        by_cam.setdefault(kf.camera_id, []).append(kf)
    nxt = {}
    for seq in by_cam.values():
        seq.sort(key=lambda k: k.timestamp)
        for a, b in zip(seq, seq[1:]):
            nxt[a.frame_id] = b
    return nxt


def _shutter_alpha(kf, next_kf, pixel_row, height):
    """Scanline interpolation fraction (mapping.py:379-387), None = global."""
    if next_kf is None or kf.shutter != ROLLING_SHUTTER:
        return None
    s = pixel_row / max(height - 1, 1)
    dt = next_kf.timestamp - kf.timestamp
    if dt <= 0:
        return None
    return float(np.clip(s * kf.exposure / dt, 0.0, 1.0))


def _needs_general(sparse_map, frames, mode):
    """True when the residuals are not all global-shutter single-pose ones:
    rig_extrinsic mode, or a rolling-shutter keyframe with a successor."""
    if mode == RIG_EXTRINSIC:
        return True
    nxt = _next_same_camera(sparse_map)
    for f in frames:
        kf = sparse_map.keyframes[f]
        if kf.shutter == ROLLING_SHUTTER and f in nxt and nxt[f].timestamp - kf.timestamp > 0:
            return True
    return False


def _check_supported(sparse_map, frames, mode):
    """The single-slot fast path (and the device-resident iterative_map)
    takes global-shutter, non-rig problems; bundle_adjust routes the rest
    to the general path (sfm_gba_solve)."""
    if _needs_general(sparse_map, frames, mode):
        raise NotImplementedError("rig / rolling-shutter residuals: use bundle_adjust "
                                  "(general two-slot path)")


_get_track = attrgetter("track")
_get_observations = attrgetter("observations")
_get_inlier_mask = attrgetter("inlier_mask")
_get_frame_id = attrgetter("frame_id")
_get_pixel = attrgetter("pixel")
_get_position = attrgetter("position")


def flatten_ba(sparse_map, config, stage=1, mode=PURE):
    """SparseMap -> (BAArrays, frames, landmark indices, loss).

    Follows the problem construction of mapping.py:399-509: frames sorted,
    fixed set (+ prior frames in localization_fixed), NoGauge check, points
    = TRIANGULATED landmarks in map order, observations = inlier obs,
    landmark-major in track order, lambda_c edges between consecutive frames
    of each camera, lambda_a priors on non-fixed frames (PURE skips prior
    provenance)."""
    loss = config.stage1.loss if stage == 1 else config.stage2.loss
    frames = sorted(sparse_map.keyframes)
    fixed = set(sparse_map.fixed_frames)
    if mode == LOCALIZATION_FIXED:
        fixed |= {f for f in frames if sparse_map.provenance.get(f) == "prior"}
    if mode != RIG_EXTRINSIC and not fixed and config.lambda_a <= 0:
        raise NoGauge("no fixed pose and no absolute prior")
    _check_supported(sparse_map, frames, mode)
    fidx = {f: i for i, f in enumerate(frames)}
    F = len(frames)
    cam_q = np.empty((F, 4))
    cam_t = np.empty((F, 3))
    for i, f in enumerate(frames):
        pose = sparse_map.keyframes[f].cam_from_world
        cam_q[i] = pose.quat
        cam_t[i] = pose.t
    models, n_models, fm = model_table([sparse_map.cameras[sparse_map.keyframes[f].camera_id]
                                        for f in frames])
    fixed_arr = np.array([1 if f in fixed else 0 for f in frames], dtype=np.uint8)
    lms = [li for li, lm in enumerate(sparse_map.landmarks) if lm.track.status == TRIANGULATED]
    sel = [sparse_map.landmarks[li] for li in lms]
    points = np.array(list(map(_get_position, sel)), dtype=np.float64).reshape(-1, 3)
    # inlier observations, landmark-major in track order (mapping.py:452-475),
    # gathered with one pass over the objects and numpy for the rest
    # (attribute getters mapped in C: the per-object Python work is the cost here)
    tracks = list(map(_get_track, sel))
    obs_lists = list(map(_get_observations, tracks))
    allobs = list(chain.from_iterable(obs_lists))
    counts = np.fromiter(map(len, obs_lists), dtype=np.int64, count=len(sel))
    keep = (np.concatenate(list(map(_get_inlier_mask, sel))).astype(bool, copy=False)
            if sel else np.zeros(0, bool))
    fids = np.fromiter(map(_get_frame_id, allobs), dtype=np.int64, count=len(allobs))
    frame_arr = np.asarray(frames, dtype=np.int64)
    at = np.searchsorted(frame_arr, fids)
    bad = (at >= len(frame_arr)) | (frame_arr[np.minimum(at, max(len(frame_arr) - 1, 0))] != fids) \
        if len(frame_arr) else np.ones(len(fids), bool)
    if np.any(bad & keep):
        raise KeyError(int(fids[np.flatnonzero(bad & keep)[0]]))
    pix = (np.array(list(map(_get_pixel, allobs)), dtype=np.float64).reshape(-1, 2) if allobs
           else np.zeros((0, 2)))
    of = at[keep]
    op = np.repeat(np.arange(len(sel), dtype=np.int64), counts)[keep]
    uv = pix[keep]
    edges = []
    if config.lambda_c > 0:
        by_cam = {}
        for f in frames:
            by_cam.setdefault(sparse_map.keyframes[f].camera_id, []).append(f)
        for seq in by_cam.values():
            edges.extend((fidx[a], fidx[b]) for a, b in zip(seq, seq[1:]))
    priors = []
    if config.lambda_a > 0:
        for f in frames:
            if f in fixed:
                continue
            if mode == PURE and sparse_map.provenance.get(f) == "prior":
                continue
            priors.append(fidx[f])
    arrays = BAArrays(
        cam_q, cam_t, fm, fixed_arr, models, n_models, np.ascontiguousarray(points),
        np.asarray(of, dtype=np.int32), np.asarray(op, dtype=np.int32),
        np.asarray(uv, dtype=np.float64).reshape(-1, 2),
        np.asarray(edges, dtype=np.int32).reshape(-1, 2), np.asarray(priors, dtype=np.int32),
        float(config.lambda_c), float(config.lambda_a))
    return arrays, frames, lms, loss


def bundle_adjust(sparse_map, config: MappingConfig = None, stage: int = 1, mode: str = PURE,
                  device: DeviceOptions = None, ctx=None):
    """mapping.py:390-527 on the B200.  Returns the SolverReport; poses and
    TRIANGULATED landmark positions are written back in place.  With a
    multi-rank context (ctx.world > 1, one process per GPU) the points are
    sharded across ranks and the camera system is all-reduced over NCCL."""
    if config is None:
        config = MappingConfig()
    if _needs_general(sparse_map, sorted(sparse_map.keyframes), mode):
        return _bundle_adjust_general(sparse_map, config, stage, mode, device, ctx)
    arrays, frames, lms, loss = flatten_ba(sparse_map, config, stage, mode)
    ctx = ctx or nat.default_context()
    sopt = SolverOptions(max_iters=config.max_solver_iters)
    if ctx.world > 1:
        q, t, X, report, _ = _solve_sharded(arrays, loss, sopt, device, ctx)
    else:
        q, t, X, report, _ = solve_arrays(arrays, loss, sopt, device, ctx)
    for i, f in enumerate(frames):
        if arrays.frame_fixed[i]:
            continue  # fixed blocks keep their (byte-identical) value
        if np.array_equal(q[i], arrays.cam_q[i]) and np.array_equal(t[i], arrays.cam_t[i]):
            continue  # never retracted: keep the entry object
        kf = sparse_map.keyframes[f]
        kf.cam_from_world = type(kf.cam_from_world)(q[i], t[i])
    # each landmark gets its own row of the (private) result array: views made
    # in C, not a Python-level copy per landmark
    landmarks = sparse_map.landmarks
    for li, row in zip(lms, list(X)):
        landmarks[li].position = row
    return report


def _bundle_adjust_general(sparse_map, config, stage, mode, device, ctx):
    """bundle_adjust (mapping.py:390-527) for rig_extrinsic mode and rolling-
    shutter keyframes: residuals over one or two SE(3) blocks, solved on the
    device by sfm_gba_solve.  Same problem construction, write-back and
    report as the reference."""
    loss = config.stage1.loss if stage == 1 else config.stage2.loss
    frames = sorted(sparse_map.keyframes)
    fixed = set(sparse_map.fixed_frames)
    if mode == LOCALIZATION_FIXED:
        fixed |= {f for f in frames if sparse_map.provenance.get(f) == "prior"}
    rig_mode = mode == RIG_EXTRINSIC
    if not rig_mode and not fixed and config.lambda_a <= 0:
        raise NoGauge("no fixed pose and no absolute prior")
    kfs = sparse_map.keyframes
    bq, bt, bfix = [], [], []
    edges, ew, priors, pw = [], [], [], []
    if rig_mode:
        if sparse_map.rig is None:
            raise NoGauge("rig_extrinsic mode needs a rig calibration")
        rig = sparse_map.rig
        instants = sorted({kfs[f].timestamp for f in frames})
        instant_id = {tm: i for i, tm in enumerate(instants)}
        vehicle_entry = {}
        for f in frames:
            i = instant_id[kfs[f].timestamp]
            if i not in vehicle_entry:
                vehicle_entry[i] = rig.extrinsic(kfs[f].camera_id).inverse() @ kfs[f].cam_from_world
        vids = sorted(vehicle_entry)
        vblock = {i: k for k, i in enumerate(vids)}
        for i in vids:
            bq.append(vehicle_entry[i].quat)
            bt.append(vehicle_entry[i].t)
            bfix.append(1 if i == 0 else 0)
        eblock = {}
        ref_id = rig.reference_id
        for cid in rig.camera_ids:
            eblock[cid] = len(bq)
            bq.append(rig.extrinsic(cid).quat)
            bt.append(rig.extrinsic(cid).t)
            bfix.append(1 if cid == ref_id else 0)
            if cid != ref_id and config.extrinsic_prior_weight > 0:
                priors.append(eblock[cid])
                pw.append(float(config.extrinsic_prior_weight))
        if config.lambda_c > 0:
            for a, b in zip(vids, vids[1:]):
                edges.append((vblock[a], vblock[b]))
                ew.append(float(config.lambda_c))
    else:
        fidx = {f: i for i, f in enumerate(frames)}
        for f in frames:
            bq.append(kfs[f].cam_from_world.quat)
            bt.append(kfs[f].cam_from_world.t)
            bfix.append(1 if f in fixed else 0)
        e_arr, p_arr = _pose_terms(frames, fidx, sparse_map, config, fixed, mode)
        edges = [tuple(e) for e in e_arr]
        ew = [float(config.lambda_c)] * len(edges)
        priors = list(p_arr)
        pw = [float(config.lambda_a)] * len(priors)
        next_of = _next_same_camera(sparse_map)
    cams = sorted({kfs[f].camera_id for f in frames})
    cam_models = [sparse_map.cameras[c] for c in cams]
    models, n_models, cam_model_idx = model_table(cam_models)
    model_of_cam = {c: int(cam_model_idx[k]) for k, c in enumerate(cams)}
    lms = [li for li, lm in enumerate(sparse_map.landmarks) if lm.track.status == TRIANGULATED]
    pts = np.array([sparse_map.landmarks[li].position for li in lms], dtype=np.float64).reshape(-1, 3)
    rp, rm, rk, rs, ra, ruv = [], [], [], [], [], []
    for pi, li in enumerate(lms):
        lm = sparse_map.landmarks[li]
        for o in lm.inlier_observations():
            kf = kfs[o.frame_id]
            rp.append(pi)
            rm.append(model_of_cam[kf.camera_id])
            ruv.append(o.pixel)
            if rig_mode:
                rk.append(nat.RES_RIG)
                rs.append((vblock[instant_id[kf.timestamp]], eblock[kf.camera_id]))
                ra.append(0.0)
                continue
            cam = sparse_map.cameras[kf.camera_id]
            alpha = _shutter_alpha(kf, next_of.get(o.frame_id), o.pixel[1], cam.height)
            if alpha is None:
                rk.append(nat.RES_GLOBAL)
                rs.append((fidx[o.frame_id], -1))
                ra.append(0.0)
            else:
                rk.append(nat.RES_ROLLING)
                rs.append((fidx[o.frame_id], fidx[next_of[o.frame_id].frame_id]))
                ra.append(alpha)
    keep = dict(
        bq=np.ascontiguousarray(np.array(bq, dtype=np.float64).reshape(-1, 4)),
        bt=np.ascontiguousarray(np.array(bt, dtype=np.float64).reshape(-1, 3)),
        bf=np.ascontiguousarray(np.array(bfix, dtype=np.uint8)), pts=np.ascontiguousarray(pts),
        rp=np.ascontiguousarray(np.array(rp, dtype=np.int32)),
        rm=np.ascontiguousarray(np.array(rm, dtype=np.int32)),
        rk=np.ascontiguousarray(np.array(rk, dtype=np.int32)),
        rs=np.ascontiguousarray(np.array(rs, dtype=np.int32).reshape(-1, 2)),
        ra=np.ascontiguousarray(np.array(ra, dtype=np.float64)),
        ruv=np.ascontiguousarray(np.array(ruv, dtype=np.float64).reshape(-1, 2)),
        eab=np.ascontiguousarray(np.array(edges, dtype=np.int32).reshape(-1, 2)),
        ew=np.ascontiguousarray(np.array(ew, dtype=np.float64)),
        pb=np.ascontiguousarray(np.array(priors, dtype=np.int32)),
        pw=np.ascontiguousarray(np.array(pw, dtype=np.float64)))
    prob = nat.GbaProblemC(
        len(keep["bf"]), n_models, nat.ptr(keep["bq"]), nat.ptr(keep["bt"]), nat.ptr(keep["bf"]),
        ctypes.addressof(models), len(keep["pts"]), nat.ptr(keep["pts"]), len(keep["rp"]),
        nat.ptr(keep["rp"]), nat.ptr(keep["rm"]), nat.ptr(keep["rk"]), nat.ptr(keep["rs"]),
        nat.ptr(keep["ra"]), nat.ptr(keep["ruv"]), len(keep["eab"]), len(keep["pb"]),
        nat.ptr(keep["eab"]), nat.ptr(keep["ew"]), nat.ptr(keep["pb"]), nat.ptr(keep["pw"]))
    opt = _options(loss, SolverOptions(max_iters=config.max_solver_iters),
                   device or DEFAULT_DEVICE_OPTIONS)
    q = keep["bq"].copy()
    t = keep["bt"].copy()
    X = keep["pts"].copy()
    rep = nat.BAReportC()
    ctx = ctx or nat.default_context()
    ctx.check(ctx.lib.sfm_gba_solve(ctx.handle, ctypes.byref(prob), ctypes.byref(opt), nat.ptr(q),
                                    nat.ptr(t), nat.ptr(X), ctypes.byref(rep)))
    pose_type = type(kfs[frames[0]].cam_from_world) if frames else Pose
    if rig_mode:
        new_extr = {cid: pose_type(q[eblock[cid]], t[eblock[cid]]) for cid in rig.camera_ids}
        sparse_map.rig = type(rig)(rig.camera_ids, new_extr)
        for f in frames:
            kf = kfs[f]
            k = vblock[instant_id[kf.timestamp]]
            kf.cam_from_world = new_extr[kf.camera_id] @ pose_type(q[k], t[k])
    else:
        for i, f in enumerate(frames):
            if bfix[i]:
                continue
            if np.array_equal(q[i], keep["bq"][i]) and np.array_equal(t[i], keep["bt"][i]):
                continue
            kfs[f].cam_from_world = pose_type(q[i], t[i])
    for pi, li in enumerate(lms):
        sparse_map.landmarks[li].position = X[pi].copy()
    return SolverReport(rep.initial_cost, rep.final_cost, rep.iterations,
                        nat.TERMINATIONS[rep.termination])


def _solve_sharded(arrays, loss, sopt, device, ctx):
    import torch.distributed as dist
    part = arrays.shard(ctx.rank, ctx.world)
    q, t, Xs, report, rep = solve_arrays(part, loss, sopt, device, ctx)
    gathered = [None] * ctx.world
    dist.all_gather_object(gathered, Xs)
    return q, t, np.concatenate(gathered, axis=0), report, rep


def solve_sharded_emulated(arrays: BAArrays, loss: RobustLoss = TRIVIAL_LOSS,
                           options: SolverOptions = None, device: DeviceOptions = None,
                           n_shards: int = 2, ctx=None):
    """The point-sharded multi-GPU solve with `n_shards` logical ranks on one
    device (sfm_ba_solve_emulated): the same shards (BAArrays.shard) and the
    same per-rank control flow and collectives as the NCCL path, the
    collectives run as fixed-rank-order reductions.  -> (cam_q, cam_t,
    points, report, raw)."""
    ctx = ctx or nat.default_context()
    options = options or SolverOptions()
    parts = [arrays.shard(r, n_shards) for r in range(n_shards)]
    structs = (nat.BAProblemC * n_shards)(*[p.struct() for p in parts])
    Xs = [np.array(p.points, dtype=np.float64, copy=True) for p in parts]
    ptrs = (ctypes.c_void_p * n_shards)(*[nat.ptr(x) for x in Xs])
    q = np.array(arrays.cam_q, dtype=np.float64, copy=True)
    t = np.array(arrays.cam_t, dtype=np.float64, copy=True)
    rep = nat.BAReportC()
    opt = _options(loss, options, device or DEFAULT_DEVICE_OPTIONS)
    ctx.check(ctx.lib.sfm_ba_solve_emulated(ctx.handle, n_shards, ctypes.addressof(structs),
                                            ctypes.byref(opt), nat.ptr(q), nat.ptr(t),
                                            ctypes.addressof(ptrs), ctypes.byref(rep)))
    report = SolverReport(rep.initial_cost, rep.final_cost, rep.iterations,
                          nat.TERMINATIONS[rep.termination])
    return q, t, np.concatenate(Xs, axis=0), report, rep


# --- tracks ------------------------------------------------------------------

def build_tracks_arrays(pair_frames, pair_ptr, match_index):
    """build_tracks (mapping.py:113-161) on arrays through the host-native
    sfm_build_tracks -> (track_ptr, obs_frame, obs_feature)."""
    lib = nat.load_library()
    pf = np.ascontiguousarray(pair_frames, dtype=np.int32).reshape(-1, 2)
    pp = np.ascontiguousarray(pair_ptr, dtype=np.int64)
    mi = np.ascontiguousarray(match_index, dtype=np.int32).reshape(-1, 2)
    nm = len(mi)
    tp = np.empty(nm + 1, np.int64)
    of = np.empty(max(2 * nm, 1), np.int32)
    fi = np.empty(max(2 * nm, 1), np.int32)
    nt, no = ctypes.c_int64(), ctypes.c_int64()
    rc = lib.sfm_build_tracks(len(pf), nat.ptr(pf), nat.ptr(pp), nat.ptr(mi), nat.ptr(tp), nat.ptr(of),
                              nat.ptr(fi), ctypes.byref(nt), ctypes.byref(no))
    if rc != nat.SFM_OK:
        from .errors import raise_for_code
        raise_for_code(rc, "sfm_build_tracks: invalid pair / match arrays")
    return tp[:nt.value + 1].copy(), of[:no.value].copy(), fi[:no.value].copy()


def build_tracks(pair_matches, features_by_frame):
    """mapping.py:113-161: connected components of the feature-match graph,
    split on conflicts -> Tracks (PENDING) in the reference's order."""
    keys = list(pair_matches)
    pf = np.array(keys, dtype=np.int32).reshape(-1, 2)
    counts = [len(pair_matches[k]) for k in keys]
    pp = np.zeros(len(keys) + 1, np.int64)
    np.cumsum(counts, out=pp[1:])
    mi = np.array([(m.index_a, m.index_b) for k in keys for m in pair_matches[k]],
                  dtype=np.int32).reshape(-1, 2)
    tp, of, fi = build_tracks_arrays(pf, pp, mi)
    tracks = []
    for t in range(len(tp) - 1):
        obs = []
        for o in range(tp[t], tp[t + 1]):
            kp = features_by_frame[int(of[o])].keypoints[int(fi[o])]
            obs.append(Observation(int(of[o]), int(fi[o]), (kp.x, kp.y)))
        tracks.append(Track(obs))
    return tracks

class TrackArrays:
    """Tracks as CSR over a frame table (sfm_tracks)."""

    def __init__(self, obs_lists, poses, cameras, active=None):
        frames = sorted(poses)
        self.fidx = {f: i for i, f in enumerate(frames)}
        F = len(frames)
        self.cam_q = np.empty((F, 4))
        self.cam_t = np.empty((F, 3))
        for i, f in enumerate(frames):
            self.cam_q[i] = poses[f].quat
            self.cam_t[i] = poses[f].t
        self.models, self.n_models, self.fm = model_table([cameras[f] for f in frames])
        counts = np.fromiter((len(o) for o in obs_lists), dtype=np.int64, count=len(obs_lists))
        self.ptr = np.zeros(len(obs_lists) + 1, dtype=np.int64)
        np.cumsum(counts, out=self.ptr[1:])
        n = int(self.ptr[-1])
        self.obs_frame = np.fromiter((self.fidx[o.frame_id] for obs in obs_lists for o in obs),
                                     dtype=np.int32, count=n)
        self.obs_uv = np.array([o.pixel for obs in obs_lists for o in obs],
                               dtype=np.float64).reshape(-1, 2)
        self.active = None if active is None else np.asarray(active, dtype=np.uint8)

    def struct(self) -> nat.TracksC:
        return nat.TracksC(len(self.fm), self.n_models, nat.ptr(self.cam_q), nat.ptr(self.cam_t),
                           nat.ptr(self.fm), ctypes.addressof(self.models), len(self.ptr) - 1,
                           len(self.obs_frame), nat.ptr(self.ptr), nat.ptr(self.obs_frame),
                           nat.ptr(self.obs_uv), nat.ptr(self.active))


def _tri_call(observations, poses, cameras, method, min_angle, ctx):
    if len(observations) < 2:
        raise ValueError("need at least two observations")
    ctx = ctx or nat.default_context()
    ta = TrackArrays([list(observations)], poses, cameras)
    X = np.empty((1, 3))
    st = np.empty(1, dtype=np.int8)
    s = ta.struct()
    ctx.check(ctx.lib.sfm_triangulate(ctx.handle, ctypes.byref(s), float(min_angle),
                                      nat.tri_method(method), nat.ptr(X), nat.ptr(st)))
    raise_for_tri_status(int(st[0]))
    return X[0].copy()


def triangulate_dlt(observations, poses, cameras, min_angle=np.radians(0.5), ctx=None):
    """mapping.py:194-221 on device."""
    return _tri_call(observations, poses, cameras, "dlt", min_angle, ctx)


def triangulate_midpoint(observations, poses, cameras, ctx=None):
    """mapping.py:224-240 on device (no parallax gate, as in the reference)."""
    return _tri_call(observations, poses, cameras, "midpoint", 0.0, ctx)


def ransac_triangulate_batch(tracks, poses, cameras, threshold_px=4.0,
                             min_angle=np.radians(0.5), method="dlt", ctx=None):
    """Batched ransac_triangulate over `tracks` in one device call.  Sets each
    track's status and returns the list of Landmark-or-None in track order."""
    ctx = ctx or nat.default_context()
    if not tracks:
        return []
    ta = TrackArrays([t.observations for t in tracks], poses, cameras)
    T = len(tracks)
    X = np.empty((T, 3))
    mask = np.empty(len(ta.obs_frame), dtype=np.uint8)
    st = np.empty(T, dtype=np.int8)
    s = ta.struct()
    ctx.check(ctx.lib.sfm_ransac_triangulate(ctx.handle, ctypes.byref(s), float(threshold_px),
                                             float(min_angle), nat.tri_method(method), nat.ptr(X),
                                             nat.ptr(mask), nat.ptr(st)))
    out = []
    for i, tr in enumerate(tracks):
        if st[i] == nat.TRI_OK:
            tr.status = TRIANGULATED
            m = mask[ta.ptr[i]:ta.ptr[i + 1]].astype(bool)
            out.append(Landmark(X[i].copy(), tr, m))
        else:
            tr.status = FAILED
            out.append(None)
    return out


def ransac_triangulate(track, poses, cameras, threshold_px=4.0, min_angle=np.radians(0.5),
                       method="dlt", seed=42, ctx=None):
    """mapping.py:255-305 on device (`seed` is unused, as in the reference)."""
    return ransac_triangulate_batch([track], poses, cameras, threshold_px, min_angle, method,
                                    ctx)[0]


def _reproj_errors(obs_lists, positions, poses, cameras, ctx):
    ctx = ctx or nat.default_context()
    ta = TrackArrays(obs_lists, poses, cameras)
    P = np.ascontiguousarray(np.asarray(positions, dtype=np.float64).reshape(-1, 3))
    err = np.empty(len(ta.obs_frame))
    s = ta.struct()
    ctx.check(ctx.lib.sfm_reprojection_errors(ctx.handle, ctypes.byref(s), nat.ptr(P),
                                              nat.ptr(err)))
    return err, ta


def reprojection_error(map_or_poses, cameras, observation, point, ctx=None):
    """mapping.py:243-252 (inf when the projection raises)."""
    poses = {observation.frame_id: map_or_poses[observation.frame_id]}
    cams = {observation.frame_id: cameras[observation.frame_id]}
    err, _ = _reproj_errors([[observation]], [point], poses, cams, ctx)
    return float(err[0])


def remove_outliers(sparse_map, threshold_px: float, ctx=None):
    """mapping.py:544-566 on device: strict `>` gate on inlier observations,
    landmarks left with < 2 inliers revert to PENDING and are dropped."""
    ctx = ctx or nat.default_context()
    poses = {f: kf.cam_from_world for f, kf in sparse_map.keyframes.items()}
    cams = {f: sparse_map.camera_of(f) for f in sparse_map.keyframes}
    tri = [lm for lm in sparse_map.landmarks if lm.track.status == TRIANGULATED]
    removed = 0
    if tri:
        ta = TrackArrays([lm.track.observations for lm in tri], poses, cams)
        mask = np.ascontiguousarray(np.concatenate([np.asarray(lm.inlier_mask, dtype=np.uint8)
                                                    for lm in tri]))
        P = np.ascontiguousarray(np.array([lm.position for lm in tri], dtype=np.float64))
        inl = np.empty(len(tri), dtype=np.int32)
        rm = ctypes.c_int64()
        s = ta.struct()
        ctx.check(ctx.lib.sfm_gate(ctx.handle, ctypes.byref(s), nat.ptr(P), float(threshold_px),
                                   nat.ptr(mask), nat.ptr(inl), ctypes.byref(rm)))
        removed = int(rm.value)
        for i, lm in enumerate(tri):
            m = mask[ta.ptr[i]:ta.ptr[i + 1]].astype(bool)
            if not np.array_equal(m, lm.inlier_mask):
                lm.inlier_mask[:] = m
            if inl[i] < 2:
                lm.track.status = PENDING
    tri_ids = {id(lm) for lm in tri}
    sparse_map.landmarks = [lm for lm in sparse_map.landmarks
                            if not (id(lm) in tri_ids and lm.track.status == PENDING)]
    return sparse_map, removed


@dataclass
class MapResult:
    """Output of iterative_map_arrays (sfm_iterative_map)."""

    cam_q: np.ndarray          # [F,4] final poses (frame order of the inputs)
    cam_t: np.ndarray          # [F,3]
    points: np.ndarray         # [T,3] per track, NaN unless a landmark
    inlier_mask: np.ndarray    # [N] bool per observation
    status: np.ndarray         # [T] int8 nat.TRACK_*
    lm_track: np.ndarray       # [L] landmarks as track ids, in map order
    round_stats: list


def _map_options(config: MappingConfig, device: DeviceOptions) -> nat.MapOptionsC:
    dev = device or DEFAULT_DEVICE_OPTIONS
    return nat.MapOptionsC(
        int(config.max_outer_iters), int(config.max_solver_iters),
        nat.LOSS_KINDS[config.stage1.loss.kind], nat.LOSS_KINDS[config.stage2.loss.kind],
        float(config.stage1.loss.param), float(config.stage2.loss.param),
        float(config.stage1.outlier_px), float(config.stage2.outlier_px),
        float(config.min_triangulation_angle), nat.tri_method(config.triangulation), 0,
        _options(TRIVIAL_LOSS, SolverOptions(max_iters=config.max_solver_iters), dev))


def iterative_map_arrays(cam_q, cam_t, frame_model, frame_fixed, models, n_models, track_ptr,
                         obs_frame, obs_uv, edge_ab=None, prior_frame=None,
                         config: MappingConfig = None, track_status=None,
                         device: DeviceOptions = None, ctx=None) -> MapResult:
    """iterative_map (mapping.py:569-624) on flattened arrays, the whole loop
    device-resident (sfm_iterative_map): frames with the fixed set resolved,
    tracks as CSR in track order, the pose terms each bundle_adjust builds
    (lambda_c / lambda_a weights from `config`)."""
    config = config or MappingConfig()
    ctx = ctx or nat.default_context()
    keep = dict(q=np.ascontiguousarray(cam_q, dtype=np.float64),
                t=np.ascontiguousarray(cam_t, dtype=np.float64),
                fm=np.ascontiguousarray(frame_model, dtype=np.int32),
                fx=np.ascontiguousarray(frame_fixed, dtype=np.uint8),
                ptr=np.ascontiguousarray(track_ptr, dtype=np.int64),
                of=np.ascontiguousarray(obs_frame, dtype=np.int32),
                uv=np.ascontiguousarray(obs_uv, dtype=np.float64).reshape(-1, 2),
                ab=np.ascontiguousarray(edge_ab if edge_ab is not None else np.zeros((0, 2)),
                                        dtype=np.int32).reshape(-1, 2),
                pf=np.ascontiguousarray(prior_frame if prior_frame is not None else np.zeros(0),
                                        dtype=np.int32))
    F, T, N = len(keep["fm"]), len(keep["ptr"]) - 1, len(keep["of"])
    st_in = None
    if track_status is not None:
        st_in = np.ascontiguousarray(track_status, dtype=np.int8)
    prob = nat.MapProblemC(
        F, n_models, nat.ptr(keep["q"]), nat.ptr(keep["t"]), nat.ptr(keep["fm"]),
        nat.ptr(keep["fx"]), ctypes.addressof(models), T, N, nat.ptr(keep["ptr"]),
        nat.ptr(keep["of"]), nat.ptr(keep["uv"]), nat.ptr(st_in), len(keep["ab"]), len(keep["pf"]),
        nat.ptr(keep["ab"]), nat.ptr(keep["pf"]),
        float(config.lambda_c) if len(keep["ab"]) else 0.0,
        float(config.lambda_a) if len(keep["pf"]) else 0.0)
    opt = _map_options(config, device)
    q = np.empty((F, 4))
    t = np.empty((F, 3))
    X = np.empty((T, 3))
    mask = np.empty(N, np.uint8)
    status = np.empty(T, np.int8)
    lm = np.empty(max(T, 1), np.int64)
    nlm = ctypes.c_int64()
    stats = (nat.RoundStatC * (int(config.max_outer_iters) + 1))()
    nst = ctypes.c_int32()
    ctx.check(ctx.lib.sfm_iterative_map(ctx.handle, ctypes.byref(prob), ctypes.byref(opt),
                                        nat.ptr(q), nat.ptr(t), nat.ptr(X), nat.ptr(mask),
                                        nat.ptr(status), nat.ptr(lm), ctypes.byref(nlm),
                                        ctypes.addressof(stats), ctypes.byref(nst)))
    rs = [{"round": (stats[i].round if stats[i].round >= 0 else "final"),
           "added": int(stats[i].added), "removed": int(stats[i].removed),
           "landmarks": int(stats[i].landmarks)} for i in range(nst.value)]
    return MapResult(q, t, X, mask.astype(bool), status, lm[:nlm.value].copy(), rs)


def _pose_terms(frames, fidx, sparse_map, config, fixed, mode):
    """The lambda_c edges / lambda_a priors bundle_adjust builds
    (mapping.py:477-509), as frame-index arrays (same as flatten_ba)."""
    edges = []
    if config.lambda_c > 0:
        by_cam = {}
        for f in frames:
            by_cam.setdefault(sparse_map.keyframes[f].camera_id, []).append(f)
        for seq in by_cam.values():
            edges.extend((fidx[a], fidx[b]) for a, b in zip(seq, seq[1:]))
    priors = []
    if config.lambda_a > 0:
        for f in frames:
            if f in fixed:
                continue
            if mode == PURE and sparse_map.provenance.get(f) == "prior":
                continue
            priors.append(fidx[f])
    return (np.asarray(edges, dtype=np.int32).reshape(-1, 2), np.asarray(priors, dtype=np.int32))


_STATUS_CODE = {PENDING: nat.TRACK_PENDING, TRIANGULATED: nat.TRACK_TRIANGULATED,
                FAILED: nat.TRACK_FAILED}
_STATUS_NAME = {v: k for k, v in _STATUS_CODE.items()}


def iterative_map(keyframes, tracks, cameras, config: MappingConfig = None, rig=None,
                  mode: str = PURE, provenance=None, fixed_frames=None, device=None,
                  ctx=None) -> SparseMap:
    """mapping.py:569-624: rounds of {RANSAC triangulation of pending tracks
    -> stage-1 BA -> 4 px gate} until a round neither adds nor removes, then
    stage-2 BA and the 2 px gate -- one device-resident call
    (iterative_map_arrays / sfm_iterative_map); the object model is read
    once and written back once."""
    if config is None:
        config = MappingConfig()
    kf_map = {kf.frame_id: kf for kf in keyframes}
    sparse_map = SparseMap(kf_map, dict(cameras), [], rig, dict(provenance or {}),
                           set(fixed_frames or ()))
    has_prior = any(sparse_map.provenance.get(f) == "prior" for f in kf_map)
    needs_anchor = not (mode == LOCALIZATION_FIXED and has_prior)
    if not sparse_map.fixed_frames and kf_map and needs_anchor:
        new = [f for f in kf_map if sparse_map.provenance.get(f) != "prior"]
        sparse_map.fixed_frames = {min(new) if new else min(kf_map)}
    frames = sorted(kf_map)
    if _needs_general(sparse_map, frames, mode):
        return _iterative_map_host(sparse_map, tracks, config, mode, device, ctx)
    fixed = set(sparse_map.fixed_frames)
    if mode == LOCALIZATION_FIXED:
        fixed |= {f for f in frames if sparse_map.provenance.get(f) == "prior"}
    # NoGauge comes out of the first bundle_adjust that has landmarks
    # (mapping.py:408-409 via :611), raised by the device loop (SFM_E_NO_GAUGE)
    fidx = {f: i for i, f in enumerate(frames)}
    cam_q = np.array([kf_map[f].cam_from_world.quat for f in frames]).reshape(-1, 4)
    cam_t = np.array([kf_map[f].cam_from_world.t for f in frames]).reshape(-1, 3)
    models, n_models, fm = model_table([sparse_map.camera_of(f) for f in frames])
    fixed_arr = np.array([1 if f in fixed else 0 for f in frames], dtype=np.uint8)
    edges, priors = _pose_terms(frames, fidx, sparse_map, config, fixed, mode)
    counts = np.fromiter((len(t.observations) for t in tracks), dtype=np.int64, count=len(tracks))
    ptr = np.zeros(len(tracks) + 1, dtype=np.int64)
    np.cumsum(counts, out=ptr[1:])
    of = np.fromiter((fidx[o.frame_id] for t in tracks for o in t.observations), dtype=np.int32,
                     count=int(ptr[-1]))
    uv = np.array([o.pixel for t in tracks for o in t.observations], dtype=np.float64).reshape(-1, 2)
    st_in = np.array([_STATUS_CODE[t.status] for t in tracks], dtype=np.int8)
    res = iterative_map_arrays(cam_q, cam_t, fm, fixed_arr, models, n_models, ptr, of, uv, edges,
                               priors, config, st_in, device, ctx)
    for i, f in enumerate(frames):
        if fixed_arr[i]:
            continue
        if np.array_equal(res.cam_q[i], cam_q[i]) and np.array_equal(res.cam_t[i], cam_t[i]):
            continue
        kf = kf_map[f]
        kf.cam_from_world = type(kf.cam_from_world)(res.cam_q[i], res.cam_t[i])
    for i, tr in enumerate(tracks):
        tr.status = _STATUS_NAME[int(res.status[i])]
    sparse_map.landmarks = [Landmark(res.points[i].copy(), tracks[i],
                                     res.inlier_mask[ptr[i]:ptr[i + 1]].copy())
                            for i in res.lm_track]
    sparse_map.round_stats = res.round_stats
    return sparse_map


def _iterative_map_host(sparse_map, tracks, config, mode, device, ctx):
    """mapping.py:596-623 driven from the host for problems the device-
    resident loop does not take (rolling-shutter keyframes, rig mode): each
    round's triangulation and gating are one batched device call, the BA the
    general two-slot solve."""
    kf_map = sparse_map.keyframes
    stats = []
    for round_idx in range(config.max_outer_iters):
        poses = {f: kf.cam_from_world for f, kf in kf_map.items()}
        cams = {f: sparse_map.camera_of(f) for f in kf_map}
        pending = [t for t in tracks if t.status == PENDING]
        results = ransac_triangulate_batch(
            pending, poses, cams, threshold_px=config.stage1.outlier_px,
            min_angle=config.min_triangulation_angle, method=config.triangulation, ctx=ctx)
        added = 0
        for lm in results:
            if lm is not None:
                sparse_map.landmarks.append(lm)
                added += 1
        if sparse_map.landmarks:
            bundle_adjust(sparse_map, config, stage=1, mode=mode, device=device, ctx=ctx)
        _, removed = remove_outliers(sparse_map, config.stage1.outlier_px, ctx=ctx)
        stats.append({"round": round_idx, "added": added, "removed": removed,
                      "landmarks": len(sparse_map.landmarks)})
        if added == 0 and removed == 0:
            break
    if sparse_map.landmarks:
        bundle_adjust(sparse_map, config, stage=2, mode=mode, device=device, ctx=ctx)
        _, removed = remove_outliers(sparse_map, config.stage2.outlier_px, ctx=ctx)
        stats.append({"round": "final", "added": 0, "removed": removed,
                      "landmarks": len(sparse_map.landmarks)})
    sparse_map.round_stats = stats
    return sparse_map


def mean_reprojection_error(sparse_map, ctx=None) -> float:
    """mapping.py:627-636."""
    poses = {f: kf.cam_from_world for f, kf in sparse_map.keyframes.items()}
    cams = {f: sparse_map.camera_of(f) for f in sparse_map.keyframes}
    lms = [lm for lm in sparse_map.landmarks if lm.track.status == TRIANGULATED]
    obs = [lm.inlier_observations() for lm in lms]
    if not any(obs):
        return 0.0
    err, _ = _reproj_errors(obs, [lm.position for lm in lms], poses, cams, ctx)
    return float(np.mean(err)) if len(err) else 0.0


__all__ = [
    "PENDING", "TRIANGULATED", "FAILED", "PURE", "LOCALIZATION_FIXED", "LOCALIZATION_ADJUST",
    "RIG_EXTRINSIC", "build_tracks", "build_tracks_arrays", "Observation", "Track", "Landmark",
    "SparseMap", "StageConfig",
    "MappingConfig", "BAArrays", "flatten_ba", "solve_arrays", "shard_ranges", "bundle_adjust",
    "triangulate_dlt", "triangulate_midpoint", "reprojection_error", "ransac_triangulate",
    "ransac_triangulate_batch", "remove_outliers", "iterative_map", "iterative_map_arrays",
    "MapResult", "mean_reprojection_error",
    "CameraModel", "Keyframe",
]


class DeviceBA:
    """Stepwise, device-resident form of solve_arrays (sfm_ba_setup /
    sfm_ba_iterate / sfm_ba_download): the problem is uploaded and its
    structure built once, then LM iterations run with no host<->device
    traffic beyond one small scalar read-back per trial."""

    def __init__(self, arrays: BAArrays, loss: RobustLoss = TRIVIAL_LOSS,
                 options: SolverOptions = None, device: DeviceOptions = None, ctx=None):
        self.ctx = ctx or nat.default_context()
        self.arrays = arrays
        self._prob = arrays.struct()
        self._opt = _options(loss, options or SolverOptions(), device or DEFAULT_DEVICE_OPTIONS)
        self.ctx.check(self.ctx.lib.sfm_ba_setup(self.ctx.handle, ctypes.byref(self._prob),
                                                 ctypes.byref(self._opt)))

    def iterate(self, n: int) -> nat.BAReportC:
        rep = nat.BAReportC()
        self.ctx.check(self.ctx.lib.sfm_ba_iterate(self.ctx.handle, int(n), ctypes.byref(rep)))
        return rep

    def restart(self):
        """A new solve from the entry state on the same device-resident
        problem (sfm_ba_restart)."""
        self.ctx.check(self.ctx.lib.sfm_ba_restart(self.ctx.handle))

    def download(self):
        a = self.arrays
        q = np.empty_like(a.cam_q)
        t = np.empty_like(a.cam_t)
        X = np.empty_like(a.points)
        self.ctx.check(self.ctx.lib.sfm_ba_download(self.ctx.handle, nat.ptr(q), nat.ptr(t),
                                                    nat.ptr(X)))
        return q, t, X
