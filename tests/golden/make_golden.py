"""Generates the golden fixtures tests/golden/*.npz by running the REFERENCE
implementation (sfmkit, imported from /root/reference/pkg/src) on seeded
synthetic inputs.  Run here (the survey container), never on the GPU box:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Each fixture stores the flattened inputs in the C-ABI layout
(include/sfm_b200.h) together with the reference outputs, so the oracle
(oracle/) and the CUDA path can both be checked against the reference
without the reference being present.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)
sys.dont_write_bytecode = True

import sfmkit.mapping as M  # noqa: E402
import sfmkit.solver as SV  # noqa: E402
from sfmkit.cameras import CameraModel, project, project_with_pose_jacobian, unproject  # noqa: E402
from sfmkit.keyframes import Keyframe  # noqa: E402
from sfmkit.posegraph import PoseEdge, _edge_residual_fn  # noqa: E402
from sfmkit.se3 import Pose, exp_map, interpolate_pose  # noqa: E402

from paper_2510_15271_b200 import mapping as D  # noqa: E402  (flattening only)

CAM = CameraModel("pinhole", 500.0, 500.0, 320.0, 240.0, 640, 480)


def models_array(arrays_models, n):
    out = np.zeros((n, 7))
    for i in range(n):
        m = arrays_models[i]
        out[i] = [m.kind, m.fx, m.fy, m.cx, m.cy, m.k1, m.k2]
    return out


def flat_dict(arrays, prefix=""):
    return {prefix + "cam_q": arrays.cam_q, prefix + "cam_t": arrays.cam_t,
            prefix + "frame_model": arrays.frame_model, prefix + "frame_fixed": arrays.frame_fixed,
            prefix + "models": models_array(arrays.models, arrays.n_models),
            prefix + "points": arrays.points, prefix + "obs_frame": arrays.obs_frame,
            prefix + "obs_point": arrays.obs_point, prefix + "obs_uv": arrays.obs_uv,
            prefix + "edge_ab": arrays.edge_ab, prefix + "prior_frame": arrays.prior_frame,
            prefix + "edge_weight": np.float64(arrays.edge_weight),
            prefix + "prior_weight": np.float64(arrays.prior_weight)}


LOSS_CODE = {"trivial": 0, "huber": 1, "cauchy": 2}


# --- scenes (pattern of test_mapping.py:24-52, :275-295) ----------------------

def cam_pose(center, rot_xi=(0.0, 0.0, 0.0)):
    R = exp_map(np.array([*rot_xi, 0, 0, 0])).R
    return Pose.from_rt(R, -R @ np.asarray(center, dtype=float))


def scene(rng, n_frames=6, n_points=40, spacing=0.8):
    points = rng.uniform([-4, -3, 6], [4, 3, 14], (n_points, 3))
    poses = {i: cam_pose([spacing * i, 0.05 * i, 0], (0.02 * i, -0.03 * i, 0.01 * i))
             for i in range(n_frames)}
    return points, poses


def observations(point, poses, noise=0.0, rng=None):
    obs = []
    for f in sorted(poses):
        pix = project(CAM, poses[f], point)
        if not (0 <= pix[0] < CAM.width and 0 <= pix[1] < CAM.height):
            continue
        if noise and rng is not None:
            pix = pix + rng.normal(0, noise, 2)
        obs.append(M.Observation(f, 0, pix))
    return obs


def map_from_scene(points, poses, perturb=0.0, rng=None, fixed_frames=(0, 1), noise=0.0,
                   outlier_every=0, outlier_px=(35.0, -25.0)):
    kfs = {f: Keyframe(f, float(f), 0, poses[f]) for f in poses}
    smap = M.SparseMap(kfs, {0: CAM}, fixed_frames=set(fixed_frames))
    for i, p in enumerate(points):
        obs = observations(p, poses, noise, rng)
        if len(obs) < 2:
            continue
        if outlier_every and i % outlier_every == 0:
            obs[1].pixel = obs[1].pixel + np.array(outlier_px)
        smap.landmarks.append(M.Landmark(p.copy(), M.Track(obs, status=M.TRIANGULATED),
                                         np.ones(len(obs), bool)))
    if perturb and rng is not None:
        for f in poses:
            if f in smap.fixed_frames:
                continue
            kfs[f].cam_from_world = exp_map(rng.normal(0, perturb, 6)) @ kfs[f].cam_from_world
        for lm in smap.landmarks:
            lm.position = lm.position + rng.normal(0, 5 * perturb, 3)
    return smap


def map_from_arrays(sc):
    """paper_2510_15271_b200.scenes.Scene -> sfmkit SparseMap."""
    kfs = {f: Keyframe(f, float(f), 0, Pose(sc.cam_q[f], sc.cam_t[f])) for f in range(sc.n_frames)}
    smap = M.SparseMap(kfs, {0: CAM}, fixed_frames={int(f) for f in np.flatnonzero(sc.frame_fixed)})
    ptr = np.searchsorted(sc.obs_point, np.arange(sc.n_points + 1))
    for p in range(sc.n_points):
        obs = [M.Observation(int(sc.obs_frame[o]), 0, sc.obs_uv[o]) for o in range(ptr[p], ptr[p + 1])]
        smap.landmarks.append(M.Landmark(sc.points[p].copy(), M.Track(obs, status=M.TRIANGULATED),
                                         np.ones(len(obs), bool)))
    return smap


# --- BA fixtures -----------------------------------------------------------------

def run_ba(name, smap, config, stage=1, mode=M.PURE, capture_jacobian=True):
    arrays, frames, lms, loss = D.flatten_ba(smap, config, stage, mode)
    captured = {}
    orig = M.solve

    def spy(problem, options):
        cost, res = problem.evaluate()
        captured["ref_initial_residual"] = res
        if capture_jacobian:
            offsets, n = SV._free_layout(problem)
            J, r = SV._assemble(problem, offsets, n)
            captured["ref_J"] = J.toarray()
            captured["ref_r"] = r
        return orig(problem, options)

    M.solve = spy
    t0 = time.time()
    out = {}
    try:
        rep = M.bundle_adjust(smap, config, stage=stage, mode=mode)
        out.update(ref_initial_cost=rep.initial_cost, ref_final_cost=rep.final_cost,
                   ref_iterations=rep.iterations, ref_termination=rep.termination,
                   ref_exception="")
    except Exception as e:  # noqa: BLE001 -- the exception class is the golden value
        out.update(ref_exception=type(e).__name__, ref_message=str(e))
    finally:
        M.solve = orig
    dt = time.time() - t0
    q = np.array([smap.keyframes[f].cam_from_world.quat for f in frames])
    t = np.array([smap.keyframes[f].cam_from_world.t for f in frames])
    X = np.array([smap.landmarks[li].position for li in lms]).reshape(-1, 3)
    out.update(ref_cam_q=q, ref_cam_t=t, ref_points=X, ref_seconds=dt)
    out.update(captured)
    out.update(flat_dict(arrays))
    out.update(loss_kind=LOSS_CODE[loss.kind], loss_param=float(loss.param),
               max_iters=config.max_solver_iters)
    np.savez_compressed(os.path.join(HERE, f"ba_{name}.npz"), **out)
    print(f"ba_{name}: N={len(arrays.obs_frame)} P={len(arrays.points)} "
          f"{out.get('ref_termination', out.get('ref_exception'))} "
          f"iters={out.get('ref_iterations')} {dt:.1f}s")


def ba_fixtures():
    rng = np.random.default_rng(42)
    pts, poses = scene(rng, 6, 40)
    run_ba("plain_stage2", map_from_scene(pts, poses, 0.01, rng),
           M.MappingConfig(lambda_a=0.0, lambda_c=0.0, max_solver_iters=100), stage=2)
    rng = np.random.default_rng(7)
    pts, poses = scene(rng, 6, 40)
    run_ba("huber_outliers", map_from_scene(pts, poses, 0.002, rng, fixed_frames=(0,), noise=0.3,
                                            outlier_every=7),
           M.MappingConfig(), stage=1)
    rng = np.random.default_rng(11)
    pts, poses = scene(rng, 7, 50)
    cfg = M.MappingConfig(stage1=M.StageConfig(4.0, SV.RobustLoss("cauchy", 1.5)), lambda_c=2.0,
                          lambda_a=0.5, max_solver_iters=30)
    run_ba("cauchy_pose_terms", map_from_scene(pts, poses, 0.005, rng, fixed_frames=(0,), noise=0.5,
                                               outlier_every=9), cfg, stage=1)
    rng = np.random.default_rng(3)
    pts, poses = scene(rng, 6, 30)
    smap = map_from_scene(pts, poses, 0.01, rng, fixed_frames=())
    smap.provenance = {f: ("prior" if f < 3 else "new") for f in poses}
    for f in range(3):
        smap.keyframes[f].cam_from_world = poses[f]
    run_ba("localization_fixed", smap,
           M.MappingConfig(lambda_a=0.0, lambda_c=0.0, max_solver_iters=100), stage=2,
           mode=M.LOCALIZATION_FIXED)
    rng = np.random.default_rng(5)
    pts, poses = scene(rng, 6, 30)
    smap = map_from_scene(pts, poses, 0.01, rng, fixed_frames=(0,))
    smap.provenance = {f: ("prior" if f < 3 else "new") for f in poses}
    run_ba("localization_adjust", smap,
           M.MappingConfig(lambda_a=1e-4, lambda_c=0.0, max_solver_iters=100), stage=2,
           mode=M.LOCALIZATION_ADJUST)
    rng = np.random.default_rng(9)
    pts, poses = scene(rng, 4, 20)
    run_ba("prior_gauge", map_from_scene(pts, poses, 0.003, rng, fixed_frames=()),
           M.MappingConfig(lambda_a=10.0, lambda_c=0.0), stage=2)
    rng = np.random.default_rng(13)
    pts, poses = scene(rng, 5, 25)
    run_ba("pure_provenance_lc", _with_provenance(map_from_scene(pts, poses, 0.004, rng,
                                                                 fixed_frames=(0,), noise=0.2)),
           M.MappingConfig(lambda_c=100.0, lambda_a=3.0), stage=1)
    # initial state with a point behind a camera: NonPositiveDepth from evaluate()
    rng = np.random.default_rng(17)
    pts, poses = scene(rng, 4, 12)
    smap = map_from_scene(pts, poses, 0.0, rng, fixed_frames=(0,))
    smap.landmarks[3].position = np.array([0.0, 0.0, -5.0])
    run_ba("depth_error", smap, M.MappingConfig(), stage=1)
    # config-1: 20 cams / ~2k pts / ~10k obs, 10 LM iterations, Huber
    from paper_2510_15271_b200.scenes import config_scene
    sc = config_scene(1, seed=1)
    smap = map_from_arrays(sc)
    run_ba("config1", smap, M.MappingConfig(max_solver_iters=10), stage=1, capture_jacobian=False)


def _with_provenance(smap):
    smap.provenance = {f: ("prior" if f in (1, 2) else "new") for f in smap.keyframes}
    return smap


# --- triangulation / gating fixtures ----------------------------------------------

def track_fixture(name, tracks, poses, thr, min_angle, method, cams_of=None, models=None):
    """cams_of: frame -> (model index, CameraModel); default all frames CAM."""
    frames = sorted(poses)
    fidx = {f: i for i, f in enumerate(frames)}
    ptr = np.zeros(len(tracks) + 1, np.int64)
    ptr[1:] = np.cumsum([len(t.observations) for t in tracks])
    of = np.array([fidx[o.frame_id] for t in tracks for o in t.observations], np.int32)
    uv = np.array([o.pixel for t in tracks for o in t.observations]).reshape(-1, 2)
    q = np.array([poses[f].quat for f in frames])
    t = np.array([poses[f].t for f in frames])
    cams = {f: (cams_of[f][1] if cams_of else CAM) for f in frames}
    frame_model = np.array([cams_of[f][0] if cams_of else 0 for f in frames], np.int32)
    if models is None:
        models = np.array([[0, 500.0, 500.0, 320.0, 240.0, 0.0, 0.0]])
    X = np.full((len(tracks), 3), np.nan)
    mask = np.zeros(len(of), np.uint8)
    status = np.zeros(len(tracks), np.int8)
    dX = np.full((len(tracks), 3), np.nan)
    dstat = np.zeros(len(tracks), np.int8)
    codes = {"InsufficientParallax": 1, "CheiralityViolation": 2, "ParallelRays": 3,
             "ValueError": 4}
    for i, tr in enumerate(tracks):
        trc = M.Track(list(tr.observations))
        lm = M.ransac_triangulate(trc, poses, cams, threshold_px=thr, min_angle=min_angle,
                                  method=method)
        if lm is None:
            status[i] = 6
        else:
            X[i] = lm.position
            mask[ptr[i]:ptr[i + 1]] = lm.inlier_mask
        try:
            if method == "dlt":
                dX[i] = M.triangulate_dlt(tr.observations, poses, cams, min_angle=min_angle)
            else:
                dX[i] = M.triangulate_midpoint(tr.observations, poses, cams)
        except Exception as e:  # noqa: BLE001
            dstat[i] = codes.get(type(e).__name__, 9)
    np.savez_compressed(os.path.join(HERE, f"tri_{name}.npz"), cam_q=q, cam_t=t,
                        frame_model=frame_model, models=models,
                        track_ptr=ptr, obs_frame=of, obs_uv=uv, threshold_px=thr,
                        min_angle=min_angle, method=method, ref_X=X, ref_mask=mask,
                        ref_status=status, ref_direct_X=dX, ref_direct_status=dstat)
    print(f"tri_{name}: T={len(tracks)} ok={int((status == 0).sum())} "
          f"direct_errors={int((dstat != 0).sum())}")


def tri_fixtures():
    for method in ("dlt", "midpoint"):
        rng = np.random.default_rng(21)
        pts, poses = scene(rng, 8, 120, spacing=0.6)
        tracks = []
        for i, p in enumerate(pts):
            obs = observations(p, poses, 0.4, rng)
            if len(obs) < 2:
                continue
            if i % 4 == 0 and len(obs) >= 3:
                k = int(rng.integers(len(obs)))
                obs[k] = M.Observation(obs[k].frame_id, 0,
                                       obs[k].pixel + rng.uniform(15, 60, 2) * rng.choice([-1, 1], 2))
            if i % 9 == 0:
                obs = [M.Observation(o.frame_id, 0, o.pixel + rng.uniform(-80, 80, 2)) for o in obs]
            tracks.append(M.Track(obs))
        # degenerate: zero baseline (InsufficientParallax / ParallelRays)
        dp = {0: cam_pose([0, 0, 0]), 1: cam_pose([0, 0, 0], (0.0, 0.05, 0))}
        for f, pz in dp.items():
            poses[100 + f] = pz
        p = np.array([0.5, -0.3, 9.0])
        tracks.append(M.Track([M.Observation(100 + f, 0, project(CAM, dp[f], p)) for f in dp]))
        # cheirality: swapped pixels
        poses[200], poses[201] = cam_pose([0, 0, 0]), cam_pose([1.0, 0, 0])
        p = np.array([0.3, 0.2, 10.0])
        pa, pb = project(CAM, poses[200], p), project(CAM, poses[201], p)
        tracks.append(M.Track([M.Observation(200, 0, pb), M.Observation(201, 0, pa)]))
        # parallel rays through the principal point
        tracks.append(M.Track([M.Observation(200, 0, (CAM.cx, CAM.cy)),
                               M.Observation(201, 0, (CAM.cx, CAM.cy))]))
        track_fixture(method, tracks, poses, 4.0, np.radians(0.5), method)


def gate_fixture():
    rng = np.random.default_rng(31)
    pts, poses = scene(rng, 6, 60)
    smap = map_from_scene(pts, poses, 0.0, rng, fixed_frames=(0,), noise=0.5)
    for i, lm in enumerate(smap.landmarks):
        if i % 5 == 0:
            lm.track.observations[1].pixel = lm.track.observations[1].pixel + np.array([10.0, 0.0])
        if i % 11 == 0:
            for o in lm.track.observations[1:]:
                o.pixel = o.pixel + np.array([25.0, 25.0])
        if i % 7 == 0:
            lm.inlier_mask[0] = False
    frames = sorted(smap.keyframes)
    fidx = {f: i for i, f in enumerate(frames)}
    tri = [lm for lm in smap.landmarks if lm.track.status == M.TRIANGULATED]
    ptr = np.zeros(len(tri) + 1, np.int64)
    ptr[1:] = np.cumsum([len(lm.track.observations) for lm in tri])
    of = np.array([fidx[o.frame_id] for lm in tri for o in lm.track.observations], np.int32)
    uv = np.array([o.pixel for lm in tri for o in lm.track.observations])
    mask_in = np.concatenate([lm.inlier_mask for lm in tri]).astype(np.uint8)
    P = np.array([lm.position for lm in tri])
    q = np.array([smap.keyframes[f].cam_from_world.quat for f in frames])
    t = np.array([smap.keyframes[f].cam_from_world.t for f in frames])
    _, removed = M.remove_outliers(smap, 2.0)
    mask_out = np.concatenate([lm.inlier_mask for lm in tri]).astype(np.uint8)
    status = np.array([1 if lm.track.status == M.TRIANGULATED else 0 for lm in tri], np.int8)
    np.savez_compressed(os.path.join(HERE, "gate.npz"), cam_q=q, cam_t=t,
                        frame_model=frame_model, models=models,
                        track_ptr=ptr, obs_frame=of, obs_uv=uv, points=P, mask_in=mask_in,
                        threshold_px=2.0, ref_mask=mask_out, ref_removed=removed,
                        ref_triangulated=status)
    print(f"gate: L={len(tri)} removed={removed} demoted={int((status == 0).sum())}")


def iterative_map_fixture(name="iterative_map", seed=42, n_frames=6, n_points=30, config=None,
                          noise=0.3, mild_every=0):
    rng = np.random.default_rng(seed)
    pts, poses = scene(rng, n_frames, n_points)
    kfs = [Keyframe(f, float(f), 0, poses[f]) for f in sorted(poses)]
    tracks = []
    for k, p in enumerate(pts):
        obs = observations(p, poses, noise, rng)
        if len(obs) < 3:
            continue
        if k % 5 == 0:
            obs[1] = M.Observation(obs[1].frame_id, 0, obs[1].pixel + np.array([40.0, 30.0]))
        if mild_every and k % mild_every == 1:
            # 2-4 px errors: inside RANSAC's 4 px bar, gated by the 2 px stage-2 gate
            # (and, on short tracks, demoted and re-triangulated)
            j = len(obs) - 1
            obs[j] = M.Observation(obs[j].frame_id, 0, obs[j].pixel + rng.uniform(2.5, 3.8, 2) *
                                   rng.choice([-1, 1], 2) / np.sqrt(2))
        tracks.append(M.Track(obs))
    # perturb the non-anchor initial poses
    for kf in kfs[1:]:
        kf.cam_from_world = exp_map(rng.normal(0, 0.003, 6)) @ kf.cam_from_world
    q0 = np.array([kf.cam_from_world.quat for kf in kfs])
    t0 = np.array([kf.cam_from_world.t for kf in kfs])
    ptr = np.zeros(len(tracks) + 1, np.int64)
    ptr[1:] = np.cumsum([len(t.observations) for t in tracks])
    of = np.array([o.frame_id for t in tracks for o in t.observations], np.int32)
    uv = np.array([o.pixel for t in tracks for o in t.observations])
    smap = M.iterative_map(kfs, tracks, {0: CAM}, config=config)
    lm_track = np.array([next(i for i, t in enumerate(tracks) if t is lm.track)
                         for lm in smap.landmarks], np.int64)
    rs = smap.round_stats
    np.savez_compressed(
        os.path.join(HERE, f"{name}.npz"), cam_q=q0, cam_t=t0, track_ptr=ptr, obs_frame=of,
        obs_uv=uv, ref_cam_q=np.array([smap.keyframes[f].cam_from_world.quat for f in sorted(poses)]),
        ref_cam_t=np.array([smap.keyframes[f].cam_from_world.t for f in sorted(poses)]),
        ref_lm_track=lm_track, ref_lm_X=np.array([lm.position for lm in smap.landmarks]),
        ref_lm_mask=np.concatenate([lm.inlier_mask for lm in smap.landmarks]).astype(np.uint8),
        ref_status=np.array([{"pending": 0, "triangulated": 1, "failed": 2}[t.status] for t in tracks]),
        ref_round_added=np.array([r["added"] for r in rs]),
        ref_round_removed=np.array([r["removed"] for r in rs]),
        ref_round_landmarks=np.array([r["landmarks"] for r in rs]),
        ref_mean_err=M.mean_reprojection_error(smap))
    print(f"{name}: tracks={len(tracks)} landmarks={len(smap.landmarks)} rounds={len(rs)} "
          f"added={[r['added'] for r in rs]} removed={[r['removed'] for r in rs]}")


# --- radial / fisheye camera kinds (cameras.py:57-125) ------

RAD = CameraModel("pinhole_radial", 480.0, 470.0, 318.0, 242.0, 640, 480, (-0.08, 0.02))
FISH = CameraModel("equidistant_fisheye", 320.0, 320.0, 320.0, 240.0, 640, 480)
KIND_MODELS = np.array([[1, 480.0, 470.0, 318.0, 242.0, -0.08, 0.02],
                        [2, 320.0, 320.0, 320.0, 240.0, 0.0, 0.0]])


def observations_cams(point, poses, cam_of, noise=0.0, rng=None):
    obs = []
    for f in sorted(poses):
        cam = cam_of[f]
        try:
            pix = project(cam, poses[f], point)
        except Exception:  # noqa: BLE001 -- outside the model domain: not observed
            continue
        if not (0 <= pix[0] < cam.width and 0 <= pix[1] < cam.height):
            continue
        if noise and rng is not None:
            pix = pix + rng.normal(0, noise, 2)
        obs.append(M.Observation(f, 0, pix))
    return obs


def camera_kinds_fixtures():
    rng = np.random.default_rng(31)
    pts, poses = scene(rng, 8, 70)
    cam_id = {f: f % 2 for f in poses}
    cams = {0: RAD, 1: FISH}
    cam_of = {f: cams[cam_id[f]] for f in poses}
    kfs = {f: Keyframe(f, float(f), cam_id[f], poses[f]) for f in poses}
    smap = M.SparseMap(kfs, cams, fixed_frames={0})
    for p in pts:
        obs = observations_cams(p, poses, cam_of, 0.3, rng)
        if len(obs) < 2:
            continue
        smap.landmarks.append(M.Landmark(p.copy(), M.Track(obs, status=M.TRIANGULATED),
                                         np.ones(len(obs), bool)))
    for f in poses:
        if f != 0:
            kfs[f].cam_from_world = exp_map(rng.normal(0, 0.003, 6)) @ kfs[f].cam_from_world
    for lm in smap.landmarks:
        lm.position = lm.position + rng.normal(0, 0.015, 3)
    run_ba("camera_kinds", smap, M.MappingConfig(max_solver_iters=30), stage=1)
    # RANSAC triangulation with the same two camera kinds
    for method in ("dlt", "midpoint"):
        rng = np.random.default_rng(37)
        pts, poses = scene(rng, 8, 90, spacing=0.6)
        cam_of = {f: (RAD if f % 2 == 0 else FISH) for f in poses}
        tracks = []
        for i, p in enumerate(pts):
            obs = observations_cams(p, poses, cam_of, 0.4, rng)
            if len(obs) < 2:
                continue
            if i % 4 == 0 and len(obs) >= 3:
                k = int(rng.integers(len(obs)))
                obs[k] = M.Observation(obs[k].frame_id, 0,
                                       obs[k].pixel + rng.uniform(15, 60, 2) * rng.choice([-1, 1], 2))
            tracks.append(M.Track(obs))
        track_fixture("kinds_" + method, tracks, poses, 4.0, np.radians(0.5), method,
                      cams_of={f: ((0, RAD) if f % 2 == 0 else (1, FISH)) for f in poses},
                      models=KIND_MODELS)


# --- build_tracks (mapping.py:113-161) ------------------------------------------

def tracks_fixture():
    from sfmkit.features import FeatureSet, Keypoint, Match
    rng = np.random.default_rng(91)
    n_frames, n_feat = 10, 60
    feats = {f: FeatureSet(f, [Keypoint(float(3 * i), float(2 * i)) for i in range(n_feat)],
                           np.tile([1.0, 0.0, 0.0, 0.0], (n_feat, 1))) for f in range(n_frames)}
    pairs = {}
    for fa in range(n_frames):
        for fb in range(fa + 1, min(n_frames, fa + 4)):
            k = int(rng.integers(15, 40))
            ia = rng.choice(n_feat, size=k, replace=False)
            # mostly consistent feature identities, with random re-links that
            # create conflicting joins
            ib = np.where(rng.random(k) < 0.8, ia, rng.integers(0, n_feat, k))
            seen, ms = set(), []
            for a, b in zip(ia, ib):
                if (a, b) not in seen:
                    seen.add((a, b))
                    ms.append(Match(int(a), int(b), 0.1))
            pairs[(fa, fb)] = ms
    # insertion order shuffled: the reference sorts the pairs itself
    keys = list(pairs)
    rng.shuffle(keys)
    pairs = {k: pairs[k] for k in keys}
    tracks = M.build_tracks(pairs, feats)
    pf = np.array(keys, np.int32)
    pp = np.zeros(len(keys) + 1, np.int64)
    pp[1:] = np.cumsum([len(pairs[k]) for k in keys])
    mi = np.array([(m.index_a, m.index_b) for k in keys for m in pairs[k]], np.int32)
    tp = np.zeros(len(tracks) + 1, np.int64)
    tp[1:] = np.cumsum([len(t.observations) for t in tracks])
    np.savez_compressed(os.path.join(HERE, "build_tracks.npz"), pair_frames=pf, pair_ptr=pp,
                        match_index=mi,
                        ref_track_ptr=tp,
                        ref_obs_frame=np.array([o.frame_id for t in tracks for o in t.observations],
                                               np.int32),
                        ref_obs_feature=np.array([o.feature_index for t in tracks
                                                  for o in t.observations], np.int32))
    print(f"build_tracks: pairs={len(keys)} matches={len(mi)} tracks={len(tracks)} "
          f"obs={int(tp[-1])}")


# --- rig-extrinsic / rolling-shutter BA (mapping.py:321-356)

KIND_CODE = {"pinhole": 0, "pinhole_radial": 1, "equidistant_fisheye": 2}


def general_ba_fixture(name, smap, config, stage, mode):
    """Serialises the object-level inputs, runs sfmkit's bundle_adjust, and
    stores its outputs."""
    frames = sorted(smap.keyframes)
    kf = [smap.keyframes[f] for f in frames]
    cids = sorted(smap.cameras)
    lms = smap.landmarks
    out = dict(
        kf_id=np.array(frames, np.int64), kf_ts=np.array([k.timestamp for k in kf]),
        kf_cam=np.array([k.camera_id for k in kf], np.int64),
        kf_q=np.array([k.cam_from_world.quat for k in kf]), kf_t=np.array([k.cam_from_world.t for k in kf]),
        kf_rolling=np.array([k.shutter == "rolling" for k in kf], np.uint8),
        kf_exposure=np.array([k.exposure for k in kf]),
        cam_id=np.array(cids, np.int64),
        cam_par=np.array([[KIND_CODE[smap.cameras[c].kind], smap.cameras[c].fx, smap.cameras[c].fy,
                           smap.cameras[c].cx, smap.cameras[c].cy, smap.cameras[c].width,
                           smap.cameras[c].height,
                           *(list(smap.cameras[c].distortion) + [0.0, 0.0])[:2]] for c in cids]),
        lm_pos=np.array([lm.position for lm in lms]),
        lm_tri=np.array([lm.track.status == "triangulated" for lm in lms], np.uint8),
        lm_ptr=np.concatenate([[0], np.cumsum([len(lm.track.observations) for lm in lms])]).astype(np.int64),
        obs_frame=np.array([o.frame_id for lm in lms for o in lm.track.observations], np.int64),
        obs_uv=np.array([o.pixel for lm in lms for o in lm.track.observations]),
        lm_mask=np.concatenate([lm.inlier_mask for lm in lms]).astype(np.uint8),
        fixed=np.array(sorted(smap.fixed_frames), np.int64),
        prior=np.array(sorted(f for f, v in smap.provenance.items() if v == "prior"), np.int64),
        stage=stage, mode=mode, loss_kind=LOSS_CODE[config.stage1.loss.kind],
        loss_param=float(config.stage1.loss.param), lambda_c=config.lambda_c,
        lambda_a=config.lambda_a, extrinsic_prior_weight=config.extrinsic_prior_weight,
        max_iters=config.max_solver_iters)
    if smap.rig is not None:
        out.update(rig_ids=np.array(smap.rig.camera_ids, np.int64),
                   rig_q=np.array([smap.rig.extrinsic(c).quat for c in smap.rig.camera_ids]),
                   rig_t=np.array([smap.rig.extrinsic(c).t for c in smap.rig.camera_ids]))
    rep = M.bundle_adjust(smap, config, stage=stage, mode=mode)
    out.update(ref_initial_cost=rep.initial_cost, ref_final_cost=rep.final_cost,
               ref_iterations=rep.iterations, ref_termination=rep.termination,
               ref_kf_q=np.array([smap.keyframes[f].cam_from_world.quat for f in frames]),
               ref_kf_t=np.array([smap.keyframes[f].cam_from_world.t for f in frames]),
               ref_lm_pos=np.array([lm.position for lm in lms]))
    if smap.rig is not None:
        out.update(ref_rig_q=np.array([smap.rig.extrinsic(c).quat for c in smap.rig.camera_ids]),
                   ref_rig_t=np.array([smap.rig.extrinsic(c).t for c in smap.rig.camera_ids]))
    np.savez_compressed(os.path.join(HERE, f"ba_{name}.npz"), **out)
    print(f"ba_{name}: {rep.termination} iters={rep.iterations} cost {rep.initial_cost:.4g} -> "
          f"{rep.final_cost:.4g}")


def rig_rs_fixtures():
    from sfmkit.cameras import RigCalibration
    from sfmkit.se3 import interpolate_pose
    # rig: test_mapping.py:420-461 scene, and a noisy Huber stage-1 variant
    for name, n_inst, n_pts, noise, seed, stage, cfg in (
            ("rig", 5, 40, 0.0, 1, 2, M.MappingConfig(lambda_a=0.0, lambda_c=10.0,
                                                      extrinsic_prior_weight=1e-6,
                                                      max_solver_iters=100)),
            ("rig_huber", 7, 70, 0.4, 2, 1, M.MappingConfig(lambda_c=5.0, extrinsic_prior_weight=1e-3,
                                                            max_solver_iters=40))):
        rng = np.random.default_rng(seed)
        true_E1 = exp_map(np.array([0.0, 0.01, 0.0, 0.5, 0.02, 0.0]))
        rig = RigCalibration((0, 1), {0: Pose.identity(), 1: true_E1})
        pts = rng.uniform([-4, -3, 6], [4, 3, 14], (n_pts, 3))
        kfs, fid, vposes = {}, 0, {}
        for i in range(n_inst):
            T_v = cam_pose([0.7 * i, 0.03 * i, 0], (0.01 * i, -0.02 * i, 0.0))
            vposes[i] = T_v
            for cid in (0, 1):
                kfs[fid] = Keyframe(fid, float(i), cid, rig.extrinsic(cid) @ T_v)
                fid += 1
        smap = M.SparseMap(kfs, {0: CAM, 1: CAM}, rig=rig)
        for p in pts:
            obs = []
            for f, kf in kfs.items():
                pix = project(CAM, kf.cam_from_world, p)
                if 0 <= pix[0] < CAM.width and 0 <= pix[1] < CAM.height:
                    obs.append(M.Observation(f, 0, pix + (rng.normal(0, noise, 2) if noise else 0.0)))
            if len(obs) >= 2:
                smap.landmarks.append(M.Landmark(p.copy(), M.Track(obs, status=M.TRIANGULATED),
                                                 np.ones(len(obs), bool)))
        bad_E1 = exp_map(np.array([0.01, -0.005, 0.008, 0.04, -0.03, 0.02])) @ true_E1
        smap.rig = RigCalibration((0, 1), {0: Pose.identity(), 1: bad_E1})
        for f, kf in kfs.items():
            if kf.camera_id == 1:
                kf.cam_from_world = bad_E1 @ vposes[int(kf.timestamp)]
        if noise:
            for lm in smap.landmarks:
                lm.position = lm.position + rng.normal(0, 0.02, 3)
        general_ba_fixture(name, smap, cfg, stage, "rig_extrinsic")
    # rolling shutter: test_mapping.py:463-498 scene, and a longer sequence
    rng = np.random.default_rng(3)
    T_a = cam_pose([0, 0, 0])
    T_b_true = cam_pose([0.6, 0.04, 0.01], (0.02, -0.01, 0.015))
    pts = rng.uniform([-3, -2, 6], [3, 2, 12], (30, 3))
    exposure, dt = 0.03, 0.1
    kfs = {0: Keyframe(0, 0.0, 0, T_a, shutter="rolling", exposure=exposure), 1: Keyframe(1, dt, 0, T_b_true)}
    smap = M.SparseMap(kfs, {0: CAM}, fixed_frames={0})
    for p in pts:
        pix = project(CAM, T_a, p)
        for _ in range(8):
            alpha = (pix[1] / (CAM.height - 1)) * exposure / dt
            pix = project(CAM, interpolate_pose(T_a, T_b_true, alpha), p)
        pix_b = project(CAM, T_b_true, p)
        if not all(0 <= q[0] < CAM.width and 0 <= q[1] < CAM.height for q in (pix, pix_b)):
            continue
        smap.landmarks.append(M.Landmark(p.copy(), M.Track([M.Observation(0, 0, pix), M.Observation(1, 0, pix_b)],
                                                           status=M.TRIANGULATED), np.ones(2, bool)))
    kfs[1].cam_from_world = exp_map(rng.normal(0, 0.005, 6)) @ T_b_true
    general_ba_fixture("rolling", smap, M.MappingConfig(lambda_a=0.0, lambda_c=0.0, max_solver_iters=100), 2,
                       "pure")
    rng = np.random.default_rng(4)
    n = 8
    poses = {i: cam_pose([0.5 * i, 0.02 * i, 0], (0.01 * i, -0.015 * i, 0.005 * i)) for i in range(n)}
    kfs = {i: Keyframe(i, 0.1 * i, 0, poses[i], shutter="rolling", exposure=0.025) for i in range(n)}
    smap = M.SparseMap(kfs, {0: CAM}, fixed_frames={0})
    pts = rng.uniform([-4, -3, 6], [8, 3, 16], (80, 3))
    for p in pts:
        obs = []
        for i in range(n):
            pix = project(CAM, poses[i], p)
            if i + 1 < n:
                for _ in range(8):
                    alpha = (pix[1] / (CAM.height - 1)) * 0.025 / 0.1
                    pix = project(CAM, interpolate_pose(poses[i], poses[i + 1], alpha), p)
            if 0 <= pix[0] < CAM.width and 0 <= pix[1] < CAM.height:
                obs.append(M.Observation(i, 0, pix + rng.normal(0, 0.3, 2)))
        if len(obs) >= 2:
            smap.landmarks.append(M.Landmark(p + rng.normal(0, 0.02, 3), M.Track(obs, status=M.TRIANGULATED),
                                             np.ones(len(obs), bool)))
    for i in range(1, n):
        kfs[i].cam_from_world = exp_map(rng.normal(0, 0.003, 6)) @ poses[i]
    general_ba_fixture("rolling_seq", smap, M.MappingConfig(max_solver_iters=40), 1, "pure")


def iterative_map_rolling_fixture(name="iterative_map_rolling"):
    """iterative_map (mapping.py:569-624) over rolling-shutter keyframes:
    observations from the interpolated-pose model (mapping.py:321-356), a
    gross outlier on every 5th track, and pending tracks throughout."""
    rng = np.random.default_rng(21)
    n, exposure, dt = 7, 0.006, 0.1
    poses = {i: cam_pose([0.5 * i, 0.02 * i, 0], (0.01 * i, -0.015 * i, 0.005 * i)) for i in range(n)}
    pts = rng.uniform([-4, -3, 6], [8, 3, 16], (60, 3))
    tracks = []
    for k, p in enumerate(pts):
        obs = []
        for i in range(n):
            pix = project(CAM, poses[i], p)
            if i + 1 < n:
                for _ in range(8):
                    alpha = (pix[1] / (CAM.height - 1)) * exposure / dt
                    pix = project(CAM, interpolate_pose(poses[i], poses[i + 1], alpha), p)
            if 0 <= pix[0] < CAM.width and 0 <= pix[1] < CAM.height:
                obs.append(M.Observation(i, 0, pix + rng.normal(0, 0.3, 2)))
        if len(obs) < 3:
            continue
        if k % 5 == 0:
            obs[1] = M.Observation(obs[1].frame_id, 0, obs[1].pixel + np.array([40.0, 30.0]))
        tracks.append(M.Track(obs))
    kfs = [Keyframe(i, dt * i, 0, poses[i], shutter="rolling", exposure=exposure) for i in range(n)]
    for kf in kfs[1:]:
        kf.cam_from_world = exp_map(rng.normal(0, 0.003, 6)) @ kf.cam_from_world
    q0 = np.array([kf.cam_from_world.quat for kf in kfs])
    t0 = np.array([kf.cam_from_world.t for kf in kfs])
    ptr = np.zeros(len(tracks) + 1, np.int64)
    ptr[1:] = np.cumsum([len(t.observations) for t in tracks])
    of = np.array([o.frame_id for t in tracks for o in t.observations], np.int32)
    uv = np.array([o.pixel for t in tracks for o in t.observations])
    config = M.MappingConfig(max_solver_iters=30)
    smap = M.iterative_map(kfs, tracks, {0: CAM}, config=config)
    lm_track = np.array([next(i for i, t in enumerate(tracks) if t is lm.track)
                         for lm in smap.landmarks], np.int64)
    rs = smap.round_stats
    np.savez_compressed(
        os.path.join(HERE, f"{name}.npz"), cam_q=q0, cam_t=t0, track_ptr=ptr, obs_frame=of,
        obs_uv=uv, kf_timestamp=np.array([kf.timestamp for kf in kfs]),
        kf_exposure=np.full(n, exposure),
        ref_cam_q=np.array([smap.keyframes[f].cam_from_world.quat for f in range(n)]),
        ref_cam_t=np.array([smap.keyframes[f].cam_from_world.t for f in range(n)]),
        ref_lm_track=lm_track, ref_lm_X=np.array([lm.position for lm in smap.landmarks]),
        ref_lm_mask=np.concatenate([lm.inlier_mask for lm in smap.landmarks]).astype(np.uint8),
        ref_status=np.array([{"pending": 0, "triangulated": 1, "failed": 2}[t.status] for t in tracks]),
        ref_round_added=np.array([r["added"] for r in rs]),
        ref_round_removed=np.array([r["removed"] for r in rs]),
        ref_round_landmarks=np.array([r["landmarks"] for r in rs]),
        ref_mean_err=M.mean_reprojection_error(smap))
    print(f"{name}: tracks={len(tracks)} landmarks={len(smap.landmarks)} rounds={len(rs)} "
          f"added={[r['added'] for r in rs]} removed={[r['removed'] for r in rs]}")


def edge_fixture():
    """Empty / degenerate inputs through the reference entry points
    (bundle_adjust without landmarks, all frames fixed, empty gate, empty and
    single-track iterative_map) -> edge_cases.npz."""
    poses = {i: exp_map(np.array([0.01 * i, -0.02 * i, 0.005 * i, 0.3 * i, 0.0, 0.0])) for i in range(4)}
    out = {"poses4": np.array([np.concatenate([poses[i].quat, poses[i].t]) for i in range(4)])}
    # E1: free frames, pose terms only
    smap = M.SparseMap({i: Keyframe(i, float(i), 0, poses[i]) for i in range(4)}, {0: CAM}, fixed_frames={0})
    rep = M.bundle_adjust(smap, M.MappingConfig(), stage=1)
    out["e1_term"], out["e1_iters"], out["e1_cost"] = rep.termination, rep.iterations, rep.final_cost
    # E2: every frame fixed, no landmarks
    smap = M.SparseMap({i: Keyframe(i, float(i), 0, poses[i]) for i in range(4)}, {0: CAM},
                       fixed_frames={0, 1, 2, 3})
    rep = M.bundle_adjust(smap, M.MappingConfig(), stage=1)
    out["e2_term"], out["e2_iters"] = rep.termination, rep.iterations
    # E3: gate on a map without landmarks
    smap = M.SparseMap({i: Keyframe(i, float(i), 0, poses[i]) for i in range(4)}, {0: CAM}, fixed_frames={0})
    out["e3_removed"] = M.remove_outliers(smap, 2.0)[1]
    # E4: iterative_map without tracks
    sm = M.iterative_map([Keyframe(i, float(i), 0, poses[i]) for i in range(4)], [], {0: CAM})
    out["e4_stats"] = np.array([[r["added"], r["removed"], r["landmarks"]] for r in sm.round_stats])
    out["e4_fixed"] = np.array(sorted(sm.fixed_frames))
    # E5: iterative_map with one two-view track
    trs = [M.Track([M.Observation(0, 0, np.array([100.0, 100.0])), M.Observation(1, 0, np.array([100.0, 100.0]))])]
    sm = M.iterative_map([Keyframe(i, float(i), 0, poses[i]) for i in range(4)], trs, {0: CAM})
    out["e5_stats"] = np.array([[r["added"], r["removed"], r["landmarks"]] for r in sm.round_stats])
    out["e5_status"] = trs[0].status
    out["e5_X"] = np.array([lm.position for lm in sm.landmarks])
    # E6: all frames fixed, landmarks free (points-only problem)
    rng = np.random.default_rng(11)
    pts, sposes = scene(rng, 5, 25)
    smap = map_from_scene(pts, sposes, 0.01, rng, fixed_frames=tuple(range(5)), noise=0.3)
    X0 = np.array([lm.position for lm in smap.landmarks])
    rep = M.bundle_adjust(smap, M.MappingConfig(max_solver_iters=30), stage=1)
    out["e6_X0"] = X0
    out["e6_X"] = np.array([lm.position for lm in smap.landmarks])
    out["e6_term"], out["e6_iters"], out["e6_cost"] = rep.termination, rep.iterations, rep.final_cost
    out["e6_poses"] = np.array([np.concatenate([sposes[f].quat, sposes[f].t]) for f in sorted(sposes)])
    out["e6_obs"] = np.array([[k, o.frame_id, o.pixel[0], o.pixel[1]] for k, lm in enumerate(smap.landmarks)
                              for o in lm.track.observations])
    np.savez_compressed(os.path.join(HERE, "edge_cases.npz"), **out)
    print("edge_cases:", {k: v for k, v in out.items() if np.ndim(v) == 0})


# --- known-answer vectors for the geometry --------------------------------------

def kat_fixture():
    rng = np.random.default_rng(55)
    cams = [CAM, CameraModel("pinhole_radial", 420.0, 410.0, 300.0, 230.0, 640, 480, (-0.12, 0.03)),
            CameraModel("equidistant_fisheye", 300.0, 300.0, 320.0, 240.0, 640, 480)]
    rows = []
    for ci, cam in enumerate(cams):
        for _ in range(60):
            pose = exp_map(rng.normal(0, [0.3, 0.3, 0.3, 1.0, 1.0, 1.0]))
            X = rng.uniform([-3, -3, 4], [3, 3, 12])
            X = pose.inverse().apply(X)  # point in front of the camera
            pix, Jp, Jx = project_with_pose_jacobian(cam, pose, X)
            ray = unproject(cam, pix)
            rows.append(np.concatenate([[ci], pose.quat, pose.t, X, pix, Jp.ravel(), Jx.ravel(), ray]))
    models = np.array([[0, 500.0, 500.0, 320.0, 240.0, 0.0, 0.0],
                       [1, 420.0, 410.0, 300.0, 230.0, -0.12, 0.03],
                       [2, 300.0, 300.0, 320.0, 240.0, 0.0, 0.0]])
    # pose terms: edge and prior residual/Jacobians (posegraph.py:195-206, mapping.py:359-368)
    prow = []
    for _ in range(40):
        Ta, Tb, Te = (exp_map(rng.normal(0, 0.4, 6)) for _ in range(3))
        lam = float(rng.uniform(0.1, 5.0))
        meas = Ta @ Tb.inverse()
        meas = exp_map(rng.normal(0, 0.05, 6)) @ meas
        fn = _edge_residual_fn(PoseEdge("sequential", 0, 1, meas, lam * np.eye(6)))
        r, (Ja, Jb) = fn(Ta, Tb)
        pfn = M.absolute_prior_residual_fn(Te, lam)
        Tc = exp_map(rng.normal(0, 0.05, 6)) @ Te
        rp, (Jpr,) = pfn(Tc)
        prow.append(np.concatenate([[lam], Ta.quat, Ta.t, Tb.quat, Tb.t, meas.quat, meas.t, r,
                                    Ja.ravel(), Jb.ravel(), Te.quat, Te.t, Tc.quat, Tc.t, rp,
                                    Jpr.ravel()]))
    np.savez_compressed(os.path.join(HERE, "kat_geometry.npz"), models=models, proj=np.array(rows),
                        pose_terms=np.array(prow))
    print(f"kat_geometry: {len(rows)} projections, {len(prow)} pose terms")


if __name__ == "__main__":
    which = sys.argv[1:] or ["kat", "tri", "gate", "imap", "ba", "kinds", "tracks", "rigrs", "edge"]
    if "kat" in which:
        kat_fixture()
    if "kinds" in which:
        camera_kinds_fixtures()
    if "tracks" in which:
        tracks_fixture()
    if "edge" in which:
        edge_fixture()
    if "rigrs" in which:
        rig_rs_fixtures()
        iterative_map_rolling_fixture()
    if "tri" in which:
        tri_fixtures()
    if "gate" in which:
        gate_fixture()
    if "imap" in which:
        iterative_map_fixture()
        # larger: 12 frames, outliers re-gated across rounds, Cauchy stage 1
        iterative_map_fixture("iterative_map_large", seed=77, n_frames=12, n_points=160,
                              config=M.MappingConfig(stage1=M.StageConfig(4.0, SV.RobustLoss("cauchy", 1.0)),
                                                     lambda_c=0.5, lambda_a=2.0, max_solver_iters=25),
                              noise=0.8, mild_every=3)
    if "ba" in which:
        ba_fixtures()
