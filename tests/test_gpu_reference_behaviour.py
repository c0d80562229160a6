"""The behaviours the reference's own hot-path tests pin
(/root/reference/pkg/tests/test_mapping.py),
restated against this package's drop-in API and run on the B200: the same
scenes (a short forward sweep of pinhole cameras over a box of points),
the same thresholds, every call through libsfm_b200.so.  Scene data is
generated with the oracle's projection (test infrastructure only).
"""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

from paper_2510_15271_b200 import (FAILED, PENDING, TRIANGULATED, CameraModel,
                                   CheiralityViolation, InsufficientParallax, Keyframe, Landmark,
                                   MappingConfig, NoGauge, Observation, ParallelRays, Pose,
                                   SparseMap, StageConfig, Track, bundle_adjust, exp_map,
                                   iterative_map, log_map, mean_reprojection_error,
                                   ransac_triangulate, remove_outliers, triangulate_dlt,
                                   triangulate_midpoint)

pytestmark = pytest.mark.gpu

CAM = CameraModel("pinhole", 500.0, 500.0, 320.0, 240.0, 640, 480)
MODEL = (0, 500.0, 500.0, 320.0, 240.0, (0.0, 0.0))


def project(pose, X):
    from oracle import geometry as G
    pix, st = G.project_cam(MODEL, (pose.R @ np.asarray(X, float) + pose.t)[None])
    assert st[0] == G.OK
    return pix[0]


def cam_pose(center, rot_xi=(0.0, 0.0, 0.0)):
    R = exp_map(np.array([*rot_xi, 0.0, 0.0, 0.0])).R
    c = np.asarray(center, float)
    from paper_2510_15271_b200.scenes import R_to_quat
    return Pose(R_to_quat(R[None])[0], -R @ c)


def scene(rng, n_frames=6, n_points=40, spacing=0.8):
    points = rng.uniform([-4, -3, 6], [4, 3, 14], (n_points, 3))
    poses = {i: cam_pose([spacing * i, 0.05 * i, 0], (0.02 * i, -0.03 * i, 0.01 * i))
             for i in range(n_frames)}
    return points, poses


def observations(point, poses):
    obs = []
    for f in sorted(poses):
        pix = project(poses[f], point)
        if 0 <= pix[0] < CAM.width and 0 <= pix[1] < CAM.height:
            obs.append(Observation(f, 0, pix))
    return obs


def cams_for(poses):
    return {f: CAM for f in poses}


def map_from_scene(points, poses, perturb=0.0, rng=None, fixed_frames=(0, 1)):
    kfs = {f: Keyframe(f, float(f), 0, poses[f]) for f in poses}
    smap = SparseMap(kfs, {0: CAM}, fixed_frames=set(fixed_frames))
    for p in points:
        obs = observations(p, poses)
        if len(obs) < 2:
            continue
        smap.landmarks.append(Landmark(p.copy(), Track(obs, status=TRIANGULATED),
                                       np.ones(len(obs), bool)))
    if perturb and rng is not None:
        for f in poses:
            if f in smap.fixed_frames:
                continue
            kfs[f].cam_from_world = exp_map(rng.normal(0, perturb, 6)) @ kfs[f].cam_from_world
        for lm in smap.landmarks:
            lm.position = lm.position + rng.normal(0, 5 * perturb, 3)
    return smap


def pose_err(a, b):
    return float(np.linalg.norm(log_map(a @ b.inverse())))


@pytest.fixture
def rng():
    return np.random.default_rng(42)


# --- triangulation (test_mapping.py:136-218) --------------------------------

def test_dlt_exact_recovery(rng):
    points, poses = scene(rng)
    for p in points[:10]:
        obs = observations(p, poses)
        assert len(obs) >= 2
        assert np.linalg.norm(triangulate_dlt(obs, poses, cams_for(poses)) - p) < 1e-6


def test_dlt_insufficient_parallax(rng):
    points, _ = scene(rng)
    poses = {0: cam_pose([0, 0, 0]), 1: cam_pose([0, 0, 0], (0.0, 0.05, 0))}
    with pytest.raises(InsufficientParallax):
        triangulate_dlt(observations(points[0], poses), poses, cams_for(poses))


def test_dlt_cheirality_violation():
    poses = {0: cam_pose([0, 0, 0]), 1: cam_pose([1.0, 0, 0])}
    p = np.array([0.3, 0.2, 10.0])
    obs = [Observation(0, 0, project(poses[1], p)), Observation(1, 0, project(poses[0], p))]
    with pytest.raises(CheiralityViolation):
        triangulate_dlt(obs, poses, cams_for(poses))


def test_midpoint_matches_dlt_noiseless(rng):
    points, poses = scene(rng)
    for p in points[:10]:
        obs = observations(p, poses)
        Xd = triangulate_dlt(obs, poses, cams_for(poses))
        Xm = triangulate_midpoint(obs, poses, cams_for(poses))
        assert np.linalg.norm(Xm - p) < 1e-6 and np.linalg.norm(Xm - Xd) < 1e-6


def test_midpoint_parallel_rays():
    poses = {0: cam_pose([0, 0, 0]), 1: cam_pose([1.0, 0, 0])}
    obs = [Observation(0, 0, (CAM.cx, CAM.cy)), Observation(1, 0, (CAM.cx, CAM.cy))]
    with pytest.raises(ParallelRays):
        triangulate_midpoint(obs, poses, cams_for(poses))


def test_ransac_rejects_outlier_observation(rng):
    points, poses = scene(rng)
    p = points[0]
    obs = observations(p, poses)
    obs[2] = Observation(obs[2].frame_id, 0, obs[2].pixel + np.array([60.0, -40.0]))
    track = Track(obs)
    lm = ransac_triangulate(track, poses, cams_for(poses), threshold_px=2.0)
    assert lm is not None and track.status == TRIANGULATED
    assert not lm.inlier_mask[2] and int(lm.inlier_mask.sum()) == len(obs) - 1
    assert np.linalg.norm(lm.position - p) < 1e-6


def test_ransac_fails_on_degenerate_track():
    poses = {0: cam_pose([0, 0, 0]), 1: cam_pose([0, 0, 0], (0, 0.05, 0))}
    p = np.array([0.5, -0.3, 9.0])
    track = Track([Observation(f, 0, project(poses[f], p)) for f in poses])
    assert ransac_triangulate(track, poses, cams_for(poses)) is None
    assert track.status == FAILED


def test_ransac_midpoint_method(rng):
    points, poses = scene(rng)
    lm = ransac_triangulate(Track(observations(points[1], poses)), poses, cams_for(poses),
                            method="midpoint")
    assert lm is not None and np.linalg.norm(lm.position - points[1]) < 1e-6


# --- residual Jacobians (test_mapping.py:221-229): device J~ vs central FD --

def test_reprojection_jacobian_fd():
    """sfm_ba_eval's analytic 2x6 (left perturbation, (phi, rho)) and 2x3
    Jacobians against central differences of its own residuals."""
    from paper_2510_15271_b200 import _native as nat
    from paper_2510_15271_b200.mapping import BAArrays, model_table
    pose = cam_pose([0.3, -0.2, 0.1], (0.05, 0.02, -0.04))
    X = np.array([0.7, -0.4, 9.0])
    pix = project(pose, X) + np.array([0.5, -0.3])
    models, n_models, fm = model_table([CAM])

    def evaluate(q, t, Xv):
        a = BAArrays(np.ascontiguousarray(q[None]), np.ascontiguousarray(t[None]), fm,
                     np.zeros(1, np.uint8), models, n_models, np.ascontiguousarray(Xv[None]),
                     np.zeros(1, np.int32), np.zeros(1, np.int32), np.ascontiguousarray(pix[None]),
                     np.zeros((0, 2), np.int32), np.zeros(0, np.int32))
        ctx = nat.default_context()
        s = a.struct()
        r = np.empty((1, 2))
        jc = np.empty((1, 2, 6))
        jp = np.empty((1, 2, 3))
        ctx.check(ctx.lib.sfm_ba_eval(ctx.handle, ctypes.byref(s), 0, 1.0, None, nat.ptr(r),
                                      nat.ptr(jc), nat.ptr(jp)))
        return r[0], jc[0], jp[0]

    r0, Jc, Jp = evaluate(pose.quat, pose.t, X)
    h = 1e-6
    for k in range(6):
        d = np.zeros(6)
        d[k] = h
        Pp, Pm = exp_map(d) @ pose, exp_map(-d) @ pose
        fd = (evaluate(Pp.quat, Pp.t, X)[0] - evaluate(Pm.quat, Pm.t, X)[0]) / (2 * h)
        assert np.abs(fd - Jc[:, k]).max() < 1e-4
    for k in range(3):
        d = np.zeros(3)
        d[k] = h
        fd = (evaluate(pose.quat, pose.t, X + d)[0] - evaluate(pose.quat, pose.t, X - d)[0]) / (2 * h)
        assert np.abs(fd - Jp[:, k]).max() < 1e-4


# --- bundle adjustment (test_mapping.py:298-417) ----------------------------

def test_no_gauge_raises(rng):
    points, poses = scene(rng, n_frames=3, n_points=10)
    smap = map_from_scene(points, poses, fixed_frames=())
    with pytest.raises(NoGauge):
        bundle_adjust(smap, MappingConfig(lambda_a=0.0, lambda_c=0.0), stage=2)


def test_ba_recovers_poses_and_points(rng):
    points, poses = scene(rng, n_frames=6, n_points=40)
    smap = map_from_scene(points, poses, perturb=0.01, rng=rng)
    bundle_adjust(smap, MappingConfig(lambda_a=0.0, lambda_c=0.0, max_solver_iters=100), stage=2)
    for f, pose in poses.items():
        assert pose_err(smap.keyframes[f].cam_from_world, pose) < 1e-6
    for lm, p in zip(smap.landmarks, points):
        assert np.linalg.norm(lm.position - p) < 1e-6
    assert mean_reprojection_error(smap) < 1e-8


def test_ba_fixed_frames_bit_identical(rng):
    points, poses = scene(rng, n_frames=5, n_points=25)
    smap = map_from_scene(points, poses, perturb=0.005, rng=rng)
    before = {f: (smap.keyframes[f].cam_from_world.quat.tobytes(),
                  smap.keyframes[f].cam_from_world.t.tobytes()) for f in smap.fixed_frames}
    bundle_adjust(smap, MappingConfig(lambda_a=0.0, lambda_c=0.0), stage=1)
    for f in smap.fixed_frames:
        after = smap.keyframes[f].cam_from_world
        assert (after.quat.tobytes(), after.t.tobytes()) == before[f]


def test_ba_absolute_prior_provides_gauge(rng):
    points, poses = scene(rng, n_frames=4, n_points=20)
    smap = map_from_scene(points, poses, fixed_frames=())
    report = bundle_adjust(smap, MappingConfig(lambda_a=10.0, lambda_c=0.0), stage=2)
    for f, pose in poses.items():
        assert smap.keyframes[f].cam_from_world.almost_equal(pose, tol=1e-6)
    assert report.final_cost <= report.initial_cost + 1e-12


def test_ba_robust_loss_resists_outliers(rng):
    points, poses = scene(rng, n_frames=6, n_points=40)

    def run(cfg, seed_rng):
        smap = map_from_scene(points, poses, perturb=0.002, rng=seed_rng)
        for lm in smap.landmarks[::7]:
            lm.track.observations[1].pixel = lm.track.observations[1].pixel + np.array([35.0, -25.0])
        bundle_adjust(smap, cfg, stage=1)
        return max(pose_err(smap.keyframes[f].cam_from_world, poses[f]) for f in poses)

    err_huber = run(MappingConfig(lambda_a=0.0, lambda_c=0.0, max_solver_iters=100),
                    np.random.default_rng(7))
    err_plain = run(MappingConfig(stage1=StageConfig(4.0), lambda_a=0.0, lambda_c=0.0,
                                  max_solver_iters=100), np.random.default_rng(7))
    assert err_huber < 0.5 * err_plain and err_huber < 0.1


def test_localization_fixed_freezes_prior_frames(rng):
    points, poses = scene(rng, n_frames=6, n_points=30)
    smap = map_from_scene(points, poses, perturb=0.01, rng=rng, fixed_frames=())
    smap.provenance = {f: ("prior" if f < 3 else "new") for f in poses}
    for f in range(3):
        smap.keyframes[f].cam_from_world = poses[f]
    bundle_adjust(smap, MappingConfig(lambda_a=0.0, lambda_c=0.0, max_solver_iters=100), stage=2,
                  mode="localization_fixed")
    for f in range(3):
        assert smap.keyframes[f].cam_from_world.almost_equal(poses[f], 1e-12)
    for f in range(3, 6):
        assert smap.keyframes[f].cam_from_world.almost_equal(poses[f], 1e-6)


def test_localization_adjust_moves_prior_frames(rng):
    points, poses = scene(rng, n_frames=6, n_points=30)
    smap = map_from_scene(points, poses, perturb=0.01, rng=rng, fixed_frames=(0,))
    smap.provenance = {f: ("prior" if f < 3 else "new") for f in poses}
    entry = {f: smap.keyframes[f].cam_from_world for f in poses}
    bundle_adjust(smap, MappingConfig(lambda_a=1e-4, lambda_c=0.0, max_solver_iters=100), stage=2,
                  mode="localization_adjust")
    assert [f for f in (1, 2) if not smap.keyframes[f].cam_from_world.almost_equal(entry[f], 1e-9)]
    total = sum(pose_err(smap.keyframes[f].cam_from_world, poses[f]) for f in poses if f)
    entry_total = sum(pose_err(entry[f], poses[f]) for f in poses if f)
    assert total < 0.35 * entry_total


def test_ba_relative_consistency_terms(rng):
    points, poses = scene(rng, n_frames=5, n_points=25)
    smap = map_from_scene(points, poses)
    bundle_adjust(smap, MappingConfig(lambda_a=0.0, lambda_c=100.0), stage=2)
    for f, pose in poses.items():
        assert smap.keyframes[f].cam_from_world.almost_equal(pose, tol=1e-8)


def test_rig_mode_without_rig_raises_no_gauge(rng):
    """mapping.py:424-425: rig_extrinsic mode needs a rig calibration."""
    points, poses = scene(rng, n_frames=3, n_points=10)
    smap = map_from_scene(points, poses)
    with pytest.raises(NoGauge):
        bundle_adjust(smap, MappingConfig(), stage=1, mode="rig_extrinsic")


# --- outlier removal (test_mapping.py:502-523) ------------------------------

def test_remove_outliers_flags_and_counts(rng):
    points, poses = scene(rng, n_frames=5, n_points=15)
    smap = map_from_scene(points, poses)
    o = smap.landmarks[0].track.observations[1]
    o.pixel = o.pixel + np.array([10.0, 0.0])
    _, removed = remove_outliers(smap, 2.0)
    assert removed == 1 and not smap.landmarks[0].inlier_mask[1]
    _, removed_again = remove_outliers(smap, 2.0)
    assert removed_again == 0


def test_remove_outliers_demotes_thin_landmarks(rng):
    points, poses = scene(rng, n_frames=5, n_points=5)
    smap = map_from_scene(points, poses)
    lm = smap.landmarks[0]
    for o in lm.track.observations[1:]:
        o.pixel = o.pixel + np.array([25.0, 25.0])
    n_before = len(smap.landmarks)
    _, removed = remove_outliers(smap, 2.0)
    assert removed == len(lm.track.observations) - 1
    assert lm.track.status == PENDING and len(smap.landmarks) == n_before - 1


# --- iterative mapping (test_mapping.py:528-581) ----------------------------

def test_iterative_map_end_to_end(rng):
    points, poses = scene(rng, n_frames=6, n_points=35)
    kfs = [Keyframe(f, float(f), 0, poses[f]) for f in sorted(poses)]
    tracks = [Track(obs) for obs in (observations(p, poses) for p in points) if len(obs) >= 2]
    smap = iterative_map(kfs, tracks, {0: CAM})
    assert len(smap.landmarks) == len(tracks)
    assert all(t.status == TRIANGULATED for t in tracks)
    assert mean_reprojection_error(smap) < 1e-6
    for lm in smap.landmarks:
        assert np.linalg.norm(points - lm.position, axis=1).min() < 1e-6
    assert smap.round_stats[-1]["round"] == "final"
    assert len(smap.round_stats) <= MappingConfig().max_outer_iters + 1


def test_iterative_map_prunes_outlier_observations(rng):
    points, poses = scene(rng, n_frames=6, n_points=30)
    kfs = [Keyframe(f, float(f), 0, poses[f]) for f in sorted(poses)]
    tracks = []
    for k, p in enumerate(points):
        obs = observations(p, poses)
        if len(obs) < 3:
            continue
        if k % 5 == 0:
            obs[1] = Observation(obs[1].frame_id, 0, obs[1].pixel + np.array([40.0, 30.0]))
        tracks.append(Track(obs))
    smap = iterative_map(kfs, tracks, {0: CAM})
    assert mean_reprojection_error(smap) < 1e-6
    for lm in smap.landmarks:
        for o, ok in zip(lm.track.observations, lm.inlier_mask):
            if ok:
                pix = project(smap.keyframes[o.frame_id].cam_from_world, lm.position)
                assert np.linalg.norm(pix - o.pixel) < 2.0


def test_iterative_map_terminates_without_progress():
    poses = {0: cam_pose([0, 0, 0]), 1: cam_pose([0, 0, 0], (0, 0.04, 0))}
    p = np.array([0.2, 0.1, 8.0])
    kfs = [Keyframe(f, float(f), 0, poses[f]) for f in poses]
    tracks = [Track([Observation(f, 0, project(poses[f], p)) for f in poses])]
    smap = iterative_map(kfs, tracks, {0: CAM})
    assert tracks[0].status == FAILED
    assert len(smap.landmarks) == 0 and len(smap.round_stats) <= 2


def test_stage_config_invariant():
    with pytest.raises(ValueError):
        MappingConfig(stage1=StageConfig(2.0), stage2=StageConfig(4.0))
