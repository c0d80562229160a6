"""Empty and degenerate inputs through the drop-in entry points, against
sfmkit's own results on the same inputs (tests/golden/make_golden.py
`edge_fixture`): bundle_adjust without landmarks (pose terms only), with
every frame fixed, and with only the points free; remove_outliers on a map
without landmarks; iterative_map without tracks and with one two-view track;
an empty RANSAC batch."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2510_15271_b200 import (CameraModel, Keyframe, Landmark, MappingConfig, Observation, Pose,
                                   SparseMap, Track, bundle_adjust, iterative_map, remove_outliers)
from paper_2510_15271_b200.mapping import ransac_triangulate_batch

pytestmark = pytest.mark.gpu

CAM = CameraModel("pinhole", 500.0, 500.0, 320.0, 240.0, 640, 480)


def _kfs(d):
    return {i: Keyframe(i, float(i), 0, Pose(d["poses4"][i][:4], d["poses4"][i][4:])) for i in range(4)}


def test_bundle_adjust_without_landmarks(golden):
    """mapping.py:390-527 with only the lambda_c / lambda_a terms: converged
    at entry (gradient_tolerance, 0 iterations)."""
    d = golden("edge_cases")
    smap = SparseMap(_kfs(d), {0: CAM}, fixed_frames={0})
    rep = bundle_adjust(smap, MappingConfig(), stage=1)
    assert rep.termination == str(d["e1_term"])
    assert rep.iterations == int(d["e1_iters"])
    assert rep.final_cost == pytest.approx(float(d["e1_cost"]), abs=1e-20)


def test_bundle_adjust_all_frames_fixed_no_landmarks(golden):
    """solver.py: no free parameter block -> 'all_fixed'."""
    d = golden("edge_cases")
    smap = SparseMap(_kfs(d), {0: CAM}, fixed_frames={0, 1, 2, 3})
    rep = bundle_adjust(smap, MappingConfig(), stage=1)
    assert rep.termination == str(d["e2_term"])
    assert rep.iterations == int(d["e2_iters"])


def test_remove_outliers_on_empty_map(golden):
    d = golden("edge_cases")
    smap = SparseMap(_kfs(d), {0: CAM}, fixed_frames={0})
    _, removed = remove_outliers(smap, 2.0)
    assert removed == int(d["e3_removed"])
    assert smap.landmarks == []


def test_iterative_map_without_tracks(golden):
    d = golden("edge_cases")
    kfs = _kfs(d)
    smap = iterative_map([kfs[i] for i in range(4)], [], {0: CAM})
    stats = np.array([[r["added"], r["removed"], r["landmarks"]] for r in smap.round_stats])
    np.testing.assert_array_equal(stats, d["e4_stats"])
    np.testing.assert_array_equal(sorted(smap.fixed_frames), d["e4_fixed"])
    assert smap.landmarks == []


def test_iterative_map_single_two_view_track(golden):
    d = golden("edge_cases")
    kfs = _kfs(d)
    tr = Track([Observation(0, 0, np.array([100.0, 100.0])), Observation(1, 0, np.array([100.0, 100.0]))])
    smap = iterative_map([kfs[i] for i in range(4)], [tr], {0: CAM})
    stats = np.array([[r["added"], r["removed"], r["landmarks"]] for r in smap.round_stats])
    np.testing.assert_array_equal(stats, d["e5_stats"])
    assert tr.status == str(d["e5_status"])
    np.testing.assert_allclose([lm.position for lm in smap.landmarks], d["e5_X"], rtol=1e-7, atol=1e-9)


def test_ransac_empty_batch():
    assert ransac_triangulate_batch([], {}, {}) == []


def test_bundle_adjust_points_only(golden):
    """Every frame fixed, landmarks free: the Schur system has no camera
    block (the point-only path), same iterations / cost / points as sfmkit."""
    d = golden("edge_cases")
    P = d["e6_poses"]
    kfs = {f: Keyframe(f, float(f), 0, Pose(P[f][:4], P[f][4:])) for f in range(len(P))}
    smap = SparseMap(kfs, {0: CAM}, fixed_frames=set(range(len(P))))
    obs = d["e6_obs"]
    for k, X in enumerate(d["e6_X0"]):
        rows = obs[obs[:, 0] == k]
        o = [Observation(int(r[1]), 0, np.array([r[2], r[3]])) for r in rows]
        smap.landmarks.append(Landmark(X.copy(), Track(o, "triangulated"), np.ones(len(o), bool)))
    rep = bundle_adjust(smap, MappingConfig(max_solver_iters=30), stage=1)
    assert rep.termination == str(d["e6_term"])
    assert rep.iterations == int(d["e6_iters"])
    assert rep.final_cost == pytest.approx(float(d["e6_cost"]), rel=1e-6)
    np.testing.assert_allclose([lm.position for lm in smap.landmarks], d["e6_X"], rtol=1e-7, atol=1e-8)


def test_iterative_map_empty_without_gauge():
    """sfmkit raises NoGauge only from a bundle_adjust that has landmarks
    (mapping.py:408-409, reached through :611): with no keyframes and
    lambda_a = 0 it returns an empty map with one empty round (sfmkit:
    [{'round': 0, 'added': 0, 'removed': 0, 'landmarks': 0}])."""
    smap = iterative_map([], [], {}, MappingConfig(lambda_a=0.0))
    assert smap.round_stats == [{"round": 0, "added": 0, "removed": 0, "landmarks": 0}]
    assert smap.landmarks == [] and smap.fixed_frames == set()


def test_triangulate_fisheye_beyond_model_domain():
    """unproject of a fisheye pixel whose distorted radius is beyond 90 deg
    raises OutOfModelDomain (cameras.py:106-108), not UndistortDiverged --
    sfmkit's triangulate_dlt on these inputs: OutOfModelDomain('distorted
    radius beyond 90 deg')."""
    from paper_2510_15271_b200 import OutOfModelDomain, triangulate_dlt, triangulate_midpoint
    cam = CameraModel("equidistant_fisheye", 300.0, 300.0, 320.0, 240.0, 640, 480)
    poses = {0: Pose(), 1: Pose(np.array([1, 0, 0, 0.0]), np.array([-1.0, 0, 0]))}
    cams = {0: cam, 1: cam}
    obs = [Observation(0, 0, np.array([320 + 300 * 1.7, 240.0])), Observation(1, 0, np.array([300.0, 240.0]))]
    with pytest.raises(OutOfModelDomain):
        triangulate_dlt(obs, poses, cams)
    with pytest.raises(OutOfModelDomain):
        triangulate_midpoint(obs, poses, cams)


def test_ransac_unknown_method_is_midpoint(golden):
    """ransac_triangulate treats every method other than "dlt" as the
    midpoint method (mapping.py:270-278)."""
    from paper_2510_15271_b200 import ransac_triangulate
    d = golden("tri_midpoint")
    cam = CameraModel("pinhole", 500.0, 500.0, 320.0, 240.0, 640, 480)
    F = len(d["cam_q"])
    poses = {f: Pose(d["cam_q"][f], d["cam_t"][f]) for f in range(F)}
    cams = {f: cam for f in range(F)}
    ptr = d["track_ptr"]
    for i in range(min(20, len(ptr) - 1)):
        obs = [Observation(int(d["obs_frame"][o]), 0, d["obs_uv"][o]) for o in range(ptr[i], ptr[i + 1])]
        a = ransac_triangulate(Track(list(obs)), poses, cams, threshold_px=float(d["threshold_px"]),
                               min_angle=float(d["min_angle"]), method="midpoint")
        b = ransac_triangulate(Track(list(obs)), poses, cams, threshold_px=float(d["threshold_px"]),
                               min_angle=float(d["min_angle"]), method="anything-else")
        assert (a is None) == (b is None)
        if a is not None:
            assert np.array_equal(a.position, b.position)
            assert np.array_equal(a.inlier_mask, b.inlier_mask)
