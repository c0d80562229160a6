"""The drop-in driven with sfmkit's OWN objects (duck typing, INTEGRATION.md
section 1): sfmkit.mapping.SparseMap / Track / Observation, sfmkit.keyframes
.Keyframe, sfmkit.se3.Pose, sfmkit.cameras.CameraModel passed straight into
this package's iterative_map / bundle_adjust, results written back into
them and compared with sfmkit's recorded outputs (tests/golden).  sfmkit is
imported from the unmodified install in baseline/_ref (bench.py's CPU
reference; git-ignored, it travels with the repo to the GPU box); skipped
when that install is absent."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")


@pytest.fixture(scope="module")
def sfmkit():
    if not os.path.isdir(os.path.join(REF, "sfmkit")):
        pytest.skip("sfmkit not installed in baseline/_ref")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    sys.dont_write_bytecode = True
    import sfmkit.cameras
    import sfmkit.keyframes
    import sfmkit.mapping
    import sfmkit.se3
    return sfmkit


def test_iterative_map_on_sfmkit_objects(golden, sfmkit):
    from paper_2510_15271_b200 import iterative_map
    SM = sfmkit.mapping
    d = golden("iterative_map")
    cam = sfmkit.cameras.CameraModel("pinhole", 500.0, 500.0, 320.0, 240.0, 640, 480)
    kfs = [sfmkit.keyframes.Keyframe(f, float(f), 0, sfmkit.se3.Pose(d["cam_q"][f], d["cam_t"][f]))
           for f in range(len(d["cam_q"]))]
    ptr = d["track_ptr"]
    tracks = [SM.Track([SM.Observation(int(d["obs_frame"][o]), 0, d["obs_uv"][o])
                        for o in range(ptr[i], ptr[i + 1])]) for i in range(len(ptr) - 1)]
    smap = iterative_map(kfs, tracks, {0: cam})
    stat = np.array([{"pending": 0, "triangulated": 1, "failed": 2}[t.status] for t in tracks])
    np.testing.assert_array_equal(stat, d["ref_status"])
    assert [r["added"] for r in smap.round_stats] == list(d["ref_round_added"])
    lm_track = [next(i for i, t in enumerate(tracks) if t is lm.track) for lm in smap.landmarks]
    np.testing.assert_array_equal(lm_track, d["ref_lm_track"])
    mask = np.concatenate([lm.inlier_mask for lm in smap.landmarks]).astype(np.uint8)
    np.testing.assert_array_equal(mask, d["ref_lm_mask"])
    np.testing.assert_allclose([lm.position for lm in smap.landmarks], d["ref_lm_X"], atol=1e-6)
    # poses written back into sfmkit's Keyframe objects as sfmkit Poses
    for f, kf in enumerate(kfs):
        assert type(kf.cam_from_world).__module__.startswith(("sfmkit", "paper_2510_15271_b200"))
        np.testing.assert_allclose(kf.cam_from_world.quat, d["ref_cam_q"][f], atol=1e-7)


def test_bundle_adjust_on_sfmkit_sparse_map(golden, sfmkit):
    """bundle_adjust(sfmkit SparseMap) -- positions and poses written back
    into sfmkit's objects, the report as sfmkit's solve returns it."""
    from paper_2510_15271_b200 import MappingConfig, bundle_adjust
    SM = sfmkit.mapping
    d = golden("ba_plain_stage2")
    cam = sfmkit.cameras.CameraModel("pinhole", 500.0, 500.0, 320.0, 240.0, 640, 480)
    F = len(d["cam_q"])
    kfs = {f: sfmkit.keyframes.Keyframe(f, float(f), 0, sfmkit.se3.Pose(d["cam_q"][f], d["cam_t"][f]))
           for f in range(F)}
    fixed = {int(f) for f in np.flatnonzero(d["frame_fixed"])}
    smap = SM.SparseMap(kfs, {0: cam}, fixed_frames=fixed)
    ptr = np.searchsorted(d["obs_point"], np.arange(len(d["points"]) + 1))
    for p in range(len(d["points"])):
        obs = [SM.Observation(int(d["obs_frame"][o]), 0, d["obs_uv"][o]) for o in range(ptr[p], ptr[p + 1])]
        smap.landmarks.append(SM.Landmark(d["points"][p], SM.Track(obs, "triangulated"), np.ones(len(obs), bool)))
    rep = bundle_adjust(smap, MappingConfig(lambda_a=0.0, lambda_c=0.0, max_solver_iters=100), stage=2)
    assert rep.termination == str(d["ref_termination"])
    assert rep.final_cost == pytest.approx(float(d["ref_final_cost"]), rel=1e-3, abs=1e-18)
    X = np.array([lm.position for lm in smap.landmarks])
    np.testing.assert_allclose(X, d["ref_points"], atol=1e-8)
