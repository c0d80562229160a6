"""CUDA path vs the reference (golden fixtures) and the oracle, through the
C-ABI.  Needs a B200: run with `pytest -m gpu`."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

BA_CASES = ["plain_stage2", "huber_outliers", "cauchy_pose_terms", "localization_fixed",
            "localization_adjust", "prior_gauge", "pure_provenance_lc", "config1", "camera_kinds"]
LOSS_NAMES = {0: "trivial", 1: "huber", 2: "cauchy"}


def arrays_from_npz(d):
    from paper_2510_15271_b200 import _native as nat
    from paper_2510_15271_b200.mapping import BAArrays
    m = d["models"]
    models = (nat.CameraModelC * len(m))(*[
        nat.CameraModelC(int(r[0]), 640, 480, 0, *[float(v) for v in r[1:7]]) for r in m])
    return BAArrays(np.ascontiguousarray(d["cam_q"]), np.ascontiguousarray(d["cam_t"]),
                    np.ascontiguousarray(d["frame_model"], dtype=np.int32),
                    np.ascontiguousarray(d["frame_fixed"], dtype=np.uint8), models, len(m),
                    np.ascontiguousarray(d["points"]), np.ascontiguousarray(d["obs_frame"]),
                    np.ascontiguousarray(d["obs_point"]), np.ascontiguousarray(d["obs_uv"]),
                    np.ascontiguousarray(d["edge_ab"], dtype=np.int32).reshape(-1, 2),
                    np.ascontiguousarray(d["prior_frame"], dtype=np.int32),
                    float(d["edge_weight"]), float(d["prior_weight"]))


def solve_case(d, linear_solver="auto"):
    from paper_2510_15271_b200.mapping import solve_arrays
    from paper_2510_15271_b200.solver import DeviceOptions, RobustLoss, SolverOptions
    loss = RobustLoss(LOSS_NAMES[int(d["loss_kind"])], float(d["loss_param"]))
    return solve_arrays(arrays_from_npz(d), loss, SolverOptions(max_iters=int(d["max_iters"])),
                        DeviceOptions(linear_solver=linear_solver))


@pytest.mark.parametrize("solver", ["dense", "pcg"])
@pytest.mark.parametrize("case", BA_CASES)
def test_ba_matches_reference(golden, case, solver):
    d = golden("ba_" + case)
    if solver == "dense" and 6 * int((d["frame_fixed"] == 0).sum()) > 210:
        pytest.skip("dense path limited to 35 free frames")
    q, t, X, rep, raw = solve_case(d, solver)
    assert raw.kernel_launches > 0
    assert rep.initial_cost == pytest.approx(float(d["ref_initial_cost"]), rel=1e-12)
    # parity bar (north star): final cost within 1e-6 relative in fp64
    assert rep.final_cost == pytest.approx(float(d["ref_final_cost"]), rel=1e-6, abs=1e-14)
    scale = max(1.0, np.abs(d["ref_points"]).max())
    np.testing.assert_allclose(X, d["ref_points"], atol=1e-6 * scale)
    np.testing.assert_allclose(t, d["ref_cam_t"], atol=1e-6 * scale)
    np.testing.assert_allclose(q, d["ref_cam_q"], atol=1e-7)
    fixed = d["frame_fixed"].astype(bool)
    assert q[fixed].tobytes() == np.ascontiguousarray(d["cam_q"][fixed]).tobytes()
    assert t[fixed].tobytes() == np.ascontiguousarray(d["cam_t"][fixed]).tobytes()
    if str(d["ref_termination"]) == "max_iterations":
        assert rep.termination == "max_iterations"
        assert rep.iterations == int(d["ref_iterations"])


def test_ba_depth_error_matches_reference(golden):
    from paper_2510_15271_b200.errors import NonPositiveDepth
    d = golden("ba_depth_error")
    with pytest.raises(NonPositiveDepth) as ei:
        solve_case(d)
    assert str(ei.value) == str(d["ref_message"])


@pytest.mark.parametrize("case", [c for c in BA_CASES if c != "config1"])
def test_eval_residuals_and_jacobians(golden, case):
    from paper_2510_15271_b200 import _native as nat
    d = golden("ba_" + case)
    a = arrays_from_npz(d)
    ctx = nat.default_context()
    N = len(a.obs_frame)
    cost, res = np.empty(N), np.empty((N, 2))
    jc, jp = np.empty((N, 2, 6)), np.empty((N, 2, 3))
    s = a.struct()
    ctx.check(ctx.lib.sfm_ba_eval(ctx.handle, ctypes.byref(s), int(d["loss_kind"]),
                                  float(d["loss_param"]), nat.ptr(cost), nat.ptr(res), nat.ptr(jc),
                                  nat.ptr(jp)))
    np.testing.assert_allclose(res.ravel(), d["ref_r"][:2 * N], rtol=1e-11, atol=1e-10)
    J = d["ref_J"]
    free = np.flatnonzero(d["frame_fixed"] == 0)
    fidx = {f: i for i, f in enumerate(free)}
    nf = len(free)
    for o in range(N):
        f = int(a.obs_frame[o])
        if f in fidx:
            np.testing.assert_allclose(jc[o], J[2 * o:2 * o + 2, 6 * fidx[f]:6 * fidx[f] + 6],
                                       rtol=1e-11, atol=1e-9)
        c = 6 * nf + 3 * int(a.obs_point[o])
        np.testing.assert_allclose(jp[o], J[2 * o:2 * o + 2, c:c + 3], rtol=1e-11, atol=1e-9)


def test_ba_is_deterministic():
    from paper_2510_15271_b200.mapping import solve_arrays
    from paper_2510_15271_b200.scenes import make_scene, scene_arrays
    from paper_2510_15271_b200.solver import DeviceOptions, RobustLoss, SolverOptions
    sc = make_scene(60, 6000, 30000, shape="venice", seed=5, outlier_frac=0.02)
    outs = [solve_arrays(scene_arrays(sc), RobustLoss("huber", 2.0), SolverOptions(max_iters=6),
                         DeviceOptions(linear_solver="pcg")) for _ in range(2)]
    for a, b in zip(outs[0][:3], outs[1][:3]):
        assert a.tobytes() == b.tobytes()
    assert outs[0][3] == outs[1][3]


def test_ba_medium_matches_oracle():
    """A 120-camera / 12k-point / 60k-observation Venice-shaped scene: PCG
    path vs the oracle's exact Schur solve, 5 LM iterations."""
    from oracle import ba as OB
    from paper_2510_15271_b200.mapping import solve_arrays
    from paper_2510_15271_b200.scenes import make_scene, scene_arrays
    from paper_2510_15271_b200.solver import DeviceOptions, RobustLoss, SolverOptions
    sc = make_scene(120, 12000, 60000, shape="venice", seed=8)
    a = scene_arrays(sc)
    q, t, X, rep, raw = solve_arrays(a, RobustLoss("huber", 2.0), SolverOptions(max_iters=5),
                                     DeviceOptions(linear_solver="pcg", pcg_rtol=1e-12))
    p = OB.BAProblem(a.cam_q, a.cam_t, a.frame_model, a.frame_fixed,
                     [(0, 500.0, 500.0, 320.0, 240.0, (0.0, 0.0))], a.points, a.obs_frame,
                     a.obs_point, a.obs_uv, a.edge_ab, a.prior_frame, a.edge_weight, a.prior_weight)
    qo, to, Xo, ro = p.solve(1, 2.0, 5)
    assert rep.initial_cost == pytest.approx(ro["initial_cost"], rel=1e-12)
    assert rep.final_cost == pytest.approx(ro["final_cost"], rel=1e-6)
    np.testing.assert_allclose(X, Xo, atol=1e-6 * np.abs(Xo).max())
    np.testing.assert_allclose(q, qo, atol=1e-7)


def tracks_struct(d):
    from paper_2510_15271_b200 import _native as nat
    m = d["models"]
    models = (nat.CameraModelC * len(m))(*[
        nat.CameraModelC(int(r[0]), 640, 480, 0, *[float(v) for v in r[1:7]]) for r in m])
    keep = dict(q=np.ascontiguousarray(d["cam_q"]), t=np.ascontiguousarray(d["cam_t"]),
                fm=np.ascontiguousarray(d["frame_model"], dtype=np.int32),
                ptr=np.ascontiguousarray(d["track_ptr"], dtype=np.int64),
                of=np.ascontiguousarray(d["obs_frame"], dtype=np.int32),
                uv=np.ascontiguousarray(d["obs_uv"]), models=models)
    s = nat.TracksC(len(keep["fm"]), len(m), nat.ptr(keep["q"]), nat.ptr(keep["t"]),
                    nat.ptr(keep["fm"]), ctypes.addressof(models), len(keep["ptr"]) - 1,
                    len(keep["of"]), nat.ptr(keep["ptr"]), nat.ptr(keep["of"]), nat.ptr(keep["uv"]),
                    None)
    return s, keep


@pytest.mark.parametrize("packed", ["0", "1"])
@pytest.mark.parametrize("case", ["dlt", "midpoint", "kinds_dlt", "kinds_midpoint"])
def test_ransac_matches_reference(golden, case, packed, monkeypatch):
    """Both RANSAC kernels (one track per warp; three short tracks per warp,
    with the in-series fallback for chunks that do not fit) against sfmkit."""
    from paper_2510_15271_b200 import _native as nat
    monkeypatch.setenv("SFM_RANSAC_PACKED", packed)
    method = case.split("_")[-1]
    d = golden("tri_" + case)
    s, keep = tracks_struct(d)
    T = len(keep["ptr"]) - 1
    X = np.empty((T, 3))
    mask = np.empty(len(keep["of"]), np.uint8)
    st = np.empty(T, np.int8)
    ctx = nat.default_context()
    ctx.check(ctx.lib.sfm_ransac_triangulate(ctx.handle, ctypes.byref(s), float(d["threshold_px"]),
                                             float(d["min_angle"]), nat.TRI_METHODS[method],
                                             nat.ptr(X), nat.ptr(mask), nat.ptr(st)))
    np.testing.assert_array_equal(st, d["ref_status"])           # bit-exact
    np.testing.assert_array_equal(mask, d["ref_mask"])          # bit-exact
    ok = st == 0
    np.testing.assert_allclose(X[ok], d["ref_X"][ok], rtol=1e-8, atol=1e-8)
    Xd = np.empty((T, 3))
    sd = np.empty(T, np.int8)
    ctx.check(ctx.lib.sfm_triangulate(ctx.handle, ctypes.byref(s), float(d["min_angle"]),
                                      nat.TRI_METHODS[method], nat.ptr(Xd), nat.ptr(sd)))
    np.testing.assert_array_equal(sd, d["ref_direct_status"])
    ok = sd == 0
    np.testing.assert_allclose(Xd[ok], d["ref_direct_X"][ok], rtol=1e-8, atol=1e-8)


def test_gate_matches_reference(golden):
    from paper_2510_15271_b200 import _native as nat
    d = golden("gate")
    s, keep = tracks_struct(d)
    mask = np.ascontiguousarray(d["mask_in"], dtype=np.uint8).copy()
    T = len(keep["ptr"]) - 1
    inl = np.empty(T, np.int32)
    rm = ctypes.c_int64()
    P = np.ascontiguousarray(d["points"])
    ctx = nat.default_context()
    ctx.check(ctx.lib.sfm_gate(ctx.handle, ctypes.byref(s), nat.ptr(P), float(d["threshold_px"]),
                               nat.ptr(mask), nat.ptr(inl), ctypes.byref(rm)))
    assert rm.value == int(d["ref_removed"])
    np.testing.assert_array_equal(mask, d["ref_mask"])
    np.testing.assert_array_equal((inl >= 2).astype(np.int8), d["ref_triangulated"])


def imap_config(case):
    from paper_2510_15271_b200 import MappingConfig, StageConfig
    from paper_2510_15271_b200.solver import RobustLoss
    if case == "iterative_map_rolling":
        return MappingConfig(max_solver_iters=30)
    if case == "iterative_map_large":  # tests/golden/make_golden.py
        return MappingConfig(stage1=StageConfig(4.0, RobustLoss("cauchy", 1.0)), lambda_c=0.5,
                             lambda_a=2.0, max_solver_iters=25)
    return MappingConfig()


@pytest.mark.parametrize("case", ["iterative_map", "iterative_map_large", "iterative_map_rolling"])
def test_iterative_map_matches_reference(golden, case):
    """The device-resident loop (sfm_iterative_map) through the object-level
    drop-in: track status, landmark order, masks, positions, poses and
    round statistics of sfmkit's iterative_map."""
    from paper_2510_15271_b200 import (CameraModel, Keyframe, Observation, Pose, Track,
                                       iterative_map, mean_reprojection_error)
    d = golden(case)
    cam = CameraModel("pinhole", 500.0, 500.0, 320.0, 240.0, 640, 480)
    if "kf_exposure" in d:  # rolling-shutter keyframes: the host-driven loop + sfm_gba_solve
        kfs = [Keyframe(f, float(d["kf_timestamp"][f]), 0, Pose(d["cam_q"][f], d["cam_t"][f]),
                        shutter="rolling", exposure=float(d["kf_exposure"][f]))
               for f in range(len(d["cam_q"]))]
    else:
        kfs = [Keyframe(f, float(f), 0, Pose(d["cam_q"][f], d["cam_t"][f]))
               for f in range(len(d["cam_q"]))]
    ptr = d["track_ptr"]
    tracks = [Track([Observation(int(d["obs_frame"][o]), 0, d["obs_uv"][o])
                     for o in range(ptr[i], ptr[i + 1])]) for i in range(len(ptr) - 1)]
    smap = iterative_map(kfs, tracks, {0: cam}, config=imap_config(case))
    stat = np.array([{"pending": 0, "triangulated": 1, "failed": 2}[t.status] for t in tracks])
    np.testing.assert_array_equal(stat, d["ref_status"])
    np.testing.assert_array_equal([r["added"] for r in smap.round_stats], d["ref_round_added"])
    np.testing.assert_array_equal([r["removed"] for r in smap.round_stats], d["ref_round_removed"])
    np.testing.assert_array_equal([r["landmarks"] for r in smap.round_stats], d["ref_round_landmarks"])
    lm_track = [next(i for i, t in enumerate(tracks) if t is lm.track) for lm in smap.landmarks]
    np.testing.assert_array_equal(lm_track, d["ref_lm_track"])
    mask = np.concatenate([lm.inlier_mask for lm in smap.landmarks]).astype(np.uint8)
    np.testing.assert_array_equal(mask, d["ref_lm_mask"])
    np.testing.assert_allclose([lm.position for lm in smap.landmarks], d["ref_lm_X"], atol=1e-6)
    q = np.array([smap.keyframes[f].cam_from_world.quat for f in sorted(smap.keyframes)])
    np.testing.assert_allclose(q, d["ref_cam_q"], atol=1e-7)
    assert mean_reprojection_error(smap) == pytest.approx(float(d["ref_mean_err"]), rel=1e-5,
                                                          abs=1e-9)


def test_dropin_bundle_adjust_objects(golden):
    """bundle_adjust on the object model: same write-back as the reference."""
    from paper_2510_15271_b200 import (CameraModel, Keyframe, Landmark, MappingConfig,
                                       Observation, Pose, SparseMap, StageConfig, Track,
                                       bundle_adjust)
    d = golden("ba_plain_stage2")
    cam = CameraModel("pinhole", 500.0, 500.0, 320.0, 240.0, 640, 480)
    F = len(d["cam_q"])
    kfs = {f: Keyframe(f, float(f), 0, Pose(d["cam_q"][f], d["cam_t"][f])) for f in range(F)}
    fixed = {int(f) for f in np.flatnonzero(d["frame_fixed"])}
    smap = SparseMap(kfs, {0: cam}, fixed_frames=fixed)
    ptr = np.searchsorted(d["obs_point"], np.arange(len(d["points"]) + 1))
    for p in range(len(d["points"])):
        obs = [Observation(int(d["obs_frame"][o]), 0, d["obs_uv"][o]) for o in range(ptr[p], ptr[p + 1])]
        smap.landmarks.append(Landmark(d["points"][p], Track(obs, "triangulated"),
                                       np.ones(len(obs), bool)))
    fixed_before = {f: smap.keyframes[f].cam_from_world for f in fixed}
    rep = bundle_adjust(smap, MappingConfig(lambda_a=0.0, lambda_c=0.0, max_solver_iters=100), stage=2)
    assert rep.termination == str(d["ref_termination"])
    assert rep.final_cost == pytest.approx(float(d["ref_final_cost"]), rel=1e-3, abs=1e-18)
    for f in fixed:
        assert smap.keyframes[f].cam_from_world is fixed_before[f]
    X = np.array([lm.position for lm in smap.landmarks])
    np.testing.assert_allclose(X, d["ref_points"], atol=1e-8)


@pytest.mark.parametrize("partition", [1, 0, 2])
@pytest.mark.parametrize("n_shards", [2, 3, 4, 8])
def test_point_sharded_solve_matches_single_rank(n_shards, partition):
    """SURVEY.md §8(e) on one B200: n logical ranks run the multi-GPU
    control flow (point shards balanced by observation count, partial Schur
    complements reduced -- reduce-scattered by block rows into the
    row-partitioned PCG (partition 1: one launch over every rank's CTAs;
    partition 2: one cooperative launch per rank meeting at the
    cross-launch barrier, the multi-device mechanism; z and the dot products
    pushed between the ranks inside the Krylov kernel, the solution
    allgathered) or all-reduced into the replicated PCG (partition 0) --
    reduced scalars); the result equals the single-rank solve and the
    oracle's."""
    from oracle import ba as OB
    from paper_2510_15271_b200.mapping import solve_arrays, solve_sharded_emulated
    from paper_2510_15271_b200.scenes import make_scene, scene_arrays
    from paper_2510_15271_b200.solver import DeviceOptions, RobustLoss, SolverOptions
    a = scene_arrays(make_scene(120, 12000, 60000, shape="venice", seed=8))
    loss, sopt = RobustLoss("huber", 2.0), SolverOptions(max_iters=5)
    dopt = DeviceOptions(linear_solver="pcg", pcg_rtol=1e-12, pcg_partition=partition)
    q1, t1, X1, r1, _ = solve_arrays(a, loss, sopt, dopt)
    qs, ts, Xs, rs, raw = solve_sharded_emulated(a, loss, sopt, dopt, n_shards)
    assert raw.kernel_launches > 0
    assert rs.iterations == r1.iterations
    assert rs.initial_cost == pytest.approx(r1.initial_cost, rel=1e-13)
    assert rs.final_cost == pytest.approx(r1.final_cost, rel=1e-10)
    scale = np.abs(X1).max()
    np.testing.assert_allclose(Xs, X1, atol=1e-9 * scale)
    np.testing.assert_allclose(qs, q1, atol=1e-10)
    p = OB.BAProblem(a.cam_q, a.cam_t, a.frame_model, a.frame_fixed,
                     [(0, 500.0, 500.0, 320.0, 240.0, (0.0, 0.0))], a.points, a.obs_frame,
                     a.obs_point, a.obs_uv, a.edge_ab, a.prior_frame, a.edge_weight, a.prior_weight)
    qo, to, Xo, ro = p.solve(1, 2.0, 5)
    assert rs.final_cost == pytest.approx(ro["final_cost"], rel=1e-9)
    np.testing.assert_allclose(Xs, Xo, atol=1e-8 * np.abs(Xo).max())


def test_point_sharded_depth_failure_matches_single_rank(golden):
    """NonPositiveDepth raised inside a sharded trial surfaces with the same
    exception class on the emulated multi-rank path."""
    from paper_2510_15271_b200.errors import NonPositiveDepth
    from paper_2510_15271_b200.mapping import solve_sharded_emulated
    from paper_2510_15271_b200.solver import DeviceOptions, RobustLoss, SolverOptions
    d = golden("ba_depth_error")
    with pytest.raises(NonPositiveDepth):
        solve_sharded_emulated(arrays_from_npz(d), RobustLoss("huber", 2.0), SolverOptions(max_iters=5),
                               DeviceOptions(linear_solver="pcg"), 2)


KIND_NAMES = {0: "pinhole", 1: "pinhole_radial", 2: "equidistant_fisheye"}


def general_map_from_npz(d):
    from paper_2510_15271_b200 import (CameraModel, Keyframe, Landmark, Observation, Pose,
                                       RigCalibration, SparseMap, Track)
    cams = {}
    for cid, par in zip(d["cam_id"], d["cam_par"]):
        kind = KIND_NAMES[int(par[0])]
        cams[int(cid)] = CameraModel(kind, *[float(v) for v in par[1:5]], int(par[5]), int(par[6]),
                                     tuple(float(v) for v in par[7:9]) if kind == "pinhole_radial" else ())
    kfs = {}
    for i, fid in enumerate(d["kf_id"]):
        kfs[int(fid)] = Keyframe(int(fid), float(d["kf_ts"][i]), int(d["kf_cam"][i]),
                                 Pose(d["kf_q"][i], d["kf_t"][i]),
                                 shutter="rolling" if d["kf_rolling"][i] else "global",
                                 exposure=float(d["kf_exposure"][i]))
    rig = None
    if "rig_ids" in d:
        rig = RigCalibration(tuple(int(c) for c in d["rig_ids"]),
                             {int(c): Pose(d["rig_q"][k], d["rig_t"][k]) for k, c in enumerate(d["rig_ids"])})
    lms = []
    ptr = d["lm_ptr"]
    for i in range(len(d["lm_pos"])):
        obs = [Observation(int(d["obs_frame"][o]), 0, d["obs_uv"][o]) for o in range(ptr[i], ptr[i + 1])]
        lms.append(Landmark(d["lm_pos"][i], Track(obs, "triangulated" if d["lm_tri"][i] else "pending"),
                            d["lm_mask"][ptr[i]:ptr[i + 1]].astype(bool)))
    return SparseMap(kfs, cams, lms, rig, {int(f): "prior" for f in d["prior"]},
                     {int(f) for f in d["fixed"]})


@pytest.mark.parametrize("case", ["rig", "rig_huber", "rolling", "rolling_seq"])
def test_rig_and_rolling_shutter_ba_match_reference(golden, case):
    """bundle_adjust with rig-extrinsic residuals
    (refine-extrinsics, mapping.py:321-333) and rolling-shutter residuals
    (mapping.py:336-356) -- two SE(3) slots per residual, solved on the
    device (sfm_gba_solve) -- against sfmkit's results."""
    from paper_2510_15271_b200 import MappingConfig, StageConfig, bundle_adjust
    from paper_2510_15271_b200.solver import RobustLoss
    d = golden("ba_" + case)
    smap = general_map_from_npz(d)
    cfg = MappingConfig(stage1=StageConfig(4.0, RobustLoss(LOSS_NAMES[int(d["loss_kind"])],
                                                           float(d["loss_param"]))),
                        lambda_c=float(d["lambda_c"]), lambda_a=float(d["lambda_a"]),
                        extrinsic_prior_weight=float(d["extrinsic_prior_weight"]),
                        max_solver_iters=int(d["max_iters"]))
    rep = bundle_adjust(smap, cfg, stage=int(d["stage"]), mode=str(d["mode"]))
    assert rep.initial_cost == pytest.approx(float(d["ref_initial_cost"]), rel=1e-10)
    assert rep.final_cost == pytest.approx(float(d["ref_final_cost"]), rel=1e-6, abs=1e-12)
    frames = sorted(smap.keyframes)
    q = np.array([smap.keyframes[f].cam_from_world.quat for f in frames])
    t = np.array([smap.keyframes[f].cam_from_world.t for f in frames])
    scale = max(1.0, np.abs(d["ref_lm_pos"]).max())
    np.testing.assert_allclose(q, d["ref_kf_q"], atol=1e-7)
    np.testing.assert_allclose(t, d["ref_kf_t"], atol=1e-6 * scale)
    np.testing.assert_allclose([lm.position for lm in smap.landmarks], d["ref_lm_pos"], atol=1e-6 * scale)
    if "ref_rig_q" in d:
        ids = [int(c) for c in d["rig_ids"]]
        np.testing.assert_allclose([smap.rig.extrinsic(c).quat for c in ids], d["ref_rig_q"], atol=1e-7)
        np.testing.assert_allclose([smap.rig.extrinsic(c).t for c in ids], d["ref_rig_t"], atol=1e-6)


def test_colmap_writer_matches_reference_bytes(tmp_path, golden):
    """paper_2510_15271_b200.io.write_colmap_sparse (reprojection errors from
    the device) writes the same three files as sfmkit's write_colmap_sparse
    (io.py:271-337) on the same map (tests/golden/make_io_golden.py)."""
    import sys
    sys.path.insert(0, __import__("os").path.dirname(__file__))
    from test_cpu_host import _io_map
    from paper_2510_15271_b200 import io as SIO
    g = golden("io_writers")
    SIO.write_colmap_sparse(_io_map(golden), tmp_path)
    for name, key in (("cameras.txt", "cameras_txt"), ("images.txt", "images_txt"),
                      ("points3D.txt", "points3d_txt")):
        assert (tmp_path / name).read_bytes() == g[key].tobytes(), name
