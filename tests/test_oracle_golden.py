"""Pins the CPU oracle (oracle/) against golden vectors produced by the
reference itself (tests/golden/make_golden.py running sfmkit)."""

import numpy as np
import pytest

from oracle import ba as OB
from oracle import geometry as G
from oracle import tri as OT

BA_CASES = ["plain_stage2", "huber_outliers", "cauchy_pose_terms", "localization_fixed",
            "localization_adjust", "prior_gauge", "pure_provenance_lc", "config1", "camera_kinds"]


def models_of(d):
    return [(int(k), fx, fy, cx, cy, (k1, k2)) for k, fx, fy, cx, cy, k1, k2 in d["models"]]


@pytest.mark.parametrize("case", BA_CASES)
def test_oracle_residual_order_and_initial_cost(golden, case):
    d = golden("ba_" + case)
    p = OB.problem_from_npz(d)
    r, st, _, _ = p.obs_project(p.q0, p.t0, p.X0)
    assert np.all(st == 0)
    stacked = [r.ravel()]
    stacked += [v for v in p.edge_terms(p.q0, p.t0)]
    stacked += [v for v in p.prior_terms(p.q0, p.t0)]
    stacked = np.concatenate(stacked)
    ref = d["ref_initial_residual"]
    assert stacked.shape == ref.shape
    # bit-for-bit observation order: residual i of the SoA == residual i of the reference
    np.testing.assert_allclose(stacked, ref, rtol=1e-11, atol=1e-11)
    c0 = p.cost(p.q0, p.t0, p.X0, int(d["loss_kind"]), float(d["loss_param"]))
    assert c0 == pytest.approx(float(d["ref_initial_cost"]), rel=1e-12)


@pytest.mark.parametrize("case", [c for c in BA_CASES if c != "config1"])
def test_oracle_jacobian_matches_reference_assembly(golden, case):
    d = golden("ba_" + case)
    p = OB.problem_from_npz(d)
    lin = p.linearize(p.q0, p.t0, p.X0, int(d["loss_kind"]), float(d["loss_param"]))
    N, nf, P = p.N, p.nf, p.P
    ncol = 6 * nf + 3 * P
    rows = [np.zeros((2 * N, ncol))]
    j = lin["j"]
    for o in range(N):
        if j[o] >= 0:
            rows[0][2 * o:2 * o + 2, 6 * j[o]:6 * j[o] + 6] = lin["Jc"][o]
        c = 6 * nf + 3 * p.op[o]
        rows[0][2 * o:2 * o + 2, c:c + 3] = lin["Jp"][o]
    for (a, b), (_, Ja, Jb) in zip(p.edges, p.edge_terms(p.q0, p.t0, True)):
        blk = np.zeros((6, ncol))
        if p.free_idx[a] >= 0:
            blk[:, 6 * p.free_idx[a]:6 * p.free_idx[a] + 6] = Ja
        if p.free_idx[b] >= 0:
            blk[:, 6 * p.free_idx[b]:6 * p.free_idx[b] + 6] = Jb
        rows.append(blk)
    for f, (_, J) in zip(p.priors, p.prior_terms(p.q0, p.t0, True)):
        blk = np.zeros((6, ncol))
        blk[:, 6 * p.free_idx[f]:6 * p.free_idx[f] + 6] = J
        rows.append(blk)
    J = np.vstack(rows)
    ref = d["ref_J"]
    assert J.shape == ref.shape
    np.testing.assert_allclose(J, ref, rtol=1e-10, atol=1e-9)


@pytest.mark.parametrize("case", BA_CASES)
def test_oracle_lm_matches_reference(golden, case):
    d = golden("ba_" + case)
    p = OB.problem_from_npz(d)
    q, t, X, rep = p.solve(int(d["loss_kind"]), float(d["loss_param"]), int(d["max_iters"]))
    ref_cost = float(d["ref_final_cost"])
    assert rep["initial_cost"] == pytest.approx(float(d["ref_initial_cost"]), rel=1e-12)
    assert rep["final_cost"] == pytest.approx(ref_cost, rel=1e-6, abs=1e-14)
    if str(d["ref_termination"]) != "max_iterations" or case == "config1":
        scale = max(1.0, np.abs(d["ref_points"]).max())
        np.testing.assert_allclose(X, d["ref_points"], atol=1e-6 * scale)
        np.testing.assert_allclose(t, d["ref_cam_t"], atol=1e-6 * scale)
        np.testing.assert_allclose(q, d["ref_cam_q"], atol=1e-7)
    fixed = d["frame_fixed"].astype(bool)
    assert q[fixed].tobytes() == d["cam_q"][fixed].tobytes()
    assert t[fixed].tobytes() == d["cam_t"][fixed].tobytes()


def test_oracle_depth_error(golden):
    d = golden("ba_depth_error")
    assert str(d["ref_exception"]) == "NonPositiveDepth"
    p = OB.problem_from_npz(d)
    with pytest.raises(OB.OracleNonPositiveDepth) as ei:
        p.solve(int(d["loss_kind"]), float(d["loss_param"]), int(d["max_iters"]))
    assert str(ei.value) == str(d["ref_message"])


def test_oracle_geometry_kat(golden):
    d = golden("kat_geometry")
    models = models_of(d)
    for row in d["proj"]:
        ci = int(row[0])
        q, t, X = row[1:5], row[5:8], row[8:11]
        pix, Jc, Jp, st = G.project_with_jacobians(models[ci], G.qmat(q)[None], t[None], X[None])
        assert st[0] == 0
        np.testing.assert_allclose(pix[0], row[11:13], rtol=1e-13, atol=1e-10)
        np.testing.assert_allclose(Jc[0].ravel(), row[13:25], rtol=1e-11, atol=1e-9)
        np.testing.assert_allclose(Jp[0].ravel(), row[25:31], rtol=1e-11, atol=1e-9)
        ray, st = G.unproject(models[ci], row[11:13])
        np.testing.assert_allclose(ray, row[31:34], rtol=1e-9, atol=1e-9)
    for row in d["pose_terms"]:
        lam = row[0]
        Ta, Tb, meas = (row[1:5], row[5:8]), (row[8:12], row[12:15]), (row[15:19], row[19:22])
        r, Ja, Jb = row[22:28], row[28:64].reshape(6, 6), row[64:100].reshape(6, 6)
        Te, Tc = (row[100:104], row[104:107]), (row[107:111], row[111:114])
        rp, Jp = row[114:120], row[120:156].reshape(6, 6)
        mi = G.pinv(meas)
        w = np.sqrt(lam)
        rr = G.log_map(G.pmul(G.pmul(mi, Ta), G.pinv(Tb)))
        np.testing.assert_allclose(w * rr, r, rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(w * G.se3_jl_inv(rr) @ G.adjoint(mi), Ja, rtol=1e-11, atol=1e-12)
        np.testing.assert_allclose(-w * G.se3_jl_inv(-rr), Jb, rtol=1e-11, atol=1e-12)
        rr = G.log_map(G.pmul(Tc, G.pinv(Te)))
        np.testing.assert_allclose(w * rr, rp, rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(w * G.se3_jl_inv(rr), Jp, rtol=1e-11, atol=1e-12)


@pytest.mark.parametrize("case", ["dlt", "midpoint", "kinds_dlt", "kinds_midpoint"])
def test_oracle_triangulation_matches_reference(golden, case):
    method = case.split("_")[-1]
    d = golden("tri_" + case)
    fr = OT.Frames(d["cam_q"], d["cam_t"], d["frame_model"], models_of(d))
    X, mask, st = OT.ransac_batch(fr, d["track_ptr"], d["obs_frame"], d["obs_uv"],
                                  float(d["threshold_px"]), float(d["min_angle"]), method)
    np.testing.assert_array_equal(st, d["ref_status"])
    np.testing.assert_array_equal(mask.astype(np.uint8), d["ref_mask"])
    ok = st == 0
    np.testing.assert_allclose(X[ok], d["ref_X"][ok], rtol=1e-9, atol=1e-9)
    ptr = d["track_ptr"]
    for i in range(len(ptr) - 1):
        b0, b1 = ptr[i], ptr[i + 1]
        frames, uvs = list(d["obs_frame"][b0:b1]), list(d["obs_uv"][b0:b1])
        if method == "dlt":
            x, s = OT.triangulate_dlt(fr, frames, uvs, float(d["min_angle"]))
        else:
            x, s = OT.triangulate_midpoint(fr, frames, uvs)
        assert s == d["ref_direct_status"][i]
        if s == 0:
            np.testing.assert_allclose(x, d["ref_direct_X"][i], rtol=1e-9, atol=1e-9)


def test_oracle_gate_matches_reference(golden):
    d = golden("gate")
    fr = OT.Frames(d["cam_q"], d["cam_t"], d["frame_model"], models_of(d))
    mask, inl, removed = OT.gate(fr, d["track_ptr"], d["obs_frame"], d["obs_uv"], d["points"],
                                 d["mask_in"].astype(bool), float(d["threshold_px"]))
    assert removed == int(d["ref_removed"])
    np.testing.assert_array_equal(mask.astype(np.uint8), d["ref_mask"])
    np.testing.assert_array_equal((inl >= 2).astype(np.int8), d["ref_triangulated"])


@pytest.mark.parametrize("case", ["dlt", "midpoint", "kinds_dlt", "kinds_midpoint"])
def test_oracle_batched_ransac_matches_reference(golden, case):
    """oracle/imap.py's track-batched RANSAC (the config-sized restatement)
    against the same sfmkit fixtures as the scalar one."""
    from oracle import imap as OI
    method = case.split("_")[-1]
    d = golden("tri_" + case)
    fr = OI.FrameArrays(d["cam_q"], d["cam_t"], d["frame_model"], models_of(d))
    X, mask, st = OI.ransac_batch(fr, d["track_ptr"], d["obs_frame"], d["obs_uv"],
                                  float(d["threshold_px"]), float(d["min_angle"]), method)
    ok = d["ref_status"] == OT.OK
    np.testing.assert_array_equal(st == OI.TRIANGULATED, ok)
    np.testing.assert_array_equal(mask.astype(np.uint8), d["ref_mask"])
    np.testing.assert_allclose(X[ok], d["ref_X"][ok], rtol=1e-9, atol=1e-9)


IMAP_CASES = {"iterative_map": {},
              "iterative_map_large": dict(stage1=(2, 1.0, 4.0), lambda_c=0.5, lambda_a=2.0,
                                          max_solver_iters=25)}


@pytest.mark.parametrize("case", sorted(IMAP_CASES))
def test_oracle_iterative_map_matches_reference(golden, case):
    """oracle/imap.py iterative_map (mapping.py:569-624) against sfmkit runs:
    statuses, landmark order, masks and round statistics bit-exact."""
    from oracle import imap as OI
    d = golden(case)
    F = len(d["cam_q"])
    fixed = np.zeros(F, np.uint8)
    fixed[0] = 1                               # anchor: min frame (mapping.py:583-593)
    edges = np.stack([np.arange(F - 1), np.arange(1, F)], 1)
    r = OI.iterative_map(d["cam_q"], d["cam_t"], np.zeros(F, int), fixed,
                         [(0, 500.0, 500.0, 320.0, 240.0, (0.0, 0.0))], d["track_ptr"],
                         d["obs_frame"], d["obs_uv"], edges, np.arange(1, F), **IMAP_CASES[case])
    np.testing.assert_array_equal(r["status"], d["ref_status"])
    np.testing.assert_array_equal(r["lm_track"], d["ref_lm_track"])
    for key in ("added", "removed", "landmarks"):
        np.testing.assert_array_equal([s[key] for s in r["round_stats"]], d["ref_round_" + key])
    ptr = d["track_ptr"]
    mask = np.concatenate([r["inlier_mask"][ptr[i]:ptr[i + 1]] for i in r["lm_track"]])
    np.testing.assert_array_equal(mask.astype(np.uint8), d["ref_lm_mask"])
    np.testing.assert_allclose(r["points"][r["lm_track"]], d["ref_lm_X"], atol=1e-6)
    np.testing.assert_allclose(r["cam_q"], d["ref_cam_q"], atol=1e-7)
