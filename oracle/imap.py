"""Vectorised restatement of the reference iterative_map (oracle only).

mapping.py:569-624 (rounds of {RANSAC-triangulate pending tracks -> stage-1
bundle_adjust -> remove_outliers at the stage-1 threshold} until a round
neither adds nor removes, then stage-2 bundle_adjust + remove_outliers at the
stage-2 threshold) on the flattened track layout of include/sfm_b200.h
(sfm_map_problem): tracks as CSR in track order, observations as (frame
index, pixel).

oracle/tri.py restates the triangulation scalar-per-track, like the
reference; it needs hours at configs[1]'s 100k tracks.  This module batches
the same arithmetic over all tracks of one length and all of their pair
hypotheses:

  * `rays`             cameras.py:150-166 unproject + mapping.py:166-174
  * `ransac_batch`     mapping.py:255-305 (triangulate_dlt :194-221 per pair,
                       exhaustive i<j pairs, strict '<' threshold, lexicographic
                       (count, -sum err) score with the first best kept,
                       refinement on the inliers, final mask recomputed)
  * `gate`             mapping.py:544-566 (strict '>' threshold; fewer than two
                       inliers -> PENDING, landmark dropped, order kept)
  * `iterative_map`    mapping.py:569-624 with bundle_adjust (mapping.py:390-527)
                       through oracle.ba.BAProblem (its own pinned restatement of
                       solver.solve)

Every per-element operation is the reference's (SVD through LAPACK like
numpy.linalg.svd in the reference, the same projection and norm), so statuses
and masks equal the scalar oracle's except on exact threshold ties.
Checked against oracle/tri.py and against the sfmkit iterative_map fixtures in
tests/test_oracle_golden.py.
"""

from __future__ import annotations

import numpy as np

from . import geometry as G
from .ba import BAProblem

PENDING, TRIANGULATED, FAILED = 0, 1, 2    # include/sfm_b200.h SFM_TRACK_*


class FrameArrays:
    """Per-frame pose + camera model (frame order of sfm_map_problem)."""

    def __init__(self, cam_q, cam_t, frame_model, models):
        self.q = np.asarray(cam_q, float).reshape(-1, 4)
        self.t = np.asarray(cam_t, float).reshape(-1, 3)
        self.fm = np.asarray(frame_model, np.int64)
        self.models = list(models)
        self.R = G.qmat(self.q)
        # pose.inverse().t = -R^T t (se3.py:127-129)
        qi = self.q * np.array([1.0, -1.0, -1.0, -1.0])
        self.center = -np.einsum("fij,fj->fi", G.qmat(qi), self.t)


def _undistort_vec(kind, dist, xd, yd):
    """cameras.py:102-125, element-wise with the scalar loop's exits."""
    st = np.zeros(xd.shape, np.int8)
    if kind == G.PINHOLE:
        return xd, yd, st
    if kind == G.FISHEYE:
        theta = np.hypot(xd, yd)
        st[theta >= np.pi / 2] = G.UNDISTORT
        small = theta < 1e-12
        ts = np.where(small | (st != 0), 1.0, theta)
        s = np.tan(ts) / ts
        x = np.where(small, xd, xd * s)
        y = np.where(small, yd, yd * s)
        return np.where(st != 0, 0.0, x), np.where(st != 0, 0.0, y), st
    k1, k2 = dist
    x, y = xd.copy(), yd.copy()
    done = np.zeros(xd.shape, bool)
    ox, oy = np.zeros_like(xd), np.zeros_like(yd)
    for _ in range(G.UNDISTORT_ITERS):
        live = ~done
        if not live.any():
            break
        r2 = x * x + y * y
        f = 1.0 + k1 * r2 + k2 * r2 * r2
        bad = live & (f <= 0)
        st[bad] = G.UNDISTORT
        done |= bad
        live = ~done
        fs = np.where(live, f, 1.0)
        xn, yn = xd / fs, yd / fs
        conv = live & (np.abs(xn - x) < G.UNDISTORT_TOL) & (np.abs(yn - y) < G.UNDISTORT_TOL)
        ox[conv], oy[conv] = xn[conv], yn[conv]
        done |= conv
        x = np.where(live & ~conv, xn, x)
        y = np.where(live & ~conv, yn, y)
    st[~done] = G.UNDISTORT
    return ox, oy, st


def rays(fr: FrameArrays, obs_frame, obs_uv):
    """unproject (cameras.py:150-166) of every observation -> (d_cam [N,3],
    world direction R^T d [N,3], ok [N])."""
    of = np.asarray(obs_frame, np.int64)
    uv = np.asarray(obs_uv, float).reshape(-1, 2)
    d = np.zeros((len(of), 3))
    ok = np.zeros(len(of), bool)
    mk = fr.fm[of]
    for m, model in enumerate(fr.models):
        sel = np.flatnonzero(mk == m)
        if len(sel) == 0:
            continue
        kind, fx, fy, cx, cy, dist = model
        x, y, st = _undistort_vec(kind, dist, (uv[sel, 0] - cx) / fx, (uv[sel, 1] - cy) / fy)
        r = np.stack([x, y, np.ones_like(x)], 1)
        d[sel] = r / np.sqrt(np.einsum("ni,ni->n", r, r))[:, None]
        ok[sel] = st == G.OK
    w = np.einsum("nji,nj->ni", fr.R[of], d)
    return d, w, ok


def reproj_errors(fr: FrameArrays, frames, uvs, X):
    """reprojection_error (mapping.py:243-252) element-wise over [..] frames /
    pixels / points: |project - pixel|, inf where projection raises."""
    frames = np.asarray(frames, np.int64)
    shp = frames.shape
    f = frames.ravel()
    Xf = np.asarray(X, float).reshape(-1, 3)
    uvf = np.asarray(uvs, float).reshape(-1, 2)
    pc = np.einsum("nij,nj->ni", fr.R[f], Xf) + fr.t[f]
    err = np.full(len(f), np.inf)
    mk = fr.fm[f]
    for m, model in enumerate(fr.models):
        sel = np.flatnonzero(mk == m)
        if len(sel) == 0:
            continue
        pix, st = G.project_cam(model, pc[sel])
        dx = pix[:, 0] - uvf[sel, 0]
        dy = pix[:, 1] - uvf[sel, 1]
        e = np.sqrt(dx * dx + dy * dy)
        err[sel] = np.where(st == G.OK, e, np.inf)
    return err.reshape(shp)


def _hat_rows(d, R, t):
    """hat(d) @ [R | t] (mapping.py:212-214), batched: d [...,3] -> [...,3,4]."""
    P = np.concatenate([R, t[..., None]], -1)
    H = np.zeros(d.shape[:-1] + (3, 3))
    H[..., 0, 1], H[..., 0, 2] = -d[..., 2], d[..., 1]
    H[..., 1, 0], H[..., 1, 2] = d[..., 2], -d[..., 0]
    H[..., 2, 0], H[..., 2, 1] = -d[..., 1], d[..., 0]
    return H @ P


def _max_angle(w, valid):
    """_max_ray_angle (mapping.py:177-183) over the valid rows of w [n,k,3]."""
    n, k, _ = w.shape
    best = np.zeros(n)
    for i in range(k):
        for j in range(i + 1, k):
            c = np.clip(np.abs(np.einsum("ni,ni->n", w[:, i], w[:, j])), -1.0, 1.0)
            a = np.arccos(c)
            use = valid[:, i] & valid[:, j]
            best = np.where(use, np.maximum(best, a), best)
    return best


def _dlt(fr, f, d, w, ok, min_angle):
    """triangulate_dlt (mapping.py:194-221) on n equally long observation sets:
    f [n,m] frames, d/w [n,m,3] camera/world rays -> (X [n,3], good [n])."""
    n, m = f.shape
    good = ok.all(1)
    good &= _max_angle(w, np.ones((n, m), bool)) >= min_angle
    A = _hat_rows(d, fr.R[f], fr.t[f]).reshape(n, 3 * m, 4)
    Xh = np.linalg.svd(A)[2][:, -1, :]
    good &= np.abs(Xh[:, 3]) >= 1e-12
    Xs = np.where(good, Xh[:, 3], 1.0)
    X = Xh[:, :3] / Xs[:, None]
    # _check_cheirality (mapping.py:186-191): p_cam . d_cam > 0 for every ray
    pc = np.einsum("nmij,nj->nmi", fr.R[f], X) + fr.t[f]
    good &= (np.einsum("nmi,nmi->nm", pc, d) > 0).all(1)
    return X, good


def _midpoint(fr, f, w, ok):
    """triangulate_midpoint (mapping.py:224-240) on n equally long sets."""
    n, m = f.shape
    good = ok.all(1)
    A = np.zeros((n, 3, 3))
    b = np.zeros((n, 3))
    c = fr.center[f]
    for i in range(m):
        M = np.eye(3)[None] - np.einsum("ni,nj->nij", w[:, i], w[:, i])
        A += M
        b += np.einsum("nij,nj->ni", M, c[:, i])
    sv = np.linalg.svd(A, compute_uv=False)
    good &= ~(sv[:, 0] / np.maximum(sv[:, -1], 1e-300) > 1e10)
    As = np.where(good[:, None, None], A, np.eye(3)[None])
    X = np.linalg.solve(As, b[..., None])[..., 0]
    return X, good


def _triangulate(fr, f, d, w, ok, method, min_angle, pair_gate=False):
    if method == "dlt":
        return _dlt(fr, f, d, w, ok, min_angle)
    good = np.ones(len(f), bool)
    if pair_gate:   # ransac's own parallax test before the midpoint (mapping.py:276-278)
        good &= ok.all(1) & (_max_angle(w, np.ones(f.shape, bool)) >= min_angle)
    X, g2 = _midpoint(fr, f, w, ok)
    pc = np.einsum("nmij,nj->nmi", fr.R[f], X) + fr.t[f]
    g2 &= (np.einsum("nmi,nmi->nm", pc, d) > 0).all(1)
    return X, good & g2


def ransac_batch(fr: FrameArrays, track_ptr, obs_frame, obs_uv, threshold_px=4.0,
                 min_angle=np.radians(0.5), method="dlt", active=None, chunk=2_000_000):
    """ransac_triangulate (mapping.py:255-305) of every active track ->
    (X [T,3] NaN unless OK, mask [N] bool, status [T]: TRIANGULATED / FAILED /
    -1 for inactive)."""
    ptr = np.asarray(track_ptr, np.int64)
    of = np.asarray(obs_frame, np.int64)
    uv = np.asarray(obs_uv, float).reshape(-1, 2)
    T = len(ptr) - 1
    X = np.full((T, 3), np.nan)
    mask = np.zeros(len(of), bool)
    status = np.full(T, -1, np.int8)
    act = np.ones(T, bool) if active is None else np.asarray(active, bool)
    klen = np.diff(ptr)
    d_all, w_all, ok_all = rays(fr, of, uv)
    for k in np.unique(klen[act]):
        trk = np.flatnonzero(act & (klen == k))
        if k < 2:
            status[trk] = FAILED
            continue
        I, J = np.triu_indices(k, 1)
        npair = len(I)
        step = max(1, chunk // (npair * k))
        for c0 in range(0, len(trk), step):
            tr = trk[c0:c0 + step]
            n = len(tr)
            O = ptr[tr][:, None] + np.arange(k)[None, :]               # [n,k]
            PO = np.stack([O[:, I], O[:, J]], -1).reshape(-1, 2)       # [n*P,2]
            Xp, good = _triangulate(fr, of[PO], d_all[PO], w_all[PO], ok_all[PO], method,
                                    min_angle, pair_gate=True)
            Xp = Xp.reshape(n, npair, 3)
            good = good.reshape(n, npair)
            errs = reproj_errors(fr, np.broadcast_to(of[O][:, None, :], (n, npair, k)),
                                 np.broadcast_to(uv[O][:, None, :, :], (n, npair, k, 2)),
                                 np.broadcast_to(Xp[:, :, None, :], (n, npair, k, 3)))
            m = errs < threshold_px
            cnt = m.sum(-1)
            ssum = np.zeros((n, npair))
            for o in range(k):            # errs[mask].sum(): masked entries in order
                ssum = np.where(m[..., o], ssum + errs[..., o], ssum)
            cand = good & (cnt >= 2)
            # lexicographic (count, -sum) maximum, first pair wins ties
            best = np.full(n, -1)
            bcnt = np.full(n, -1)
            bsum = np.full(n, np.inf)
            for p in range(npair):
                better = cand[:, p] & ((cnt[:, p] > bcnt) |
                                       ((cnt[:, p] == bcnt) & (-ssum[:, p] > -bsum)))
                best = np.where(better, p, best)
                bcnt = np.where(better, cnt[:, p], bcnt)
                bsum = np.where(better, ssum[:, p], bsum)
            has = best >= 0
            status[tr[~has]] = FAILED
            if not has.any():
                continue
            rows = np.flatnonzero(has)
            nin = m[rows, best[rows]].sum(1)
            for kin in np.unique(nin):
                sel = rows[nin == kin]
                sub = m[sel, best[sel]]
                Oi = O[sel][sub].reshape(len(sel), kin)
                Xr, g = _triangulate(fr, of[Oi], d_all[Oi], w_all[Oi], ok_all[Oi], method,
                                     min_angle)
                e2 = reproj_errors(fr, of[O[sel]], uv[O[sel]],
                                   np.broadcast_to(Xr[:, None, :], (len(sel), k, 3)))
                m2 = e2 < threshold_px
                g &= m2.sum(1) >= 2
                tsel = tr[sel]
                status[tsel[~g]] = FAILED
                ts = tsel[g]
                status[ts] = TRIANGULATED
                X[ts] = Xr[g]
                mask[O[sel][g]] = m2[g]
    return X, mask, status


def gate(fr: FrameArrays, track_ptr, obs_frame, obs_uv, lm_track, points, mask, threshold_px):
    """remove_outliers (mapping.py:544-566) over the landmarks (track ids in
    map order) -> (mask, surviving landmark track ids, demoted track ids,
    removed)."""
    ptr = np.asarray(track_ptr, np.int64)
    lm = np.asarray(lm_track, np.int64)
    mask = mask.copy()
    k = np.diff(ptr)[lm]
    o = np.repeat(ptr[lm], k) + (np.arange(k.sum()) - np.repeat(np.cumsum(k) - k, k))
    li = np.repeat(np.arange(len(lm)), k)
    live = mask[o]
    e = reproj_errors(fr, np.asarray(obs_frame)[o[live]], np.asarray(obs_uv)[o[live]],
                      points[lm[li[live]]])
    drop = o[live][e > threshold_px]
    mask[drop] = False
    inl = np.bincount(li, weights=mask[o].astype(float), minlength=len(lm))
    keep = inl >= 2
    return mask, lm[keep], lm[~keep], int(len(drop))


def bundle_adjust(fr, cam_q, cam_t, frame_fixed, models, ptr, obs_frame, obs_uv, lm_track,
                  points, mask, edge_ab, prior_frame, lambda_c, lambda_a, loss_kind, loss_param,
                  max_iters):
    """bundle_adjust (mapping.py:390-527) in pure mode over the landmarks in
    map order and their inlier observations (mapping.py:452-475)."""
    lm = np.asarray(lm_track, np.int64)
    k = np.diff(ptr)[lm]
    o = np.repeat(ptr[lm], k) + (np.arange(k.sum()) - np.repeat(np.cumsum(k) - k, k))
    li = np.repeat(np.arange(len(lm)), k)
    keep = mask[o]
    prob = BAProblem(cam_q, cam_t, fr.fm, frame_fixed, models, points[lm],
                     np.asarray(obs_frame)[o[keep]], li[keep], np.asarray(obs_uv)[o[keep]],
                     edge_ab, prior_frame, lambda_c if len(edge_ab) else 0.0,
                     lambda_a if len(prior_frame) else 0.0)
    q, t, X, rep = prob.solve(loss_kind, loss_param, max_iters)
    return q, t, X, rep


def iterative_map(cam_q, cam_t, frame_model, frame_fixed, models, track_ptr, obs_frame, obs_uv,
                  edge_ab, prior_frame, lambda_c=1.0, lambda_a=1.0, stage1=(1, 2.0, 4.0),
                  stage2=(0, 1.0, 2.0), max_outer_iters=10, max_solver_iters=50,
                  min_angle=np.radians(0.5), method="dlt", track_status=None, log=None):
    """iterative_map (mapping.py:569-624) on arrays; the fixed set (anchor)
    is resolved by the caller as in sfm_map_problem.  stageN = (loss kind,
    loss param, outlier px).  Returns dict(cam_q, cam_t, points [T,3],
    inlier_mask [N], status [T], lm_track [L], round_stats, reports)."""
    q = np.asarray(cam_q, float).reshape(-1, 4).copy()
    t = np.asarray(cam_t, float).reshape(-1, 3).copy()
    ptr = np.asarray(track_ptr, np.int64)
    of = np.asarray(obs_frame, np.int64)
    uv = np.asarray(obs_uv, float).reshape(-1, 2)
    T = len(ptr) - 1
    edges = np.asarray(edge_ab, np.int64).reshape(-1, 2)
    priors = np.asarray(prior_frame, np.int64)
    status = np.zeros(T, np.int8) if track_status is None else np.asarray(track_status,
                                                                          np.int8).copy()
    points = np.full((T, 3), np.nan)
    mask = np.zeros(len(of), bool)
    lm = np.zeros(0, np.int64)
    stats, reports = [], []

    def ba(stage):
        nonlocal q, t
        kind, param, _ = stage
        fr = FrameArrays(q, t, frame_model, models)
        q, t, X, rep = bundle_adjust(fr, q, t, frame_fixed, models, ptr, of, uv, lm, points,
                                     mask, edges, priors, lambda_c, lambda_a, kind, param,
                                     max_solver_iters)
        points[lm] = X
        reports.append(rep)
        if log:
            log(f"  BA stage {1 if stage is stage1 else 2}: {rep}")

    for r in range(max_outer_iters):
        fr = FrameArrays(q, t, frame_model, models)
        pend = status == PENDING
        Xn, mn, st = ransac_batch(fr, ptr, of, uv, stage1[2], min_angle, method, active=pend)
        newly = np.flatnonzero(pend & (st == TRIANGULATED))
        status[pend & (st == FAILED)] = FAILED
        status[newly] = TRIANGULATED
        points[newly] = Xn[newly]
        for i in newly:
            mask[ptr[i]:ptr[i + 1]] = mn[ptr[i]:ptr[i + 1]]
        lm = np.concatenate([lm, newly])
        added = len(newly)
        if len(lm):
            ba(stage1)
        fr = FrameArrays(q, t, frame_model, models)
        mask, lm, demoted, removed = gate(fr, ptr, of, uv, lm, points, mask, stage1[2])
        status[demoted] = PENDING
        for i in demoted:
            mask[ptr[i]:ptr[i + 1]] = False
            points[i] = np.nan
        stats.append({"round": r, "added": added, "removed": removed, "landmarks": len(lm)})
        if log:
            log(f"round {r}: {stats[-1]}")
        if added == 0 and removed == 0:
            break
    if len(lm):
        ba(stage2)
        fr = FrameArrays(q, t, frame_model, models)
        mask, lm, demoted, removed = gate(fr, ptr, of, uv, lm, points, mask, stage2[2])
        status[demoted] = PENDING
        for i in demoted:
            mask[ptr[i]:ptr[i + 1]] = False
            points[i] = np.nan
        stats.append({"round": "final", "added": 0, "removed": removed, "landmarks": len(lm)})
    return dict(cam_q=q, cam_t=t, points=points, inlier_mask=mask, status=status, lm_track=lm,
                round_stats=stats, reports=reports)
