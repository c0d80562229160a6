"""Restatement of the reference triangulation and gating (oracle only).

mapping.py:166-305 (world rays, max ray angle, cheirality, DLT via SVD,
midpoint, reprojection error, exhaustive pair RANSAC) and mapping.py:544-566
(remove_outliers) on the CSR track layout of include/sfm_b200.h.  Per-track
Python loops with numpy linear algebra, like the reference: small cases.
"""

from __future__ import annotations

import numpy as np

from . import geometry as G

OK, PARALLAX, CHEIRALITY, PARALLEL, TOO_FEW, CAMERA, FAILED, SKIPPED = range(8)


class Frames:
    def __init__(self, cam_q, cam_t, frame_model, models):
        self.q = np.asarray(cam_q, float).reshape(-1, 4)
        self.t = np.asarray(cam_t, float).reshape(-1, 3)
        self.fm = np.asarray(frame_model, np.int64)
        self.models = list(models)
        self.R = G.qmat(self.q)

    def model(self, f):
        return self.models[self.fm[f]]


def world_rays(fr: Frames, frames, uvs):
    """mapping.py:166-174 -> (centers, dirs, status)"""
    centers, dirs = [], []
    for f, uv in zip(frames, uvs):
        d, st = G.unproject(fr.model(f), uv)
        if st != G.OK:
            return None, None, CAMERA
        qi = np.array([fr.q[f][0], -fr.q[f][1], -fr.q[f][2], -fr.q[f][3]])
        centers.append(-(G.qmat(qi) @ fr.t[f]))
        dirs.append(fr.R[f].T @ d)
    return np.array(centers), np.array(dirs), OK


def max_ray_angle(dirs):
    """mapping.py:177-183"""
    best = 0.0
    for i in range(len(dirs)):
        for j in range(i + 1, len(dirs)):
            best = max(best, np.arccos(np.clip(abs(dirs[i] @ dirs[j]), -1.0, 1.0)))
    return best


def cheirality_ok(fr, frames, uvs, X):
    """mapping.py:186-191"""
    for f, uv in zip(frames, uvs):
        d, _ = G.unproject(fr.model(f), uv)
        if (fr.R[f] @ X + fr.t[f]) @ d <= 0:
            return False
    return True


def triangulate_dlt(fr, frames, uvs, min_angle=np.radians(0.5)):
    """mapping.py:194-221 -> (X, status)"""
    if len(frames) < 2:
        return None, TOO_FEW
    _, dirs, st = world_rays(fr, frames, uvs)
    if st != OK:
        return None, st
    if max_ray_angle(dirs) < min_angle:
        return None, PARALLAX
    rows = []
    for f, uv in zip(frames, uvs):
        d, _ = G.unproject(fr.model(f), uv)
        P = np.hstack([fr.R[f], fr.t[f].reshape(3, 1)])
        rows.append(G.hat(d) @ P)
    _, _, Vt = np.linalg.svd(np.vstack(rows))
    Xh = Vt[-1]
    if abs(Xh[3]) < 1e-12:
        return None, PARALLAX
    X = Xh[:3] / Xh[3]
    if not cheirality_ok(fr, frames, uvs, X):
        return None, CHEIRALITY
    return X, OK


def triangulate_midpoint(fr, frames, uvs):
    """mapping.py:224-240 -> (X, status)"""
    if len(frames) < 2:
        return None, TOO_FEW
    centers, dirs, st = world_rays(fr, frames, uvs)
    if st != OK:
        return None, st
    A = np.zeros((3, 3))
    b = np.zeros(3)
    for c, w in zip(centers, dirs):
        M = np.eye(3) - np.outer(w, w)
        A += M
        b += M @ c
    sv = np.linalg.svd(A, compute_uv=False)
    if sv[0] / max(sv[-1], 1e-300) > 1e10:
        return None, PARALLEL
    X = np.linalg.solve(A, b)
    if not cheirality_ok(fr, frames, uvs, X):
        return None, CHEIRALITY
    return X, OK


def reprojection_error(fr, f, uv, X):
    """mapping.py:243-252"""
    pc = fr.R[f] @ X + fr.t[f]
    pix, st = G.project_cam(fr.model(f), pc[None, :])
    if st[0] != G.OK:
        return np.inf
    return float(np.linalg.norm(pix[0] - uv))


def ransac_triangulate(fr, frames, uvs, threshold_px=4.0, min_angle=np.radians(0.5),
                       method="dlt"):
    """mapping.py:255-305 -> (X or None, mask, status OK/FAILED)"""
    k = len(frames)
    best = None
    for i in range(k):
        for j in range(i + 1, k):
            pf, pu = [frames[i], frames[j]], [uvs[i], uvs[j]]
            if method == "dlt":
                X, st = triangulate_dlt(fr, pf, pu, min_angle)
            else:
                _, dirs, st = world_rays(fr, pf, pu)
                if st != OK or max_ray_angle(dirs) < min_angle:
                    continue
                X, st = triangulate_midpoint(fr, pf, pu)
            if st != OK:
                continue
            errs = np.array([reprojection_error(fr, f, uv, X) for f, uv in zip(frames, uvs)])
            mask = errs < threshold_px
            score = (int(mask.sum()), -float(errs[mask].sum()))
            if mask.sum() >= 2 and (best is None or score > best[0]):
                best = (score, mask, X)
    if best is None:
        return None, np.zeros(k, bool), FAILED
    _, mask, X = best
    inl = np.flatnonzero(mask)
    pf, pu = [frames[i] for i in inl], [uvs[i] for i in inl]
    if method == "dlt":
        X, st = triangulate_dlt(fr, pf, pu, min_angle)
    else:
        X, st = triangulate_midpoint(fr, pf, pu)
    if st != OK:
        return None, np.zeros(k, bool), FAILED
    errs = np.array([reprojection_error(fr, f, uv, X) for f, uv in zip(frames, uvs)])
    mask = errs < threshold_px
    if mask.sum() < 2:
        return None, np.zeros(k, bool), FAILED
    return X, mask, OK


def ransac_batch(fr, track_ptr, obs_frame, obs_uv, threshold_px, min_angle, method,
                 active=None):
    T = len(track_ptr) - 1
    X = np.full((T, 3), np.nan)
    mask = np.zeros(len(obs_frame), bool)
    status = np.full(T, SKIPPED, np.int8)
    for i in range(T):
        if active is not None and not active[i]:
            continue
        b0, b1 = track_ptr[i], track_ptr[i + 1]
        x, m, st = ransac_triangulate(fr, list(obs_frame[b0:b1]), list(obs_uv[b0:b1]),
                                      threshold_px, min_angle, method)
        status[i] = st
        if st == OK:
            X[i] = x
            mask[b0:b1] = m
    return X, mask, status


def gate(fr, track_ptr, obs_frame, obs_uv, points, mask, threshold_px):
    """remove_outliers (mapping.py:544-566) over TRIANGULATED landmarks ->
    (new mask, inlier counts, removed)."""
    mask = np.array(mask, bool, copy=True)
    T = len(track_ptr) - 1
    inl = np.zeros(T, np.int64)
    removed = 0
    for i in range(T):
        for o in range(track_ptr[i], track_ptr[i + 1]):
            if not mask[o]:
                continue
            if reprojection_error(fr, obs_frame[o], obs_uv[o], points[i]) > threshold_px:
                mask[o] = False
                removed += 1
        inl[i] = int(mask[track_ptr[i]:track_ptr[i + 1]].sum())
    return mask, inl, removed
