"""Vectorised numpy restatement of the reference geometry (oracle only).

se3.py:20-267 (quaternions, exp/log, Jacobians, adjoint) and
cameras.py:57-179 (distortion, projection, unprojection and the
reprojection Jacobians).  Batched over observations so the oracle can run
config-sized samples.
"""

from __future__ import annotations

import numpy as np

MIN_DEPTH = 1e-9                      # cameras.py:28
UNDISTORT_ITERS = 50                  # cameras.py:29
UNDISTORT_TOL = 1e-10                 # cameras.py:30
MAX_FISHEYE_ANGLE = np.deg2rad(89.9)  # cameras.py:32

PINHOLE, RADIAL, FISHEYE = 0, 1, 2
OK, DEPTH, DOMAIN, UNDISTORT = 0, 1, 2, 3


# --- SE(3), scalar (se3.py) ---------------------------------------------------

def qnormalize(q):
    """se3.py:20-29"""
    q = np.asarray(q, dtype=float)
    q = q / np.linalg.norm(q)
    lead = q[0] if q[0] != 0 else next((c for c in q[1:] if c != 0), 0.0)
    return -q if lead < 0 else q


def qmul(a, b):
    """se3.py:39-47"""
    aw, ax, ay, az = a
    bw, bx, by, bz = b
    return np.array([aw * bw - ax * bx - ay * by - az * bz,
                     aw * bx + ax * bw + ay * bz - az * by,
                     aw * by - ax * bz + ay * bw + az * bx,
                     aw * bz + ax * by - ay * bx + az * bw])


def qmat(q):
    """se3.py:50-56 (batched over leading axes)."""
    q = np.asarray(q, dtype=float)
    w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    R = np.empty(q.shape[:-1] + (3, 3))
    R[..., 0, 0] = 1 - 2 * (y * y + z * z)
    R[..., 0, 1] = 2 * (x * y - w * z)
    R[..., 0, 2] = 2 * (x * z + w * y)
    R[..., 1, 0] = 2 * (x * y + w * z)
    R[..., 1, 1] = 1 - 2 * (x * x + z * z)
    R[..., 1, 2] = 2 * (y * z - w * x)
    R[..., 2, 0] = 2 * (x * z - w * y)
    R[..., 2, 1] = 2 * (y * z + w * x)
    R[..., 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def hat(v):
    return np.array([[0.0, -v[2], v[1]], [v[2], 0.0, -v[0]], [-v[1], v[0], 0.0]])


def pose(q, t):
    """Pose(q, t) construction: normalises q (se3.py:96-98)."""
    return qnormalize(q), np.asarray(t, dtype=float).reshape(3)


def pinv(p):
    """Pose.inverse (se3.py:127-129)."""
    q, t = p
    qi = np.array([q[0], -q[1], -q[2], -q[3]])
    return pose(qi, -(qmat(qi) @ t))


def pmul(a, b):
    """compose (se3.py:138-140)."""
    return pose(qmul(a[0], b[0]), qmat(a[0]) @ b[1] + a[1])


def so3_exp(phi):
    """se3.py:143-154"""
    theta = np.linalg.norm(phi)
    half = 0.5 * theta
    if theta < 1e-8:
        w, s = 1.0 - half * half / 2.0, 0.5 - half * half / 12.0
    else:
        w, s = np.cos(half), np.sin(half) / theta
    return qnormalize(np.concatenate(([w], s * phi)))


def so3_log(q):
    """se3.py:157-168"""
    v = np.asarray(q[1:])
    n = np.linalg.norm(v)
    if n < 1e-10:
        return 2.0 * v
    return (2.0 * np.arctan2(n, q[0]) / n) * v


def so3_jl(phi):
    """se3.py:171-178"""
    theta = np.linalg.norm(phi)
    P = hat(phi)
    if theta < 1e-6:
        return np.eye(3) + 0.5 * P + (P @ P) / 6.0
    return (np.eye(3) + (1.0 - np.cos(theta)) / theta ** 2 * P
            + (theta - np.sin(theta)) / theta ** 3 * (P @ P))


def so3_jl_inv(phi):
    """se3.py:181-187"""
    theta = np.linalg.norm(phi)
    P = hat(phi)
    if theta < 1e-6:
        return np.eye(3) - 0.5 * P + (P @ P) / 12.0
    c = 1.0 / theta ** 2 - (1.0 + np.cos(theta)) / (2.0 * theta * np.sin(theta))
    return np.eye(3) - 0.5 * P + c * (P @ P)


def exp_map(xi):
    """se3.py:190-194"""
    xi = np.asarray(xi, dtype=float)
    return pose(so3_exp(xi[:3]), so3_jl(xi[:3]) @ xi[3:])


def log_map(p):
    """se3.py:197-201"""
    phi = so3_log(p[0])
    return np.concatenate([phi, so3_jl_inv(phi) @ p[1]])


def adjoint(p):
    """se3.py:204-211"""
    R = qmat(p[0])
    A = np.zeros((6, 6))
    A[:3, :3] = R
    A[3:, :3] = hat(p[1]) @ R
    A[3:, 3:] = R
    return A


def se3_Q(phi, rho):
    """se3.py:214-235"""
    theta = np.linalg.norm(phi)
    P, Rh = hat(phi), hat(rho)
    PR, RP = P @ Rh, Rh @ P
    PRP = PR @ P
    if theta < 1e-4:
        t2 = theta * theta
        c1, c2, c3 = 1 / 6 - t2 / 120, 1 / 24 - t2 / 720, 1 / 120 - t2 / 2520
    else:
        c1 = (theta - np.sin(theta)) / theta ** 3
        c2 = (1.0 - theta ** 2 / 2.0 - np.cos(theta)) / theta ** 4
        c3 = (theta - np.sin(theta) - theta ** 3 / 6.0) / theta ** 5
    return (0.5 * Rh + c1 * (PR + RP + PRP) - c2 * (P @ PR + RP @ P - 3.0 * PRP)
            - 0.5 * (c2 - 3.0 * c3) * (PRP @ P + P @ PRP))


def se3_jl_inv(xi):
    """se3.py:250-259"""
    xi = np.asarray(xi, dtype=float)
    Ji = so3_jl_inv(xi[:3])
    Q = se3_Q(xi[:3], xi[3:])
    out = np.zeros((6, 6))
    out[:3, :3] = Ji
    out[3:, :3] = -Ji @ Q @ Ji
    out[3:, 3:] = Ji
    return out


# --- camera models, batched (cameras.py) ----------------------------------------

def distort(kind, dist, x, y):
    """cameras.py:57-73 -> (xd, yd, status)"""
    st = np.zeros(x.shape, dtype=np.int8)
    if kind == PINHOLE:
        return x, y, st
    if kind == RADIAL:
        k1, k2 = dist
        r2 = x * x + y * y
        f = 1.0 + k1 * r2 + k2 * r2 * r2
        return x * f, y * f, st
    r = np.hypot(x, y)
    theta = np.arctan(r)
    st[theta > MAX_FISHEYE_ANGLE] = DOMAIN
    with np.errstate(divide="ignore", invalid="ignore"):
        s = np.where(r < 1e-12, 1.0, theta / np.where(r < 1e-12, 1.0, r))
    return x * s, y * s, st


def distort_jacobian(kind, dist, x, y):
    """cameras.py:75-100 -> [...,2,2]"""
    J = np.zeros(x.shape + (2, 2))
    if kind == PINHOLE:
        J[..., 0, 0] = 1.0
        J[..., 1, 1] = 1.0
        return J
    r2 = x * x + y * y
    if kind == RADIAL:
        k1, k2 = dist
        f = 1.0 + k1 * r2 + k2 * r2 * r2
        g = 2.0 * (k1 + 2.0 * k2 * r2)
    else:
        r = np.sqrt(r2)
        small = r < 1e-4
        rs = np.where(small, 1.0, r)
        theta = np.arctan(rs)
        f = np.where(small, 1.0 - r2 / 3.0, theta / rs)
        g = np.where(small, -2.0 / 3.0 + 0.8 * r2, (1.0 / (1.0 + r2) - theta / rs) / np.where(small, 1.0, r2))
    J[..., 0, 0] = f + x * x * g
    J[..., 0, 1] = x * y * g
    J[..., 1, 0] = x * y * g
    J[..., 1, 1] = f + y * y * g
    return J


def project_cam(model, pc):
    """cameras.py:129-135 batched: camera-frame points [n,3] -> (pix, status)."""
    kind, fx, fy, cx, cy, dist = model
    Z = pc[:, 2]
    st = np.where(Z <= MIN_DEPTH, DEPTH, OK).astype(np.int8)
    Zs = np.where(st == DEPTH, 1.0, Z)
    xd, yd, st2 = distort(kind, dist, pc[:, 0] / Zs, pc[:, 1] / Zs)
    st = np.where(st == OK, st2, st)
    return np.stack([fx * xd + cx, fy * yd + cy], axis=1), st


def project_with_jacobians(model, R, t, X):
    """cameras.py:169-179 batched: R [n,3,3], t [n,3], X [n,3] ->
    (pix [n,2], Jc [n,2,6], Jp [n,2,3], status [n])."""
    kind, fx, fy, cx, cy, dist = model
    pc = np.einsum("nij,nj->ni", R, X) + t
    pix, st = project_cam(model, pc)
    Z = np.where(st == OK, pc[:, 2], 1.0)
    x, y = pc[:, 0] / Z, pc[:, 1] / Z
    Jn = np.zeros((len(X), 2, 3))
    Jn[:, 0, 0] = 1.0 / Z
    Jn[:, 0, 2] = -pc[:, 0] / (Z * Z)
    Jn[:, 1, 1] = 1.0 / Z
    Jn[:, 1, 2] = -pc[:, 1] / (Z * Z)
    Jd = distort_jacobian(kind, dist, x, y)
    Jpc = np.array([fx, fy])[None, :, None] * np.einsum("nij,njk->nik", Jd, Jn)
    mh = np.zeros((len(X), 3, 3))  # -hat(p)
    mh[:, 0, 1], mh[:, 0, 2] = pc[:, 2], -pc[:, 1]
    mh[:, 1, 0], mh[:, 1, 2] = -pc[:, 2], pc[:, 0]
    mh[:, 2, 0], mh[:, 2, 1] = pc[:, 1], -pc[:, 0]
    Jc = np.concatenate([np.einsum("nij,njk->nik", Jpc, mh), Jpc], axis=2)
    Jp = np.einsum("nij,njk->nik", Jpc, R)
    return pix, Jc, Jp, st


def undistort(kind, dist, xd, yd):
    """cameras.py:102-125 (scalar) -> (x, y, status)"""
    if kind == PINHOLE:
        return xd, yd, OK
    if kind == FISHEYE:
        theta = np.hypot(xd, yd)
        if theta >= np.pi / 2:
            return 0.0, 0.0, DOMAIN
        if theta < 1e-12:
            return xd, yd, OK
        s = np.tan(theta) / theta
        return xd * s, yd * s, OK
    k1, k2 = dist
    x, y = xd, yd
    for _ in range(UNDISTORT_ITERS):
        r2 = x * x + y * y
        f = 1.0 + k1 * r2 + k2 * r2 * r2
        if f <= 0:
            return 0.0, 0.0, UNDISTORT
        xn, yn = xd / f, yd / f
        if abs(xn - x) < UNDISTORT_TOL and abs(yn - y) < UNDISTORT_TOL:
            return xn, yn, OK
        x, y = xn, yn
    return 0.0, 0.0, UNDISTORT


def unproject(model, pixel):
    """cameras.py:150-166 (scalar) -> (unit ray, status)"""
    kind, fx, fy, cx, cy, dist = model
    x, y, st = undistort(kind, dist, (pixel[0] - cx) / fx, (pixel[1] - cy) / fy)
    if st != OK:
        return None, st
    r = np.array([x, y, 1.0])
    return r / np.linalg.norm(r), OK


def model_tuple(m):
    """sfm_camera_model-like record -> (kind, fx, fy, cx, cy, (k1, k2))."""
    return (int(m["kind"]), float(m["fx"]), float(m["fy"]), float(m["cx"]), float(m["cy"]),
            (float(m["k1"]), float(m["k2"])))


def loss_rho(kind, param, s):
    """solver.py:32-41 (vectorised)"""
    if kind == 0:
        return s
    if kind == 1:
        d2 = param * param
        return np.where(s <= d2, s, 2.0 * param * np.sqrt(s) - d2)
    c2 = param * param
    return c2 * np.log1p(s / c2)


def loss_rho_prime(kind, param, s):
    """solver.py:43-51 (vectorised)"""
    if kind == 0:
        return np.ones_like(s)
    if kind == 1:
        d2 = param * param
        with np.errstate(divide="ignore"):
            return np.where(s <= d2, 1.0, param / np.sqrt(np.where(s <= d2, 1.0, s)))
    return 1.0 / (1.0 + s / (param * param))
