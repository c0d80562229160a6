// sfm_math.cuh -- fp64 SE(3) / camera math for the sm_100a kernels.
//
// Device restatement of the reference geometry the hot path touches:
//   se3.py:20-29   _quat_normalize (canonical sign w >= 0)
//   se3.py:39-56   quat_multiply, quat_to_matrix
//   se3.py:138-201 compose, so3_exp/log, so3 left Jacobian (+inverse),
//                  exp_map, log_map
//   se3.py:204-267 adjoint, _se3_Q, se3_left_jacobian_inv
//   cameras.py:57-179 distortion, projection, projection Jacobian,
//                  unprojection, project_with_pose_jacobian
// Everything is straight-line register code; no memory traffic.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/sfm_b200.h"

#define SFM_HD __host__ __device__ __forceinline__

namespace sfm {

constexpr double kMinDepth = 1e-9;            // cameras.py:28
constexpr int kUndistortIters = 50;           // cameras.py:29
constexpr double kUndistortTol = 1e-10;       // cameras.py:30
constexpr double kMaxFisheyeAngle = 1.5690509975429023;  // deg2rad(89.9), cameras.py:32

// Projection status codes (device side).
enum : int { PROJ_OK = 0, PROJ_DEPTH = 1, PROJ_DOMAIN = 2, PROJ_UNDISTORT = 3 };

struct Quat { double w, x, y, z; };
struct Vec3 { double x, y, z; };
struct Mat3 { double m[9]; };  // row-major

// Rigid transform with its rotation matrix materialised (quat kept for
// retraction/composition).
struct Pose {
  Quat q;
  Vec3 t;
  Mat3 R;
};

SFM_HD Vec3 v3(double x, double y, double z) { return Vec3{x, y, z}; }
SFM_HD Vec3 add(Vec3 a, Vec3 b) { return v3(a.x + b.x, a.y + b.y, a.z + b.z); }
SFM_HD Vec3 sub(Vec3 a, Vec3 b) { return v3(a.x - b.x, a.y - b.y, a.z - b.z); }
SFM_HD Vec3 scale(Vec3 a, double s) { return v3(a.x * s, a.y * s, a.z * s); }
SFM_HD double dot(Vec3 a, Vec3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
SFM_HD double norm(Vec3 a) { return sqrt(dot(a, a)); }
SFM_HD Vec3 cross(Vec3 a, Vec3 b) {
  return v3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
SFM_HD Vec3 mul(const Mat3& A, Vec3 v) {
  return v3(A.m[0] * v.x + A.m[1] * v.y + A.m[2] * v.z,
            A.m[3] * v.x + A.m[4] * v.y + A.m[5] * v.z,
            A.m[6] * v.x + A.m[7] * v.y + A.m[8] * v.z);
}
SFM_HD Vec3 mulT(const Mat3& A, Vec3 v) {  // A^T v
  return v3(A.m[0] * v.x + A.m[3] * v.y + A.m[6] * v.z,
            A.m[1] * v.x + A.m[4] * v.y + A.m[7] * v.z,
            A.m[2] * v.x + A.m[5] * v.y + A.m[8] * v.z);
}
SFM_HD Mat3 matmul(const Mat3& A, const Mat3& B) {
  Mat3 C;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      C.m[i * 3 + j] = A.m[i * 3 + 0] * B.m[0 * 3 + j] + A.m[i * 3 + 1] * B.m[1 * 3 + j] +
                       A.m[i * 3 + 2] * B.m[2 * 3 + j];
  return C;
}
SFM_HD Mat3 hat(Vec3 v) {
  Mat3 H;
  H.m[0] = 0.0;  H.m[1] = -v.z; H.m[2] = v.y;
  H.m[3] = v.z;  H.m[4] = 0.0;  H.m[5] = -v.x;
  H.m[6] = -v.y; H.m[7] = v.x;  H.m[8] = 0.0;
  return H;
}
SFM_HD Mat3 eye3() {
  Mat3 I;
#pragma unroll
  for (int i = 0; i < 9; ++i) I.m[i] = (i % 4 == 0) ? 1.0 : 0.0;
  return I;
}

// se3.py:20-29 -- unit norm, canonical sign (w >= 0; ties by first nonzero).
SFM_HD Quat quat_normalize(Quat q) {
  double n = sqrt(q.w * q.w + q.x * q.x + q.y * q.y + q.z * q.z);
  q.w /= n; q.x /= n; q.y /= n; q.z /= n;
  bool neg = q.w < 0.0;
  if (q.w == 0.0) {
    if (q.x != 0.0) neg = q.x < 0.0;
    else if (q.y != 0.0) neg = q.y < 0.0;
    else if (q.z != 0.0) neg = q.z < 0.0;
  }
  if (neg) { q.w = -q.w; q.x = -q.x; q.y = -q.y; q.z = -q.z; }
  return q;
}

// se3.py:39-47
SFM_HD Quat quat_mul(Quat a, Quat b) {
  return Quat{a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z,
              a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y,
              a.w * b.y - a.x * b.z + a.y * b.w + a.z * b.x,
              a.w * b.z + a.x * b.y - a.y * b.x + a.z * b.w};
}

// se3.py:50-56
SFM_HD Mat3 quat_to_matrix(Quat q) {
  const double w = q.w, x = q.x, y = q.y, z = q.z;
  Mat3 R;
  R.m[0] = 1 - 2 * (y * y + z * z); R.m[1] = 2 * (x * y - w * z);     R.m[2] = 2 * (x * z + w * y);
  R.m[3] = 2 * (x * y + w * z);     R.m[4] = 1 - 2 * (x * x + z * z); R.m[5] = 2 * (y * z - w * x);
  R.m[6] = 2 * (x * z - w * y);     R.m[7] = 2 * (y * z + w * x);     R.m[8] = 1 - 2 * (x * x + y * y);
  return R;
}

SFM_HD Pose make_pose(Quat q, Vec3 t) {  // Pose.__post_init__ (se3.py:96-98)
  Pose p;
  p.q = quat_normalize(q);
  p.t = t;
  p.R = quat_to_matrix(p.q);
  return p;
}

// se3.py:127-129 -- Pose.inverse
SFM_HD Pose pose_inverse(const Pose& p) {
  Quat qi{p.q.w, -p.q.x, -p.q.y, -p.q.z};
  Mat3 Ri = quat_to_matrix(qi);
  Vec3 t = mul(Ri, p.t);
  return make_pose(qi, v3(-t.x, -t.y, -t.z));
}

// se3.py:138-140 -- compose(a, b) = a @ b
SFM_HD Pose compose(const Pose& a, const Pose& b) {
  return make_pose(quat_mul(a.q, b.q), add(mul(a.R, b.t), a.t));
}

// se3.py:143-154
SFM_HD Quat so3_exp(Vec3 phi) {
  double theta = norm(phi);
  double half = 0.5 * theta;
  double w, s;
  if (theta < 1e-8) {
    w = 1.0 - half * half / 2.0;
    s = 0.5 - half * half / 12.0;
  } else {
    w = cos(half);
    s = sin(half) / theta;
  }
  return quat_normalize(Quat{w, s * phi.x, s * phi.y, s * phi.z});
}

// se3.py:157-168
SFM_HD Vec3 so3_log(Quat q) {
  Vec3 v = v3(q.x, q.y, q.z);
  double n = norm(v);
  if (n < 1e-10) return scale(v, 2.0);
  double angle = 2.0 * atan2(n, q.w);
  return scale(v, angle / n);
}

// se3.py:171-178
SFM_HD Mat3 so3_left_jacobian(Vec3 phi) {
  double theta = norm(phi);
  Mat3 P = hat(phi), PP = matmul(P, P), J = eye3();
  double a, b;
  if (theta < 1e-6) { a = 0.5; b = 1.0 / 6.0; }
  else {
    a = (1.0 - cos(theta)) / (theta * theta);
    b = (theta - sin(theta)) / (theta * theta * theta);
  }
#pragma unroll
  for (int i = 0; i < 9; ++i) J.m[i] += a * P.m[i] + b * PP.m[i];
  return J;
}

// se3.py:181-187
SFM_HD Mat3 so3_left_jacobian_inv(Vec3 phi) {
  double theta = norm(phi);
  Mat3 P = hat(phi), PP = matmul(P, P), J = eye3();
  double c;
  if (theta < 1e-6) c = 1.0 / 12.0;
  else c = 1.0 / (theta * theta) - (1.0 + cos(theta)) / (2.0 * theta * sin(theta));
#pragma unroll
  for (int i = 0; i < 9; ++i) J.m[i] += -0.5 * P.m[i] + c * PP.m[i];
  return J;
}

// se3.py:190-194 -- exp_map(xi), xi = (phi, rho)
SFM_HD Pose se3_exp(const double xi[6]) {
  Vec3 phi = v3(xi[0], xi[1], xi[2]), rho = v3(xi[3], xi[4], xi[5]);
  Quat q = so3_exp(phi);
  Vec3 t = mul(so3_left_jacobian(phi), rho);
  return make_pose(q, t);
}

// se3.py:197-201
SFM_HD void se3_log(const Pose& p, double xi[6]) {
  Vec3 phi = so3_log(p.q);
  Vec3 rho = mul(so3_left_jacobian_inv(phi), p.t);
  xi[0] = phi.x; xi[1] = phi.y; xi[2] = phi.z;
  xi[3] = rho.x; xi[4] = rho.y; xi[5] = rho.z;
}

// se3.py:214-235 -- coupling block Q(phi, rho)
SFM_HD Mat3 se3_Q(Vec3 phi, Vec3 rho) {
  double theta = norm(phi);
  Mat3 P = hat(phi), Rh = hat(rho);
  Mat3 PR = matmul(P, Rh), RP = matmul(Rh, P), PRP = matmul(PR, P);
  double c1, c2, c3;
  if (theta < 1e-4) {
    double t2 = theta * theta;
    c1 = 1.0 / 6.0 - t2 / 120.0;
    c2 = 1.0 / 24.0 - t2 / 720.0;
    c3 = 1.0 / 120.0 - t2 / 2520.0;
  } else {
    double t2 = theta * theta, t3 = t2 * theta;
    c1 = (theta - sin(theta)) / t3;
    c2 = (1.0 - t2 / 2.0 - cos(theta)) / (t2 * t2);
    c3 = (theta - sin(theta) - t3 / 6.0) / (t3 * t2);
  }
  Mat3 PPR = matmul(P, PR), RPP = matmul(RP, P), PRPP = matmul(PRP, P), PPRP = matmul(P, PRP);
  Mat3 Q;
#pragma unroll
  for (int i = 0; i < 9; ++i)
    Q.m[i] = 0.5 * Rh.m[i] + c1 * (PR.m[i] + RP.m[i] + PRP.m[i]) -
             c2 * (PPR.m[i] + RPP.m[i] - 3.0 * PRP.m[i]) -
             0.5 * (c2 - 3.0 * c3) * (PRPP.m[i] + PPRP.m[i]);
  return Q;
}

// se3.py:250-259 -- 6x6 row-major J_l^{-1}(xi)
SFM_HD void se3_left_jacobian_inv(const double xi[6], double out[36]) {
  Vec3 phi = v3(xi[0], xi[1], xi[2]), rho = v3(xi[3], xi[4], xi[5]);
  Mat3 Ji = so3_left_jacobian_inv(phi);
  Mat3 Q = se3_Q(phi, rho);
  Mat3 B = matmul(matmul(Ji, Q), Ji);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      out[i * 6 + j] = Ji.m[i * 3 + j];
      out[i * 6 + j + 3] = 0.0;
      out[(i + 3) * 6 + j] = -B.m[i * 3 + j];
      out[(i + 3) * 6 + j + 3] = Ji.m[i * 3 + j];
    }
}

// se3.py:204-211 -- 6x6 row-major Adj(T)
SFM_HD void se3_adjoint(const Pose& p, double out[36]) {
  Mat3 tR = matmul(hat(p.t), p.R);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      out[i * 6 + j] = p.R.m[i * 3 + j];
      out[i * 6 + j + 3] = 0.0;
      out[(i + 3) * 6 + j] = tR.m[i * 3 + j];
      out[(i + 3) * 6 + j + 3] = p.R.m[i * 3 + j];
    }
}

// ---------------------------------------------------------------------------
// Camera models (cameras.py:57-166)
// ---------------------------------------------------------------------------

// cameras.py:57-73 -- normalized -> distorted; returns PROJ_* code.
SFM_HD int distort(const sfm_camera_model& c, double x, double y, double& xd, double& yd) {
  if (c.kind == SFM_CAM_PINHOLE) { xd = x; yd = y; return PROJ_OK; }
  if (c.kind == SFM_CAM_PINHOLE_RADIAL) {
    double r2 = x * x + y * y;
    double f = 1.0 + c.k1 * r2 + c.k2 * r2 * r2;
    xd = x * f; yd = y * f;
    return PROJ_OK;
  }
  double r = hypot(x, y);
  double theta = atan(r);
  if (theta > kMaxFisheyeAngle) return PROJ_DOMAIN;
  if (r < 1e-12) { xd = x; yd = y; return PROJ_OK; }
  double s = theta / r;
  xd = x * s; yd = y * s;
  return PROJ_OK;
}

// cameras.py:75-100 -- 2x2 d(distorted)/d(normalized), row-major
SFM_HD void distort_jacobian(const sfm_camera_model& c, double x, double y, double J[4]) {
  if (c.kind == SFM_CAM_PINHOLE) { J[0] = 1.0; J[1] = 0.0; J[2] = 0.0; J[3] = 1.0; return; }
  double f, g;
  double r2 = x * x + y * y;
  if (c.kind == SFM_CAM_PINHOLE_RADIAL) {
    f = 1.0 + c.k1 * r2 + c.k2 * r2 * r2;
    g = 2.0 * (c.k1 + 2.0 * c.k2 * r2);
  } else {
    double r = sqrt(r2);
    if (r < 1e-4) { f = 1.0 - r2 / 3.0; g = -2.0 / 3.0 + 0.8 * r2; }
    else {
      double theta = atan(r);
      f = theta / r;
      g = (1.0 / (1.0 + r2) - f) / r2;
    }
  }
  J[0] = f + x * x * g; J[1] = x * y * g;
  J[2] = x * y * g;     J[3] = f + y * y * g;
}

// cameras.py:102-125 -- distorted -> normalized
SFM_HD int undistort(const sfm_camera_model& c, double xd, double yd, double& x, double& y) {
  if (c.kind == SFM_CAM_PINHOLE) { x = xd; y = yd; return PROJ_OK; }
  if (c.kind == SFM_CAM_EQUIDISTANT_FISHEYE) {
    double theta = hypot(xd, yd);
    if (theta >= 1.5707963267948966) return PROJ_DOMAIN;
    if (theta < 1e-12) { x = xd; y = yd; return PROJ_OK; }
    double s = tan(theta) / theta;
    x = xd * s; y = yd * s;
    return PROJ_OK;
  }
  double cx = xd, cy = yd;
  for (int it = 0; it < kUndistortIters; ++it) {
    double r2 = cx * cx + cy * cy;
    double f = 1.0 + c.k1 * r2 + c.k2 * r2 * r2;
    if (f <= 0.0) return PROJ_UNDISTORT;
    double xn = xd / f, yn = yd / f;
    if (fabs(xn - cx) < kUndistortTol && fabs(yn - cy) < kUndistortTol) {
      x = xn; y = yn;
      return PROJ_OK;
    }
    cx = xn; cy = yn;
  }
  return PROJ_UNDISTORT;
}

// cameras.py:162-166 -- pixel -> unit ray in the camera frame
SFM_HD int unproject(const sfm_camera_model& c, double u, double v, Vec3& ray) {
  double x, y;
  int st = undistort(c, (u - c.cx) / c.fx, (v - c.cy) / c.fy, x, y);
  if (st != PROJ_OK) return st;
  Vec3 r = v3(x, y, 1.0);
  ray = scale(r, 1.0 / norm(r));
  return PROJ_OK;
}

// cameras.py:129-135 -- camera-frame point -> pixel
SFM_HD int project_point(const sfm_camera_model& c, Vec3 p, double& u, double& v) {
  if (p.z <= kMinDepth) return PROJ_DEPTH;
  double xd, yd;
  int st = distort(c, p.x / p.z, p.y / p.z, xd, yd);
  if (st != PROJ_OK) return st;
  u = c.fx * xd + c.cx;
  v = c.fy * yd + c.cy;
  return PROJ_OK;
}

// cameras.py:169-179 -- pixel, J_pose (2x6, left perturbation, (phi,rho)),
// J_point (2x3).  Jc/Jp row-major.
SFM_HD int project_with_jacobians(const sfm_camera_model& c, const Mat3& R, Vec3 t, Vec3 X,
                                  double& u, double& v, double Jc[12], double Jp[6]) {
  Vec3 p = add(mul(R, X), t);
  int st = project_point(c, p, u, v);
  if (st != PROJ_OK) return st;
  const double iz = 1.0 / p.z;
  const double x = p.x * iz, y = p.y * iz;
  double Jd[4];
  distort_jacobian(c, x, y, Jd);
  // J_norm = [[1/Z, 0, -X/Z^2], [0, 1/Z, -Y/Z^2]]
  const double n02 = -p.x * iz * iz, n12 = -p.y * iz * iz;
  // J_pc = diag(fx,fy) * Jd * J_norm
  double A[6];
  A[0] = c.fx * (Jd[0] * iz);
  A[1] = c.fx * (Jd[1] * iz);
  A[2] = c.fx * (Jd[0] * n02 + Jd[1] * n12);
  A[3] = c.fy * (Jd[2] * iz);
  A[4] = c.fy * (Jd[3] * iz);
  A[5] = c.fy * (Jd[2] * n02 + Jd[3] * n12);
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const double a = A[r * 3 + 0], b = A[r * 3 + 1], cc = A[r * 3 + 2];
    // row r of J_pc @ (-hat(p))
    Jc[r * 6 + 0] = -b * p.z + cc * p.y;
    Jc[r * 6 + 1] = a * p.z - cc * p.x;
    Jc[r * 6 + 2] = -a * p.y + b * p.x;
    Jc[r * 6 + 3] = a;
    Jc[r * 6 + 4] = b;
    Jc[r * 6 + 5] = cc;
    // row r of J_pc @ R
#pragma unroll
    for (int j = 0; j < 3; ++j)
      Jp[r * 3 + j] = a * R.m[0 * 3 + j] + b * R.m[1 * 3 + j] + cc * R.m[2 * 3 + j];
  }
  return PROJ_OK;
}

// solver.py:32-51 -- rho(s) and rho'(s)
SFM_HD double loss_rho(int kind, double param, double s) {
  if (kind == SFM_LOSS_TRIVIAL) return s;
  if (kind == SFM_LOSS_HUBER) {
    double d2 = param * param;
    return s <= d2 ? s : 2.0 * param * sqrt(s) - d2;
  }
  double c2 = param * param;
  return c2 * log1p(s / c2);
}
SFM_HD double loss_rho_prime(int kind, double param, double s) {
  if (kind == SFM_LOSS_TRIVIAL) return 1.0;
  if (kind == SFM_LOSS_HUBER) {
    double d2 = param * param;
    return s <= d2 ? 1.0 : param / sqrt(s);
  }
  return 1.0 / (1.0 + s / (param * param));
}

// Inverse of a symmetric positive-definite 6x6 block (row-major) through
// its Cholesky factor, fully unrolled (block and factors stay in
// registers).  Returns false (and a finite substitute) if A is not PD.
__device__ __forceinline__ bool spd6_inverse(const double A[36], double* __restrict__ M) {
  double L[36];
#pragma unroll
  for (int i = 0; i < 36; ++i) L[i] = 0.0;
  bool ok = true;
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    double s = A[c * 6 + c];
#pragma unroll
    for (int k = 0; k < c; ++k) s -= L[c * 6 + k] * L[c * 6 + k];
    if (!(s > 0.0)) { ok = false; s = 1.0; }
    double d = sqrt(s);
    L[c * 6 + c] = d;
#pragma unroll
    for (int r = c + 1; r < 6; ++r) {
      double v = A[r * 6 + c];
#pragma unroll
      for (int k = 0; k < c; ++k) v -= L[r * 6 + k] * L[c * 6 + k];
      L[r * 6 + c] = v / d;
    }
  }
  double Li[36];
#pragma unroll
  for (int i = 0; i < 36; ++i) Li[i] = 0.0;
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    Li[c * 6 + c] = 1.0 / L[c * 6 + c];
#pragma unroll
    for (int r = c + 1; r < 6; ++r) {
      double s = 0.0;
#pragma unroll
      for (int k = c; k < r; ++k) s += L[r * 6 + k] * Li[k * 6 + c];
      Li[r * 6 + c] = -s / L[r * 6 + r];
    }
  }
#pragma unroll
  for (int r = 0; r < 6; ++r)
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      double s = 0.0;
#pragma unroll
      for (int k = (r > c ? r : c); k < 6; ++k) s += Li[k * 6 + r] * Li[k * 6 + c];
      M[r * 6 + c] = s;
    }
  return ok;
}

}  // namespace sfm
