// tri.cu -- batched multi-view triangulation, RANSAC over observation pairs
// and reprojection gating (sm_100a, fp64).
//
// Reference path being replaced:
//   mapping.py:166-191  _world_rays, _max_ray_angle, _check_cheirality
//   mapping.py:194-221  triangulate_dlt (SVD of the stacked hat(d)[R|t] rows)
//   mapping.py:224-240  triangulate_midpoint (cond > 1e10 -> ParallelRays)
//   mapping.py:243-252  reprojection_error (inf when projection raises)
//   mapping.py:255-305  ransac_triangulate (exhaustive i<j pairs, strict <,
//                       lexicographic (count, -sum err), first best wins)
//   mapping.py:544-566  remove_outliers (strict >)
//
// DLT: the 3k x 4 system is reduced by streaming Givens rotations to a 4x4
// upper-triangular R (same right singular vectors as A, no squaring of the
// condition number), whose smallest right singular vector comes from a
// one-sided (Hestenes) Jacobi SVD.  RANSAC is warp-per-track: lanes split
// the pair hypotheses, a warp arg-max with a lowest-index tie-break
// reproduces the reference's sequential "first best" rule.
#include <cmath>
#include <cstdlib>

#include "sfm_math.cuh"
#include "tri.cuh"

namespace sfm {

namespace {

struct TriData {
  const int* of;              // [N] frame per observation
  const double* uv;           // [N*2]
  const double* ray;          // [N*3] unit camera-frame ray (unproject)
  const int* ray_st;          // [N] PROJ_* of unproject
  const double* Rt;           // [F*12]
  const int* fm;
  const sfm_camera_model* models;
};

__device__ __forceinline__ void cam_of(const TriData& d, int f, Mat3& R, Vec3& t) {
  const double* p = d.Rt + (int64_t)f * 12;
#pragma unroll
  for (int i = 0; i < 9; ++i) R.m[i] = p[i];
  t = v3(p[9], p[10], p[11]);
}

__global__ void k_rt(int F, const double* q, const double* t, double* Rt) {
  int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  Mat3 R = quat_to_matrix(Quat{q[f * 4], q[f * 4 + 1], q[f * 4 + 2], q[f * 4 + 3]});
  for (int i = 0; i < 9; ++i) Rt[f * 12 + i] = R.m[i];
  for (int i = 0; i < 3; ++i) Rt[f * 12 + 9 + i] = t[f * 3 + i];
}

// unproject every observation once (cameras.py:162-166)
__global__ void k_rays(int64_t N, TriData d, double* ray, int* st) {
  int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= N) return;
  const sfm_camera_model cm = d.models[d.fm[d.of[o]]];
  Vec3 r = v3(0, 0, 0);
  int s = unproject(cm, d.uv[o * 2], d.uv[o * 2 + 1], r);
  ray[o * 3] = r.x; ray[o * 3 + 1] = r.y; ray[o * 3 + 2] = r.z;
  st[o] = s;
}

// Observation selection inside a track.
struct Sel {
  int64_t b0, b1;
  int i, j;               // pair mode when i >= 0 (local indices)
  const uint8_t* mask;    // mask mode when non-null (indexed by global obs)
  __device__ __forceinline__ bool operator()(int64_t o) const {
    if (i >= 0) return o == b0 + i || o == b0 + j;
    if (mask) return mask[o] != 0;
    return true;
  }
};

__device__ __forceinline__ Vec3 world_dir(const TriData& d, int64_t o, Mat3& R, Vec3& t) {
  cam_of(d, d.of[o], R, t);
  Vec3 r = v3(d.ray[o * 3], d.ray[o * 3 + 1], d.ray[o * 3 + 2]);
  return mulT(R, r);
}

// mapping.py:177-183: max pairwise arccos(clip(|di.dj|)) == arccos(min |.|)
__device__ double max_ray_angle(const TriData& d, const Sel& s) {
  double mind = 2.0;
  for (int64_t a = s.b0; a < s.b1; ++a) {
    if (!s(a)) continue;
    Mat3 R; Vec3 t;
    Vec3 da = world_dir(d, a, R, t);
    for (int64_t b = a + 1; b < s.b1; ++b) {
      if (!s(b)) continue;
      Vec3 db = world_dir(d, b, R, t);
      double c = fabs(dot(da, db));
      mind = fmin(mind, c);
    }
  }
  if (mind > 1.0) mind = 1.0;
  return acos(mind);
}

__device__ __forceinline__ void givens_add(double Rm[10], double v[4]) {
  // Rm packed upper triangle row-major: (0,0)(0,1)(0,2)(0,3)(1,1)(1,2)(1,3)(2,2)(2,3)(3,3)
  int base = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int len = 4 - c;
    double rc = Rm[base];
    double vc = v[c];
    if (vc != 0.0) {
      double r = hypot(rc, vc);
      double cs = rc / r, sn = vc / r;
      Rm[base] = r;
      for (int j = 1; j < len; ++j) {
        double a = Rm[base + j], b = v[c + j];
        Rm[base + j] = cs * a + sn * b;
        v[c + j] = -sn * a + cs * b;
      }
    }
    base += len;
  }
}

// Smallest right singular vector of the 4x4 upper-triangular R
// (one-sided Jacobi on the columns).
__device__ __forceinline__ void smallest_right_sv(const double Rm[10], double out[4]) {
  // every index below is a compile-time constant after unrolling, so A and
  // V stay in registers (a runtime column index would put them in local
  // memory for the whole sweep loop)
  double A[4][4];
  int base = 0;
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) A[r][c] = 0.0;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
#pragma unroll
    for (int c = r; c < 4; ++c) A[r][c] = Rm[base + (c - r)];
    base += 4 - r;
  }
  double V[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) V[r][c] = (r == c) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 40; ++sweep) {
    bool rotated = false;
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int q = p + 1; q < 4; ++q) {
        double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          al += A[r][p] * A[r][p];
          be += A[r][q] * A[r][q];
          ga += A[r][p] * A[r][q];
        }
        if (ga == 0.0 || fabs(ga) <= 1e-17 * sqrt(al * be)) continue;
        rotated = true;
        double zeta = (be - al) / (2.0 * ga);
        double tt = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        double cs = 1.0 / sqrt(1.0 + tt * tt), sn = cs * tt;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          double a = A[r][p], b = A[r][q];
          A[r][p] = cs * a - sn * b;
          A[r][q] = sn * a + cs * b;
          double va = V[r][p], vb = V[r][q];
          V[r][p] = cs * va - sn * vb;
          V[r][q] = sn * va + cs * vb;
        }
      }
    if (!rotated) break;
  }
  // smallest column norm (first on ties), its V column selected by value
  double bn = 1e308, v0 = 0.0, v1 = 0.0, v2 = 0.0, v3_ = 0.0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    double n = 0.0;
#pragma unroll
    for (int r = 0; r < 4; ++r) n += A[r][c] * A[r][c];
    if (n < bn) { bn = n; v0 = V[0][c]; v1 = V[1][c]; v2 = V[2][c]; v3_ = V[3][c]; }
  }
  double nv = 0.0;
  nv += v0 * v0;
  nv += v1 * v1;
  nv += v2 * v2;
  nv += v3_ * v3_;
  nv = sqrt(nv);
  out[0] = v0 / nv; out[1] = v1 / nv; out[2] = v2 / nv; out[3] = v3_ / nv;
}

// Eigenvalues of a symmetric 3x3 (cyclic Jacobi) -> condition estimate.
__device__ double sym3_cond(const double S[9]) {
  double A[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) A[r][c] = S[r * 3 + c];
  for (int sweep = 0; sweep < 50; ++sweep) {
    double off = fabs(A[0][1]) + fabs(A[0][2]) + fabs(A[1][2]);
    if (off == 0.0) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        if (A[p][q] == 0.0) continue;
        double theta = (A[q][q] - A[p][p]) / (2.0 * A[p][q]);
        double t = copysign(1.0, theta) / (fabs(theta) + sqrt(theta * theta + 1.0));
        double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < 3; ++k) {
          double akp = A[k][p], akq = A[k][q];
          A[k][p] = c * akp - s * akq;
          A[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < 3; ++k) {
          double apk = A[p][k], aqk = A[q][k];
          A[p][k] = c * apk - s * aqk;
          A[q][k] = s * apk + c * aqk;
        }
      }
  }
  double e0 = fabs(A[0][0]), e1 = fabs(A[1][1]), e2 = fabs(A[2][2]);
  double mx = fmax(e0, fmax(e1, e2)), mn = fmin(e0, fmin(e1, e2));
  return mx / fmax(mn, 1e-300);
}

// LU with partial pivoting (numpy.linalg.solve / LAPACK gesv).
__device__ bool solve3(double A[9], double b[3], double x[3]) {
  int piv[3] = {0, 1, 2};
  for (int k = 0; k < 3; ++k) {
    int p = k;
    double mx = fabs(A[piv[k] * 3 + k]);
    for (int i = k + 1; i < 3; ++i)
      if (fabs(A[piv[i] * 3 + k]) > mx) { mx = fabs(A[piv[i] * 3 + k]); p = i; }
    if (mx == 0.0) return false;
    int tmp = piv[k]; piv[k] = piv[p]; piv[p] = tmp;
    for (int i = k + 1; i < 3; ++i) {
      double f = A[piv[i] * 3 + k] / A[piv[k] * 3 + k];
      A[piv[i] * 3 + k] = f;
      for (int j = k + 1; j < 3; ++j) A[piv[i] * 3 + j] -= f * A[piv[k] * 3 + j];
    }
  }
  double y[3];
  for (int i = 0; i < 3; ++i) {
    double s = b[piv[i]];
    for (int j = 0; j < i; ++j) s -= A[piv[i] * 3 + j] * y[j];
    y[i] = s;
  }
  for (int i = 2; i >= 0; --i) {
    double s = y[i];
    for (int j = i + 1; j < 3; ++j) s -= A[piv[i] * 3 + j] * x[j];
    x[i] = s / A[piv[i] * 3 + i];
  }
  return true;
}

// Triangulates the selected observations (mapping.py:194-240).  Returns a
// SFM_TRI_* status.  check_angle applies the min_angle parallax gate.
__device__ int tri_solve(const TriData& d, const Sel& s, int method, double min_angle, bool check_angle,
                         Vec3& X) {
  int n = 0;
  for (int64_t o = s.b0; o < s.b1; ++o) {
    if (!s(o)) continue;
    ++n;
    if (d.ray_st[o] != PROJ_OK) return d.ray_st[o] == PROJ_DOMAIN ? SFM_TRI_CAMERA_DOMAIN : SFM_TRI_CAMERA_ERROR;
  }
  if (n < 2) return SFM_TRI_TOO_FEW_OBS;
  if (check_angle && max_ray_angle(d, s) < min_angle) return SFM_TRI_INSUFFICIENT_PARALLAX;
  if (method == SFM_TRI_DLT) {
    double Rm[10];
    for (int i = 0; i < 10; ++i) Rm[i] = 0.0;
    for (int64_t o = s.b0; o < s.b1; ++o) {
      if (!s(o)) continue;
      Mat3 R; Vec3 t;
      cam_of(d, d.of[o], R, t);
      const double dx = d.ray[o * 3], dy = d.ray[o * 3 + 1], dz = d.ray[o * 3 + 2];
      double P[3][4];
      for (int i = 0; i < 3; ++i) {
        P[i][0] = R.m[i * 3]; P[i][1] = R.m[i * 3 + 1]; P[i][2] = R.m[i * 3 + 2];
      }
      P[0][3] = t.x; P[1][3] = t.y; P[2][3] = t.z;
      double row[4];
      for (int c = 0; c < 4; ++c) row[c] = -dz * P[1][c] + dy * P[2][c];
      givens_add(Rm, row);
      for (int c = 0; c < 4; ++c) row[c] = dz * P[0][c] - dx * P[2][c];
      givens_add(Rm, row);
      for (int c = 0; c < 4; ++c) row[c] = -dy * P[0][c] + dx * P[1][c];
      givens_add(Rm, row);
    }
    double Xh[4];
    smallest_right_sv(Rm, Xh);
    if (fabs(Xh[3]) < 1e-12) return SFM_TRI_INSUFFICIENT_PARALLAX;
    X = v3(Xh[0] / Xh[3], Xh[1] / Xh[3], Xh[2] / Xh[3]);
  } else {
    double A[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, b[3] = {0, 0, 0};
    for (int64_t o = s.b0; o < s.b1; ++o) {
      if (!s(o)) continue;
      Mat3 R; Vec3 t;
      Vec3 w = world_dir(d, o, R, t);
      Vec3 c = mulT(R, t);
      c = v3(-c.x, -c.y, -c.z);
      const double wv[3] = {w.x, w.y, w.z}, cv[3] = {c.x, c.y, c.z};
      for (int i = 0; i < 3; ++i) {
        double bi = 0.0;
        for (int j = 0; j < 3; ++j) {
          double m = (i == j ? 1.0 : 0.0) - wv[i] * wv[j];
          A[i * 3 + j] += m;
          bi += m * cv[j];
        }
        b[i] += bi;
      }
    }
    if (sym3_cond(A) > 1e10) return SFM_TRI_PARALLEL_RAYS;
    double x[3];
    if (!solve3(A, b, x)) return SFM_TRI_PARALLEL_RAYS;
    X = v3(x[0], x[1], x[2]);
  }
  // cheirality (mapping.py:186-191)
  for (int64_t o = s.b0; o < s.b1; ++o) {
    if (!s(o)) continue;
    Mat3 R; Vec3 t;
    cam_of(d, d.of[o], R, t);
    Vec3 pc = add(mul(R, X), t);
    Vec3 r = v3(d.ray[o * 3], d.ray[o * 3 + 1], d.ray[o * 3 + 2]);
    if (dot(pc, r) <= 0.0) return SFM_TRI_CHEIRALITY;
  }
  if (!(isfinite(X.x) && isfinite(X.y) && isfinite(X.z))) return SFM_TRI_INSUFFICIENT_PARALLAX;
  return SFM_TRI_OK;
}

// mapping.py:243-252
__device__ __forceinline__ double reproj_err(const TriData& d, int64_t o, Vec3 X) {
  Mat3 R; Vec3 t;
  const int f = d.of[o];
  cam_of(d, f, R, t);
  Vec3 pc = add(mul(R, X), t);
  double u, v;
  if (project_point(d.models[d.fm[f]], pc, u, v) != PROJ_OK) return INFINITY;
  double du = u - d.uv[o * 2], dv = v - d.uv[o * 2 + 1];
  return sqrt(du * du + dv * dv);
}

// numpy's pairwise summation order (numpy/_core/src/umath/loops_utils.h
// pairwise_sum) for n <= 128 elements streamed in order; longer arrays fall
// back to a sequential sum.
struct NpSum {
  int n, m = 0;
  double r[8];
  double res = 0.0;
  __device__ explicit NpSum(int n_) : n(n_) {}
  __device__ void add(double v) {
    if (n < 8 || n > 128) { res += v; ++m; return; }
    const int blocks = n - (n % 8);
    if (m < 8) r[m] = v;
    else if (m < blocks) r[m % 8] += v;
    else res += v;
    ++m;
    if (m == blocks) res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7])) + res;
  }
  __device__ double value() const { return res; }
};

// Score of one hypothesis: inlier count and -sum(err[inliers]).
__device__ void score_hyp(const TriData& d, int64_t b0, int64_t b1, Vec3 X, double thr, int& cnt,
                          double& negsum) {
  cnt = 0;
  for (int64_t o = b0; o < b1; ++o) cnt += reproj_err(d, o, X) < thr;
  NpSum s(cnt);
  for (int64_t o = b0; o < b1; ++o) {
    double e = reproj_err(d, o, X);
    if (e < thr) s.add(e);
  }
  negsum = -s.value();
}

struct TrackArgs {
  int64_t T;
  const int64_t* ptr;
  const uint8_t* active;
  TriData d;
  double thr, min_angle;
  int method;
  double* X;
  uint8_t* mask;
  int8_t* status;
};

__device__ __forceinline__ void pair_of(int k, int pi, int& i, int& j) {
  i = 0;
  int rem = pi;
  while (rem >= k - 1 - i) { rem -= k - 1 - i; ++i; }
  j = i + 1 + rem;
}

// Warp per track, observations read from global memory: ransac_triangulate
// (mapping.py:255-305) for tracks longer than the staged kernel takes.
__device__ void ransac_track_global(const TrackArgs& a, int64_t t, int lane) {
  const int64_t b0 = a.ptr[t], b1 = a.ptr[t + 1];
  const int k = (int)(b1 - b0);
  const int npairs = k * (k - 1) / 2;
  int bcnt = -1, bidx = 0x7fffffff;
  double bneg = -INFINITY;
  for (int pi = lane; pi < npairs; pi += 32) {
    int i, j;
    pair_of(k, pi, i, j);
    Sel s{b0, b1, i, j, nullptr};
    Vec3 X;
    int st;
    if (a.method == SFM_TRI_DLT) {
      st = tri_solve(a.d, s, SFM_TRI_DLT, a.min_angle, true, X);
    } else {
      st = tri_solve(a.d, s, SFM_TRI_MIDPOINT, a.min_angle, true, X);
    }
    if (st != SFM_TRI_OK) continue;
    int cnt;
    double neg;
    score_hyp(a.d, b0, b1, X, a.thr, cnt, neg);
    if (cnt >= 2 && (cnt > bcnt || (cnt == bcnt && neg > bneg))) {
      bcnt = cnt; bneg = neg; bidx = pi;
    }
  }
  // warp arg-max: (count, -sum) lexicographic, lowest pair index on ties
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    int oc = __shfl_down_sync(0xffffffffu, bcnt, off);
    double on = __shfl_down_sync(0xffffffffu, bneg, off);
    int oi = __shfl_down_sync(0xffffffffu, bidx, off);
    bool take = oc > bcnt || (oc == bcnt && (on > bneg || (on == bneg && oi < bidx)));
    if (take) { bcnt = oc; bneg = on; bidx = oi; }
  }
  if (lane != 0) return;
  int status = SFM_TRI_FAILED;
  Vec3 X = v3(NAN, NAN, NAN);
  if (bcnt >= 2) {
    int i, j;
    pair_of(k, bidx, i, j);
    Sel s{b0, b1, i, j, nullptr};
    Vec3 Xb;
    tri_solve(a.d, s, a.method, a.min_angle, true, Xb);
    for (int64_t o = b0; o < b1; ++o) a.mask[o] = reproj_err(a.d, o, Xb) < a.thr;
    Sel si{b0, b1, -1, -1, a.mask};
    // refinement on the inliers (midpoint has no parallax gate, :295)
    int st = tri_solve(a.d, si, a.method, a.min_angle, a.method == SFM_TRI_DLT, X);
    if (st == SFM_TRI_OK) {
      int cnt = 0;
      for (int64_t o = b0; o < b1; ++o) {
        uint8_t m = reproj_err(a.d, o, X) < a.thr;
        a.mask[o] = m;
        cnt += m;
      }
      if (cnt >= 2) status = SFM_TRI_OK;
    }
  }
  if (status != SFM_TRI_OK) {
    for (int64_t o = b0; o < b1; ++o) a.mask[o] = 0;
    X = v3(NAN, NAN, NAN);
  }
  a.status[t] = (int8_t)status;
  a.X[t * 3] = X.x; a.X[t * 3 + 1] = X.y; a.X[t * 3 + 2] = X.z;
}

// ---- staged RANSAC: a track's observations (camera record, ray, world
// direction, pixel, model, unproject status) copied into the warp's shared
// memory once, lane o <- observation o, so every hypothesis of the track
// reads them from shared memory instead of re-gathering camera records from
// L2 for each of its ~k^2 uses.  Same arithmetic, in the same order, as
// tri_solve / reproj_err / score_hyp above -- the masks, statuses and
// positions are bit-identical -- plus: a pair hypothesis touches only its two
// observations (no filtered loop over the track), and the refinement's
// per-observation errors run across the lanes.
constexpr int kRansacMaxK = 32;
constexpr int kRansacWarps = 4;

struct ObsSm {
  double R[9], t[3], ray[3], w[3], uv[2];
  int model, st;
};

__device__ __forceinline__ double reproj_sm(const ObsSm& ob, const sfm_camera_model* models, Vec3 X) {
  Mat3 R;
#pragma unroll
  for (int i = 0; i < 9; ++i) R.m[i] = ob.R[i];
  const Vec3 pc = add(mul(R, X), v3(ob.t[0], ob.t[1], ob.t[2]));
  double u, v;
  if (project_point(models[ob.model], pc, u, v) != PROJ_OK) return INFINITY;
  const double du = u - ob.uv[0], dv = v - ob.uv[1];
  return sqrt(du * du + dv * dv);
}

__device__ __forceinline__ void dlt_rows_sm(const ObsSm& ob, double Rm[10]) {
  const double dx = ob.ray[0], dy = ob.ray[1], dz = ob.ray[2];
  double P[3][4];
  for (int i = 0; i < 3; ++i) {
    P[i][0] = ob.R[i * 3]; P[i][1] = ob.R[i * 3 + 1]; P[i][2] = ob.R[i * 3 + 2];
  }
  P[0][3] = ob.t[0]; P[1][3] = ob.t[1]; P[2][3] = ob.t[2];
  double row[4];
  for (int c = 0; c < 4; ++c) row[c] = -dz * P[1][c] + dy * P[2][c];
  givens_add(Rm, row);
  for (int c = 0; c < 4; ++c) row[c] = dz * P[0][c] - dx * P[2][c];
  givens_add(Rm, row);
  for (int c = 0; c < 4; ++c) row[c] = -dy * P[0][c] + dx * P[1][c];
  givens_add(Rm, row);
}

__device__ __forceinline__ void midpoint_add_sm(const ObsSm& ob, double A[9], double b[3]) {
  Mat3 R;
#pragma unroll
  for (int i = 0; i < 9; ++i) R.m[i] = ob.R[i];
  Vec3 c = mulT(R, v3(ob.t[0], ob.t[1], ob.t[2]));
  c = v3(-c.x, -c.y, -c.z);
  const double wv[3] = {ob.w[0], ob.w[1], ob.w[2]}, cv[3] = {c.x, c.y, c.z};
  for (int i = 0; i < 3; ++i) {
    double bi = 0.0;
    for (int j = 0; j < 3; ++j) {
      double m = (i == j ? 1.0 : 0.0) - wv[i] * wv[j];
      A[i * 3 + j] += m;
      bi += m * cv[j];
    }
    b[i] += bi;
  }
}

// tri_solve over the observations in `sel` (bit o = observation o of the
// track, visited in ascending order), from the staged records.
__device__ int tri_solve_sm(const ObsSm* ob, unsigned sel, const sfm_camera_model* models, int method,
                            double min_angle, bool check_angle, Vec3& X) {
  (void)models;
  const int n = __popc(sel);
  for (unsigned m = sel; m; m &= m - 1) {
    const int o = __ffs(m) - 1;
    if (ob[o].st != PROJ_OK) return ob[o].st == PROJ_DOMAIN ? SFM_TRI_CAMERA_DOMAIN : SFM_TRI_CAMERA_ERROR;
  }
  if (n < 2) return SFM_TRI_TOO_FEW_OBS;
  if (check_angle) {  // max_ray_angle: arccos of the smallest |da.db| over pairs
    double mind = 2.0;
    for (unsigned ma = sel; ma; ma &= ma - 1) {
      const int oa = __ffs(ma) - 1;
      const Vec3 da = v3(ob[oa].w[0], ob[oa].w[1], ob[oa].w[2]);
      for (unsigned mb = ma & (ma - 1); mb; mb &= mb - 1) {
        const int b = __ffs(mb) - 1;
        mind = fmin(mind, fabs(dot(da, v3(ob[b].w[0], ob[b].w[1], ob[b].w[2]))));
      }
    }
    if (mind > 1.0) mind = 1.0;
    if (acos(mind) < min_angle) return SFM_TRI_INSUFFICIENT_PARALLAX;
  }
  if (method == SFM_TRI_DLT) {
    double Rm[10];
    for (int i = 0; i < 10; ++i) Rm[i] = 0.0;
    for (unsigned m = sel; m; m &= m - 1) dlt_rows_sm(ob[__ffs(m) - 1], Rm);
    double Xh[4];
    smallest_right_sv(Rm, Xh);
    if (fabs(Xh[3]) < 1e-12) return SFM_TRI_INSUFFICIENT_PARALLAX;
    X = v3(Xh[0] / Xh[3], Xh[1] / Xh[3], Xh[2] / Xh[3]);
  } else {
    double A[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, b[3] = {0, 0, 0};
    for (unsigned m = sel; m; m &= m - 1) midpoint_add_sm(ob[__ffs(m) - 1], A, b);
    if (sym3_cond(A) > 1e10) return SFM_TRI_PARALLEL_RAYS;
    double x[3];
    if (!solve3(A, b, x)) return SFM_TRI_PARALLEL_RAYS;
    X = v3(x[0], x[1], x[2]);
  }
  for (unsigned m = sel; m; m &= m - 1) {  // cheirality (mapping.py:186-191)
    const ObsSm& o = ob[__ffs(m) - 1];
    Mat3 R;
#pragma unroll
    for (int i = 0; i < 9; ++i) R.m[i] = o.R[i];
    const Vec3 pc = add(mul(R, X), v3(o.t[0], o.t[1], o.t[2]));
    if (dot(pc, v3(o.ray[0], o.ray[1], o.ray[2])) <= 0.0) return SFM_TRI_CHEIRALITY;
  }
  if (!(isfinite(X.x) && isfinite(X.y) && isfinite(X.z))) return SFM_TRI_INSUFFICIENT_PARALLAX;
  return SFM_TRI_OK;
}

// One track by the whole warp: ransac_triangulate (mapping.py:255-305).
__device__ void ransac_track(const TrackArgs& a, int64_t t, int lane, ObsSm* ob) {
  const int64_t b0 = a.ptr[t], b1 = a.ptr[t + 1];
  const int k = (int)(b1 - b0);
  if (a.active && !a.active[t]) {
    for (int64_t o = b0 + lane; o < b1; o += 32) a.mask[o] = 0;
    if (lane == 0) {
      a.status[t] = SFM_TRI_SKIPPED;
      a.X[t * 3] = a.X[t * 3 + 1] = a.X[t * 3 + 2] = NAN;
    }
    return;
  }
  if (k > kRansacMaxK) {
    ransac_track_global(a, t, lane);
    return;
  }
  __syncwarp();  // the previous track's readers of ob are done
  if (lane < k) {  // stage observation lane
    const int64_t o = b0 + lane;
    const int f = a.d.of[o];
    ObsSm& m = ob[lane];
    const double* p = a.d.Rt + (int64_t)f * 12;
#pragma unroll
    for (int i = 0; i < 9; ++i) m.R[i] = p[i];
    m.t[0] = p[9]; m.t[1] = p[10]; m.t[2] = p[11];
    m.ray[0] = a.d.ray[o * 3]; m.ray[1] = a.d.ray[o * 3 + 1]; m.ray[2] = a.d.ray[o * 3 + 2];
    Mat3 R;
#pragma unroll
    for (int i = 0; i < 9; ++i) R.m[i] = m.R[i];
    const Vec3 w = mulT(R, v3(m.ray[0], m.ray[1], m.ray[2]));  // world_dir
    m.w[0] = w.x; m.w[1] = w.y; m.w[2] = w.z;
    m.uv[0] = a.d.uv[o * 2]; m.uv[1] = a.d.uv[o * 2 + 1];
    m.model = a.d.fm[f];
    m.st = a.d.ray_st[o];
  }
  __syncwarp();
  const sfm_camera_model* models = a.d.models;
  const int npairs = k * (k - 1) / 2;
  int bcnt = -1, bidx = 0x7fffffff;
  double bneg = -INFINITY;
  Vec3 bX = v3(0.0, 0.0, 0.0);  // this lane's best hypothesis (the winner is not re-solved)
  for (int pi = lane; pi < npairs; pi += 32) {
    int i, j;
    pair_of(k, pi, i, j);
    Vec3 X;
    if (tri_solve_sm(ob, (1u << i) | (1u << j), models, a.method, a.min_angle, true, X) != SFM_TRI_OK) continue;
    // score_hyp: inlier count, then numpy's pairwise sum of their errors.
    // Fewer than 8 inliers sum sequentially (NpSum's short path), so a
    // track of k < 8 observations needs one pass over them, not two.
    int cnt = 0;
    double neg;
    if (k < 8) {
      double res = 0.0;
      for (int o = 0; o < k; ++o) {
        const double e = reproj_sm(ob[o], models, X);
        if (e < a.thr) { ++cnt; res += e; }
      }
      neg = -res;
    } else {
      for (int o = 0; o < k; ++o) cnt += reproj_sm(ob[o], models, X) < a.thr;
      NpSum acc(cnt);
      for (int o = 0; o < k; ++o) {
        const double e = reproj_sm(ob[o], models, X);
        if (e < a.thr) acc.add(e);
      }
      neg = -acc.value();
    }
    if (cnt >= 2 && (cnt > bcnt || (cnt == bcnt && neg > bneg))) {
      bcnt = cnt; bneg = neg; bidx = pi; bX = X;
    }
  }
  // warp arg-max: (count, -sum) lexicographic, lowest pair index on ties
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    int oc = __shfl_down_sync(0xffffffffu, bcnt, off);
    double on = __shfl_down_sync(0xffffffffu, bneg, off);
    int oi = __shfl_down_sync(0xffffffffu, bidx, off);
    bool take = oc > bcnt || (oc == bcnt && (on > bneg || (on == bneg && oi < bidx)));
    if (take) { bcnt = oc; bneg = on; bidx = oi; }
  }
  bcnt = __shfl_sync(0xffffffffu, bcnt, 0);
  bidx = __shfl_sync(0xffffffffu, bidx, 0);
  int status = SFM_TRI_FAILED;
  Vec3 X = v3(NAN, NAN, NAN);
  unsigned inl = 0;
  if (bcnt >= 2) {
    // the winning hypothesis from the lane that scored it (pair bidx ran on
    // lane bidx % 32), its inlier set across lanes
    const int wl = bidx & 31;
    const Vec3 Xb = v3(__shfl_sync(0xffffffffu, bX.x, wl), __shfl_sync(0xffffffffu, bX.y, wl),
                       __shfl_sync(0xffffffffu, bX.z, wl));
    const unsigned sel = __ballot_sync(0xffffffffu, lane < k && reproj_sm(ob[lane < k ? lane : 0], models, Xb) < a.thr);
    // refinement on the inliers (midpoint has no parallax gate, :295)
    int st = SFM_TRI_FAILED;
    if (lane == 0) st = tri_solve_sm(ob, sel, models, a.method, a.min_angle, a.method == SFM_TRI_DLT, X);
    st = __shfl_sync(0xffffffffu, st, 0);
    if (st == SFM_TRI_OK) {
      X = v3(__shfl_sync(0xffffffffu, X.x, 0), __shfl_sync(0xffffffffu, X.y, 0), __shfl_sync(0xffffffffu, X.z, 0));
      inl = __ballot_sync(0xffffffffu, lane < k && reproj_sm(ob[lane < k ? lane : 0], models, X) < a.thr);
      if (__popc(inl) >= 2) status = SFM_TRI_OK;
    }
  }
  if (status != SFM_TRI_OK) {
    inl = 0;
    X = v3(NAN, NAN, NAN);
  }
  if (lane < k) a.mask[b0 + lane] = (inl >> lane) & 1u;
  if (lane == 0) {
    a.status[t] = (int8_t)status;
    a.X[t * 3] = X.x; a.X[t * 3 + 1] = X.y; a.X[t * 3 + 2] = X.z;
  }
}


// Warp per track.
__global__ void __launch_bounds__(kRansacWarps * 32) k_ransac(TrackArgs a) {
  __shared__ ObsSm obs[kRansacWarps][kRansacMaxK];
  const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (t >= a.T) return;
  ransac_track(a, t, lane, obs[warp]);
}

// Short tracks share a warp.  Warp w takes tracks 3w .. 3w+2: when their
// observations fit the warp's staging slots (sum k <= 32) and the active
// tracks' pair hypotheses fit its lanes (sum k(k-1)/2 <= 32), all three run
// in one pass -- each track's hypotheses on a contiguous lane range, a
// segmented arg-max per range, the refinements on the ranges' first lanes in
// parallel -- with each track's arithmetic exactly as in ransac_track, so the
// statuses, masks and positions are the same bits.  Otherwise the warp runs
// the three tracks one after another.  (configs[3]: k = 5, 10 hypotheses a
// track, a third of the lanes busy one track per warp.)
constexpr int kPack = 3;
__global__ void __launch_bounds__(kRansacWarps * 32) k_ransac_packed(TrackArgs a) {
  __shared__ ObsSm obs[kRansacWarps][kRansacMaxK];
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t t0 = w * kPack;
  if (t0 >= a.T) return;
  const int nt = a.T - t0 < kPack ? (int)(a.T - t0) : kPack;
  ObsSm* ob = obs[warp];
  int kk[kPack], off[kPack + 1], hoff[kPack + 1];
  bool act[kPack];
  const int64_t base = a.ptr[t0];
  off[0] = 0;
  hoff[0] = 0;
#pragma unroll
  for (int q = 0; q < kPack; ++q) {
    const bool in = q < nt;
    kk[q] = in ? (int)(a.ptr[t0 + q + 1] - a.ptr[t0 + q]) : 0;
    act[q] = in && (!a.active || a.active[t0 + q]);
    off[q + 1] = off[q] + kk[q];
    hoff[q + 1] = hoff[q] + (act[q] ? kk[q] * (kk[q] - 1) / 2 : 0);
  }
  if (off[kPack] > kRansacMaxK || hoff[kPack] > 32) {
    for (int q = 0; q < nt; ++q) ransac_track(a, t0 + q, lane, ob);
    return;
  }
  // stage the chunk's observations (one contiguous range), lane o <- observation o
  const int ktot = off[kPack];
  if (lane < ktot) {
    const int64_t o = base + lane;
    const int f = a.d.of[o];
    ObsSm& m = ob[lane];
    const double* p = a.d.Rt + (int64_t)f * 12;
#pragma unroll
    for (int i = 0; i < 9; ++i) m.R[i] = p[i];
    m.t[0] = p[9]; m.t[1] = p[10]; m.t[2] = p[11];
    m.ray[0] = a.d.ray[o * 3]; m.ray[1] = a.d.ray[o * 3 + 1]; m.ray[2] = a.d.ray[o * 3 + 2];
    Mat3 R;
#pragma unroll
    for (int i = 0; i < 9; ++i) R.m[i] = m.R[i];
    const Vec3 wd = mulT(R, v3(m.ray[0], m.ray[1], m.ray[2]));  // world_dir
    m.w[0] = wd.x; m.w[1] = wd.y; m.w[2] = wd.z;
    m.uv[0] = a.d.uv[o * 2]; m.uv[1] = a.d.uv[o * 2 + 1];
    m.model = a.d.fm[f];
    m.st = a.d.ray_st[o];
  }
  __syncwarp();
  const sfm_camera_model* models = a.d.models;
  // this lane's hypothesis: track hq, pair index pi within it
  int hq = -1;
#pragma unroll
  for (int q = 0; q < kPack; ++q)
    if (lane >= hoff[q] && lane < hoff[q + 1]) hq = q;
  int qo = 0, qk = 0, hs = 0, he = 0;  // the lane's track: staging offset, k, lane range
#pragma unroll
  for (int q = 0; q < kPack; ++q)
    if (q == hq) { qo = off[q]; qk = kk[q]; hs = hoff[q]; he = hoff[q + 1]; }
  int bcnt = -1, bidx = 0x7fffffff;
  double bneg = -INFINITY;
  Vec3 bX = v3(0.0, 0.0, 0.0);
  if (hq >= 0) {
    const int pi = lane - hs;
    const ObsSm* tob = ob + qo;
    int i, j;
    pair_of(qk, pi, i, j);
    Vec3 X;
    if (tri_solve_sm(tob, (1u << i) | (1u << j), models, a.method, a.min_angle, true, X) == SFM_TRI_OK) {
      int cnt = 0;
      double neg;
      if (qk < 8) {
        double res = 0.0;
        for (int o = 0; o < qk; ++o) {
          const double e = reproj_sm(tob[o], models, X);
          if (e < a.thr) { ++cnt; res += e; }
        }
        neg = -res;
      } else {
        for (int o = 0; o < qk; ++o) cnt += reproj_sm(tob[o], models, X) < a.thr;
        NpSum acc(cnt);
        for (int o = 0; o < qk; ++o) {
          const double e = reproj_sm(tob[o], models, X);
          if (e < a.thr) acc.add(e);
        }
        neg = -acc.value();
      }
      if (cnt >= 2) { bcnt = cnt; bneg = neg; bidx = pi; bX = X; }
    }
  }
  // segmented arg-max over each track's lane range: (count, -sum)
  // lexicographic, lowest pair index on ties; the range's first lane ends
  // with its track's winner
#pragma unroll
  for (int sh = 16; sh > 0; sh >>= 1) {
    const int oc = __shfl_down_sync(0xffffffffu, bcnt, sh);
    const double on = __shfl_down_sync(0xffffffffu, bneg, sh);
    const int oi = __shfl_down_sync(0xffffffffu, bidx, sh);
    const bool same = hq >= 0 && lane + sh < he;
    const bool take = same && (oc > bcnt || (oc == bcnt && (on > bneg || (on == bneg && oi < bidx))));
    if (take) { bcnt = oc; bneg = on; bidx = oi; }
  }
  // per observation lane: its track, that track's winner
  int oq = -1;
#pragma unroll
  for (int q = 0; q < kPack; ++q)
    if (lane >= off[q] && lane < off[q + 1]) oq = q;
  int ohs = 0;
  bool oact = false;
#pragma unroll
  for (int q = 0; q < kPack; ++q)
    if (q == oq) { ohs = hoff[q]; oact = act[q]; }
  const int wcnt = __shfl_sync(0xffffffffu, bcnt, ohs & 31);
  const int widx = __shfl_sync(0xffffffffu, bidx, ohs & 31);
  const int wl = (ohs + (wcnt >= 2 ? widx : 0)) & 31;
  const Vec3 Xb = v3(__shfl_sync(0xffffffffu, bX.x, wl), __shfl_sync(0xffffffffu, bX.y, wl),
                     __shfl_sync(0xffffffffu, bX.z, wl));
  const bool obs_in = oq >= 0 && oact && wcnt >= 2;
  const unsigned selall = __ballot_sync(0xffffffffu, obs_in && reproj_sm(ob[obs_in ? lane : 0], models, Xb) < a.thr);
  // refinement on each track's inliers, on its range's first lane
  int st = SFM_TRI_FAILED;
  Vec3 X = v3(NAN, NAN, NAN);
  const bool head = hq >= 0 && lane == hs;
  if (head && bcnt >= 2) {
    const unsigned sel = (selall >> qo) & ((qk >= 32) ? 0xffffffffu : ((1u << qk) - 1u));
    st = tri_solve_sm(ob + qo, sel, models, a.method, a.min_angle, a.method == SFM_TRI_DLT, X);
  }
  // the track's refined position to its observation lanes
  const int hl = ohs & 31;
  const int rst = __shfl_sync(0xffffffffu, st, hl);
  const Vec3 Xr = v3(__shfl_sync(0xffffffffu, X.x, hl), __shfl_sync(0xffffffffu, X.y, hl),
                     __shfl_sync(0xffffffffu, X.z, hl));
  const bool refined = obs_in && rst == SFM_TRI_OK;
  const unsigned inlall = __ballot_sync(0xffffffffu, refined && reproj_sm(ob[refined ? lane : 0], models, Xr) < a.thr);
  // per track: status from its inlier count, mask bits, position
#pragma unroll
  for (int q = 0; q < kPack; ++q) {
    if (q >= nt) break;
    const int64_t t = t0 + q;
    const unsigned bits = (inlall >> off[q]) & ((kk[q] >= 32) ? 0xffffffffu : ((1u << kk[q]) - 1u));
    if (!act[q]) {
      if (lane < kk[q]) a.mask[base + off[q] + lane] = 0;
      if (lane == 0) {
        a.status[t] = SFM_TRI_SKIPPED;
        a.X[t * 3] = a.X[t * 3 + 1] = a.X[t * 3 + 2] = NAN;
      }
      continue;
    }
    const int hl_q = hoff[q] & 31;
    const int rq = __shfl_sync(0xffffffffu, st, hl_q);
    const int cq = __shfl_sync(0xffffffffu, bcnt, hl_q);
    const Vec3 Xq = v3(__shfl_sync(0xffffffffu, X.x, hl_q), __shfl_sync(0xffffffffu, X.y, hl_q),
                       __shfl_sync(0xffffffffu, X.z, hl_q));
    const bool ok = cq >= 2 && rq == SFM_TRI_OK && __popc(bits) >= 2;
    const unsigned mk = ok ? bits : 0u;
    if (lane < kk[q]) a.mask[base + off[q] + lane] = (mk >> lane) & 1u;
    if (lane == 0) {
      a.status[t] = (int8_t)(ok ? SFM_TRI_OK : SFM_TRI_FAILED);
      a.X[t * 3] = ok ? Xq.x : NAN; a.X[t * 3 + 1] = ok ? Xq.y : NAN; a.X[t * 3 + 2] = ok ? Xq.z : NAN;
    }
  }
}

#ifndef SFM_RANSAC_PACK
#define SFM_RANSAC_PACK 1
#endif
// Packed warps when the mean track is short enough that three tracks' pair
// hypotheses usually fit 32 lanes (mean k <= 5.5); otherwise most packed
// warps would fall back to three tracks in series, which measured slower
// than one track per warp (configs[1], k ~ 9: 47.8 vs 38.8 ms; configs[3],
// k ~ 5: 191 vs 395 ms packed).
void launch_ransac(const TrackArgs& a, int64_t n_obs, cudaStream_t s) {
  bool packed = SFM_RANSAC_PACK && 2 * n_obs <= 11 * a.T;
  if (const char* e = std::getenv("SFM_RANSAC_PACKED")) packed = std::atoi(e) != 0;  // tests: force either kernel
  if (packed) {
    const int64_t warps = (a.T + kPack - 1) / kPack;
    k_ransac_packed<<<grid_for(warps * 32, kRansacWarps * 32), kRansacWarps * 32, 0, s>>>(a);
  } else {
    k_ransac<<<grid_for(a.T * 32, kRansacWarps * 32), kRansacWarps * 32, 0, s>>>(a);
  }
  SFM_CHECK_LAUNCH();
}

__global__ void k_direct(TrackArgs a) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.T) return;
  if (a.active && !a.active[t]) { a.status[t] = SFM_TRI_SKIPPED; return; }
  Sel s{a.ptr[t], a.ptr[t + 1], -1, -1, nullptr};
  Vec3 X = v3(NAN, NAN, NAN);
  int st = tri_solve(a.d, s, a.method, a.min_angle, a.method == SFM_TRI_DLT, X);
  if (st != SFM_TRI_OK) X = v3(NAN, NAN, NAN);
  a.status[t] = (int8_t)st;
  a.X[t * 3] = X.x; a.X[t * 3 + 1] = X.y; a.X[t * 3 + 2] = X.z;
}

__global__ void k_gate(int64_t T, const int64_t* ptr, TriData d, const double* P, double thr, uint8_t* mask,
                       int* inliers, unsigned long long* removed) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long rm = 0;
  if (t < T) {
    Vec3 X = v3(P[t * 3], P[t * 3 + 1], P[t * 3 + 2]);
    int cnt = 0;
    for (int64_t o = ptr[t]; o < ptr[t + 1]; ++o) {
      if (!mask[o]) continue;
      if (reproj_err(d, o, X) > thr) { mask[o] = 0; ++rm; }
      else ++cnt;
    }
    inliers[t] = cnt;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) rm += __shfl_down_sync(0xffffffffu, rm, o);
  if ((threadIdx.x & 31) == 0 && rm) atomicAdd(removed, rm);  // integer: order-free
}

__global__ void k_errs(int64_t T, const int64_t* ptr, TriData d, const double* P, double* err) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  Vec3 X = v3(P[t * 3], P[t * 3 + 1], P[t * 3 + 2]);
  for (int64_t o = ptr[t]; o < ptr[t + 1]; ++o) err[o] = reproj_err(d, o, X);
}

// Device copies of a track set.
struct TrackDev {
  DevBuf<sfm_camera_model> models;
  DevBuf<int> fm, of, st;
  DevBuf<double> q, t, Rt, uv, ray;
  DevBuf<int64_t> ptr;
  DevBuf<uint8_t> active;
  TriData d{};
  void load(const sfm_tracks& tr, cudaStream_t s, Profiler* prof, bool rays) {
    SFM_REQUIRE(tr.n_tracks >= 0 && tr.n_obs >= 0 && tr.n_frames >= 0, "negative sizes");
    models.upload(tr.models, tr.n_models, s);
    fm.upload(tr.frame_model, tr.n_frames, s);
    q.upload(tr.cam_q, (size_t)tr.n_frames * 4, s);
    t.upload(tr.cam_t, (size_t)tr.n_frames * 3, s);
    Rt.resize((size_t)tr.n_frames * 12);
    if (tr.n_frames) {
      ProfScope ps(*prof, "tri_rt", 0.0, s);
      k_rt<<<grid_for(tr.n_frames, 128), 128, 0, s>>>(tr.n_frames, q.get(), t.get(), Rt.get());
    }
    ptr.upload(tr.track_ptr, tr.n_tracks + 1, s);
    of.upload(tr.obs_frame, tr.n_obs, s);
    uv.upload(tr.obs_uv, (size_t)tr.n_obs * 2, s);
    if (tr.active) active.upload(tr.active, tr.n_tracks, s);
    d.of = of.get(); d.uv = uv.get(); d.Rt = Rt.get(); d.fm = fm.get(); d.models = models.get();
    if (rays) {
      ray.resize((size_t)tr.n_obs * 3);
      st.resize(tr.n_obs);
      d.ray = ray.get();
      d.ray_st = st.get();
      if (tr.n_obs) {
        ProfScope ps(*prof, "tri_rays", 48.0 * tr.n_obs, s);
        k_rays<<<grid_for(tr.n_obs, 128), 128, 0, s>>>(tr.n_obs, d, ray.get(), st.get());
      }
    }
  }
};

void validate(const sfm_tracks& tr) {
  for (int f = 0; f < tr.n_frames; ++f)
    SFM_REQUIRE(tr.frame_model[f] >= 0 && tr.frame_model[f] < tr.n_models, "frame_model out of range");
  SFM_REQUIRE(tr.track_ptr[0] == 0 && tr.track_ptr[tr.n_tracks] == tr.n_obs, "track_ptr must span obs");
  for (int64_t i = 0; i < tr.n_tracks; ++i)
    SFM_REQUIRE(tr.track_ptr[i + 1] >= tr.track_ptr[i], "track_ptr must be non-decreasing");
  for (int64_t o = 0; o < tr.n_obs; ++o)
    SFM_REQUIRE(tr.obs_frame[o] >= 0 && tr.obs_frame[o] < tr.n_frames, "obs_frame out of range");
}

}  // namespace

void tri_ransac(cudaStream_t s, Profiler* prof, const sfm_tracks& tr, double thr, double min_angle, int method,
                double* out_X, uint8_t* out_mask, int8_t* out_status) {
  validate(tr);
  TrackDev dev;
  dev.load(tr, s, prof, true);
  DevBuf<double> X;
  DevBuf<uint8_t> mask;
  DevBuf<int8_t> st;
  X.resize((size_t)tr.n_tracks * 3);
  mask.resize(tr.n_obs);
  st.resize(tr.n_tracks);
  TrackArgs a{};
  a.T = tr.n_tracks; a.ptr = dev.ptr.get(); a.active = tr.active ? dev.active.get() : nullptr; a.d = dev.d;
  a.thr = thr; a.min_angle = min_angle; a.method = method; a.X = X.get(); a.mask = mask.get(); a.status = st.get();
  if (tr.n_tracks) {
    ProfScope ps(*prof, "tri_ransac", 24.0 * tr.n_obs + 24.0 * tr.n_tracks + tr.n_obs, s);
    launch_ransac(a, tr.n_obs, s);
  }
  X.download(out_X, (size_t)tr.n_tracks * 3, s);
  mask.download(out_mask, tr.n_obs, s);
  st.download(out_status, tr.n_tracks, s);
  SFM_CUDA(cudaStreamSynchronize(s));
}

void tri_direct(cudaStream_t s, Profiler* prof, const sfm_tracks& tr, double min_angle, int method, double* out_X,
                int8_t* out_status) {
  validate(tr);
  TrackDev dev;
  dev.load(tr, s, prof, true);
  DevBuf<double> X;
  DevBuf<int8_t> st;
  X.resize((size_t)tr.n_tracks * 3);
  st.resize(tr.n_tracks);
  TrackArgs a{};
  a.T = tr.n_tracks; a.ptr = dev.ptr.get(); a.active = tr.active ? dev.active.get() : nullptr; a.d = dev.d;
  a.min_angle = min_angle; a.method = method; a.X = X.get(); a.status = st.get();
  if (tr.n_tracks) {
    ProfScope ps(*prof, "tri_direct", 0.0, s);
    k_direct<<<grid_for(tr.n_tracks, 128), 128, 0, s>>>(a);
  }
  X.download(out_X, (size_t)tr.n_tracks * 3, s);
  st.download(out_status, tr.n_tracks, s);
  SFM_CUDA(cudaStreamSynchronize(s));
}

void tri_gate(cudaStream_t s, Profiler* prof, const sfm_tracks& tr, const double* points, double thr,
              uint8_t* mask_inout, int32_t* out_inliers, int64_t* out_removed) {
  validate(tr);
  TrackDev dev;
  dev.load(tr, s, prof, false);
  DevBuf<double> P;
  DevBuf<uint8_t> mask;
  DevBuf<int> inl;
  DevBuf<unsigned long long> rm;
  P.upload(points, (size_t)tr.n_tracks * 3, s);
  mask.upload(mask_inout, tr.n_obs, s);
  inl.resize(tr.n_tracks);
  rm.resize(1);
  rm.zero(s);
  if (tr.n_tracks) {
    ProfScope ps(*prof, "gate", 24.0 * tr.n_obs + 24.0 * tr.n_tracks + 2.0 * tr.n_obs, s);
    k_gate<<<grid_for(tr.n_tracks, 128), 128, 0, s>>>(tr.n_tracks, dev.ptr.get(), dev.d, P.get(), thr, mask.get(),
                                                       inl.get(), rm.get());
  }
  unsigned long long h = 0;
  mask.download(mask_inout, tr.n_obs, s);
  if (out_inliers) inl.download(out_inliers, tr.n_tracks, s);
  rm.download(&h, 1, s);
  SFM_CUDA(cudaStreamSynchronize(s));
  if (out_removed) *out_removed = (int64_t)h;
}

namespace {
TriData tri_data(const TriDeviceTracks& tr) {
  TriData d{};
  d.of = tr.obs_frame; d.uv = tr.obs_uv; d.ray = tr.ray; d.ray_st = tr.ray_st; d.Rt = tr.Rt;
  d.fm = tr.frame_model; d.models = tr.models;
  return d;
}
}  // namespace

void tri_rt_device(cudaStream_t s, int F, const double* q, const double* t, double* Rt) {
  if (F) k_rt<<<grid_for(F, 128), 128, 0, s>>>(F, q, t, Rt);
  SFM_CHECK_LAUNCH();
}

void tri_rays_device(cudaStream_t s, Profiler* prof, const TriDeviceTracks& tr, double* ray, int* ray_st) {
  if (!tr.n_obs) return;
  ProfScope ps(*prof, "tri_rays", 48.0 * tr.n_obs, s);
  k_rays<<<grid_for(tr.n_obs, 128), 128, 0, s>>>(tr.n_obs, tri_data(tr), ray, ray_st);
}

void tri_ransac_device(cudaStream_t s, Profiler* prof, const TriDeviceTracks& tr, const uint8_t* active,
                       double thr, double min_angle, int method, double* X, uint8_t* mask, int8_t* status) {
  if (!tr.n_tracks) return;
  TrackArgs a{};
  a.T = tr.n_tracks; a.ptr = tr.ptr; a.active = active; a.d = tri_data(tr);
  a.thr = thr; a.min_angle = min_angle; a.method = method; a.X = X; a.mask = mask; a.status = status;
  ProfScope ps(*prof, "tri_ransac", 24.0 * tr.n_obs + 24.0 * tr.n_tracks + tr.n_obs, s);
  launch_ransac(a, tr.n_obs, s);
}

void tri_gate_device(cudaStream_t s, Profiler* prof, const TriDeviceTracks& tr, const double* P, double thr,
                     uint8_t* mask, int* inliers, unsigned long long* removed) {
  if (!tr.n_tracks) return;
  ProfScope ps(*prof, "gate", 24.0 * tr.n_obs + 24.0 * tr.n_tracks + 2.0 * tr.n_obs, s);
  k_gate<<<grid_for(tr.n_tracks, 128), 128, 0, s>>>(tr.n_tracks, tr.ptr, tri_data(tr), P, thr, mask, inliers,
                                                     removed);
}

void tri_reproj_errors(cudaStream_t s, Profiler* prof, const sfm_tracks& tr, const double* points,
                       double* out_err) {
  validate(tr);
  TrackDev dev;
  dev.load(tr, s, prof, false);
  DevBuf<double> P, err;
  P.upload(points, (size_t)tr.n_tracks * 3, s);
  err.resize(tr.n_obs);
  if (tr.n_tracks) {
    ProfScope ps(*prof, "reproj_errors", 0.0, s);
    k_errs<<<grid_for(tr.n_tracks, 128), 128, 0, s>>>(tr.n_tracks, dev.ptr.get(), dev.d, P.get(), err.get());
  }
  err.download(out_err, tr.n_obs, s);
  SFM_CUDA(cudaStreamSynchronize(s));
}

}  // namespace sfm
