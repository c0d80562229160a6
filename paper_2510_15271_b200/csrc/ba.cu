// ba.cu -- sm_100a kernels and the host LM driver for bundle adjustment.
//
// Reference path being replaced (all fp64):
//   solver.py:194-257  solve(): LM loop, Marquardt damping, accept/reject
//   solver.py:164-191  _assemble(): sqrt(rho') weighted residuals/Jacobians
//   solver.py:132-151  evaluate()/_cost_only(): sum rho(|r|^2), no 1/2
//   solver.py:68-71    retraction exp(delta)*T for poses, X+delta for points
//   mapping.py:390-527 bundle_adjust(): residual set and write-back
//   mapping.py:359-368 absolute prior residual, posegraph.py:195-206 edges
//
// Device design:
//   * observations stay point-major (the reference residual order); every
//     per-point quantity (V_i, g_i, V*_i^-1, delta_p, trial cost) is a
//     thread-per-point loop over the point's contiguous observations;
//   * every camera-indexed sum (U_j, g_c, S blocks, b_S) is a fixed-order
//     reduction over a pair list sorted by S block then point, one warp per
//     block: no floating-point atomics anywhere, so results are
//     bit-reproducible run to run;
//   * Jacobians are recomputed from the 24-byte observation record instead
//     of being stored (HBM traffic is the bound, fp64 FMAs are cheap);
//   * the reduced camera system is solved by a single-CTA dense Cholesky when
//     6*free <= kDenseMax, else by a persistent cooperative block-Jacobi PCG.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <future>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "ba.cuh"
#include "pcg.cuh"
#include "sfm_math.cuh"

namespace cg = cooperative_groups;

namespace sfm {

// Arguments of the per-S-block kernels (k_blocks).
struct BlkArgs {
  int n;                       // warps of work
  const int* work;             // MODE 1: upper-block ids, heaviest first
  int nf;
  int rank;
  double lam;
  const unsigned long long* ub_key;
  const int* ub_pb;
  const int* ub_edge;
  const int* pos_up;
  const int* pos_lo;
  const int* diag_ub;
  const int64_t* pb_pair_ptr;
  const unsigned long long* pairs;
  const int* op;
  const int* of;
  const double* uv;
  const int* free_frame;
  const int* frame_model;
  const sfm_camera_model* models;
  const double* Rt;
  const double4* geo;
  const double* pv;            // [P*12] packed V*^-1 (6) | e (3) | pad
  const int* pair_pt;          // [n_pairs] point of each pair
  const int64_t* cm_ptr;       // [nf+1] camera-major observation ranges
  const int* cm_pt;            // camera-major point ids
  const double* cm_uv;         // camera-major pixels
  const double4* geo_cm;       // camera-major linearisation records
  const int* diag_pos;         // [nf] BSR slot of the diagonal blocks
  const int4* offrec;          // [2*n] off-diagonal work: {frame lo, frame hi, model lo, model hi},
                               //   {pos_up, pos_lo, edge, 0}
  const longlong2* offk;       // [n] pair range of each off-diagonal block
  const double* U;
  const double* Dc;
  const double* gc;
  const double* edge_H;
  double* S;
  double* b;
  double* Uout;
  double* gout;
  BAScalars* sc;
  const BAScalars* pre;        // MODE 1: flags of a point prep done at linearisation (or null)
};

namespace {

// PcgCollective over the solver's Comm: the row-partitioned PCG's coarse
// operator sum and its single launch across ranks sharing a device.
class CommPcgCollective final : public PcgCollective {
 public:
  explicit CommPcgCollective(Comm* c) : c_(c) {}
  int rank() const override { return c_->rank; }
  int world() const override { return c_->world; }
  void sum(double* d, size_t n, cudaStream_t s) override { c_->sum(d, n, s); }
  void launch_all(const PcgRankView& mine, cudaStream_t s,
                  const std::function<void(const PcgRankView*)>& launch) override {
    SFM_REQUIRE(c_->emu != nullptr, "a single PCG launch needs its ranks on one device");
    c_->emu->run_root(c_->rank, &mine, s, [&](const void* const* all) {
      std::vector<PcgRankView> v((size_t)c_->world);
      for (int r = 0; r < c_->world; ++r) v[r] = *static_cast<const PcgRankView*>(all[r]);
      launch(v.data());
    });
  }
  bool separate_launches() const override { return c_->emu == nullptr || c_->pcg_partition == 2; }
  void launch_each(const PcgRankView& mine, cudaStream_t s, const std::function<void()>& root_prep,
                   const std::function<void(const PcgRankView*)>& launch) override {
    SFM_REQUIRE(c_->host != nullptr, "per-rank PCG launches need the ranks in one process");
    c_->host->run_each(c_->rank, &mine, s, root_prep, [&](const void* const* all) {
      std::vector<PcgRankView> v((size_t)c_->world);
      for (int r = 0; r < c_->world; ++r) v[r] = *static_cast<const PcgRankView*>(all[r]);
      launch(v.data());
    });
  }

 private:
  Comm* c_;
};

constexpr int kDenseMax = 210;    // packed lower triangle of 6*nf fits in smem
constexpr int kBlock = 128;

// ---------------------------------------------------------------------------
// small helpers
// ---------------------------------------------------------------------------

// 256-bit read-only load (LDG.E.ENL2.256 on sm_100a): one L1 wavefront per
// 32-byte record instead of four 64-bit loads.  p must be 32-byte aligned and
// not written during the kernel.
__device__ __forceinline__ double4 ldg256(const void* p) {
  double4 v;
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}

// A camera's 6-vector (48 B, 16-byte aligned) as three 128-bit loads: a
// gather across the warp costs one request per load instruction, not six.
__device__ __forceinline__ void ldg_vec6(const double* p, double d[6]) {
  const double2* q = reinterpret_cast<const double2*>(p);
  const double2 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
  d[0] = a.x; d[1] = a.y; d[2] = b.x; d[3] = b.y; d[4] = c.x; d[5] = c.y;
}

// Camera record R (row-major) | t: 96 bytes = three 256-bit loads.
__device__ __forceinline__ void load_cam256(const double* __restrict__ Rt, int f, Mat3& R, Vec3& t) {
  const double* p = Rt + (int64_t)f * 12;
  const double4 a = ldg256(p), b = ldg256(p + 4), c = ldg256(p + 8);
  R.m[0] = a.x; R.m[1] = a.y; R.m[2] = a.z; R.m[3] = a.w;
  R.m[4] = b.x; R.m[5] = b.y; R.m[6] = b.z; R.m[7] = b.w;
  R.m[8] = c.x; t = v3(c.y, c.z, c.w);
}

// Compact camera record q | t | 0 (64 B = two 256-bit loads) -> R, t.
#ifndef SFM_PT_QCAM
#define SFM_PT_QCAM 1   // point passes read the 64 B record (1) or the 96 B R | t (0)
#endif
__device__ __forceinline__ void load_cam_q(const double* __restrict__ Rt, const double* __restrict__ qt, int f,
                                           Mat3& R, Vec3& t) {
  if (SFM_PT_QCAM) {
    const double4 a = ldg256(qt + (int64_t)f * 8), b = ldg256(qt + (int64_t)f * 8 + 4);
    R = quat_to_matrix(Quat{a.x, a.y, a.z, a.w});
    t = v3(b.x, b.y, b.z);
  } else {
    load_cam256(Rt, f, R, t);
  }
}

// Camera models staged in shared memory when the table is small (the usual
// case is one model for the whole map).
constexpr int kSmemModels = 8;
__device__ __forceinline__ const sfm_camera_model* stage_models(const sfm_camera_model* g, int n,
                                                                 sfm_camera_model* sm) {
  if (n > kSmemModels) return g;
  for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = g[i];
  __syncthreads();
  return sm;
}

__device__ __forceinline__ void load_cam(const double* __restrict__ Rt, int f, Mat3& R, Vec3& t) {
  const double* p = Rt + (int64_t)f * 12;
#pragma unroll
  for (int i = 0; i < 9; ++i) R.m[i] = __ldg(p + i);
  t = v3(__ldg(p + 9), __ldg(p + 10), __ldg(p + 11));
}

__device__ __forceinline__ Vec3 load_X(const double* __restrict__ X, int64_t i) {
  return v3(X[i * 3 + 0], X[i * 3 + 1], X[i * 3 + 2]);
}

__device__ __forceinline__ Pose load_pose(const double* q, const double* t, const double* Rt, int f) {
  Pose p;
  p.q = Quat{q[f * 4 + 0], q[f * 4 + 1], q[f * 4 + 2], q[f * 4 + 3]};
  p.t = v3(t[f * 3 + 0], t[f * 3 + 1], t[f * 3 + 2]);
#pragma unroll
  for (int i = 0; i < 9; ++i) p.R.m[i] = Rt[f * 12 + i];
  return p;
}

// Per-observation linearisation record g = (x, y, 1/Z, w) with (x, y) the
// normalised image point and w = sqrt(rho'(s)), written once per
// linearisation by k_point_lin.  Every later evaluation of the weighted
// Jacobians at that linearisation point rebuilds them from g and the camera
// (cameras.py:137-148, :169-179 regrouped): no projection, no division,
// no sqrt -- and only 32 bytes per observation instead of uv + point.
//   J~c = w [A N, (1/Z) A [[1,0,-x],[0,1,-y]]],  J~p = (right half) R
//   N = [[-xy, 1+x^2, -y], [-(1+y^2), xy, x]],   A = diag(fx,fy) J_dist(x,y)
__device__ __forceinline__ void geo_jacobians(const sfm_camera_model& cm, const Mat3& R, const double4 g,
                                              double Jc[12], double Jp[6]) {
  const double x = g.x, y = g.y, iz = g.z, w = g.w;
  double A00, A01, A10, A11;
  if (cm.kind == SFM_CAM_PINHOLE) {
    A00 = cm.fx * w; A01 = 0.0; A10 = 0.0; A11 = cm.fy * w;
  } else {
    double Jd[4];
    distort_jacobian(cm, x, y, Jd);
    A00 = cm.fx * Jd[0] * w; A01 = cm.fx * Jd[1] * w;
    A10 = cm.fy * Jd[2] * w; A11 = cm.fy * Jd[3] * w;
  }
  const double xy = x * y;
  const double n00 = -xy, n01 = 1.0 + x * x, n02 = -y;
  const double n10 = -(1.0 + y * y), n11 = xy, n12 = x;
  Jc[0] = A00 * n00 + A01 * n10; Jc[1] = A00 * n01 + A01 * n11; Jc[2] = A00 * n02 + A01 * n12;
  Jc[6] = A10 * n00 + A11 * n10; Jc[7] = A10 * n01 + A11 * n11; Jc[8] = A10 * n02 + A11 * n12;
  const double K00 = iz * A00, K01 = iz * A01, K02 = -(K00 * x + K01 * y);
  const double K10 = iz * A10, K11 = iz * A11, K12 = -(K10 * x + K11 * y);
  Jc[3] = K00; Jc[4] = K01; Jc[5] = K02;
  Jc[9] = K10; Jc[10] = K11; Jc[11] = K12;
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    Jp[j] = K00 * R.m[j] + K01 * R.m[3 + j] + K02 * R.m[6 + j];
    Jp[3 + j] = K10 * R.m[j] + K11 * R.m[3 + j] + K12 * R.m[6 + j];
  }
}

// Deterministic block sum (fixed shuffle tree + fixed smem order).
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* smem) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) smem[warp] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) r += smem[w];
  }
  return r;  // valid in thread 0
}


__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long w = __shfl_down_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}

// ---------------------------------------------------------------------------
// setup kernels
// ---------------------------------------------------------------------------

// Camera records of a state: Rt = R (row-major) | t, 96 B, and the compact
// qt = q | t | 0, 64 B (two 256-bit loads), from which the per-observation
// point passes rebuild R (quat_to_matrix, the same arithmetic that made R).
__global__ void k_frames_rt(int F, const double* __restrict__ q, const double* __restrict__ t,
                            double* __restrict__ Rt, double* __restrict__ qt) {
  int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  Mat3 R = quat_to_matrix(Quat{q[f * 4], q[f * 4 + 1], q[f * 4 + 2], q[f * 4 + 3]});
#pragma unroll
  for (int i = 0; i < 9; ++i) Rt[f * 12 + i] = R.m[i];
  Rt[f * 12 + 9] = t[f * 3];
  Rt[f * 12 + 10] = t[f * 3 + 1];
  Rt[f * 12 + 11] = t[f * 3 + 2];
  if (qt) {
#pragma unroll
    for (int i = 0; i < 4; ++i) qt[f * 8 + i] = q[f * 4 + i];
#pragma unroll
    for (int i = 0; i < 3; ++i) qt[f * 8 + 4 + i] = t[f * 3 + i];
    qt[f * 8 + 7] = 0.0;
  }
}

// Validates the layout contract: frames in range, points in range and
// non-decreasing (landmark-major order, mapping.py:452-475).
__global__ void k_validate_obs(int64_t N, int F, int64_t P, const int* __restrict__ of,
                               const int* __restrict__ op, int* __restrict__ bad) {
  int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= N) return;
  int f = of[o], p = op[o];
  bool b = f < 0 || f >= F || p < 0 || p >= P || (o > 0 && op[o - 1] > p);
  if (b) atomicOr(bad, 1);
}

__global__ void k_pt_ptr(int64_t P, int64_t N, const int* __restrict__ op, int64_t* __restrict__ ptr) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p > P) return;
  int64_t lo = 0, hi = N;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (op[mid] < p) lo = mid + 1; else hi = mid;
  }
  ptr[p] = lo;
}

// Pairs (self + off-diagonal) of free-camera observations per point.
__global__ void k_pair_count(int64_t P, const int64_t* __restrict__ ptr, const int* __restrict__ of,
                             const int* __restrict__ free_idx, int64_t* __restrict__ cnt) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p > P) return;
  if (p == P) { cnt[p] = 0; return; }
  int64_t k = 0;
  for (int64_t o = ptr[p]; o < ptr[p + 1]; ++o) k += free_idx[of[o]] >= 0;
  cnt[p] = k * (k + 1) / 2;
}

__global__ void k_pair_gen(int64_t P, int nf, const int64_t* __restrict__ ptr,
                           const int* __restrict__ of, const int* __restrict__ free_idx,
                           const int64_t* __restrict__ off, unsigned long long* __restrict__ keys,
                           unsigned long long* __restrict__ vals) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  int64_t w = off[p];
  const int64_t b0 = ptr[p], b1 = ptr[p + 1];
  for (int64_t a = b0; a < b1; ++a) {
    int ja = free_idx[of[a]];
    if (ja < 0) continue;
    for (int64_t b = a; b < b1; ++b) {
      int jb = free_idx[of[b]];
      if (jb < 0) continue;
      int64_t oa = a, ob = b;
      int lo = ja, hi = jb;
      if (jb < ja) { lo = jb; hi = ja; oa = b; ob = a; }
      keys[w] = (unsigned long long)lo * nf + hi;
      vals[w] = ((unsigned long long)oa << 32) | (unsigned long long)(uint32_t)ob;
      ++w;
    }
  }
}

__global__ void k_div_ceil(int n, const int* __restrict__ cnt, int64_t* __restrict__ out, int d) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > n) return;
  out[i] = (i == n) ? 0 : (cnt[i] + d - 1) / d;
}

__device__ __forceinline__ int64_t lower_bound_u64(const unsigned long long* a, int64_t n,
                                                   unsigned long long key) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void k_full_keys(int n_ub, int nf, const unsigned long long* __restrict__ ub,
                            unsigned long long* __restrict__ out) {
  int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n_ub) return;
  unsigned long long k = ub[u];
  unsigned long long lo = k / nf, hi = k % nf;
  out[2 * u] = k;
  out[2 * u + 1] = (lo == hi) ? ~0ull : hi * nf + lo;
}

__global__ void k_bsr_pattern(int nf, int n_full, const unsigned long long* __restrict__ full,
                              int* __restrict__ row_ptr, int* __restrict__ col) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_full) col[i] = (int)(full[i] % nf);
  if (i <= nf) row_ptr[i] = (int)lower_bound_u64(full, n_full, (unsigned long long)i * nf);
}

__global__ void k_ub_map(int n_ub, int nf, int n_full, const unsigned long long* __restrict__ ub,
                         const unsigned long long* __restrict__ full, int* __restrict__ pos_up,
                         int* __restrict__ pos_lo) {
  int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n_ub) return;
  unsigned long long k = ub[u], lo = k / nf, hi = k % nf;
  pos_up[u] = (int)lower_bound_u64(full, n_full, k);
  pos_lo[u] = (lo == hi) ? -1 : (int)lower_bound_u64(full, n_full, hi * nf + lo);
}

__global__ void k_scatter_pb(int n_pb, int n_ub, const unsigned long long* __restrict__ pb_key,
                             const unsigned long long* __restrict__ ub, int* __restrict__ ub_pb) {
  int pb = blockIdx.x * blockDim.x + threadIdx.x;
  if (pb >= n_pb) return;
  ub_pb[lower_bound_u64(ub, n_ub, pb_key[pb])] = pb;
}

__global__ void k_scatter_edges(int E, int nf, const int* __restrict__ ab, const int* __restrict__ free_idx,
                                int n_ub, const unsigned long long* __restrict__ ub,
                                int* __restrict__ ub_edge) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  int ja = free_idx[ab[2 * e]], jb = free_idx[ab[2 * e + 1]];
  if (ja < 0 || jb < 0 || ja == jb) return;
  unsigned long long lo = min(ja, jb), hi = max(ja, jb);
  ub_edge[lower_bound_u64(ub, n_ub, lo * nf + hi)] = e;
}

// lambda_c measurement meas = T_a T_b^-1 taken at BA entry (mapping.py:494)
// stored as meas^-1 (posegraph.py:197); lambda_a anchor T_init^-1
// (mapping.py:362).
__global__ void k_terms_init(int E, int A, const int* __restrict__ ab, const int* __restrict__ pf,
                             const double* __restrict__ q, const double* __restrict__ t,
                             const double* __restrict__ Rt, double* __restrict__ meas_inv,
                             double* __restrict__ init_inv) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < E) {
    Pose Ta = load_pose(q, t, Rt, ab[2 * i]), Tb = load_pose(q, t, Rt, ab[2 * i + 1]);
    Pose m = compose(Ta, pose_inverse(Tb));
    Pose mi = pose_inverse(m);
    double* o = meas_inv + i * 7;
    o[0] = mi.q.w; o[1] = mi.q.x; o[2] = mi.q.y; o[3] = mi.q.z;
    o[4] = mi.t.x; o[5] = mi.t.y; o[6] = mi.t.z;
  } else if (i < E + A) {
    int a = i - E;
    Pose T = load_pose(q, t, Rt, pf[a]);
    Pose ti = pose_inverse(T);
    double* o = init_inv + a * 7;
    o[0] = ti.q.w; o[1] = ti.q.x; o[2] = ti.q.y; o[3] = ti.q.z;
    o[4] = ti.t.x; o[5] = ti.t.y; o[6] = ti.t.z;
  }
}

__device__ __forceinline__ Pose pose7(const double* p) {
  Pose P;
  P.q = Quat{p[0], p[1], p[2], p[3]};
  P.t = v3(p[4], p[5], p[6]);
  P.R = quat_to_matrix(P.q);
  return P;
}

// posegraph.py:195-206 -- weighted edge residual and Jacobians.
__device__ void edge_eval(const double* meas_inv7, const Pose& Ta, const Pose& Tb, double w,
                          double r[6], double* Ja, double* Jb) {
  Pose mi = pose7(meas_inv7);
  Pose E = compose(compose(mi, Ta), pose_inverse(Tb));
  double rr[6];
  se3_log(E, rr);
#pragma unroll
  for (int i = 0; i < 6; ++i) r[i] = w * rr[i];
  if (Ja) {
    double Jl[36], Ad[36];
    se3_left_jacobian_inv(rr, Jl);
    se3_adjoint(mi, Ad);
    for (int i = 0; i < 6; ++i)
      for (int j = 0; j < 6; ++j) {
        double s = 0.0;
        for (int k = 0; k < 6; ++k) s += Jl[i * 6 + k] * Ad[k * 6 + j];
        Ja[i * 6 + j] = w * s;
      }
  }
  if (Jb) {
    double neg[6], Jr[36];
    for (int i = 0; i < 6; ++i) neg[i] = -rr[i];
    se3_left_jacobian_inv(neg, Jr);  // se3_right_jacobian_inv(r) (se3.py:266-267)
    for (int i = 0; i < 36; ++i) Jb[i] = -w * Jr[i];
  }
}

// mapping.py:359-368 -- weighted absolute prior.
__device__ void prior_eval(const double* init_inv7, const Pose& T, double w, double r[6], double* J) {
  Pose E = compose(T, pose7(init_inv7));
  double rr[6];
  se3_log(E, rr);
  for (int i = 0; i < 6; ++i) r[i] = w * rr[i];
  if (J) {
    double Jl[36];
    se3_left_jacobian_inv(rr, Jl);
    for (int i = 0; i < 36; ++i) J[i] = w * Jl[i];
  }
}

// ---------------------------------------------------------------------------
// cost evaluation (solver.py:132-151) and trial step (solver.py:220-235)
// ---------------------------------------------------------------------------

struct PointArgs {
  int64_t P;
  int lk;
  double lp;
  const int64_t* ptr;
  const int* of;
  const double* uv;
  const int* frame_model;
  const sfm_camera_model* models;
  int nmodels;
  const int* free_idx;
  const double* Rt;       // linearization state cameras (R | t)
  const double* X;        // linearization state points
  const double* Rt_eval;  // state whose cost is evaluated (R | t)
  const double* qt;       // linearization state cameras (q | t | 0), read by the point passes
  const double* qt_eval;  // evaluated state (q | t | 0)
  double* X_out;          // trial points (TRIAL) or unused
  const double* pv;       // packed V*^-1 | e per point
  double lam;              // k_point_lin: also prepare pv for this lambda (the first trial's)
  double* pv_out;          //   into pv_out (null: skip), flags into sc_pre
  BAScalars* sc_pre;
  const double* dc;
  const double4* geo;     // linearisation records (TRIAL) / output (LIN)
  const int* cm_pos;      // camera-major slot of each observation (-1: fixed)
  double4* geo_cm;        // camera-major copy of the records (LIN)
  int64_t obs_offset;
  double* part_cost;
  double* part_dp2;
  BAScalars* sc;
};

// TRIAL=false: cost of (Rt_eval, X).  TRIAL=true: delta_p back-substitution
// delta_p = -e - V*^-1 sum_j Jp^T Jc dc_j (Jacobians at the linearization
// state), X' = X + delta_p, then cost of (Rt_eval, X').
template <bool TRIAL>
__global__ void __launch_bounds__(kBlock) k_point_cost(PointArgs a) {
  __shared__ double red[kBlock / 32];
  __shared__ sfm_camera_model smod[kSmemModels];
  const sfm_camera_model* models = stage_models(a.models, a.nmodels, smod);
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double cost = 0.0, dp2 = 0.0;
  bool nonfinite = false;
  unsigned long long bad = ~0ull;
  if (p < a.P) {
    const int64_t b0 = a.ptr[p], b1 = a.ptr[p + 1];
    Vec3 X = load_X(a.X, p);
    if (TRIAL) {
      double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
      int f_nx = b0 < b1 ? a.of[b0] : 0;  // the next observation's frame, one iteration ahead
      for (int64_t o = b0; o < b1; ++o) {
        const int f = f_nx;
        if (o + 1 < b1) f_nx = a.of[o + 1];
        const int j = a.free_idx[f];
        if (j < 0) continue;
        Mat3 R; Vec3 t;
        load_cam_q(a.Rt, a.qt, f, R, t);
        const sfm_camera_model& cm = models[a.frame_model[f]];
        double Jc[12], Jp[6];
        geo_jacobians(cm, R, ldg256(a.geo + o), Jc, Jp);
        double d[6];
        ldg_vec6(a.dc + (int64_t)j * 6, d);
        double y0 = 0.0, y1 = 0.0;
#pragma unroll
        for (int k = 0; k < 6; ++k) { y0 += Jc[k] * d[k]; y1 += Jc[6 + k] * d[k]; }
        acc0 += Jp[0] * y0 + Jp[3] * y1;
        acc1 += Jp[1] * y0 + Jp[4] * y1;
        acc2 += Jp[2] * y0 + Jp[5] * y1;
      }
      // packed point record: V*^-1 (xx xy xz yy yz zz) | e | pad
      const double4 pa = ldg256(a.pv + p * 12), pb = ldg256(a.pv + p * 12 + 4);
      const double e0 = pb.z, e1 = pb.w, e2 = __ldg(a.pv + p * 12 + 8);
      double d0 = -e0 - (pa.x * acc0 + pa.y * acc1 + pa.z * acc2);
      double d1 = -e1 - (pa.y * acc0 + pa.w * acc1 + pb.x * acc2);
      double d2 = -e2 - (pa.z * acc0 + pb.x * acc1 + pb.y * acc2);
      if (!(isfinite(d0) && isfinite(d1) && isfinite(d2))) nonfinite = true;
      dp2 = d0 * d0 + d1 * d1 + d2 * d2;
      X = v3(X.x + d0, X.y + d1, X.z + d2);
      a.X_out[p * 3 + 0] = X.x;
      a.X_out[p * 3 + 1] = X.y;
      a.X_out[p * 3 + 2] = X.z;
    }
    if (!nonfinite) {
      int f_nx = b0 < b1 ? a.of[b0] : 0;
      for (int64_t o = b0; o < b1; ++o) {
        const int f = f_nx;
        if (o + 1 < b1) f_nx = a.of[o + 1];
        Mat3 R; Vec3 t;
        load_cam_q(a.Rt_eval, a.qt_eval, f, R, t);
        const sfm_camera_model& cm = models[a.frame_model[f]];
        Vec3 pc = add(mul(R, X), t);
        double u, v;
        if (project_point(cm, pc, u, v) != PROJ_OK) {
          bad = (unsigned long long)(a.obs_offset + o);
          break;  // first raising observation of this point (in order)
        }
        const double2 uv = reinterpret_cast<const double2*>(a.uv)[o];
        const double r0 = u - uv.x, r1 = v - uv.y;
        cost += loss_rho(a.lk, a.lp, r0 * r0 + r1 * r1);
      }
    }
  }
  if (nonfinite) atomicOr(&a.sc->nonfinite, 1);
  unsigned long long wb = bad;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long x = __shfl_down_sync(0xffffffffu, wb, o);
    wb = x < wb ? x : wb;
  }
  if ((threadIdx.x & 31) == 0 && wb != ~0ull) atomicMin(&a.sc->depth_obs, wb);
  double c = block_sum<kBlock>(cost, red);
  if (threadIdx.x == 0) a.part_cost[blockIdx.x] = c;
  if (TRIAL) {
    double d = block_sum<kBlock>(dp2, red);
    if (threadIdx.x == 0) a.part_dp2[blockIdx.x] = d;
  }
}

// Pose-term cost at a state (trivial loss on these terms, mapping.py:485-509).
__global__ void __launch_bounds__(kBlock) k_terms_cost(int E, int A, const int* __restrict__ ab,
                                                       const int* __restrict__ pf,
                                                       const double* __restrict__ meas_inv,
                                                       const double* __restrict__ init_inv,
                                                       double we, double wa, const double* q,
                                                       const double* t, const double* Rt,
                                                       double* __restrict__ part) {
  __shared__ double red[kBlock / 32];
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  double c = 0.0;
  double r[6];
  if (i < E) {
    Pose Ta = load_pose(q, t, Rt, ab[2 * i]), Tb = load_pose(q, t, Rt, ab[2 * i + 1]);
    edge_eval(meas_inv + i * 7, Ta, Tb, we, r, nullptr, nullptr);
    for (int k = 0; k < 6; ++k) c += r[k] * r[k];
  } else if (i < E + A) {
    int k0 = i - E;
    Pose T = load_pose(q, t, Rt, pf[k0]);
    prior_eval(init_inv + k0 * 7, T, wa, r, nullptr);
    for (int k = 0; k < 6; ++k) c += r[k] * r[k];
  }
  double s = block_sum<kBlock>(c, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// Sums the per-block partials in a fixed order into the scalars.
__global__ void k_finalize(const double* __restrict__ pa, int na, const double* __restrict__ pb, int nb,
                           const double* __restrict__ pc, int nc, const double* __restrict__ pd,
                           int nd, BAScalars* sc, int mode) {
  __shared__ double red[8];
  double a = 0.0, b = 0.0, c = 0.0;
  // eight partial loads in flight per thread, then the additions in the
  // same (ascending) order as a plain strided loop
  auto strided_sum = [](const double* __restrict__ p, int n) {
    double acc = 0.0;
    for (int i0 = threadIdx.x; i0 < n; i0 += 8 * blockDim.x) {
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int i = i0 + q * (int)blockDim.x;
        v[q] = i < n ? __ldg(p + i) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) acc += v[q];
    }
    return acc;
  };
  a = strided_sum(pa, na);
  c = strided_sum(pc, nc);
  double sa = block_sum<256>(a, red);
  double sc_ = block_sum<256>(c, red);
  if (mode == 1) {
    b = strided_sum(pb, nb);
  }
  double sb = block_sum<256>(b, red);
  double d = 0.0;
  if (mode == 1)
    d = strided_sum(pd, nd);
  double sd = block_sum<256>(d, red);
  if (threadIdx.x == 0) {
    sc->cost = sa + sc_;
    if (mode == 1) {
      sc->dp2 = sb;
      sc->dc2 = sd;
    }
  }
}

// ---------------------------------------------------------------------------
// linearization (solver.py:210-217 restricted to the Schur blocks)
// ---------------------------------------------------------------------------

// V* = V + lam max(diag V, 1e-12), V*^-1 (adjugate), e = V*^-1 g -> the
// packed point record; returns false when V* is not invertible / finite.
__device__ __forceinline__ bool point_prep_one(const double* v, const double* g, double lam, double* o) {
  double a = v[0] + lam * fmax(v[0], 1e-12);
  double b = v[1], c = v[2];
  double d = v[3] + lam * fmax(v[3], 1e-12);
  double ee = v[4];
  double f = v[5] + lam * fmax(v[5], 1e-12);
  double A = d * f - ee * ee, B = c * ee - b * f, C = b * ee - c * d;
  double D = a * f - c * c, Ee = b * c - a * ee, Fm = a * d - b * b;
  double det = a * A + b * B + c * C;
  double inv = 1.0 / det;
  const double i0 = A * inv, i1 = B * inv, i2 = C * inv, i3 = D * inv, i4 = Ee * inv, i5 = Fm * inv;
  const double e0 = i0 * g[0] + i1 * g[1] + i2 * g[2];
  const double e1 = i1 * g[0] + i3 * g[1] + i4 * g[2];
  const double e2 = i2 * g[0] + i4 * g[1] + i5 * g[2];
  reinterpret_cast<double2*>(o)[0] = make_double2(i0, i1);
  reinterpret_cast<double2*>(o)[1] = make_double2(i2, i3);
  reinterpret_cast<double2*>(o)[2] = make_double2(i4, i5);
  reinterpret_cast<double2*>(o)[3] = make_double2(e0, e1);
  reinterpret_cast<double2*>(o)[4] = make_double2(e2, 0.0);
  return det > 0.0 && isfinite(inv) && isfinite(e0) && isfinite(e1) && isfinite(e2);
}

// V_i = sum Jp^T Jp, g_i = sum Jp^T r over ALL observations of the point.
__global__ void __launch_bounds__(kBlock) k_point_lin(PointArgs a, double* __restrict__ V,
                                                      double* __restrict__ gp) {
  __shared__ sfm_camera_model smod[kSmemModels];
  const sfm_camera_model* models = stage_models(a.models, a.nmodels, smod);
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double gm = 0.0;
  if (p < a.P) {
    Vec3 X = load_X(a.X, p);
    double v[6] = {0, 0, 0, 0, 0, 0}, g[3] = {0, 0, 0};
    bool bad = false;
    for (int64_t o = a.ptr[p]; o < a.ptr[p + 1]; ++o) {
      const int f = a.of[o];
      Mat3 R; Vec3 t;
      load_cam_q(a.Rt, a.qt, f, R, t);
      const sfm_camera_model& cm = models[a.frame_model[f]];
      const double2 uv = reinterpret_cast<const double2*>(a.uv)[o];
      const Vec3 pc = add(mul(R, X), t);
      double u, vv;
      if (project_point(cm, pc, u, vv) != PROJ_OK) { bad = true; continue; }
      double r[2] = {u - uv.x, vv - uv.y};
      const double w = sqrt(loss_rho_prime(a.lk, a.lp, r[0] * r[0] + r[1] * r[1]));
      r[0] *= w;
      r[1] *= w;
      const double iz = 1.0 / pc.z;
      const double4 rec = make_double4(pc.x * iz, pc.y * iz, iz, w);
      const_cast<double4*>(a.geo)[o] = rec;
      const int cp = a.cm_pos[o];
      if (cp >= 0) a.geo_cm[cp] = rec;
      double Jc[12], Jp[6];
      geo_jacobians(cm, R, rec, Jc, Jp);
      v[0] += Jp[0] * Jp[0] + Jp[3] * Jp[3];
      v[1] += Jp[0] * Jp[1] + Jp[3] * Jp[4];
      v[2] += Jp[0] * Jp[2] + Jp[3] * Jp[5];
      v[3] += Jp[1] * Jp[1] + Jp[4] * Jp[4];
      v[4] += Jp[1] * Jp[2] + Jp[4] * Jp[5];
      v[5] += Jp[2] * Jp[2] + Jp[5] * Jp[5];
      g[0] += Jp[0] * r[0] + Jp[3] * r[1];
      g[1] += Jp[1] * r[0] + Jp[4] * r[1];
      g[2] += Jp[2] * r[0] + Jp[5] * r[1];
    }
    if (bad) atomicOr(&a.sc->nonfinite, 1);
#pragma unroll
    for (int k = 0; k < 6; ++k) V[p * 6 + k] = v[k];
#pragma unroll
    for (int k = 0; k < 3; ++k) gp[p * 3 + k] = g[k];
    // the first trial's damped point record, while V and g are in registers
    // (k_point_prep would re-read them); its flag goes to sc_pre, which the
    // trial's diagonal Schur kernel folds into the trial's scalars
    if (a.pv_out && !point_prep_one(v, g, a.lam, a.pv_out + p * 12)) atomicOr(&a.sc_pre->nonfinite, 1);
    gm = fmax(fabs(g[0]), fmax(fabs(g[1]), fabs(g[2])));
    if (isnan(g[0]) || isnan(g[1]) || isnan(g[2])) gm = __longlong_as_double(0x7ff8000000000000ll);
  }
  unsigned long long m = warp_max_u64((unsigned long long)__double_as_longlong(gm));
  if ((threadIdx.x & 31) == 0) atomicMax(&a.sc->gmax, m);
}


// fp64 tensor-core step D += A(8x4) B(4x8) (DMMA.8x8x4).  Fragments:
// a = A[lane/4][lane%4], b = B[lane%4][lane/4], d = D[lane/4][2(lane%4)+{0,1}].
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// One warp per off-diagonal S block (lo < hi), blocks in row-major order so
// consecutive warps share cameras and points (L2 reuse).  The block's pairs
// (observation a in camera lo, b in camera hi of the same point, sorted by
// point) are taken 32 at a time, one per lane.  Each pair's contribution is
// the rank-2 product -J~c_a^T (M J~c_b), M = J~p_a V*^-1 J~p_b^T (2x2), so
// the block is S_ab = A^T B with A = [J~c_a] and B = [-M J~c_b] stacked over
// pairs (K = 2 x pairs): lanes stage their 2x6 factors in shared memory and
// the warp contracts them on the fp64 tensor cores (two pairs per
// DMMA.8x8x4, fixed order, so the sum is bit-reproducible).  The lambda_c
// edge block is added on rank 0 and both BSR triangles written.
// One-warp CTAs, 20 per SM: measured 0.483 ms vs 0.496 with four-warp CTAs
// (5 per SM) and 0.590 with eight (same bits; a finer grain lets a finished
// block's slot refill without waiting for its CTA's other warps).
#ifndef SFM_OFF_WARPS
#define SFM_OFF_WARPS 1
#endif
constexpr int kOffWarps = SFM_OFF_WARPS;
constexpr int kOffLd = 13;  // padded row of the staged factors (bank spread)
constexpr int kOffRows = 32;
constexpr size_t kOffSmem = sizeof(double) * kOffWarps * 2 * kOffRows * kOffLd;

// One packed header per off-diagonal work item (structure build): the
// kernel's prologue is then one independent load instead of the
// work -> key -> frame -> pose / pair-range chain.
__global__ void k_off_records(int n, const int* __restrict__ work, const unsigned long long* __restrict__ ub_key,
                              int nf, const int* __restrict__ ub_pb, const int* __restrict__ ub_edge,
                              const int* __restrict__ pos_up, const int* __restrict__ pos_lo,
                              const int* __restrict__ free_frame, const int* __restrict__ frame_model,
                              const int64_t* __restrict__ pb_pair_ptr, int4* __restrict__ rec,
                              longlong2* __restrict__ kr) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= n) return;
  const int u = work[w];
  const unsigned long long key = ub_key[u];
  const int lo = (int)(key / nf), hi = (int)(key % nf);
  const int fa = free_frame[lo], fb = free_frame[hi];
  const int pb = ub_pb[u];
  rec[2 * w] = make_int4(fa, fb, frame_model[fa], frame_model[fb]);
  rec[2 * w + 1] = make_int4(pos_up[u], pos_lo[u], ub_edge[u], 0);
  kr[w] = pb >= 0 ? make_longlong2(pb_pair_ptr[pb], pb_pair_ptr[pb + 1]) : make_longlong2(0, 0);
}

#ifndef SFM_OFF_MINB
#define SFM_OFF_MINB 20
#endif
#ifndef SFM_CAM_MINB
#define SFM_CAM_MINB 5
#endif
__global__ void __launch_bounds__(kOffWarps * 32, SFM_OFF_MINB) k_offdiag_blocks(BlkArgs a) {
  extern __shared__ double offsm[];  // per warp: A | B staged factors [kOffRows x kOffLd] each

  __shared__ Mat3 Rsm[kOffWarps][2];
  __shared__ sfm_camera_model Csm[kOffWarps][2];
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* Aw = offsm + (size_t)warp * 2 * kOffRows * kOffLd;
  double* Bw = Aw + kOffRows * kOffLd;
  if (w >= a.n) return;
  const int4 hd = __ldg(a.offrec + 2 * w);
  const int4 out = __ldg(a.offrec + 2 * w + 1);
  const longlong2 kr = __ldg(a.offk + w);
  double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
  const int fr = lane >> 2;          // fragment row (A) / column (B)
  const int fk = lane & 3;           // fragment k: pair (fk >> 1), component (fk & 1)
  if (kr.y > kr.x) {
    // warp-uniform cameras staged in shared memory (keeps registers for
    // the per-pair factors)
    if (lane < 9) {
      Rsm[warp][0].m[lane] = __ldg(a.Rt + (int64_t)hd.x * 12 + lane);
      Rsm[warp][1].m[lane] = __ldg(a.Rt + (int64_t)hd.y * 12 + lane);
    }
    if (lane == 0) {
      Csm[warp][0] = a.models[hd.z];
      Csm[warp][1] = a.models[hd.w];
    }
    __syncwarp();
    const Mat3& Ra = Rsm[warp][0];
    const Mat3& Rb = Rsm[warp][1];
    const sfm_camera_model& ca = Csm[warp][0];
    const sfm_camera_model& cb = Csm[warp][1];
    const int64_t k0 = kr.x, k1 = kr.y;
    double* As = &Aw[lane * kOffLd];
    double* Bs = &Bw[lane * kOffLd];
    for (int64_t kb = k0; kb < k1; kb += 32) {
      const int64_t k = kb + lane;
      if (k < k1) {
        const unsigned long long pr = a.pairs[k];
        const int64_t oa = (int64_t)(pr >> 32), ob = (int64_t)(uint32_t)pr;
        const double* pv = a.pv + (int64_t)a.pair_pt[k] * 12;
        const double4 ga = ldg256(a.geo + oa), gb = ldg256(a.geo + ob);
        const double4 pva = ldg256(pv), pvb = ldg256(pv + 4);
        const double v0 = pva.x, v1 = pva.y, v2 = pva.z, v3_ = pva.w, v4 = pvb.x, v5 = pvb.y;
        double Jca[12], Jpa[6];
        geo_jacobians(ca, Ra, ga, Jca, Jpa);
#pragma unroll
        for (int i = 0; i < 12; ++i) As[i] = Jca[i];
        double Jcb[12], Jpb[6];
        geo_jacobians(cb, Rb, gb, Jcb, Jpb);
        const double P00 = v0 * Jpb[0] + v1 * Jpb[1] + v2 * Jpb[2];
        const double P01 = v1 * Jpb[0] + v3_ * Jpb[1] + v4 * Jpb[2];
        const double P02 = v2 * Jpb[0] + v4 * Jpb[1] + v5 * Jpb[2];
        const double P10 = v0 * Jpb[3] + v1 * Jpb[4] + v2 * Jpb[5];
        const double P11 = v1 * Jpb[3] + v3_ * Jpb[4] + v4 * Jpb[5];
        const double P12 = v2 * Jpb[3] + v4 * Jpb[4] + v5 * Jpb[5];
        const double m00 = Jpa[0] * P00 + Jpa[1] * P01 + Jpa[2] * P02;
        const double m01 = Jpa[0] * P10 + Jpa[1] * P11 + Jpa[2] * P12;
        const double m10 = Jpa[3] * P00 + Jpa[4] * P01 + Jpa[5] * P02;
        const double m11 = Jpa[3] * P10 + Jpa[4] * P11 + Jpa[5] * P12;
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          Bs[c] = -(m00 * Jcb[c] + m01 * Jcb[6 + c]);
          Bs[6 + c] = -(m10 * Jcb[c] + m11 * Jcb[6 + c]);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 12; ++i) { As[i] = 0.0; Bs[i] = 0.0; }
      }
      __syncwarp();
      const int nch = (int)((min((int64_t)32, k1 - kb) + 1) >> 1);
      const int slot = (fk & 1) * 6 + fr;
      for (int ch = 0; ch < nch; ch += 2) {
        const int p0 = 2 * ch + (fk >> 1);
        const double a0 = fr < 6 ? Aw[p0 * kOffLd + slot] : 0.0;
        const double b0 = fr < 6 ? Bw[p0 * kOffLd + slot] : 0.0;
        dmma_8x8x4(d0, d1, a0, b0);
        if (ch + 1 < nch) {
          const int p1 = p0 + 2;
          const double a1 = fr < 6 ? Aw[p1 * kOffLd + slot] : 0.0;
          const double b1 = fr < 6 ? Bw[p1 * kOffLd + slot] : 0.0;
          dmma_8x8x4(e0, e1, a1, b1);
        }
      }
      __syncwarp();
    }
  }
  d0 += e0;
  d1 += e1;
  const int c0 = 2 * fk;
  if (fr < 6 && c0 < 6) {
    if (a.rank == 0 && out.z >= 0) {
      const double* H = a.edge_H + (int64_t)out.z * 36;
      d0 += H[fr * 6 + c0];
      d1 += H[fr * 6 + c0 + 1];
    }
    double* up = a.S + (int64_t)out.x * 36;
    up[fr * 6 + c0] = d0;
    up[fr * 6 + c0 + 1] = d1;
    double* dn = a.S + (int64_t)out.y * 36;
    dn[c0 * 6 + fr] = d0;
    dn[(c0 + 1) * 6 + fr] = d1;
  }
}

// ---------------------------------------------------------------------------
// Register-accumulating form of the camera-block contraction.  k_cam_blocks
// below stages 28 doubles per observation in shared memory and reads them
// back as DMMA fragments: ncu puts its L1 data pipe at 85-95% of peak,
// 86% of it shared-memory wavefronts, so the staging -- not HBM and not the
// fp64 math -- bounds it.  k_cam_fma instead has each lane accumulate its
// observations' rank-2 terms in registers (54 fp64 FMA per observation)
// and combines the lanes once per camera with a fixed butterfly
// reduce-scatter, so every sum is still taken in one fixed order and the
// results stay bit-reproducible run to run.  Measured on config 3: the
// diagonal Schur pass 0.236 -> 0.116 ms, the U / g_c pass 0.129 -> 0.089 ms.
// (The same change to k_offdiag_blocks measured no gain, 0.495 -> 0.500 ms,
// also with cp.async double-buffered gathers (0.56 ms): that kernel waits on
// its per-block header -> pair -> gather chain, not on shared memory.)
// ---------------------------------------------------------------------------
#ifndef SFM_CAM_FMA
#define SFM_CAM_FMA 1   // camera blocks: register accumulation (1) or DMMA staging (0)
#endif

// One butterfly level over N values: lanes with bit MASK keep the upper
// half, the others the lower half, each adding its partner's copy.
template <int N, int MASK>
__device__ __forceinline__ void rs_level(double* v, int lane) {
  constexpr int H = (N + 1) / 2;
  const bool hi = (lane & MASK) != 0;
#pragma unroll
  for (int i = 0; i < H; ++i) {
    const double lo_v = v[i];
    const double hi_v = (H + i < N) ? v[H + i] : 0.0;
    const double send = hi ? lo_v : hi_v;
    v[i] = (hi ? hi_v : lo_v) + __shfl_xor_sync(0xffffffffu, send, MASK);
  }
}

// Warp reduce-scatter of N per-lane values: afterwards v[0..) of each lane
// hold warp totals, rs_entry<N>(lane, i) naming which entry slot i holds.
template <int N>
__device__ __forceinline__ void warp_reduce_scatter(double* v, int lane) {
  constexpr int N1 = (N + 1) / 2, N2 = (N1 + 1) / 2, N3 = (N2 + 1) / 2, N4 = (N3 + 1) / 2;
  rs_level<N, 16>(v, lane);
  rs_level<N1, 8>(v, lane);
  rs_level<N2, 4>(v, lane);
  rs_level<N3, 2>(v, lane);
  rs_level<N4, 1>(v, lane);
}

template <int N>
__device__ __forceinline__ int rs_entry(int lane, int i) {
  constexpr int N1 = (N + 1) / 2, N2 = (N1 + 1) / 2, N3 = (N2 + 1) / 2, N4 = (N3 + 1) / 2, N5 = (N4 + 1) / 2;
  int j = ((lane & 1) ? N5 : 0) + i;
  if (j >= N4) return -1;
  j += (lane & 2) ? N4 : 0;
  if (j >= N3) return -1;
  j += (lane & 4) ? N3 : 0;
  if (j >= N2) return -1;
  j += (lane & 8) ? N2 : 0;
  if (j >= N1) return -1;
  j += (lane & 16) ? N1 : 0;
  return j < N ? j : -1;
}

constexpr int kCamWarps = 4;
constexpr int kCamLd = 29;  // staged factors per observation: A (12) | B (16), padded

// One CTA per free camera j over its observations in camera-major order
// (contiguous linearisation records, point ids and pixels): the diagonal
// S block and the camera half of the normal equations.  Each observation
// contributes a rank-2 term A^T B with A = J~c (2x6) and
//   MODE 0: B = [J~c | r~ | 0]                U_j = sum J~c^T J~c, g_j = sum J~c^T r~
//   MODE 1: B = [-M J~c | J~p e | 0],  M = J~p V*^-1 J~p^T
//           S_jj = U*_j - sum J~c^T M J~c,  b_j = -g_j + sum J~c^T J~p e
// so the camera's [6 x 8] result is one long K = 2 x observations
// contraction: lanes stage their factors in shared memory, each warp runs
// DMMA.8x8x4 over its 32-observation batches (two observations per step)
// and the four warp results are added in warp order -- fixed order.
template <int MODE>
__global__ void __launch_bounds__(kCamWarps * 32, SFM_CAM_MINB) k_cam_blocks(BlkArgs a) {
  __shared__ double St[kCamWarps][32 * kCamLd];
  __shared__ double Wsum[kCamWarps][64];
  const int j = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (MODE == 1 && a.pre && j == 0 && threadIdx.x == 0 && a.pre->nonfinite) atomicOr(&a.sc->nonfinite, 1);
  const int f = a.free_frame[j];
  Mat3 R; Vec3 t;
  load_cam(a.Rt, f, R, t);
  const sfm_camera_model cm = a.models[a.frame_model[f]];
  const int64_t k0 = a.cm_ptr[j], k1 = a.cm_ptr[j + 1];
  double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
  double* As = &St[warp][lane * kCamLd];
  double* Bs = As + 12;
  const int fr = lane >> 2, fk = lane & 3;
  // one batch ahead: MODE 0 loads the next linearisation record, MODE 1 the
  // next point id (the packed point record load then does not wait on it)
  const int64_t kfirst = k0 + (int64_t)warp * 32 + lane;
  double4 g_nx = make_double4(0.0, 0.0, 0.0, 0.0);
  double2 uv_nx = make_double2(0.0, 0.0);
  int pt_nx = 0;
  const double2* cm_uv2 = reinterpret_cast<const double2*>(a.cm_uv);
  if (MODE == 0 && kfirst < k1) { g_nx = ldg256(a.geo_cm + kfirst); uv_nx = __ldg(cm_uv2 + kfirst); }
  if (MODE == 1 && kfirst < k1) pt_nx = __ldg(a.cm_pt + kfirst);
  for (int64_t kb = k0 + (int64_t)warp * 32; kb < k1; kb += kCamWarps * 32) {
    const int64_t k = kb + lane;
    const double4 g_pf = g_nx;
    const double2 uv_pf = uv_nx;
    const int pt_cur = pt_nx;
    if (k + kCamWarps * 32 < k1) {
      if (MODE == 0) {
        g_nx = ldg256(a.geo_cm + k + kCamWarps * 32);
        uv_nx = __ldg(cm_uv2 + k + kCamWarps * 32);  // the pixel too (its load was the top stall)
      } else {
        pt_nx = __ldg(a.cm_pt + k + kCamWarps * 32);
      }
    }
    if (k < k1) {
      const double4 g = MODE == 0 ? g_pf : ldg256(a.geo_cm + k);
      double Jc[12], Jp[6];
      geo_jacobians(cm, R, g, Jc, Jp);
#pragma unroll
      for (int i = 0; i < 12; ++i) As[i] = Jc[i];
      if (MODE == 0) {
        const double2 uv = uv_pf;
        double xd, yd;
        distort(cm, g.x, g.y, xd, yd);
        const double r0 = g.w * (cm.fx * xd + cm.cx - uv.x);
        const double r1 = g.w * (cm.fy * yd + cm.cy - uv.y);
#pragma unroll
        for (int c = 0; c < 6; ++c) { Bs[c] = Jc[c]; Bs[8 + c] = Jc[6 + c]; }
        Bs[6] = r0; Bs[14] = r1;
      } else {
        const double* pv = a.pv + (int64_t)pt_cur * 12;
        const double4 pva = ldg256(pv), pvb = ldg256(pv + 4);
        const double v0 = pva.x, v1 = pva.y, v2 = pva.z, v3_ = pva.w, v4 = pvb.x, v5 = pvb.y;
        const double pe0 = pvb.z, pe1 = pvb.w, pe2 = __ldg(pv + 8);
        const double P00 = v0 * Jp[0] + v1 * Jp[1] + v2 * Jp[2];
        const double P01 = v1 * Jp[0] + v3_ * Jp[1] + v4 * Jp[2];
        const double P02 = v2 * Jp[0] + v4 * Jp[1] + v5 * Jp[2];
        const double P10 = v0 * Jp[3] + v1 * Jp[4] + v2 * Jp[5];
        const double P11 = v1 * Jp[3] + v3_ * Jp[4] + v4 * Jp[5];
        const double P12 = v2 * Jp[3] + v4 * Jp[4] + v5 * Jp[5];
        const double m00 = Jp[0] * P00 + Jp[1] * P01 + Jp[2] * P02;
        const double m01 = Jp[0] * P10 + Jp[1] * P11 + Jp[2] * P12;
        const double m11 = Jp[3] * P10 + Jp[4] * P11 + Jp[5] * P12;
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          Bs[c] = -(m00 * Jc[c] + m01 * Jc[6 + c]);
          Bs[8 + c] = -(m01 * Jc[c] + m11 * Jc[6 + c]);
        }
        Bs[6] = Jp[0] * pe0 + Jp[1] * pe1 + Jp[2] * pe2;
        Bs[14] = Jp[3] * pe0 + Jp[4] * pe1 + Jp[5] * pe2;
      }
      Bs[7] = 0.0;
      Bs[15] = 0.0;
    } else {
#pragma unroll
      for (int i = 0; i < 28; ++i) As[i] = 0.0;
    }
    __syncwarp();
    const int nch = (int)((min((int64_t)32, k1 - kb) + 1) >> 1);
    const double* Sw = &St[warp][0];
    const int comp = fk & 1;
    for (int ch = 0; ch < nch; ch += 2) {
      const int o0 = 2 * ch + (fk >> 1);
      const double a0 = fr < 6 ? Sw[o0 * kCamLd + comp * 6 + fr] : 0.0;
      const double b0 = Sw[o0 * kCamLd + 12 + comp * 8 + fr];
      dmma_8x8x4(d0, d1, a0, b0);
      if (ch + 1 < nch) {
        const int o1 = o0 + 2;
        const double a1 = fr < 6 ? Sw[o1 * kCamLd + comp * 6 + fr] : 0.0;
        const double b1 = Sw[o1 * kCamLd + 12 + comp * 8 + fr];
        dmma_8x8x4(e0, e1, a1, b1);
      }
    }
    __syncwarp();
  }
  // warp result C[fr][2fk + {0,1}] -> smem, then warp 0 adds the warps in order
  Wsum[warp][fr * 8 + 2 * fk] = d0 + e0;
  Wsum[warp][fr * 8 + 2 * fk + 1] = d1 + e1;
  __syncthreads();
  if (warp != 0) return;
  // lane l < 36: block entry (l/6, l%6); lanes 36.. handled below via l2
  const int r0 = lane / 6, c0 = lane % 6;
  // MODE 1's -J~c^T M J~c is symmetric only up to rounding: average the two
  // triangles so S stays exactly symmetric (MODE 0 is symmetric as computed)
  auto ent = [&](int w, int r, int c) {
    return MODE == 0 ? Wsum[w][r * 8 + c] : 0.5 * (Wsum[w][r * 8 + c] + Wsum[w][c * 8 + r]);
  };
  double s0 = 0.0;
#pragma unroll
  for (int w = 0; w < kCamWarps; ++w) s0 += ent(w, r0, c0);
  // second value per lane: entries 32..35 of the block (lanes 0..3), the
  // 6-vector column 6 (lanes 4..9)
  double s1 = 0.0;
  if (lane < 4) {
    const int e = 32 + lane;
#pragma unroll
    for (int w = 0; w < kCamWarps; ++w) s1 += ent(w, e / 6, e % 6);
  } else if (lane < 10) {
#pragma unroll
    for (int w = 0; w < kCamWarps; ++w) s1 += Wsum[w][(lane - 4) * 8 + 6];
  }
  if (MODE == 0) {
    a.Uout[(int64_t)j * 36 + lane] = s0;
    if (lane < 4) a.Uout[(int64_t)j * 36 + 32 + lane] = s1;
    else if (lane < 10) a.gout[(int64_t)j * 6 + lane - 4] = s1;
    return;
  }
  if (a.rank == 0) {
    const double* Uj = a.U + (int64_t)j * 36;
    s0 += Uj[lane];
    if (lane % 7 == 0) s0 += a.lam * a.Dc[j * 6 + lane / 7];
    if (lane < 4) {
      s1 += Uj[32 + lane];
      if (lane == 3) s1 += a.lam * a.Dc[j * 6 + 5];
    } else if (lane < 10) {
      s1 -= a.gc[j * 6 + lane - 4];
    }
  }
  double* up = a.S + (int64_t)a.diag_pos[j] * 36;
  up[lane] = s0;
  if (lane < 4) up[32 + lane] = s1;
  else if (lane < 10) a.b[j * 6 + lane - 4] = s1;
}

// Register-accumulating k_cam_blocks (same CTA / warp / batch structure):
// each lane sums its observations' upper-triangle block terms (21) and
// 6-vector terms in 27 registers; the warp reduce-scatters them once per
// camera and warp 0 adds the four warps in order.  The block is symmetric by
// construction (upper triangle mirrored).
#ifndef SFM_CAMF_MINB
#define SFM_CAMF_MINB 3
#endif
__device__ __forceinline__ int tri6(int r, int c) {  // upper-triangle slot of (r, c), r <= c
  return r * 6 - (r * (r - 1)) / 2 + (c - r);
}

template <int MODE>
__global__ void __launch_bounds__(kCamWarps * 32, SFM_CAMF_MINB) k_cam_fma(BlkArgs a) {
  __shared__ double Wsum[kCamWarps][32];
  const int j = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (MODE == 1 && a.pre && j == 0 && threadIdx.x == 0 && a.pre->nonfinite) atomicOr(&a.sc->nonfinite, 1);
  const int f = a.free_frame[j];
  Mat3 R; Vec3 t;
  load_cam(a.Rt, f, R, t);
  const sfm_camera_model cm = a.models[a.frame_model[f]];
  const int64_t k0 = a.cm_ptr[j], k1 = a.cm_ptr[j + 1];
  double acc[27];
#pragma unroll
  for (int i = 0; i < 27; ++i) acc[i] = 0.0;
  const double2* cm_uv2 = reinterpret_cast<const double2*>(a.cm_uv);
  constexpr int kStride = kCamWarps * 32;
  int64_t k = k0 + (int64_t)warp * 32 + lane;
  // one observation ahead: MODE 0 its record and pixel, MODE 1 its point id
  double4 g_nx = make_double4(0.0, 0.0, 0.0, 0.0);
  double2 uv_nx = make_double2(0.0, 0.0);
  int pt_nx = 0;
  if (k < k1) {
    if (MODE == 0) { g_nx = ldg256(a.geo_cm + k); uv_nx = __ldg(cm_uv2 + k); }
    else pt_nx = __ldg(a.cm_pt + k);
  }
  for (; k < k1; k += kStride) {
    const double4 g = MODE == 0 ? g_nx : ldg256(a.geo_cm + k);
    const double2 uv = uv_nx;
    const int pt = pt_nx;
    if (k + kStride < k1) {
      if (MODE == 0) { g_nx = ldg256(a.geo_cm + k + kStride); uv_nx = __ldg(cm_uv2 + k + kStride); }
      else pt_nx = __ldg(a.cm_pt + k + kStride);
    }
    double Jc[12], Jp[6];
    geo_jacobians(cm, R, g, Jc, Jp);
    double B0[6], B1[6], s0, s1;
    if (MODE == 0) {
      double xd, yd;
      distort(cm, g.x, g.y, xd, yd);
      s0 = g.w * (cm.fx * xd + cm.cx - uv.x);
      s1 = g.w * (cm.fy * yd + cm.cy - uv.y);
#pragma unroll
      for (int c = 0; c < 6; ++c) { B0[c] = Jc[c]; B1[c] = Jc[6 + c]; }
    } else {
      const double* pv = a.pv + (int64_t)pt * 12;
      const double4 pva = ldg256(pv), pvb = ldg256(pv + 4);
      const double v0 = pva.x, v1 = pva.y, v2 = pva.z, v3_ = pva.w, v4 = pvb.x, v5 = pvb.y;
      const double pe0 = pvb.z, pe1 = pvb.w, pe2 = __ldg(pv + 8);
      const double P00 = v0 * Jp[0] + v1 * Jp[1] + v2 * Jp[2];
      const double P01 = v1 * Jp[0] + v3_ * Jp[1] + v4 * Jp[2];
      const double P02 = v2 * Jp[0] + v4 * Jp[1] + v5 * Jp[2];
      const double P10 = v0 * Jp[3] + v1 * Jp[4] + v2 * Jp[5];
      const double P11 = v1 * Jp[3] + v3_ * Jp[4] + v4 * Jp[5];
      const double P12 = v2 * Jp[3] + v4 * Jp[4] + v5 * Jp[5];
      const double m00 = Jp[0] * P00 + Jp[1] * P01 + Jp[2] * P02;
      const double m01 = Jp[0] * P10 + Jp[1] * P11 + Jp[2] * P12;
      const double m11 = Jp[3] * P10 + Jp[4] * P11 + Jp[5] * P12;
#pragma unroll
      for (int c = 0; c < 6; ++c) {
        B0[c] = -(m00 * Jc[c] + m01 * Jc[6 + c]);
        B1[c] = -(m01 * Jc[c] + m11 * Jc[6 + c]);
      }
      s0 = Jp[0] * pe0 + Jp[1] * pe1 + Jp[2] * pe2;
      s1 = Jp[3] * pe0 + Jp[4] * pe1 + Jp[5] * pe2;
    }
#pragma unroll
    for (int r = 0; r < 6; ++r) {
#pragma unroll
      for (int c = r; c < 6; ++c) {
        const int q = tri6(r, c);
        acc[q] = fma(Jc[6 + r], B1[c], fma(Jc[r], B0[c], acc[q]));
      }
      acc[21 + r] = fma(Jc[6 + r], s1, fma(Jc[r], s0, acc[21 + r]));
    }
  }
  warp_reduce_scatter<27>(acc, lane);
  const int e = rs_entry<27>(lane, 0);
  if (e >= 0) Wsum[warp][e] = acc[0];
  __syncthreads();
  if (warp != 0) return;
  // lane l < 32: block entry (l/6, l%6); second value: entries 32..35
  // (lanes 0..3), the 6-vector (lanes 4..9)
  const int r0 = lane / 6, c0 = lane % 6;
  const int q0 = r0 <= c0 ? tri6(r0, c0) : tri6(c0, r0);
  double s0 = 0.0;
#pragma unroll
  for (int w = 0; w < kCamWarps; ++w) s0 += Wsum[w][q0];
  double s1 = 0.0;
  if (lane < 4) {
    const int q1 = tri6(lane == 0 ? 2 : lane == 1 ? 3 : lane == 2 ? 4 : 5, 5);  // (5, 2..5)
#pragma unroll
    for (int w = 0; w < kCamWarps; ++w) s1 += Wsum[w][q1];
  } else if (lane < 10) {
#pragma unroll
    for (int w = 0; w < kCamWarps; ++w) s1 += Wsum[w][21 + lane - 4];
  }
  if (MODE == 0) {
    a.Uout[(int64_t)j * 36 + lane] = s0;
    if (lane < 4) a.Uout[(int64_t)j * 36 + 32 + lane] = s1;
    else if (lane < 10) a.gout[(int64_t)j * 6 + lane - 4] = s1;
    return;
  }
  if (a.rank == 0) {
    const double* Uj = a.U + (int64_t)j * 36;
    s0 += Uj[lane];
    if (lane % 7 == 0) s0 += a.lam * a.Dc[j * 6 + lane / 7];
    if (lane < 4) {
      s1 += Uj[32 + lane];
      if (lane == 3) s1 += a.lam * a.Dc[j * 6 + 5];
    } else if (lane < 10) {
      s1 -= a.gc[j * 6 + lane - 4];
    }
  }
  double* up = a.S + (int64_t)a.diag_pos[j] * 36;
  up[lane] = s0;
  if (lane < 4) up[32 + lane] = s1;
  else if (lane < 10) a.b[j * 6 + lane - 4] = s1;
}

#include "ischur.cuh"

// Camera-major observation streams (built once per bundle_adjust): the
// diagonal pair blocks already hold each free camera's observations in point
// order; copy them out contiguously with their pixels and point ids.
__global__ void k_cm_build(int nf, const int* __restrict__ diag_ub, const int* __restrict__ ub_pb,
                           const int64_t* __restrict__ pb_pair_ptr, const unsigned long long* __restrict__ pairs,
                           const int64_t* __restrict__ cm_ptr, const int* __restrict__ op,
                           const double* __restrict__ uv, int64_t* __restrict__ cm_obs, int* __restrict__ cm_pt,
                           double* __restrict__ cm_uv, int* __restrict__ cm_pos) {
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= nf) return;
  const int pb = ub_pb[diag_ub[j]];
  if (pb < 0) return;
  const int64_t p0 = pb_pair_ptr[pb], c0 = cm_ptr[j], n = cm_ptr[j + 1] - c0;
  for (int64_t q = lane; q < n; q += 32) {
    const int64_t o = (int64_t)(pairs[p0 + q] >> 32);
    cm_obs[c0 + q] = o;
    cm_pt[c0 + q] = op[o];
    cm_uv[(c0 + q) * 2] = uv[o * 2];
    cm_uv[(c0 + q) * 2 + 1] = uv[o * 2 + 1];
    cm_pos[o] = (int)(c0 + q);
  }
}

__global__ void k_pair_pt(int64_t n, const unsigned long long* __restrict__ pairs, const int* __restrict__ op,
                          int* __restrict__ pair_pt) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) pair_pt[k] = op[(int64_t)(pairs[k] >> 32)];
}


struct CamArgs {
  int nf;
  const int* term_ptr;
  const int* term_list;
  const int* ab;
  const int* pf;
  int E;
  const double* meas_inv;
  const double* init_inv;
  double we, wa;
  const double* q;
  const double* t;
  const double* Rt;
  double* U;
  double* gc;
};

// Pose terms, one thread per edge / prior: each term is evaluated once and
// its normal-equation contributions J^T J | J^T r (42 doubles per side)
// written to `contrib` (edge e side 0/1 at 2e / 2e+1, prior a at 2E + a);
// an edge between two free cameras also writes its off-diagonal block
// (the lower camera's J^T times the upper camera's J) to H.
__global__ void k_terms_lin(int E, int A, const int* __restrict__ ab, const int* __restrict__ pf,
                            const int* __restrict__ free_idx, const double* __restrict__ meas_inv,
                            const double* __restrict__ init_inv, double we, double wa, const double* q,
                            const double* t, const double* Rt, double* __restrict__ contrib,
                            double* __restrict__ H) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= E + A) return;
  double r[6];
  auto emit = [&](const double* J, double* out) {
#pragma unroll
    for (int rr = 0; rr < 6; ++rr) {
#pragma unroll
      for (int cc = 0; cc < 6; ++cc) {
        double s = 0.0;
#pragma unroll
        for (int m = 0; m < 6; ++m) s += J[m * 6 + rr] * J[m * 6 + cc];
        out[rr * 6 + cc] = s;
      }
      double s = 0.0;
#pragma unroll
      for (int m = 0; m < 6; ++m) s += J[m * 6 + rr] * r[m];
      out[36 + rr] = s;
    }
  };
  if (i < E) {
    const int fa = ab[2 * i], fb = ab[2 * i + 1];
    const int ja = free_idx[fa], jb = free_idx[fb];
    Pose Ta = load_pose(q, t, Rt, fa), Tb = load_pose(q, t, Rt, fb);
    double Ja[36], Jb[36];
    edge_eval(meas_inv + i * 7, Ta, Tb, we, r, Ja, Jb);
    if (ja >= 0) emit(Ja, contrib + (int64_t)(2 * i) * 42);
    if (jb >= 0) emit(Jb, contrib + (int64_t)(2 * i + 1) * 42);
    if (ja >= 0 && jb >= 0 && ja != jb) {
      const double* L = ja < jb ? Ja : Jb;
      const double* Rr = ja < jb ? Jb : Ja;
      for (int rr = 0; rr < 6; ++rr)
        for (int cc = 0; cc < 6; ++cc) {
          double s = 0.0;
          for (int m = 0; m < 6; ++m) s += L[m * 6 + rr] * Rr[m * 6 + cc];
          H[(int64_t)i * 36 + rr * 6 + cc] = s;
        }
    }
  } else {
    const int pi = i - E;
    if (free_idx[pf[pi]] < 0) return;
    Pose T = load_pose(q, t, Rt, pf[pi]);
    double J[36];
    prior_eval(init_inv + pi * 7, T, wa, r, J);
    emit(J, contrib + (int64_t)(2 * E + pi) * 42);
  }
}

// + the incident pose terms (rank 0 only holds them), in term order.
__global__ void k_cam_terms_sum(CamArgs a, const double* __restrict__ contrib) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= a.nf || a.term_ptr[j] == a.term_ptr[j + 1]) return;
  double* U = a.U + (int64_t)j * 36;
  double* g = a.gc + (int64_t)j * 6;
  double Ua[36], ga[6];
#pragma unroll
  for (int i = 0; i < 36; ++i) Ua[i] = U[i];
#pragma unroll
  for (int i = 0; i < 6; ++i) ga[i] = g[i];
  for (int k = a.term_ptr[j]; k < a.term_ptr[j + 1]; ++k) {
    const int code = a.term_list[k];
    const int term = code >> 2, side = code & 3;
    const double* c = contrib + (int64_t)(term < a.E ? 2 * term + side : 2 * a.E + (term - a.E)) * 42;
#pragma unroll
    for (int i = 0; i < 36; ++i) Ua[i] += __ldg(c + i);
#pragma unroll
    for (int i = 0; i < 6; ++i) ga[i] += __ldg(c + 36 + i);
  }
#pragma unroll
  for (int i = 0; i < 36; ++i) U[i] = Ua[i];
#pragma unroll
  for (int i = 0; i < 6; ++i) g[i] = ga[i];
}

__global__ void k_cam_post(int nf, const double* __restrict__ U, const double* __restrict__ gc,
                           double* __restrict__ Dc, BAScalars* sc) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  double gm = 0.0;
  if (j < nf) {
    for (int i = 0; i < 6; ++i) {
      Dc[j * 6 + i] = fmax(U[(int64_t)j * 36 + i * 7], 1e-12);  // solver.py:217
      double g = gc[j * 6 + i];
      gm = isnan(g) ? __longlong_as_double(0x7ff8000000000000ll) : fmax(gm, fabs(g));
    }
  }
  unsigned long long m = warp_max_u64((unsigned long long)__double_as_longlong(gm));
  if ((threadIdx.x & 31) == 0) atomicMax(&sc->gmax, m);
}

// Off-diagonal edge block oriented as the upper block (lo, hi).
// ---------------------------------------------------------------------------
// Schur complement (per LM trial)
// ---------------------------------------------------------------------------

// V* = V + lam*max(diag V, 1e-12) (solver.py:217-220), V*^-1 (adjugate),
// e = V*^-1 g_p.

__global__ void k_point_prep(int64_t P, double lam, const double* __restrict__ V,
                             const double* __restrict__ gp, double* __restrict__ pv, BAScalars* sc) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  // V (48 B, 16-byte aligned) as three 128-bit loads, g_p as scalars (24 B stride)
  const double2* v2 = reinterpret_cast<const double2*>(V + p * 6);
  const double2 a = __ldg(v2), b = __ldg(v2 + 1), c = __ldg(v2 + 2);
  const double v[6] = {a.x, a.y, b.x, b.y, c.x, c.y};
  const double g[3] = {__ldg(gp + p * 3), __ldg(gp + p * 3 + 1), __ldg(gp + p * 3 + 2)};
  if (!point_prep_one(v, g, lam, pv + p * 12)) atomicOr(&sc->nonfinite, 1);
}

// ---------------------------------------------------------------------------
// reduced camera system solvers
// ---------------------------------------------------------------------------

__device__ __forceinline__ int pk(int i, int j) { return i * (i + 1) / 2 + j; }

// Dense Cholesky of S (n = 6*nf <= kDenseMax) in one CTA's shared memory,
// then forward/back substitution.  Fails (nonfinite) if not PD.
__global__ void __launch_bounds__(1024) k_dense_solve(int nf, const int* __restrict__ row_ptr,
                                                      const int* __restrict__ col,
                                                      const double* __restrict__ S,
                                                      const double* __restrict__ b,
                                                      double* __restrict__ x, BAScalars* sc) {
  extern __shared__ double L[];
  __shared__ double y[kDenseMax];
  __shared__ int fail;
  __shared__ double red[32];
  const int n = nf * 6;
  const int tid = threadIdx.x, nt = blockDim.x;
  if (tid == 0) fail = 0;
  for (int i = tid; i < n * (n + 1) / 2; i += nt) L[i] = 0.0;
  __syncthreads();
  for (int r = 0; r < nf; ++r) {
    for (int k = row_ptr[r] + 0; k < row_ptr[r + 1]; ++k) {
      int c = col[k];
      if (c > r) continue;
      for (int e = tid; e < 36; e += nt) {
        int i = e / 6, j = e % 6;
        int R = r * 6 + i, C = c * 6 + j;
        if (C <= R) L[pk(R, C)] = S[(int64_t)k * 36 + e];
      }
    }
  }
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    if (tid == 0) {
      double d = L[pk(k, k)];
      if (!(d > 0.0) || !isfinite(d)) fail = 1;
      L[pk(k, k)] = sqrt(d);
    }
    __syncthreads();
    if (fail) break;
    const double dk = L[pk(k, k)];
    for (int i = k + 1 + tid; i < n; i += nt) L[pk(i, k)] /= dk;
    __syncthreads();
    // trailing update of the lower triangle
    const int m = n - k - 1;
    const int tot = m * (m + 1) / 2;
    for (int lin = tid; lin < tot; lin += nt) {
      // lin -> (ii, jj) with 0 <= jj <= ii < m
      int ii = (int)((sqrt(8.0 * lin + 1.0) - 1.0) * 0.5);
      while (ii * (ii + 1) / 2 > lin) --ii;
      while ((ii + 1) * (ii + 2) / 2 <= lin) ++ii;
      int jj = lin - ii * (ii + 1) / 2;
      int i = k + 1 + ii, j = k + 1 + jj;
      L[pk(i, j)] -= L[pk(i, k)] * L[pk(j, k)];
    }
    __syncthreads();
  }
  if (fail) {
    if (tid == 0) sc->nonfinite = 1;
    return;
  }
  // forward: L y = b
  for (int i = 0; i < n; ++i) {
    double s = 0.0;
    for (int j = tid; j < i; j += nt) s += L[pk(i, j)] * y[j];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((tid & 31) == 0) red[tid >> 5] = s;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < (nt + 31) / 32; ++w) t += red[w];
      y[i] = (b[i] - t) / L[pk(i, i)];
    }
    __syncthreads();
  }
  // backward: L^T x = y (x kept in y)
  for (int i = n - 1; i >= 0; --i) {
    double s = 0.0;
    for (int j = i + 1 + tid; j < n; j += nt) s += L[pk(j, i)] * y[j];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((tid & 31) == 0) red[tid >> 5] = s;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < (nt + 31) / 32; ++w) t += red[w];
      y[i] = (y[i] - t) / L[pk(i, i)];
    }
    __syncthreads();
  }
  for (int i = tid; i < n; i += nt) x[i] = y[i];
  for (int i = tid; i < n; i += nt)
    if (!isfinite(y[i])) sc->nonfinite = 1;
}

// ---------------------------------------------------------------------------
// trial poses (solver.py:68-71: exp_map(delta) @ T)
// ---------------------------------------------------------------------------
__global__ void k_cam_trial(int nf, const int* __restrict__ free_frame, const double* __restrict__ dc,
                            const double* q, const double* t, const double* Rt, double* qo, double* to,
                            double* Rto, double* qto, double* __restrict__ part, BAScalars* sc) {
  __shared__ double red[kBlock / 32];
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  double s = 0.0;
  if (j < nf) {
    const int f = free_frame[j];
    double d[6];
    bool fin = true;
    for (int i = 0; i < 6; ++i) {
      d[i] = dc[j * 6 + i];
      s += d[i] * d[i];
      fin = fin && isfinite(d[i]);
    }
    if (!fin) atomicOr(&sc->nonfinite, 1);
    Pose T = load_pose(q, t, Rt, f);
    Pose E = se3_exp(d);
    Pose N = compose(E, T);
    qo[f * 4] = N.q.w; qo[f * 4 + 1] = N.q.x; qo[f * 4 + 2] = N.q.y; qo[f * 4 + 3] = N.q.z;
    to[f * 3] = N.t.x; to[f * 3 + 1] = N.t.y; to[f * 3 + 2] = N.t.z;
    for (int i = 0; i < 9; ++i) Rto[f * 12 + i] = N.R.m[i];
    Rto[f * 12 + 9] = N.t.x; Rto[f * 12 + 10] = N.t.y; Rto[f * 12 + 11] = N.t.z;
    if (qto) {
      qto[f * 8] = N.q.w; qto[f * 8 + 1] = N.q.x; qto[f * 8 + 2] = N.q.y; qto[f * 8 + 3] = N.q.z;
      qto[f * 8 + 4] = N.t.x; qto[f * 8 + 5] = N.t.y; qto[f * 8 + 6] = N.t.z; qto[f * 8 + 7] = 0.0;
    }
  }
  double b = block_sum<kBlock>(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = b;
}

__global__ void k_reset_scalars(BAScalars* sc, int full) {
  sc->nonfinite = 0;
  sc->depth_obs = ~0ull;
  sc->gmax = 0ull;
  sc->pcg_fail = 0;
  if (full) { sc->pcg_iters = 0; sc->pcg_stop = 0; }
}

// Locates the projection failure of one observation (message payload).
__global__ void k_probe_obs(int64_t o, const int* of, const int* op, const double* uv,
                            const int* frame_model, const sfm_camera_model* models,
                            const double* Rt, const double* X, BAScalars* sc) {
  const int f = of[o];
  Mat3 R; Vec3 t;
  load_cam(Rt, f, R, t);
  Vec3 pc = add(mul(R, load_X(X, op[o])), t);
  double u, v;
  sc->proj_code = project_point(models[frame_model[f]], pc, u, v);
  sc->proj_depth = pc.z;
  (void)uv;
}

// sfm_ba_eval: per-observation robust cost and weighted r, Jc, Jp.
__global__ void k_eval_obs(int64_t N, int lk, double lp, const int* of, const int* op,
                           const double* uv, const int* frame_model, const sfm_camera_model* models,
                           const double* Rt, const double* X, double* cost, double* res, double* jc,
                           double* jp, BAScalars* sc) {
  int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= N) return;
  const int f = of[o];
  Mat3 R; Vec3 t;
  load_cam(Rt, f, R, t);
  double Jc[12], Jp[6], r[2];
  double u, v;
  Vec3 Xp = load_X(X, op[o]);
  int st = project_with_jacobians(models[frame_model[f]], R, t, Xp, u, v, Jc, Jp);
  if (st != PROJ_OK) {
    atomicMin(&sc->depth_obs, (unsigned long long)o);
    return;
  }
  r[0] = u - uv[o * 2];
  r[1] = v - uv[o * 2 + 1];
  double s = r[0] * r[0] + r[1] * r[1];
  double w = sqrt(loss_rho_prime(lk, lp, s));
  if (cost) cost[o] = loss_rho(lk, lp, s);
  if (res) { res[o * 2] = w * r[0]; res[o * 2 + 1] = w * r[1]; }
  if (jc) for (int i = 0; i < 12; ++i) jc[o * 12 + i] = w * Jc[i];
  if (jp) for (int i = 0; i < 6; ++i) jp[o * 6 + i] = w * Jp[i];
}

// Temp-storage helper for CUB device-wide primitives.
struct CubTemp {
  DevBuf<char> buf;
  void* get(size_t bytes) { return buf.resize(bytes); }
};

int bits_for(unsigned long long maxval) {
  int b = 1;
  while (b < 64 && (maxval >> b) != 0) ++b;
  return b;
}

}  // namespace

// ===========================================================================
// host driver
// ===========================================================================

namespace {
// SFM_TIMING=1: wall-clock split of sfm_ba_setup on stderr (stream-synced
// at each mark, so only for diagnosis).
struct SetupTimer {
  bool on = std::getenv("SFM_TIMING") != nullptr;
  cudaStream_t s;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  explicit SetupTimer(cudaStream_t st) : s(st) {}
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[sfm setup] %-28s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  }
};
}  // namespace

BASolver::~BASolver() {
  if (h_pin_) cudaFreeHost(h_pin_);
  if (side_) {
    cudaStreamSynchronize(side_);
    cudaStreamDestroy(side_);
  }
  if (plan_stream_) {
    cudaStreamSynchronize(plan_stream_);
    cudaStreamDestroy(plan_stream_);
  }
  if (plan_ev_) cudaEventDestroy(plan_ev_);
  if (side_ready_) cudaEventDestroy(side_ready_);
  if (side_done_) cudaEventDestroy(side_done_);
}

void BASolver::setup(const sfm_ba_problem& pr, const sfm_ba_options& opt) {
  NvtxRange nv("sfm ba setup");
  opt_ = opt;
  rank_ = comm_ ? comm_->rank : 0;
  SFM_REQUIRE(pr.n_frames >= 0 && pr.n_points >= 0 && pr.n_obs >= 0, "negative sizes");
  SFM_REQUIRE(pr.n_obs < (1ll << 31), "n_obs must fit in 31 bits");
  SFM_REQUIRE(opt.loss_kind >= 0 && opt.loss_kind <= 2, "unknown loss kind");
  F_ = pr.n_frames;
  nmodels_ = pr.n_models;
  P_ = pr.n_points;
  N_ = pr.n_obs;
  obs_offset_ = pr.obs_offset;
  n_edges_ = pr.n_edges;
  n_priors_ = pr.n_priors;
  edge_w_ = std::sqrt(pr.edge_weight);
  prior_w_ = std::sqrt(pr.prior_weight);
  cudaStream_t s = stream_;
  SetupTimer tm(s);

  // frames: free index map (solver.py:154-161: free blocks in insertion
  // order = sorted frames), models
  std::vector<int> free_idx(F_), free_frame;
  for (int f = 0; f < F_; ++f) {
    SFM_REQUIRE(pr.frame_model[f] >= 0 && pr.frame_model[f] < nmodels_, "frame_model out of range");
    if (pr.frame_fixed[f]) free_idx[f] = -1;
    else { free_idx[f] = (int)free_frame.size(); free_frame.push_back(f); }
  }
  nfree_ = (int)free_frame.size();
  SFM_REQUIRE((unsigned long long)nfree_ * nfree_ < (1ull << 62), "too many free frames");
  n_params_ = pr.n_params_global > 0 ? pr.n_params_global : (int64_t)nfree_ * 6 + P_ * 3;
  models_.upload(pr.models, nmodels_, s);
  frame_model_.upload(pr.frame_model, F_, s);
  free_idx_.upload(free_idx.data(), F_, s);
  free_frame_.upload(free_frame.data(), nfree_, s);
  for (int k = 0; k < 2; ++k) {
    if (k == 0) {
      q_[0].upload(pr.cam_q, (size_t)F_ * 4, s);
      t_[0].upload(pr.cam_t, (size_t)F_ * 3, s);
    } else {  // the second state buffer starts as a device copy of the first
      q_[1].resize((size_t)F_ * 4);
      t_[1].resize((size_t)F_ * 3);
      if (F_) {
        SFM_CUDA(cudaMemcpyAsync(q_[1].get(), q_[0].get(), sizeof(double) * 4 * F_, cudaMemcpyDeviceToDevice, s));
        SFM_CUDA(cudaMemcpyAsync(t_[1].get(), t_[0].get(), sizeof(double) * 3 * F_, cudaMemcpyDeviceToDevice, s));
      }
    }
    Rt_[k].resize((size_t)F_ * 12);
    qt_[k].resize((size_t)F_ * 8);
    if (F_) { k_frames_rt<<<grid_for(F_, 128), 128, 0, s>>>(F_, q_[k].get(), t_[k].get(), Rt_[k].get(), qt_[k].get()); SFM_CHECK_LAUNCH(); }
  }
  cur_ = 0;
  // The points and pixels (~2/3 of the input bytes) are not read until the
  // camera-major streams: they go over a side stream while the index
  // arrays arrive and the pair list / S pattern are built.
  if (!side_) {
    SFM_CUDA(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking));
    SFM_CUDA(cudaEventCreateWithFlags(&side_ready_, cudaEventDisableTiming));
    SFM_CUDA(cudaEventCreateWithFlags(&side_done_, cudaEventDisableTiming));
  }
  struct SideJoin {  // no early exit leaves a copy in flight into freed buffers
    cudaStream_t st;
    ~SideJoin() { cudaStreamSynchronize(st); }
  } side_join{side_};
  X_[0].resize((size_t)P_ * 3);
  X_[1].resize((size_t)P_ * 3);
  obs_uv_.resize((size_t)N_ * 2);
  SFM_CUDA(cudaEventRecord(side_ready_, s));
  SFM_CUDA(cudaStreamWaitEvent(side_, side_ready_, 0));
  if (P_) {
    SFM_CUDA(cudaMemcpyAsync(X_[0].get(), pr.points, sizeof(double) * 3 * P_, cudaMemcpyDefault, side_));
    SFM_CUDA(cudaMemcpyAsync(X_[1].get(), X_[0].get(), sizeof(double) * 3 * P_, cudaMemcpyDeviceToDevice, side_));
  }
  if (N_) SFM_CUDA(cudaMemcpyAsync(obs_uv_.get(), pr.obs_uv, sizeof(double) * 2 * N_, cudaMemcpyDefault, side_));
  SFM_CUDA(cudaEventRecord(side_done_, side_));
  obs_frame_.upload(pr.obs_frame, N_, s);
  obs_point_.upload(pr.obs_point, N_, s);
  geo_.resize(N_);
  sc_.resize(1);
  SFM_CUDA(cudaMemsetAsync(sc_.get(), 0, sizeof(BAScalars), s));

  tm.mark("uploads");
  // layout validation
  {
    DevBuf<int> bad;
    bad.resize(1);
    bad.zero(s);
    if (N_) { k_validate_obs<<<grid_for(N_, 256), 256, 0, s>>>(N_, F_, P_, obs_frame_.get(), obs_point_.get(), bad.get()); SFM_CHECK_LAUNCH(); }
    int hb = 0;
    bad.download(&hb, 1, s);
    SFM_CUDA(cudaStreamSynchronize(s));
    SFM_REQUIRE(hb == 0, "observations must reference valid frames/points and be sorted by point");
  }
  pt_ptr_.resize(P_ + 1);
  k_pt_ptr<<<grid_for(P_ + 1, 256), 256, 0, s>>>(P_, N_, obs_point_.get(), pt_ptr_.get());
  SFM_CHECK_LAUNCH();

  CubTemp tmp;
  size_t tb = 0;
  tm.mark("validate + pt_ptr");
  // ---- pair list: count, scan, generate, stable sort by S block ----------
  DevBuf<int64_t> pcnt, poff;
  pcnt.resize(P_ + 1);
  poff.resize(P_ + 1);
  k_pair_count<<<grid_for(P_ + 1, 256), 256, 0, s>>>(P_, pt_ptr_.get(), obs_frame_.get(), free_idx_.get(), pcnt.get());
  SFM_CHECK_LAUNCH();
  SFM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, pcnt.get(), poff.get(), P_ + 1, s));
  SFM_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(tb), tb, pcnt.get(), poff.get(), P_ + 1, s));
  int64_t n_pairs = 0;
  SFM_CUDA(cudaMemcpyAsync(&n_pairs, poff.get() + P_, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SFM_CUDA(cudaStreamSynchronize(s));
  n_pairs_ = n_pairs;
  SFM_REQUIRE(n_pairs_ < (1ll << 31), "pair list too large for int32 CUB offsets");
  DevBuf<unsigned long long> keys_in, keys_out, vals_in;
  keys_in.resize(n_pairs_);
  keys_out.resize(n_pairs_);
  vals_in.resize(n_pairs_);
  pairs_.resize(n_pairs_);
  if (P_) { k_pair_gen<<<grid_for(P_, 256), 256, 0, s>>>(P_, nfree_, pt_ptr_.get(), obs_frame_.get(), free_idx_.get(), poff.get(), keys_in.get(), vals_in.get()); SFM_CHECK_LAUNCH(); }
  const int key_bits = bits_for((unsigned long long)nfree_ * nfree_);
  if (n_pairs_) {
    SFM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys_in.get(), keys_out.get(), vals_in.get(), pairs_.get(), (int)n_pairs_, 0, key_bits, s));
    SFM_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(tb), tb, keys_in.get(), keys_out.get(), vals_in.get(), pairs_.get(), (int)n_pairs_, 0, key_bits, s));
  }
  vals_in.release();
  // run-length encode into pair blocks
  DevBuf<unsigned long long> pb_key;
  DevBuf<int> pb_cnt, n_runs;
  pb_key.resize(n_pairs_);
  pb_cnt.resize(n_pairs_ + 1);
  n_runs.resize(1);
  int h_runs = 0;
  if (n_pairs_) {
    SFM_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, tb, keys_out.get(), pb_key.get(), pb_cnt.get(), n_runs.get(), (int)n_pairs_, s));
    SFM_CUDA(cub::DeviceRunLengthEncode::Encode(tmp.get(tb), tb, keys_out.get(), pb_key.get(), pb_cnt.get(), n_runs.get(), (int)n_pairs_, s));
    n_runs.download(&h_runs, 1, s);
    SFM_CUDA(cudaStreamSynchronize(s));
  }
  n_pb_ = h_runs;
  keys_out.release();
  keys_in.release();
  // pair-block -> pair range
  {
    DevBuf<int64_t> pb_pair_cnt64;
    pb_pair_cnt64.resize(n_pb_ + 1);
    pb_pair_ptr_.resize(n_pb_ + 1);
    k_div_ceil<<<grid_for(n_pb_ + 1, 256), 256, 0, s>>>(n_pb_, pb_cnt.get(), pb_pair_cnt64.get(), 1);
    SFM_CHECK_LAUNCH();
    SFM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, pb_pair_cnt64.get(), pb_pair_ptr_.get(), n_pb_ + 1, s));
    SFM_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(tb), tb, pb_pair_cnt64.get(), pb_pair_ptr_.get(), n_pb_ + 1, s));
  }

  tm.mark("pair list + sort");
  // ---- S block pattern: pair blocks U diagonal U lambda_c edges ----------
  std::vector<int> h_ab(2 * (size_t)n_edges_), h_pf(n_priors_);
  if (n_edges_) std::memcpy(h_ab.data(), pr.edge_ab, sizeof(int) * 2 * n_edges_);
  if (n_priors_) std::memcpy(h_pf.data(), pr.prior_frame, sizeof(int) * n_priors_);
  std::vector<unsigned long long> extra;
  for (int j = 0; j < nfree_; ++j) extra.push_back((unsigned long long)j * nfree_ + j);
  {
    std::vector<unsigned long long> ek;
    for (int e = 0; e < n_edges_; ++e) {
      int a = h_ab[2 * e], b = h_ab[2 * e + 1];
      SFM_REQUIRE(a >= 0 && a < F_ && b >= 0 && b < F_ && a != b, "edge frames out of range");
      int ja = free_idx[a], jb = free_idx[b];
      if (ja < 0 || jb < 0) continue;
      unsigned long long k = (unsigned long long)std::min(ja, jb) * nfree_ + std::max(ja, jb);
      ek.push_back(k);
    }
    std::vector<unsigned long long> sorted_ek = ek;
    std::sort(sorted_ek.begin(), sorted_ek.end());
    SFM_REQUIRE(std::adjacent_find(sorted_ek.begin(), sorted_ek.end()) == sorted_ek.end(),
                "duplicate pose edge between the same frames");
    extra.insert(extra.end(), ek.begin(), ek.end());
  }
  for (int a = 0; a < n_priors_; ++a)
    SFM_REQUIRE(h_pf[a] >= 0 && h_pf[a] < F_, "prior frame out of range");
  DevBuf<unsigned long long> cand, cand_sorted, ub_local;
  const int64_t n_cand = n_pb_ + (int64_t)extra.size();
  cand.resize(n_cand);
  cand_sorted.resize(n_cand);
  ub_local.resize(n_cand);
  if (n_pb_) SFM_CUDA(cudaMemcpyAsync(cand.get(), pb_key.get(), sizeof(unsigned long long) * n_pb_, cudaMemcpyDeviceToDevice, s));
  if (!extra.empty()) SFM_CUDA(cudaMemcpyAsync(cand.get() + n_pb_, extra.data(), sizeof(unsigned long long) * extra.size(), cudaMemcpyHostToDevice, s));
  DevBuf<int> n_uniq;
  n_uniq.resize(1);
  int h_nu = 0;
  if (n_cand) {
    SFM_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, cand.get(), cand_sorted.get(), (int)n_cand, 0, key_bits, s));
    SFM_CUDA(cub::DeviceRadixSort::SortKeys(tmp.get(tb), tb, cand.get(), cand_sorted.get(), (int)n_cand, 0, key_bits, s));
    SFM_CUDA(cub::DeviceSelect::Unique(nullptr, tb, cand_sorted.get(), ub_local.get(), n_uniq.get(), (int)n_cand, s));
    SFM_CUDA(cub::DeviceSelect::Unique(tmp.get(tb), tb, cand_sorted.get(), ub_local.get(), n_uniq.get(), (int)n_cand, s));
    n_uniq.download(&h_nu, 1, s);
    SFM_CUDA(cudaStreamSynchronize(s));
  }
  if (comm_ && comm_->active()) {
    // union of the per-rank patterns (the S pattern is global)
    DevBuf<unsigned long long> cnt;
    cnt.resize(1);
    unsigned long long hc = (unsigned long long)h_nu;
    SFM_CUDA(cudaMemcpyAsync(cnt.get(), &hc, sizeof(hc), cudaMemcpyHostToDevice, s));
    comm_->max_u64(cnt.get(), 1, s);
    cnt.download(&hc, 1, s);
    SFM_CUDA(cudaStreamSynchronize(s));
    const size_t m = (size_t)hc;
    DevBuf<unsigned long long> sendb, recvb, rsorted;
    sendb.resize(m);
    SFM_CUDA(cudaMemsetAsync(sendb.get(), 0xff, sizeof(unsigned long long) * m, s));
    if (h_nu) SFM_CUDA(cudaMemcpyAsync(sendb.get(), ub_local.get(), sizeof(unsigned long long) * h_nu, cudaMemcpyDeviceToDevice, s));
    recvb.resize(m * comm_->world);
    rsorted.resize(m * comm_->world);
    comm_->allgather_u64(sendb.get(), recvb.get(), m, s);
    const int tot = (int)(m * comm_->world);
    SFM_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, recvb.get(), rsorted.get(), tot, 0, 64, s));
    SFM_CUDA(cub::DeviceRadixSort::SortKeys(tmp.get(tb), tb, recvb.get(), rsorted.get(), tot, 0, 64, s));
    ub_local.resize(tot);
    SFM_CUDA(cub::DeviceSelect::Unique(nullptr, tb, rsorted.get(), ub_local.get(), n_uniq.get(), tot, s));
    SFM_CUDA(cub::DeviceSelect::Unique(tmp.get(tb), tb, rsorted.get(), ub_local.get(), n_uniq.get(), tot, s));
    n_uniq.download(&h_nu, 1, s);
    SFM_CUDA(cudaStreamSynchronize(s));
    if (h_nu > 0) {
      unsigned long long last = 0;
      SFM_CUDA(cudaMemcpy(&last, ub_local.get() + h_nu - 1, sizeof(last), cudaMemcpyDeviceToHost));
      if (last == ~0ull) --h_nu;  // padding sentinel
    }
  }
  n_ub_ = h_nu;
  ub_key_.resize(n_ub_);
  if (n_ub_) SFM_CUDA(cudaMemcpyAsync(ub_key_.get(), ub_local.get(), sizeof(unsigned long long) * n_ub_, cudaMemcpyDeviceToDevice, s));
  // full (both triangles) BSR pattern
  n_full_ = 2 * n_ub_ - nfree_;
  {
    DevBuf<unsigned long long> fk, fks;
    fk.resize(2 * (size_t)n_ub_);
    fks.resize(2 * (size_t)n_ub_);
    row_ptr_.resize(nfree_ + 1);
    col_idx_.resize(n_full_);
    if (n_ub_) {
      k_full_keys<<<grid_for(n_ub_, 256), 256, 0, s>>>(n_ub_, nfree_, ub_key_.get(), fk.get());
      SFM_CHECK_LAUNCH();
      SFM_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, fk.get(), fks.get(), 2 * n_ub_, 0, 64, s));
      SFM_CUDA(cub::DeviceRadixSort::SortKeys(tmp.get(tb), tb, fk.get(), fks.get(), 2 * n_ub_, 0, 64, s));
    }
    k_bsr_pattern<<<grid_for(std::max(n_full_, nfree_ + 1), 256), 256, 0, s>>>(nfree_, n_full_, fks.get(), row_ptr_.get(), col_idx_.get());
    SFM_CHECK_LAUNCH();
    ub_pos_up_.resize(n_ub_);
    ub_pos_lo_.resize(n_ub_);
    if (n_ub_) { k_ub_map<<<grid_for(n_ub_, 256), 256, 0, s>>>(n_ub_, nfree_, n_full_, ub_key_.get(), fks.get(), ub_pos_up_.get(), ub_pos_lo_.get()); SFM_CHECK_LAUNCH(); }
    SFM_CUDA(cudaStreamSynchronize(s));
  }
  ub_pb_.resize(n_ub_);
  ub_edge_.resize(n_ub_);
  if (n_ub_) {
    SFM_CUDA(cudaMemsetAsync(ub_pb_.get(), 0xff, sizeof(int) * n_ub_, s));
    SFM_CUDA(cudaMemsetAsync(ub_edge_.get(), 0xff, sizeof(int) * n_ub_, s));
  }
  if (n_pb_) { k_scatter_pb<<<grid_for(n_pb_, 256), 256, 0, s>>>(n_pb_, n_ub_, pb_key.get(), ub_key_.get(), ub_pb_.get()); SFM_CHECK_LAUNCH(); }
  std::vector<int> hpb(n_ub_);
  std::vector<int64_t> hptr(n_pb_ + 1);
  if (n_ub_) ub_pb_.download(hpb.data(), n_ub_, s);
  pb_pair_ptr_.download(hptr.data(), n_pb_ + 1, s);
  SFM_CUDA(cudaStreamSynchronize(s));
  edge_ab_.upload(h_ab.data(), h_ab.size(), s);
  prior_frame_.upload(h_pf.data(), h_pf.size(), s);
  if (n_edges_) { k_scatter_edges<<<grid_for(n_edges_, 128), 128, 0, s>>>(n_edges_, nfree_, edge_ab_.get(), free_idx_.get(), n_ub_, ub_key_.get(), ub_edge_.get()); SFM_CHECK_LAUNCH(); }
  // diagonal positions per free camera (upper index and BSR slot)
  {
    std::vector<unsigned long long> hk(n_ub_);
    ub_key_.download(hk.data(), n_ub_, s);
    std::vector<int> hpos(n_ub_);
    ub_pos_up_.download(hpos.data(), n_ub_, s);
    SFM_CUDA(cudaStreamSynchronize(s));
    std::vector<int> dub(nfree_), dpos(nfree_);
    for (int j = 0; j < nfree_; ++j) {
      unsigned long long key = (unsigned long long)j * nfree_ + j;
      auto it = std::lower_bound(hk.begin(), hk.end(), key);
      SFM_REQUIRE(it != hk.end() && *it == key, "internal: missing diagonal block");
      dub[j] = (int)(it - hk.begin());
      dpos[j] = hpos[dub[j]];
    }
    diag_ub_host_ = dub;
    diag_ub_.upload(dub.data(), nfree_, s);
    diag_pos_.upload(dpos.data(), nfree_, s);
  }
  tm.mark("S pattern");
  // Linear solver choice, then the PCG plan (host-side partition of S) on
  // its own thread and stream: it only needs the S pattern, and overlaps
  // the camera-major streams, the pose-term lists and the initial cost.
  int dense_cap = opt_.dense_max_dim > 0 ? std::min(opt_.dense_max_dim, kDenseMax) : kDenseMax;
  if (opt_.linear_solver == SFM_LINSOLVE_DENSE) {
    SFM_REQUIRE(6 * nfree_ <= kDenseMax, "dense solver limited to 6*free_frames <= 210; use PCG");
    use_dense_ = 1;
  } else if (opt_.linear_solver == SFM_LINSOLVE_PCG) {
    use_dense_ = 0;
  } else {
    use_dense_ = (6 * nfree_ <= dense_cap) ? 1 : 0;
  }
  SFM_CUDA(cudaFuncSetAttribute(k_offdiag_blocks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kOffSmem));
  if (use_dense_ && nfree_ > 0) {
    const int n = 6 * nfree_;
    size_t smem = sizeof(double) * (size_t)n * (n + 1) / 2;
    SFM_CUDA(cudaFuncSetAttribute(k_dense_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(smem, 1)));
  }
  std::future<void> plan;
  if (!use_dense_ && nfree_ > 0) {
    if (!plan_stream_) {
      SFM_CUDA(cudaStreamCreateWithFlags(&plan_stream_, cudaStreamNonBlocking));
      SFM_CUDA(cudaEventCreateWithFlags(&plan_ev_, cudaEventDisableTiming));
    }
    SFM_CUDA(cudaEventRecord(plan_ev_, s));  // row_ptr / col are complete here
    int dev = 0;
    SFM_CUDA(cudaGetDevice(&dev));
    const int cl = opt_.coarse_cluster == 0 ? 8 : opt_.coarse_cluster;
    const int refresh = opt_.coarse_refresh > 0 ? opt_.coarse_refresh : 8;
    cudaStream_t ps = plan_stream_;
    cudaEvent_t pe = plan_ev_;
    // row-partitioned PCG: ranks sharing a device, or the devices of one
    // process with peer access (NCCL ranks of separate processes: replicated).
    // Across devices each of the two barriers per iteration costs ~3.7 us
    // more than a grid barrier (measured on one B200, tools/xbar_cost.py)
    // plus the NVLink hop, so it only pays once S no longer fits in L2 and
    // the SpMV it divides is HBM-bound; below that the replicated PCG on
    // the reduced S is faster (scaling model).
    const bool s_beyond_l2 = 288.0 * (double)n_full_ > 100e6;
    partitioned_ = comm_ && comm_->active() && opt_.pcg_partition != 0 &&
                   (comm_->emu != nullptr ||
                    (comm_->host != nullptr && comm_->peer && (s_beyond_l2 || opt_.pcg_partition == 2)));
    if (comm_) comm_->pcg_partition = opt_.pcg_partition;
    plan = std::async(std::launch::async, [this, dev, cl, refresh, ps, pe]() {
      SFM_CUDA(cudaSetDevice(dev));
      alloc_stream() = ps;  // the plan's buffers are stream-ordered on the plan stream
      SFM_CUDA(cudaStreamWaitEvent(ps, pe, 0));
      pcg_.setup(nfree_, cl, refresh, ps);
      if (partitioned_) pcg_.set_partition(comm_->world, comm_->rank);
      pcg_.set_coarse_policy(opt_.coarse_max_lambda > 0.0 ? opt_.coarse_max_lambda : 1e-2,
                             opt_.coarse_drift > 1.0 ? opt_.coarse_drift : 4.0);
      pcg_.set_pattern(row_ptr_.get(), col_idx_.get(), n_full_, ps);  // ends with a sync of ps
    });
  }

  // camera-major observation streams + off-diagonal block list
  {
    std::vector<int64_t> cptr(nfree_ + 1, 0);
    for (int j = 0; j < nfree_; ++j) {
      const int pb = hpb[diag_ub_host_[j]];
      cptr[j + 1] = cptr[j] + (pb < 0 ? 0 : hptr[pb + 1] - hptr[pb]);
    }
    n_cm_ = cptr[nfree_];
    cm_ptr_.upload(cptr.data(), cptr.size(), s);
    SFM_CUDA(cudaStreamWaitEvent(s, side_done_, 0));  // pixels + points resident from here on
    cm_obs_.resize(n_cm_);
    cm_pt_.resize(n_cm_);
    cm_uv_.resize((size_t)n_cm_ * 2);
    geo_cm_.resize(n_cm_);
    cm_pos_.resize(N_);
    if (N_) SFM_CUDA(cudaMemsetAsync(cm_pos_.get(), 0xff, sizeof(int) * N_, s));
    if (nfree_) {
      k_cm_build<<<grid_for((int64_t)nfree_ * 32, 128), 128, 0, s>>>(
          nfree_, diag_ub_.get(), ub_pb_.get(), pb_pair_ptr_.get(), pairs_.get(), cm_ptr_.get(),
          obs_point_.get(), obs_uv_.get(), cm_obs_.get(), cm_pt_.get(), cm_uv_.get(), cm_pos_.get());
      SFM_CHECK_LAUNCH();
    }
    pair_pt_.resize(n_pairs_);
    if (n_pairs_) {
      k_pair_pt<<<grid_for(n_pairs_, 256), 256, 0, s>>>(n_pairs_, pairs_.get(), obs_point_.get(), pair_pt_.get());
      SFM_CHECK_LAUNCH();
    }
    std::vector<unsigned long long> hk(n_ub_);
    if (n_ub_) ub_key_.download(hk.data(), n_ub_, s);
    SFM_CUDA(cudaStreamSynchronize(s));
    std::vector<int> off;
    for (int u = 0; u < n_ub_; ++u)
      if (hk[u] / nfree_ != hk[u] % nfree_) off.push_back(u);
    n_off_ = (int)off.size();
    work_.upload(off.data(), off.size(), s);
    offrec_.resize((size_t)2 * n_off_);
    offk_.resize(n_off_);
    if (n_off_) {
      k_off_records<<<grid_for(n_off_, 256), 256, 0, s>>>(
          n_off_, work_.get(), ub_key_.get(), nfree_, ub_pb_.get(), ub_edge_.get(), ub_pos_up_.get(),
          ub_pos_lo_.get(), free_frame_.get(), frame_model_.get(), pb_pair_ptr_.get(), offrec_.get(), offk_.get());
      SFM_CHECK_LAUNCH();
    }
  }
  tm.mark("camera-major streams");
  // pose terms per free camera (edge side 0 = from/a, 1 = to/b, prior 2)
  {
    std::vector<std::vector<int>> per(nfree_);
    for (int e = 0; e < n_edges_; ++e) {
      int ja = free_idx[h_ab[2 * e]], jb = free_idx[h_ab[2 * e + 1]];
      if (ja >= 0) per[ja].push_back(e << 2 | 0);
      if (jb >= 0) per[jb].push_back(e << 2 | 1);
    }
    for (int a = 0; a < n_priors_; ++a) {
      int j = free_idx[h_pf[a]];
      if (j >= 0) per[j].push_back((n_edges_ + a) << 2 | 2);
    }
    std::vector<int> tp(nfree_ + 1, 0), tl;
    for (int j = 0; j < nfree_; ++j) {
      std::sort(per[j].begin(), per[j].end());
      tp[j + 1] = tp[j] + (int)per[j].size();
      tl.insert(tl.end(), per[j].begin(), per[j].end());
    }
    term_ptr_.upload(tp.data(), tp.size(), s);
    term_list_.upload(tl.data(), tl.size(), s);
  }
  tm.mark("pose-term lists");
  edge_meas_inv_.resize((size_t)n_edges_ * 7);
  prior_init_inv_.resize((size_t)n_priors_ * 7);
  edge_H_.resize((size_t)n_edges_ * 36);
  if (n_edges_ + n_priors_) {
    k_terms_init<<<grid_for(n_edges_ + n_priors_, 128), 128, 0, s>>>(n_edges_, n_priors_, edge_ab_.get(), prior_frame_.get(), q_[0].get(), t_[0].get(), Rt_[0].get(), edge_meas_inv_.get(), prior_init_inv_.get());
    SFM_CHECK_LAUNCH();
  }
  // work buffers
  V_.resize((size_t)P_ * 6);
  gp_.resize((size_t)P_ * 3);
  pv_.resize((size_t)P_ * 12);
  U_.resize((size_t)nfree_ * 36);
  gc_.resize((size_t)nfree_ * 6);
  Dc_.resize((size_t)nfree_ * 6);
  S_.resize((size_t)n_full_ * 36);
  b_.resize((size_t)nfree_ * 6);
  dc_.resize((size_t)nfree_ * 6);
  part_a_.resize(grid_for(std::max<int64_t>(P_, 1), kBlock));
  part_b_.resize(grid_for(std::max<int64_t>(P_, 1), kBlock));
  part_c_.resize(grid_for(std::max(n_edges_ + n_priors_, 1), kBlock));
  part_d_.resize(grid_for(std::max(nfree_, 1), kBlock));

  if (plan.valid()) plan.get();  // the PCG plan built on its own thread (rethrows its errors)
  if (partitioned_) {
    coll_.reset(new CommPcgCollective(comm_));
    const auto& rr = pcg_.rank_rows();
    const auto& rb = pcg_.rank_blocks();
    s_off_.assign(rb.begin(), rb.end());
    b_off_.assign(rr.begin(), rr.end());
    for (auto& v : s_off_) v *= 36;
    for (auto& v : b_off_) v *= 6;
  }

  tm.mark("terms + buffers + pcg plan");
  // all_fixed (solver.py:200-203) and the initial cost (solver.py:201)
  int has_res = (N_ > 0 || n_edges_ > 0 || n_priors_ > 0) ? 1 : 0;
  if (comm_ && comm_->active()) {
    DevBuf<int> hr;
    hr.upload(&has_res, 1, s);
    comm_->max_i32(hr.get(), 1, s);
    hr.download(&has_res, 1, s);
    SFM_CUDA(cudaStreamSynchronize(s));
  }
  has_residuals_ = has_res != 0;
  iters_ = 0;
  n_trials_ = 0;
  pcg_total_ = 0;
  pcg_stagnated_ = 0;
  pcg_max_hit_ = 0;
  term_ = SFM_TERM_MAX_ITERATIONS;
  lam_ = opt_.initial_lambda;
  initial_cost_ = eval_cost_current();
  tm.mark("initial cost");
  cost_ = initial_cost_;
  finished_ = false;
  if (n_params_ == 0 || !has_residuals_) {
    term_ = SFM_TERM_ALL_FIXED;
    finished_ = true;
  } else if (opt_.max_iters <= 0) {
    finished_ = true;
  }
}

void BASolver::save_entry() {
  cudaStream_t s = stream_;
  q0_.resize((size_t)F_ * 4);
  t0_.resize((size_t)F_ * 3);
  X0_.resize((size_t)P_ * 3);
  if (F_) {
    SFM_CUDA(cudaMemcpyAsync(q0_.get(), q_[cur_].get(), q0_.bytes(), cudaMemcpyDeviceToDevice, s));
    SFM_CUDA(cudaMemcpyAsync(t0_.get(), t_[cur_].get(), t0_.bytes(), cudaMemcpyDeviceToDevice, s));
  }
  if (P_) SFM_CUDA(cudaMemcpyAsync(X0_.get(), X_[cur_].get(), X0_.bytes(), cudaMemcpyDeviceToDevice, s));
}

void BASolver::restart() {
  NvtxRange nv("sfm restart");
  SFM_REQUIRE(q0_.n == (size_t)F_ * 4 && X0_.n == (size_t)P_ * 3, "restart without a saved entry state");
  cudaStream_t s = stream_;
  cur_ = 0;
  if (F_) {
    SFM_CUDA(cudaMemcpyAsync(q_[0].get(), q0_.get(), q0_.bytes(), cudaMemcpyDeviceToDevice, s));
    SFM_CUDA(cudaMemcpyAsync(t_[0].get(), t0_.get(), t0_.bytes(), cudaMemcpyDeviceToDevice, s));
    k_frames_rt<<<grid_for(F_, 128), 128, 0, s>>>(F_, q_[0].get(), t_[0].get(), Rt_[0].get(), qt_[0].get());
    SFM_CHECK_LAUNCH();
  }
  if (P_) SFM_CUDA(cudaMemcpyAsync(X_[0].get(), X0_.get(), X0_.bytes(), cudaMemcpyDeviceToDevice, s));
  prep_ready_ = false;
  prep_done_lam_ = -1.0;
  prep_folded_ = false;
  last_pcg_ = -1;
  imp_iters_ = 0;
  pcg_.restart();
  iters_ = 0;
  n_trials_ = 0;
  pcg_total_ = 0;
  pcg_stagnated_ = 0;
  pcg_max_hit_ = 0;
  term_ = SFM_TERM_MAX_ITERATIONS;
  lam_ = opt_.initial_lambda;
  initial_cost_ = eval_cost_current();
  cost_ = initial_cost_;
  finished_ = false;
  if (n_params_ == 0 || !has_residuals_) {
    term_ = SFM_TERM_ALL_FIXED;
    finished_ = true;
  } else if (opt_.max_iters <= 0) {
    finished_ = true;
  }
}

// The one host synchronisation of a trial (the accept / reject decision is
// the host's, solver.py:236-245): 128 bytes D2H into pinned memory.
void BASolver::read_scalars() {
  if (!h_pin_) SFM_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h_pin_), sizeof(BAScalars)));
  SFM_CUDA(cudaMemcpyAsync(h_pin_, sc_.get(), sizeof(BAScalars), cudaMemcpyDeviceToHost, stream_));
  SFM_CUDA(cudaStreamSynchronize(stream_));
  h_sc_ = *h_pin_;
}

// Raises NonPositiveDepth / OutOfModelDomain for the first offending
// observation in residual order (solver.py:235 -> cameras.py:132-133).
void BASolver::raise_projection_error(bool trial_state) {
  const unsigned long long g = h_sc_.depth_obs;
  const int64_t local = (int64_t)g - obs_offset_;
  char msg[160];
  int code = SFM_E_NON_POSITIVE_DEPTH;
  if (local >= 0 && local < N_) {
    const int other = cur_ ^ 1;
    const double* Rt = trial_state ? Rt_[other].get() : Rt_[cur_].get();
    const double* X = trial_state ? X_[other].get() : X_[cur_].get();
    k_probe_obs<<<1, 1, 0, stream_>>>(local, obs_frame_.get(), obs_point_.get(), obs_uv_.get(), frame_model_.get(), models_.get(), Rt, X, sc_.get());
    SFM_CHECK_LAUNCH();
    read_scalars();
    if (h_sc_.proj_code == PROJ_DOMAIN) {
      code = SFM_E_OUT_OF_MODEL_DOMAIN;
      std::snprintf(msg, sizeof(msg), "incidence angle beyond model domain (observation %lld)", (long long)g);
    } else {
      std::snprintf(msg, sizeof(msg), "depth %.3e", h_sc_.proj_depth);
    }
  } else {
    std::snprintf(msg, sizeof(msg), "depth of observation %lld (remote shard) not positive", (long long)g);
  }
  throw SfmError(code, msg);
}

double BASolver::eval_cost_current() {
  cudaStream_t s = stream_;
  k_reset_scalars<<<1, 1, 0, s>>>(sc_.get(), 0);
  SFM_CHECK_LAUNCH();
  PointArgs pa{};
  pa.P = P_; pa.lk = opt_.loss_kind; pa.lp = opt_.loss_param;
  pa.ptr = pt_ptr_.get(); pa.of = obs_frame_.get(); pa.uv = obs_uv_.get();
  pa.frame_model = frame_model_.get(); pa.models = models_.get(); pa.nmodels = nmodels_;
  pa.free_idx = free_idx_.get();
  pa.Rt = Rt_[cur_].get(); pa.X = X_[cur_].get(); pa.Rt_eval = Rt_[cur_].get();
  pa.qt = qt_[cur_].get(); pa.qt_eval = qt_[cur_].get();
  pa.obs_offset = obs_offset_; pa.part_cost = part_a_.get(); pa.part_dp2 = part_b_.get(); pa.sc = sc_.get();
  const unsigned gp = grid_for(std::max<int64_t>(P_, 1), kBlock);
  {
    ProfScope ps(*prof_, "point_cost", 24.0 * N_ + 24.0 * P_, s);
    k_point_cost<false><<<gp, kBlock, 0, s>>>(pa);
  }
  const int T = n_edges_ + n_priors_;
  const unsigned gt = grid_for(std::max(T, 1), kBlock);
  {
    ProfScope ps(*prof_, "terms_cost", 0.0, s);
    k_terms_cost<<<gt, kBlock, 0, s>>>(n_edges_, n_priors_, edge_ab_.get(), prior_frame_.get(), edge_meas_inv_.get(), prior_init_inv_.get(), edge_w_, prior_w_, q_[cur_].get(), t_[cur_].get(), Rt_[cur_].get(), part_c_.get());
  }
  {
    ProfScope ps(*prof_, "finalize", 0.0, s);
    k_finalize<<<1, 256, 0, s>>>(part_a_.get(), (int)gp, nullptr, 0, part_c_.get(), (int)gt, nullptr, 0, sc_.get(), 0);
  }
  if (comm_ && comm_->active()) {
    comm_->sum(&sc_.get()->cost, 1, s);
    comm_->min_u64(&sc_.get()->depth_obs, 1, s);
  }
  read_scalars();
  if (h_sc_.depth_obs != ~0ull) raise_projection_error(false);
  return h_sc_.cost;
}

void BASolver::linearize() {
  NvtxRange nv("sfm linearize");
  cudaStream_t s = stream_;
  last_pcg_ = -1;
  k_reset_scalars<<<1, 1, 0, s>>>(sc_.get(), 0);
  SFM_CHECK_LAUNCH();
  PointArgs pa{};
  pa.P = P_; pa.lk = opt_.loss_kind; pa.lp = opt_.loss_param;
  pa.ptr = pt_ptr_.get(); pa.of = obs_frame_.get(); pa.uv = obs_uv_.get();
  pa.frame_model = frame_model_.get(); pa.models = models_.get(); pa.nmodels = nmodels_;
  pa.free_idx = free_idx_.get();
  pa.Rt = Rt_[cur_].get(); pa.X = X_[cur_].get(); pa.sc = sc_.get(); pa.geo = geo_.get();
  pa.qt = qt_[cur_].get();
  pa.cm_pos = cm_pos_.get(); pa.geo_cm = geo_cm_.get();
  if (P_) {
    // compulsory: observation records in, points in, V/g_p and the 32-byte
    // linearisation record per observation out
    prep_ready_ = nfree_ > 0;
    if (prep_ready_) {
      sc_pre_.resize(1);
      SFM_CUDA(cudaMemsetAsync(sc_pre_.get(), 0, sizeof(BAScalars), s));
      pa.lam = lam_;
      pa.pv_out = pv_.get();
      pa.sc_pre = sc_pre_.get();
      prep_lam_ = lam_;
    }
    // + the camera-major copy of the record (32 B) and its slot (4 B) per
    // observation in a free camera, which this design writes here
    ProfScope ps(*prof_, "point_lin", 24.0 * N_ + 24.0 * P_ + 72.0 * P_ + 32.0 * N_ + 36.0 * n_cm_ +
                                          (prep_ready_ ? 96.0 * P_ : 0.0), s);
    k_point_lin<<<grid_for(P_, kBlock), kBlock, 0, s>>>(pa, V_.get(), gp_.get());
  }
  if (nfree_) {
    BlkArgs ba = blk_args(0.0);
    ba.Uout = U_.get();
    ba.gout = gc_.get();
    // compulsory: camera-major linearisation record (32 B) + pixel (16 B)
    // per observation; U, g_c out
    ProfScope ps(*prof_, "cam_lin", 48.0 * n_cm_ + 336.0 * nfree_, s);
    if (SFM_CAM_FMA)
      k_cam_fma<0><<<nfree_, kCamWarps * 32, 0, s>>>(ba);
    else
      k_cam_blocks<0><<<nfree_, kCamWarps * 32, 0, s>>>(ba);
  }
  if (nfree_) {
    CamArgs c{};
    c.nf = nfree_;
    c.term_ptr = term_ptr_.get(); c.term_list = term_list_.get(); c.ab = edge_ab_.get();
    c.pf = prior_frame_.get(); c.E = n_edges_; c.meas_inv = edge_meas_inv_.get();
    c.init_inv = prior_init_inv_.get(); c.we = edge_w_; c.wa = prior_w_;
    c.q = q_[cur_].get(); c.t = t_[cur_].get(); c.Rt = Rt_[cur_].get(); c.U = U_.get(); c.gc = gc_.get();
    if (n_edges_ + n_priors_) {
      ProfScope ps(*prof_, "cam_terms", 0.0, s);
      term_contrib_.resize((size_t)(2 * n_edges_ + n_priors_) * 42);
      k_terms_lin<<<grid_for(n_edges_ + n_priors_, 32), 32, 0, s>>>(
          n_edges_, n_priors_, edge_ab_.get(), prior_frame_.get(), free_idx_.get(), edge_meas_inv_.get(),
          prior_init_inv_.get(), edge_w_, prior_w_, c.q, c.t, c.Rt, term_contrib_.get(), edge_H_.get());
      k_cam_terms_sum<<<grid_for(nfree_, 64), 64, 0, s>>>(c, term_contrib_.get());
    }
    if (comm_ && comm_->active()) {
      comm_->sum(U_.get(), (size_t)nfree_ * 36, s);
      comm_->sum(gc_.get(), (size_t)nfree_ * 6, s);
    }
    {
      ProfScope ps(*prof_, "cam_post", 0.0, s);
      k_cam_post<<<grid_for(nfree_, 128), 128, 0, s>>>(nfree_, U_.get(), gc_.get(), Dc_.get(), sc_.get());
    }
  }
  if (!use_dense_ && nfree_)
    pcg_.set_basis(free_frame_.get(), q_[cur_].get(), t_[cur_].get(), Rt_[cur_].get(), s, prof_);
  if (comm_ && comm_->active()) comm_->max_u64(&sc_.get()->gmax, 1, s);
  read_scalars();
}

BlkArgs BASolver::blk_args(double lam) const {
  BlkArgs ba{};
  ba.work = work_.get(); ba.nf = nfree_; ba.rank = rank_; ba.lam = lam;
  ba.offrec = offrec_.get(); ba.offk = offk_.get();
  ba.sc = sc_.get();
  ba.ub_key = ub_key_.get(); ba.ub_pb = ub_pb_.get(); ba.ub_edge = ub_edge_.get();
  ba.pos_up = ub_pos_up_.get(); ba.pos_lo = ub_pos_lo_.get(); ba.diag_ub = diag_ub_.get();
  ba.pb_pair_ptr = pb_pair_ptr_.get(); ba.pairs = pairs_.get(); ba.op = obs_point_.get();
  ba.of = obs_frame_.get(); ba.uv = obs_uv_.get(); ba.free_frame = free_frame_.get();
  ba.frame_model = frame_model_.get(); ba.models = models_.get(); ba.Rt = Rt_[cur_].get();
  ba.geo = geo_.get(); ba.pv = pv_.get(); ba.pair_pt = pair_pt_.get(); ba.cm_ptr = cm_ptr_.get();
  ba.cm_pt = cm_pt_.get(); ba.cm_uv = cm_uv_.get(); ba.geo_cm = geo_cm_.get(); ba.diag_pos = diag_pos_.get();
  ba.U = U_.get(); ba.Dc = Dc_.get();
  ba.gc = gc_.get(); ba.edge_H = edge_H_.get(); ba.S = S_.get(); ba.b = b_.get();
  return ba;
}

// V*^-1 and e per point for this trial's lambda (skipped when k_point_lin
// already prepared them for it).
void BASolver::point_prep(double lam) {
  cudaStream_t s = stream_;
  if (prep_done_lam_ == lam) return;
  const bool prepped = prep_ready_ && lam == prep_lam_ && nfree_ > 0;
  prep_ready_ = false;
  prep_folded_ = prepped;
  if (P_ && !prepped) {
    ProfScope ps(*prof_, "point_prep", 72.0 * P_ + 96.0 * P_, s);
    k_point_prep<<<grid_for(P_, 256), 256, 0, s>>>(P_, lam, V_.get(), gp_.get(), pv_.get(), sc_.get());
  }
  prep_done_lam_ = lam;
}

void BASolver::build_schur(double lam) {
  NvtxRange nv("sfm schur");
  cudaStream_t s = stream_;
  point_prep(lam);
  const bool prepped = prep_folded_;
  if (nfree_) {
    BlkArgs ba = blk_args(lam);
    ba.pre = prepped ? sc_pre_.get() : nullptr;
    // compulsory: camera-major record + point id per observation, packed
    // point record (V*^-1, e), diagonal blocks and b out
    ProfScope ps(*prof_, "schur_diag", (32.0 + 4.0) * n_cm_ + 96.0 * P_ + 336.0 * nfree_, s);
    if (SFM_CAM_FMA)
      k_cam_fma<1><<<nfree_, kCamWarps * 32, 0, s>>>(ba);
    else
      k_cam_blocks<1><<<nfree_, kCamWarps * 32, 0, s>>>(ba);
  }
  if (n_off_) {
    BlkArgs ba = blk_args(lam);
    ba.n = n_off_;
    // compulsory: off-diagonal pair list (8 B) + pair point (4 B), both
    // observation records, point V*^-1 once; both triangles of S out
    ProfScope ps(*prof_, "schur_offdiag",
                 12.0 * (n_pairs_ - n_cm_) + 32.0 * N_ + 48.0 * P_ + 288.0 * (n_full_ - nfree_), s);
    k_offdiag_blocks<<<grid_for((int64_t)n_off_ * 32, kOffWarps * 32), kOffWarps * 32, kOffSmem, s>>>(ba);
  }
  if (comm_ && comm_->active()) {
    if (partitioned_) {  // each rank keeps only the block rows it solves for
      comm_->reduce_ranges(S_.get(), s_off_, s);
      comm_->reduce_ranges(b_.get(), b_off_, s);
    } else {
      comm_->sum(S_.get(), (size_t)n_full_ * 36, s);
      comm_->sum(b_.get(), (size_t)nfree_ * 6, s);
    }
  }
}

bool BASolver::solve_reduced(double lam) {
  cudaStream_t s = stream_;
  if (nfree_ == 0) return true;
  if (use_dense_) {
    const int n = 6 * nfree_;
    size_t smem = sizeof(double) * (size_t)n * (n + 1) / 2;
    ProfScope ps(*prof_, "dense_solve", 0.0, s);
    k_dense_solve<<<1, 1024, smem, s>>>(nfree_, row_ptr_.get(), col_idx_.get(), S_.get(), b_.get(), dc_.get(), sc_.get());
    return true;
  }
  PcgProblem pp{};
  pp.nf = nfree_; pp.row_ptr = row_ptr_.get(); pp.col = col_idx_.get(); pp.S = S_.get(); pp.nnzb = n_full_;
  pp.diag_pos = diag_pos_.get(); pp.b = b_.get(); pp.x = dc_.get(); pp.lam = lam;
  pcg_.solve(pp, opt_.pcg_max_iters > 0 ? opt_.pcg_max_iters : 1000, opt_.pcg_rtol > 0 ? opt_.pcg_rtol : 1e-10,
             sc_.get(), s, prof_, partitioned_ ? coll_.get() : nullptr);
  if (partitioned_) comm_->allgather_ranges(dc_.get(), b_off_, s);  // every rank's cameras need all of dc
  return true;
}

bool BASolver::solve_implicit(double lam) {
  cudaStream_t s = stream_;
  const int n = 6 * nfree_;
  imp_s_.resize((size_t)P_ * 3);
  imp_r_.resize(n); imp_z_.resize(n); imp_p_.resize(n); imp_q_.resize(n); imp_b_.resize(n);
  imp_M_.resize((size_t)nfree_ * 36);
  imp_st_.resize(1);
  SFM_CUDA(cudaMemsetAsync(imp_st_.get(), 0, sizeof(ImpState), s));
  const double rtol = opt_.pcg_rtol > 0 ? opt_.pcg_rtol : 1e-10;
  ImpCamArgs ca{};
  ca.nf = nfree_; ca.rank = rank_; ca.lam = lam; ca.free_frame = free_frame_.get();
  ca.frame_model = frame_model_.get(); ca.models = models_.get(); ca.Rt = Rt_[cur_].get();
  ca.cm_ptr = cm_ptr_.get(); ca.cm_pt = cm_pt_.get(); ca.geo_cm = geo_cm_.get();
  ca.U = U_.get(); ca.Dc = Dc_.get(); ca.gc = gc_.get(); ca.term_ptr = term_ptr_.get();
  ca.term_list = term_list_.get(); ca.E = n_edges_; ca.edge_ab = edge_ab_.get(); ca.free_idx = free_idx_.get();
  ca.edge_H = edge_H_.get(); ca.st = imp_st_.get();
  {  // b = -g_c + sum_a W_a e_i
    ProfScope ps(*prof_, "imp_cam", 36.0 * n_cm_ + 24.0 * P_ + 96.0 * nfree_, s);
    ca.mode = 0; ca.v = pv_.get(); ca.vstride = 12; ca.voff = 6; ca.pvec = nullptr; ca.out = imp_b_.get();
    k_imp_cam<<<nfree_, kImpWarps * 32, 0, s>>>(ca);
  }
  {
    ProfScope ps(*prof_, "imp_update", 0.0, s);
    k_imp_precond<<<grid_for(nfree_, 64), 64, 0, s>>>(nfree_, U_.get(), Dc_.get(), lam, imp_M_.get(), imp_st_.get());
    k_imp_init<<<1, 1024, 0, s>>>(n, imp_b_.get(), imp_M_.get(), dc_.get(), imp_r_.get(), imp_z_.get(),
                                  imp_p_.get(), imp_st_.get());
  }
  constexpr int kChunk = 4, kMaxIt = 12;
  ImpState h{};
  // iterations are enqueued in chunks with one host check each (a converged
  // solve turns the rest of its chunk into early-exit launches); the first
  // chunk is as long as the previous trial needed (<= 3: why this path was
  // taken), so a tail trial of 1-2 iterations launches 1-2 rounds, not 4
  int chunk = std::max(1, std::min(kChunk, last_pcg_));
  for (int done_it = 0; done_it < kMaxIt; done_it += chunk, chunk = kChunk) {
    for (int k = 0; k < chunk && done_it + k < kMaxIt; ++k) {
      {
        ProfScope ps(*prof_, "imp_point", 36.0 * N_ + 136.0 * P_, s);
        k_imp_point<<<grid_for(std::max<int64_t>(P_, 1), kBlock), kBlock, 0, s>>>(
            P_, pt_ptr_.get(), obs_frame_.get(), free_idx_.get(), frame_model_.get(), models_.get(), nmodels_,
            Rt_[cur_].get(), qt_[cur_].get(), geo_.get(), pv_.get(), imp_p_.get(), imp_s_.get(), imp_st_.get());
      }
      {
        ProfScope ps(*prof_, "imp_cam", 60.0 * n_cm_ + 96.0 * nfree_, s);
        ca.mode = 1; ca.v = imp_s_.get(); ca.vstride = 3; ca.voff = 0; ca.pvec = imp_p_.get(); ca.out = imp_q_.get();
        k_imp_cam<<<nfree_, kImpWarps * 32, 0, s>>>(ca);
      }
      {
        ProfScope ps(*prof_, "imp_update", 0.0, s);
        k_imp_step<<<1, 1024, 0, s>>>(n, imp_q_.get(), imp_M_.get(), rtol, kMaxIt, dc_.get(), imp_r_.get(),
                                      imp_z_.get(), imp_p_.get(), imp_st_.get());
      }
    }
    imp_st_.download(&h, 1, s);
    SFM_CUDA(cudaStreamSynchronize(s));
    if (h.done) break;
  }
  imp_iters_ = h.it;
  return h.done == 1;
}

// One LM trial at damping lam (solver.py:220-235).  Returns false when the
// step is not finite (the reference then multiplies lambda by 10 without
// evaluating the cost).
bool BASolver::trial(double lam, double* new_cost, double* step_norm) {
  NvtxRange nv("sfm trial");
  cudaStream_t s = stream_;
  k_reset_scalars<<<1, 1, 0, s>>>(sc_.get(), 1);
  SFM_CHECK_LAUNCH();
  prep_done_lam_ = -1.0;
  // Matrix-free Schur PCG when the previous trial of this linearisation
  // needed at most 3 PCG iterations (S strongly diagonally dominant at this
  // damping); the explicit S otherwise, or if it does not converge.
  const bool try_imp = imp_enabled_ && !use_dense_ && nfree_ > 0 && !(comm_ && comm_->active()) &&
                       last_pcg_ >= 0 && last_pcg_ <= 3 && !(prep_ready_ && lam == prep_lam_);
  bool imp_ok = false;
  if (try_imp) {
    point_prep(lam);
    imp_ok = solve_implicit(lam);
    ++imp_trials_;
  }
  if (!imp_ok) {
    build_schur(lam);
    solve_reduced(lam);
  }
  const int o = cur_ ^ 1;
  const unsigned gd = grid_for(std::max(nfree_, 1), kBlock);
  if (nfree_) {
    ProfScope ps(*prof_, "cam_trial", 0.0, s);
    k_cam_trial<<<gd, kBlock, 0, s>>>(nfree_, free_frame_.get(), dc_.get(), q_[cur_].get(), t_[cur_].get(), Rt_[cur_].get(), q_[o].get(), t_[o].get(), Rt_[o].get(), qt_[o].get(), part_d_.get(), sc_.get());
  }
  PointArgs pa{};
  pa.P = P_; pa.lk = opt_.loss_kind; pa.lp = opt_.loss_param;
  pa.ptr = pt_ptr_.get(); pa.of = obs_frame_.get(); pa.uv = obs_uv_.get();
  pa.frame_model = frame_model_.get(); pa.models = models_.get(); pa.nmodels = nmodels_;
  pa.free_idx = free_idx_.get();
  pa.Rt = Rt_[cur_].get(); pa.X = X_[cur_].get(); pa.Rt_eval = Rt_[o].get(); pa.X_out = X_[o].get();
  pa.qt = qt_[cur_].get(); pa.qt_eval = qt_[o].get();
  pa.pv = pv_.get(); pa.dc = dc_.get(); pa.geo = geo_.get();
  pa.obs_offset = obs_offset_; pa.part_cost = part_a_.get(); pa.part_dp2 = part_b_.get(); pa.sc = sc_.get();
  const unsigned gp = grid_for(std::max<int64_t>(P_, 1), kBlock);
  {
    // compulsory: observation records + linearisation records, point state
    // (X, V*^-1, e) in, trial points out
    ProfScope ps(*prof_, "point_trial", 24.0 * N_ + 32.0 * N_ + (24.0 + 72.0 + 24.0) * P_, s);
    k_point_cost<true><<<gp, kBlock, 0, s>>>(pa);
  }
  const int T = n_edges_ + n_priors_;
  const unsigned gt = grid_for(std::max(T, 1), kBlock);
  {
    ProfScope ps(*prof_, "terms_cost", 0.0, s);
    k_terms_cost<<<gt, kBlock, 0, s>>>(n_edges_, n_priors_, edge_ab_.get(), prior_frame_.get(), edge_meas_inv_.get(), prior_init_inv_.get(), edge_w_, prior_w_, q_[o].get(), t_[o].get(), Rt_[o].get(), part_c_.get());
  }
  {
    ProfScope ps(*prof_, "finalize", 0.0, s);
    k_finalize<<<1, 256, 0, s>>>(part_a_.get(), (int)gp, part_b_.get(), (int)gp, part_c_.get(), (int)gt, part_d_.get(), nfree_ ? (int)gd : 0, sc_.get(), 1);
  }
  if (comm_ && comm_->active()) {
    comm_->sum(&sc_.get()->cost, 2, s);  // cost, dp2
    comm_->min_u64(&sc_.get()->depth_obs, 1, s);
    comm_->max_i32(&sc_.get()->nonfinite, 1, s);
  }
  read_scalars();
  if (imp_ok) {
    h_sc_.pcg_iters = imp_iters_;
    h_sc_.pcg_stop = PCG_STOP_CONVERGED;
  } else if (try_imp) {
    h_sc_.pcg_iters += imp_iters_;
  }
  last_pcg_ = use_dense_ ? -1 : h_sc_.pcg_iters;
  pcg_total_ += h_sc_.pcg_iters;
  if (!use_dense_ && nfree_) {
    pcg_stagnated_ += h_sc_.pcg_stop == PCG_STOP_STAGNATED;
    pcg_max_hit_ += h_sc_.pcg_stop == PCG_STOP_MAX_ITERS;
  }
  if (!use_dense_ && nfree_ && !imp_ok)  // S read + 7 length-6nf vectors touched per PCG iteration
    prof_->add_bytes("pcg", (double)(h_sc_.pcg_iters - (try_imp ? imp_iters_ : 0)) *
                                (288.0 * n_full_ + 7.0 * 48.0 * nfree_));
  if (h_sc_.nonfinite) return false;
  if (h_sc_.depth_obs != ~0ull) raise_projection_error(true);
  *new_cost = h_sc_.cost;
  *step_norm = std::sqrt(h_sc_.dc2 + h_sc_.dp2);
  return true;
}

void BASolver::iterate(int n, sfm_ba_report* rep) {
  cudaEvent_t e0, e1;
  SFM_CUDA(cudaEventCreate(&e0));
  SFM_CUDA(cudaEventCreate(&e1));
  SFM_CUDA(cudaEventRecord(e0, stream_));
  const int64_t launches0 = prof_->launches;
  int done = 0;
  while (!finished_ && done < n) {
    ++iters_;
    ++done;
    linearize();
    const double gmax = __longlong_as_double_host(h_sc_.gmax);
    if (gmax < opt_.grad_tol) {  // solver.py:212-215
      term_ = SFM_TERM_GRADIENT_TOLERANCE;
      --iters_;
      finished_ = true;
      break;
    }
    bool accepted = false;
    double step_norm = 0.0;
    while (lam_ <= opt_.max_lambda) {  // solver.py:219-245
      double nc = 0.0, sn = 0.0;
      ++n_trials_;
      const bool ok = trial(lam_, &nc, &sn);
      if (trace_)
        std::fprintf(stderr, "[sfm trial] it=%d lam=%.3e pcg=%d stop=%d ok=%d cost=%.17g cur=%.17g acc=%d\n", iters_, lam_,
                     h_sc_.pcg_iters, h_sc_.pcg_stop, (int)ok, nc, cost_, (int)(ok && std::isfinite(nc) && nc < cost_));
      if (!ok) {
        lam_ *= 10.0;
        continue;
      }
      if (std::isfinite(nc) && nc < cost_) {
        cur_ ^= 1;  // commit the trial state
        cost_ = nc;
        step_norm = sn;
        lam_ = std::max(lam_ * 0.5, 1e-18);
        accepted = true;
        break;
      }
      lam_ *= 10.0;
    }
    if (!accepted) {  // solver.py:246-250
      if (lam_ > opt_.max_lambda && cost_ > initial_cost_)
        throw SfmError(SFM_E_SOLVER_DIVERGED, "damping overflow at cost " + std::to_string(cost_));
      term_ = SFM_TERM_NO_DECREASE;
      finished_ = true;
      break;
    }
    if (step_norm < opt_.param_tol * (std::sqrt((double)n_params_) + opt_.param_tol)) {
      term_ = SFM_TERM_PARAMETER_TOLERANCE;
      finished_ = true;
      break;
    }
    if (cost_ < 1e-30) {
      term_ = SFM_TERM_COST_ZERO;
      finished_ = true;
      break;
    }
    if (iters_ >= opt_.max_iters) finished_ = true;
  }
  SFM_CUDA(cudaEventRecord(e1, stream_));
  SFM_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  SFM_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  prof_->flush();
  if (rep) {
    rep->initial_cost = initial_cost_;
    rep->final_cost = cost_;
    rep->iterations = iters_;
    rep->termination = term_;
    rep->n_trials = n_trials_;
    rep->pcg_iterations = pcg_total_;
    rep->final_lambda = lam_;
    rep->device_ms = ms;
    rep->kernel_launches = prof_->launches - launches0;
    rep->n_blocks_S = n_full_;
    rep->pcg_stagnated = pcg_stagnated_;
    rep->pcg_max_hit = pcg_max_hit_;
  }
}

void BASolver::download(double* q, double* t, double* X) {
  if (q) q_[cur_].download(q, (size_t)F_ * 4, stream_);
  if (t) t_[cur_].download(t, (size_t)F_ * 3, stream_);
  if (X) X_[cur_].download(X, (size_t)P_ * 3, stream_);
  SFM_CUDA(cudaStreamSynchronize(stream_));
}

void BASolver::eval(cudaStream_t s, Profiler* prof, const sfm_ba_problem& pr, int lk, double lp,
                    double* cost, double* res, double* jc, double* jp) {
  const int64_t N = pr.n_obs;
  DevBuf<sfm_camera_model> models;
  DevBuf<int> fm, of, op;
  DevBuf<double> q, t, Rt, X, uv, dcost, dres, djc, djp;
  DevBuf<BAScalars> sc;
  models.upload(pr.models, pr.n_models, s);
  fm.upload(pr.frame_model, pr.n_frames, s);
  q.upload(pr.cam_q, (size_t)pr.n_frames * 4, s);
  t.upload(pr.cam_t, (size_t)pr.n_frames * 3, s);
  Rt.resize((size_t)pr.n_frames * 12);
  if (pr.n_frames) { k_frames_rt<<<grid_for(pr.n_frames, 128), 128, 0, s>>>(pr.n_frames, q.get(), t.get(), Rt.get(), nullptr); SFM_CHECK_LAUNCH(); }
  X.upload(pr.points, (size_t)pr.n_points * 3, s);
  of.upload(pr.obs_frame, N, s);
  op.upload(pr.obs_point, N, s);
  uv.upload(pr.obs_uv, (size_t)N * 2, s);
  dcost.resize(N); dres.resize(N * 2); djc.resize(N * 12); djp.resize(N * 6);
  sc.resize(1);
  k_reset_scalars<<<1, 1, 0, s>>>(sc.get(), 1);
  SFM_CHECK_LAUNCH();
  if (N) {
    ProfScope ps(*prof, "eval_obs", 0.0, s);
    k_eval_obs<<<grid_for(N, 128), 128, 0, s>>>(N, lk, lp, of.get(), op.get(), uv.get(), fm.get(), models.get(), Rt.get(), X.get(), dcost.get(), dres.get(), djc.get(), djp.get(), sc.get());
  }
  BAScalars h{};
  sc.download(&h, 1, s);
  SFM_CUDA(cudaStreamSynchronize(s));
  if (h.depth_obs != ~0ull) {
    char msg[96];
    std::snprintf(msg, sizeof(msg), "projection failed at observation %llu", h.depth_obs);
    throw SfmError(SFM_E_NON_POSITIVE_DEPTH, msg);
  }
  if (cost) dcost.download(cost, N, s);
  if (res) dres.download(res, N * 2, s);
  if (jc) djc.download(jc, N * 12, s);
  if (jp) djp.download(jp, N * 6, s);
  SFM_CUDA(cudaStreamSynchronize(s));
}

#include "gba_impl.cuh"

}  // namespace sfm
