// pcg.cu -- two-level preconditioned CG on the reduced camera system
// (see pcg.cuh).  sm_100a, fp64, deterministic.
#include <cooperative_groups.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <array>
#include <cstdlib>
#include <vector>

#include "ba.cuh"
#include "pcg.cuh"
#include "sfm_math.cuh"

namespace cg = cooperative_groups;

namespace sfm {

namespace {

constexpr int kNB = 48;          // Gauss-Jordan tile
#ifndef SFM_GJ_SYM
#define SFM_GJ_SYM 1  // upper-tile Gauss-Jordan on the symmetric coarse operator
#endif
constexpr int kGJThreads = 256;
#ifndef SFM_PCG_MAXT
#define SFM_PCG_MAXT 512
#endif
constexpr int kPcgMaxThreads = SFM_PCG_MAXT;  // CTA size chosen at setup (512 or 1024)
#define kPcgThreads ((int)blockDim.x)
#define kPcgWarps ((int)(blockDim.x >> 5))

// Block-Jacobi: inverse of each 6x6 diagonal block of S (Cholesky).
__global__ void k_block_jacobi(int r0, int r1, const int* __restrict__ diag_pos, const double* __restrict__ S,
                               double* __restrict__ Minv, BAScalars* sc) {
  int j = r0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= r1) return;
  const double* Ag = S + (int64_t)diag_pos[j] * 36;
  double A[36];
#pragma unroll
  for (int i = 0; i < 36; ++i) A[i] = __ldg(Ag + i);
  const bool ok = spd6_inverse(A, Minv + (int64_t)j * 36);
  if (!ok) atomicOr(&sc->nonfinite, 1);
}

// Centroid of cluster k's camera centres C_j = -R_j^T t_j (frames
// [cluster_row0[k], cluster_row0[k+1])), in frame order.
__global__ void k_cluster_centroid(int nc, const int* __restrict__ cluster_row0, const int* __restrict__ free_frame,
                                   const double* __restrict__ t, const double* __restrict__ Rt, double* __restrict__ cen) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nc) return;
  double sx = 0.0, sy = 0.0, sz = 0.0;
  const int j0 = cluster_row0[k], j1 = cluster_row0[k + 1];
  for (int j = j0; j < j1; ++j) {
    const int f = free_frame[j];
    const double* R = Rt + (int64_t)f * 12;
    const double tx = t[f * 3], ty = t[f * 3 + 1], tz = t[f * 3 + 2];
    sx -= R[0] * tx + R[3] * ty + R[6] * tz;
    sy -= R[1] * tx + R[4] * ty + R[7] * tz;
    sz -= R[2] * tx + R[5] * ty + R[8] * tz;
  }
  const double inv = j1 > j0 ? 1.0 / (j1 - j0) : 0.0;
  cen[k * 3] = sx * inv;
  cen[k * 3 + 1] = sy * inv;
  cen[k * 3 + 2] = sz * inv;
}

// Camera j's coarse basis, row-major 6 x kCoarseDim: its cluster's world
// rigid motions about the cluster centroid c, as left perturbations
// (Adj(T_j) [[I, 0], [hat(c), I]], se3.py:204-211), and the cluster's
// scaling about c (t_j -> t_j + s (t_j + R_j c): the translation part of the
// perturbation, rotation-first ordering).  About the centroid rather than the
// world origin: the same span, but a cluster far from the origin would
// otherwise see its rotations and its scale as near-translations and A_c
// would lose the precision its Gauss-Jordan inverse needs.
__global__ void k_coarse_basis(int nf, const int* __restrict__ free_frame, const int* __restrict__ frame_cluster,
                               const double* __restrict__ cen, const double* q, const double* t,
                               const double* Rt, double* __restrict__ Pm) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nf) return;
  const int f = free_frame[j];
  Pose T;
  T.q = Quat{q[f * 4], q[f * 4 + 1], q[f * 4 + 2], q[f * 4 + 3]};
  T.t = v3(t[f * 3], t[f * 3 + 1], t[f * 3 + 2]);
  for (int i = 0; i < 9; ++i) T.R.m[i] = Rt[f * 12 + i];
  double A[36];
  se3_adjoint(T, A);
  const int k = frame_cluster[j];
  const double c[3] = {cen[k * 3], cen[k * 3 + 1], cen[k * 3 + 2]};
  const double hc[9] = {0.0, -c[2], c[1], c[2], 0.0, -c[0], -c[1], c[0], 0.0};  // hat(c)
  double* P = Pm + (int64_t)j * 6 * kCoarseDim;
  for (int r = 0; r < 6; ++r) {
    for (int i = 0; i < 3; ++i) {
      double v = A[r * 6 + i];
      for (int m = 0; m < 3; ++m) v += A[r * 6 + 3 + m] * hc[m * 3 + i];
      P[r * kCoarseDim + i] = v;
      P[r * kCoarseDim + 3 + i] = A[r * 6 + 3 + i];
    }
  }
  if (kCoarseDim > 6) {
    const Vec3 Rc = mul(T.R, v3(c[0], c[1], c[2]));
    const double sc[6] = {0.0, 0.0, 0.0, T.t.x + Rc.x, T.t.y + Rc.y, T.t.z + Rc.z};
    for (int r = 0; r < 6; ++r) P[r * kCoarseDim + 6] = sc[r];
  }
}

// A_c = P^T S P, dense [npad x npad] row-major (zeroed beforehand).  Warp
// per nonzero coarse block (c, d); its runs (row i of cluster c, the
// contiguous blocks of row i whose columns fall in cluster d) are visited in
// row order.  Inside a run the lanes take one S block each (T_k = S_k P_j,
// 6 x kCoarseDim), the products are summed over lanes in lane order through
// shared memory, then acc += P_i^T T (kCoarseDim x kCoarseDim).
constexpr int kCD = kCoarseDim, kT = 6 * kCoarseDim, kA = kCoarseDim * kCoarseDim;
__global__ void __launch_bounds__(128) k_coarse_assemble(int npairs, int npad, const int2* __restrict__ pair_cd,
                                                         const int* __restrict__ pair_run_ptr,
                                                         const int4* __restrict__ runs,
                                                         const int* __restrict__ col,
                                                         const double* __restrict__ S,
                                                         const double* __restrict__ Pm,
                                                         double* __restrict__ Ac) {
  __shared__ double Tsm[4][32][kT + 1];
  __shared__ double Tsum[4][kT];
  const int pi = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (pi >= npairs) return;
  // T entries this lane sums: lane, lane + 32 (< kT); A_c entries: lane, lane + 32 (< kA)
  const int te1 = lane + 32;
  const int e0 = lane, e1 = lane + 32;
  const int r0 = e0 / kCD, cc0 = e0 % kCD, r1 = e1 / kCD, cc1 = e1 % kCD;
  double acc0 = 0.0, acc1 = 0.0;
  for (int q = pair_run_ptr[pi]; q < pair_run_ptr[pi + 1]; ++q) {
    const int4 run = runs[q];  // (row i, k0, k1, -)
    double t0 = 0.0, t1 = 0.0;
    for (int kb = run.y; kb < run.z; kb += 32) {
      const int k = kb + lane;
      const int nv = min(32, run.z - kb);
      if (k < run.z) {
        const double* Sb = S + (int64_t)k * 36;
        const double* Pj = Pm + (int64_t)col[k] * kT;
        double Pc[kT];
#pragma unroll
        for (int m = 0; m < kT; ++m) Pc[m] = __ldg(Pj + m);
#pragma unroll
        for (int r = 0; r < 6; ++r) {
          double sr[6];
#pragma unroll
          for (int m = 0; m < 6; ++m) sr[m] = __ldg(Sb + r * 6 + m);
#pragma unroll
          for (int c = 0; c < kCD; ++c) {
            double v = 0.0;
#pragma unroll
            for (int m = 0; m < 6; ++m) v += sr[m] * Pc[m * kCD + c];
            Tsm[warp][lane][r * kCD + c] = v;
          }
        }
      }
      __syncwarp();
      for (int l = 0; l < nv; ++l) {
        t0 += Tsm[warp][l][lane];
        if (te1 < kT) t1 += Tsm[warp][l][te1];
      }
      __syncwarp();
    }
    Tsum[warp][lane] = t0;
    if (te1 < kT) Tsum[warp][te1] = t1;
    __syncwarp();
    const double* Pi = Pm + (int64_t)run.x * kT;
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int m = 0; m < 6; ++m) {
      s0 += __ldg(Pi + m * kCD + r0) * Tsum[warp][m * kCD + cc0];
      if (e1 < kA) s1 += __ldg(Pi + m * kCD + r1) * Tsum[warp][m * kCD + cc1];
    }
    acc0 += s0;
    acc1 += s1;
    __syncwarp();
  }
  const int2 cd = pair_cd[pi];
  Ac[(int64_t)(kCD * cd.x + r0) * npad + kCD * cd.y + cc0] = acc0;
  if (e1 < kA) Ac[(int64_t)(kCD * cd.x + r1) * npad + kCD * cd.y + cc1] = acc1;
}

__global__ void k_pad_identity(int first, int npad, double* Ac) {
  int i = first + blockIdx.x * blockDim.x + threadIdx.x;
  if (i < npad) Ac[(int64_t)i * npad + i] = 1.0;
}

// Blocked Gauss-Jordan inversion of the SPD coarse matrix (no pivoting).
// Ping-pongs between two buffers so each block step reads one and writes
// the other: one grid barrier per step.  Result in buf[T & 1].  256
// threads as 16x16, each owning a 3x3 patch of a 48x48 tile; the tile
// updates are register-blocked 48x48x48 products.  The 48x48 pivot inverse
// of step K+1 is computed once, by the CTA that writes tile (K+1, K+1) in
// step K (it does that tile first and inverts it in registers while the
// other CTAs finish their tiles), and handed over through `pivg` -- the
// sequential 48-column elimination runs in one CTA per step, not in all.
__device__ __forceinline__ void tile_mm(const double* __restrict__ A, const double* __restrict__ B, int ty,
                                        int tx, double acc[3][3]) {
#pragma unroll 4
  for (int m = 0; m < kNB; ++m) {
    double a0 = A[(ty * 3 + 0) * kNB + m], a1 = A[(ty * 3 + 1) * kNB + m], a2 = A[(ty * 3 + 2) * kNB + m];
    double b0 = B[m * kNB + tx * 3 + 0], b1 = B[m * kNB + tx * 3 + 1], b2 = B[m * kNB + tx * 3 + 2];
    acc[0][0] += a0 * b0; acc[0][1] += a0 * b1; acc[0][2] += a0 * b2;
    acc[1][0] += a1 * b0; acc[1][1] += a1 * b1; acc[1][2] += a1 * b2;
    acc[2][0] += a2 * b0; acc[2][1] += a2 * b1; acc[2][2] += a2 * b2;
  }
}

// acc += A^T B over 48x48 tiles (A read column-wise: a warp's lanes share
// its rows, so the reads broadcast)
__device__ __forceinline__ void tile_mm_at(const double* __restrict__ A, const double* __restrict__ B, int ty,
                                           int tx, double acc[3][3]) {
#pragma unroll 4
  for (int m = 0; m < kNB; ++m) {
    double a0 = A[m * kNB + ty * 3 + 0], a1 = A[m * kNB + ty * 3 + 1], a2 = A[m * kNB + ty * 3 + 2];
    double b0 = B[m * kNB + tx * 3 + 0], b1 = B[m * kNB + tx * 3 + 1], b2 = B[m * kNB + tx * 3 + 2];
    acc[0][0] += a0 * b0; acc[0][1] += a0 * b1; acc[0][2] += a0 * b2;
    acc[1][0] += a1 * b0; acc[1][1] += a1 * b1; acc[1][2] += a1 * b2;
    acc[2][0] += a2 * b0; acc[2][1] += a2 * b1; acc[2][2] += a2 * b2;
  }
}

// In-register Gauss-Jordan inverse of the CTA's 48x48 tile P (thread
// (ty, tx) holds rows 3ty.., columns 3tx..); one barrier per column, the
// pivot row / column double-buffered in smem.  Writes the inverse to g.
__device__ __forceinline__ void gj_invert_tile(double P[3][3], double* cbuf, double* rbuf, int* bad, double* g) {
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
#pragma unroll
  for (int a = 0; a < 3; ++a)
    if (tx == 0) cbuf[ty * 3 + a] = P[a][0];
#pragma unroll
  for (int b = 0; b < 3; ++b)
    if (ty == 0) rbuf[tx * 3 + b] = P[0][b];
  __syncthreads();
  for (int k = 0; k < kNB; ++k) {
    const double* ck = cbuf + (k & 1) * kNB;
    const double* rk = rbuf + (k & 1) * kNB;
    const double pk = ck[k];
    if (tid == 0 && !(pk > 0.0)) *bad = 1;
    const double ip = 1.0 / pk;
    // branch-free update (selects, not divergent branches: this loop is the
    // inversion's sequential critical path)
    double rj[3];
#pragma unroll
    for (int b = 0; b < 3; ++b) rj[b] = rk[tx * 3 + b] * ip;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int i = ty * 3 + a;
      const double ci = ck[i];
      const double cip = -ci * ip;
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        const int j = tx * 3 + b;
        const double gen = fma(-ci, rj[b], P[a][b]);
        const double rowk = (j == k) ? ip : rj[b];
        const double other = (j == k) ? cip : gen;
        P[a][b] = (i == k) ? rowk : other;
      }
    }
    if (k + 1 < kNB) {
      double* cn = cbuf + ((k + 1) & 1) * kNB;
      double* rn = rbuf + ((k + 1) & 1) * kNB;
      const int kk = k + 1;
      const int km = kk % 3;
      if (tx == kk / 3) {
#pragma unroll
        for (int a = 0; a < 3; ++a) cn[ty * 3 + a] = km == 0 ? P[a][0] : (km == 1 ? P[a][1] : P[a][2]);
      }
      if (ty == kk / 3) {
#pragma unroll
        for (int b = 0; b < 3; ++b) rn[tx * 3 + b] = km == 0 ? P[0][b] : (km == 1 ? P[1][b] : P[2][b]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) g[(ty * 3 + a) * kNB + tx * 3 + b] = P[a][b];
}

// 48x48 tile (row stride n) -> shared memory: all nine loads per thread in
// flight before the first store (the generic-pointer stores would otherwise
// order each load behind the previous store).
__device__ __forceinline__ void load_tile(const double* src, int64_t n, double* dst) {
  constexpr int kPer = kNB * kNB / kGJThreads;
  static_assert(kPer * kGJThreads == kNB * kNB, "tile / CTA size");
  double v[kPer];
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int e = threadIdx.x + q * kGJThreads;
    v[q] = __ldcg(src + (e / kNB) * n + e % kNB);
  }
#pragma unroll
  for (int q = 0; q < kPer; ++q) dst[threadIdx.x + q * kGJThreads] = v[q];
}

__global__ void __launch_bounds__(kGJThreads) k_gj_inverse(double* A0, double* A1, int n, double* pivg,
                                                          BAScalars* sc) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double gsm[];
  double* piv = gsm;                      // 48x48 (inverted pivot tile)
  double* tKJ = piv + kNB * kNB;          // 48x48
  double* tIK = tKJ + kNB * kNB;          // 48x48
  double* tM = tIK + kNB * kNB;           // 48x48
  double* cbuf = tM + kNB * kNB;          // [2][48] pivot column k
  double* rbuf = cbuf + 2 * kNB;          // [2][48] pivot row k
  __shared__ int bad;
  const int T = n / kNB;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  if (tid == 0) bad = 0;
  __syncthreads();
  if (blockIdx.x == 0) {  // pivot 0 straight from the input
    double P[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) P[a][b] = __ldcg(A0 + (int64_t)(ty * 3 + a) * n + tx * 3 + b);
    gj_invert_tile(P, cbuf, rbuf, &bad, pivg);
  }
  grid.sync();
#ifdef SFM_GJ_PHASES
  long long gt[6] = {0, 0, 0, 0, 0, 0}, g0 = clock64();
#define GJP(k) do { const long long t_ = clock64(); gt[k] += t_ - g0; g0 = t_; } while (0)
#else
#define GJP(k) do {} while (0)
#endif
#if SFM_GJ_SYM
  // A_c is symmetric, and so is every Gauss-Jordan iterate up to sign: with
  // the swept pivots S = {0..K-1} and the rest U, M_SS = A_SS^-1 and
  // M_UU = A_UU - A_US A_SS^-1 A_SU are symmetric and M_US = -M_SU^T.  So
  // only the upper tiles (I <= J) are updated -- half the tile products --
  // and a lower tile a step needs is read as its transposed upper partner:
  // M(K,J) = -M(J,K)^T for J < K, M(I,K) = M(K,I)^T for I > K.  The last
  // step's upper triangle is mirrored at the end.
  auto upper_of = [&](int u, int& I, int& J) {
    I = 0;
    while (u >= T - I) { u -= T - I; ++I; }
    J = I + u;
  };
  auto upper_idx = [&](int I, int J) { return I * T - (I * (I - 1)) / 2 + (J - I); };
  for (int K = 0; K < T; ++K) {
    const double* src = (K & 1) ? A1 : A0;
    double* dst = (K & 1) ? A0 : A1;
    const double* pg = pivg + (K & 1) * kNB * kNB;
    double* pg_next = pivg + ((K + 1) & 1) * kNB * kNB;
    load_tile(pg, kNB, piv);
    __syncthreads();
    GJP(0);
    const int nt = T * (T + 1) / 2;
    const int next_diag = K + 1 < T ? upper_idx(K + 1, K + 1) : -1;
    const int owner = next_diag >= 0 ? next_diag % (int)gridDim.x : -1;
    const int G = (int)gridDim.x, bx = (int)blockIdx.x;
    for (int it = bx - (owner == bx ? G : 0); it < nt; it += G) {
      const bool first = it < 0;
      const int tile = first ? next_diag : it;
      if (!first && tile == next_diag) continue;  // done first
      int I, J;
      upper_of(tile, I, J);
      double* out = dst;
      double acc[3][3];
      auto zero = [&]() {
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b) acc[a][b] = 0.0;
      };
      auto store = [&](int ti, int tj, double sgn) {
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b)
            out[(int64_t)(ti * kNB + ty * 3 + a) * n + tj * kNB + tx * 3 + b] = sgn * acc[a][b];
      };
      if (I == K && J == K) {
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b) acc[a][b] = piv[(ty * 3 + a) * kNB + tx * 3 + b];
        store(K, K, 1.0);
        continue;
      }
      if (I == K) {  // row K (J > K): piv M(K,J)
        load_tile(src + (int64_t)(K * kNB) * n + J * kNB, n, tKJ);
        __syncthreads();
        zero();
        tile_mm(piv, tKJ, ty, tx, acc);
        store(K, J, 1.0);
        __syncthreads();
        continue;
      }
      if (J == K) {  // column K (I < K): -M(I,K) piv
        load_tile(src + (int64_t)(I * kNB) * n + K * kNB, n, tIK);
        __syncthreads();
        zero();
        tile_mm(tIK, piv, ty, tx, acc);
        store(I, K, -1.0);
        __syncthreads();
        continue;
      }
      // tM = piv M(K,J)
      if (J > K) {
        load_tile(src + (int64_t)(K * kNB) * n + J * kNB, n, tKJ);
        __syncthreads();
        zero();
        tile_mm(piv, tKJ, ty, tx, acc);
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b) tM[(ty * 3 + a) * kNB + tx * 3 + b] = acc[a][b];
      } else {  // M(K,J) = -M(J,K)^T: tM = -(M(J,K) piv)^T (piv symmetric)
        load_tile(src + (int64_t)(J * kNB) * n + K * kNB, n, tKJ);
        __syncthreads();
        zero();
        tile_mm(tKJ, piv, ty, tx, acc);
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b) tM[(tx * 3 + b) * kNB + ty * 3 + a] = -acc[a][b];
      }
      double old_ij[3][3];
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
          old_ij[a][b] = __ldcg(src + (int64_t)(I * kNB + ty * 3 + a) * n + J * kNB + tx * 3 + b);
      // M(I,K): stored for I < K, M(K,I)^T for I > K
      const bool iT = I > K;
      load_tile(iT ? src + (int64_t)(K * kNB) * n + I * kNB : src + (int64_t)(I * kNB) * n + K * kNB, n, tIK);
      __syncthreads();
      zero();
      if (iT) tile_mm_at(tIK, tM, ty, tx, acc);
      else tile_mm(tIK, tM, ty, tx, acc);
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) acc[a][b] = old_ij[a][b] - acc[a][b];
      store(I, J, 1.0);
      GJP(1);
      if (first) {  // the next step's pivot tile: invert it now
        __syncthreads();
        gj_invert_tile(acc, cbuf, rbuf, &bad, pg_next);
        GJP(2);
      }
      __syncthreads();
    }
    GJP(3);
    grid.sync();
    GJP(4);
  }
  {  // mirror the inverse's upper tiles into the lower ones
    double* res = (T & 1) ? A1 : A0;
    const int G = (int)gridDim.x, bx = (int)blockIdx.x;
    for (int tile = bx; tile < T * (T + 1) / 2; tile += G) {
      int I, J;
      upper_of(tile, I, J);
      if (I == J) continue;
      load_tile(res + (int64_t)(I * kNB) * n + J * kNB, n, tKJ);
      __syncthreads();
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
          res[(int64_t)(J * kNB + ty * 3 + a) * n + I * kNB + tx * 3 + b] = tKJ[(tx * 3 + b) * kNB + ty * 3 + a];
      __syncthreads();
    }
  }
#else
  for (int K = 0; K < T; ++K) {
    const double* src = (K & 1) ? A1 : A0;
    double* dst = (K & 1) ? A0 : A1;
    const double* pg = pivg + (K & 1) * kNB * kNB;
    double* pg_next = pivg + ((K + 1) & 1) * kNB * kNB;
    load_tile(pg, kNB, piv);
    __syncthreads();
    GJP(0);
    // tile (K+1, K+1) first: its owner inverts it for the next step
    const int nt = T * T;
    const int next_diag = K + 1 < T ? (K + 1) * T + (K + 1) : -1;
    const int owner = next_diag >= 0 ? next_diag % (int)gridDim.x : -1;
    const int G = (int)gridDim.x, bx = (int)blockIdx.x;
    for (int it = bx - (owner == bx ? G : 0); it < nt; it += G) {
      const bool first = it < 0;
      const int tile = first ? next_diag : it;
      if (!first && tile == next_diag) continue;  // done first
      const int I = tile / T, J = tile % T;
      double* out = dst;
      if (I == K && J == K) {
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b)
            out[(int64_t)(K * kNB + ty * 3 + a) * n + K * kNB + tx * 3 + b] = piv[(ty * 3 + a) * kNB + tx * 3 + b];
        continue;
      }
      double acc[3][3];
      if (I == K || J != K) {  // tM = KKinv * src_KJ
        load_tile(src + (int64_t)(K * kNB) * n + J * kNB, n, tKJ);
        __syncthreads();
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b) acc[a][b] = 0.0;
        tile_mm(piv, tKJ, ty, tx, acc);
        if (I == K) {
#pragma unroll
          for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b)
              out[(int64_t)(K * kNB + ty * 3 + a) * n + J * kNB + tx * 3 + b] = acc[a][b];
          __syncthreads();
          continue;
        }
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b) tM[(ty * 3 + a) * kNB + tx * 3 + b] = acc[a][b];
      }
      load_tile(src + (int64_t)(I * kNB) * n + K * kNB, n, tIK);
      double old_ij[3][3];
      if (J != K) {
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b)
            old_ij[a][b] = __ldcg(src + (int64_t)(I * kNB + ty * 3 + a) * n + J * kNB + tx * 3 + b);
      }
      __syncthreads();
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) acc[a][b] = 0.0;
      if (J == K) {
        tile_mm(tIK, piv, ty, tx, acc);
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b)
            out[(int64_t)(I * kNB + ty * 3 + a) * n + K * kNB + tx * 3 + b] = -acc[a][b];
      } else {
        tile_mm(tIK, tM, ty, tx, acc);
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b) {
            const int64_t g = (int64_t)(I * kNB + ty * 3 + a) * n + J * kNB + tx * 3 + b;
            acc[a][b] = old_ij[a][b] - acc[a][b];
            out[g] = acc[a][b];
          }
        GJP(1);
        if (first) {  // the next step's pivot tile: invert it now
          __syncthreads();
          gj_invert_tile(acc, cbuf, rbuf, &bad, pg_next);
          GJP(2);
        }
      }
      __syncthreads();
    }
    GJP(3);
    grid.sync();
    GJP(4);
  }
#endif
#ifdef SFM_GJ_PHASES
  if (tid == 0 && (blockIdx.x < 2 || blockIdx.x == 100))
    printf("GJ cta %d T=%d piv=%lld tiles=%lld inv=%lld tail=%lld sync=%lld\n", blockIdx.x, T, gt[0] / T, gt[1] / T,
           gt[2] / T, gt[3] / T, gt[4] / T);
#endif
  if (bad && tid == 0) atomicOr(&sc->nonfinite, 1);
}

// ---------------------------------------------------------------------------
// Persistent two-level PCG.
//
// Partition (built on the host once per BSR pattern, set_pattern): G CTAs
// (one 512-thread CTA per SM by default, all co-resident) own contiguous block-row ranges of S
// balanced by stored blocks; inside a CTA the range's blocks are cut into
// kPcgWarps contiguous chunks, one per warp, so every warp streams the same
// number of S blocks whatever the row lengths.  A warp's chunk meets one or
// more rows; each (warp, row) meeting is a "segment" whose 6-vector partial
// product goes to shared memory, and a row's result is the sum of its
// segments in warp order -- a fixed order, so the solve is bit-reproducible.
// Coarse clusters are groups of consecutive CTAs, so the restriction P^T q
// of a cluster is a fixed-order sum of per-CTA partials.
// Two grid barriers per iteration (after p.q / P^T q, after r.z / r.r).
// ---------------------------------------------------------------------------

struct Pcg3Args {
  int nf, G, nc, npad, maxrows, maxsegs;
  const int* row_ptr;
  const int* col;
  int two;                 // coarse level on (every rank's view has Aci)
  const int* cta_row0;     // [G+1]
  const int4* wchunk;      // [G*kPcgWarps] (k_begin, k_end, first row, first segment)
  const int2* wres;        // [G*kPcgWarps] (resident blocks at the chunk head, smem slot)
  int resblocks;           // smem capacity for resident S blocks
  const int* lcol;         // [nnzb] column of each block as an index into its CTA's z list
  const int* zl_ptr;       // [G+1] per-CTA distinct columns
  const int* zl;           // distinct frame ids, CTA by CTA
  int maxblk, maxdist;     // per-CTA maxima (shared-memory sizing)
  const int2* rowseg;      // [nf] (first segment local to the CTA, count)
  const int* cta_cluster;  // [G]
  const int* cluster_cta0; // [nc+1]
  int R;                   // ranks (1: single device)
  int rcta0[kPcgMaxRanks + 1];  // first CTA of each rank
  int cta_base;            // global index of this launch's first CTA (per-rank launches)
  unsigned* xbar;          // [2] cross-launch barrier counter | abort flag (null: grid.sync)
  long long xbar_limit;    // spin budget of one cross-launch barrier, in clock64 cycles
  PcgRankView v[kPcgMaxRanks];  // per-rank buffers (pcg.cuh)
  int max_it;
  double rtol;
  int fuse_zc;
  int warm;                // start from the energy-optimal multiple of the previous solution
  double stag_slack;       // stagnation stop only once |r| <= stag_slack * rtol * |b|
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double2 ldg2(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }
__device__ __forceinline__ double2 ldcg2(const double* p) { return __ldcg(reinterpret_cast<const double2*>(p)); }

__device__ __forceinline__ double dot6_sg(const double* s, const double* v) {  // S global, z smem
  const double2 s0 = ldg2(s), s1 = ldg2(s + 2), s2 = ldg2(s + 4);
  const double2 v0 = *reinterpret_cast<const double2*>(v);
  const double2 v1 = *reinterpret_cast<const double2*>(v + 2);
  const double2 v2 = *reinterpret_cast<const double2*>(v + 4);
  double acc = s0.x * v0.x;
  acc = fma(s0.y, v0.y, acc);
  acc = fma(s1.x, v1.x, acc);
  acc = fma(s1.y, v1.y, acc);
  acc = fma(s2.x, v2.x, acc);
  return fma(s2.y, v2.y, acc);
}
__device__ __forceinline__ double dot6_ss(const double* s, const double* v) {  // both smem
  const double2 s0 = *reinterpret_cast<const double2*>(s);
  const double2 s1 = *reinterpret_cast<const double2*>(s + 2);
  const double2 s2 = *reinterpret_cast<const double2*>(s + 4);
  const double2 v0 = *reinterpret_cast<const double2*>(v);
  const double2 v1 = *reinterpret_cast<const double2*>(v + 2);
  const double2 v2 = *reinterpret_cast<const double2*>(v + 4);
  double acc = s0.x * v0.x;
  acc = fma(s0.y, v0.y, acc);
  acc = fma(s1.x, v1.x, acc);
  acc = fma(s1.y, v1.y, acc);
  acc = fma(s2.x, v2.x, acc);
  return fma(s2.y, v2.y, acc);
}

// w = S z over the CTA's rows; writes one 6-vector per segment to seg[].
// z is read from the CTA's shared-memory z cache (zc, the distinct columns
// of its rows, gathered once per iteration) through the block's local
// column index (lc, staged once per solve), so the only global traffic in
// the loop is the S stream itself: independent loads, no index -> z chain.
// The head of every warp's chunk (wres.x blocks) is resident in shared
// memory for the whole solve (Ssm).
__device__ __forceinline__ void spmv_segments(const Pcg3Args& a, int cta, const double* __restrict__ S,
                                              const double* zc, const int* lc, int kc0, double* seg,
                                              const double* Ssm, const int* rpl) {
  const unsigned full = 0xffffffffu;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / 6, comp = lane % 6;
  const int4 ch = a.wchunk[cta * kPcgWarps + warp];
  const int2 wr = a.wres[cta * kPcgWarps + warp];
  int kb = ch.x, r = ch.z, sidx = ch.w;
  const int ke = ch.y;
  // an empty chunk (a CTA with fewer blocks than warps) owns no segment:
  // its sidx is the next warp's (compute-sanitizer racecheck)
  if (kb >= ke) return;
  const int kres = ch.x + wr.x;                    // first non-resident block
  const double* Sres = Ssm + ((int64_t)wr.y - ch.x) * 36 + comp * 6;  // Sres + k*36 for resident k
  const int* lcb = lc - kc0;                       // lcb[k] for global block k
  // Chunks over one or two rows (nearly all of them) stream all their blocks
  // in one loop: a block's product goes to the accumulators of its row, so
  // the loads do not stop and restart at the row boundary.
  const int rb = rpl[r + 1];  // end of the first row
  if (wr.x == 0 && (rb >= ke || rpl[r + 2] >= ke)) {
    const int bnd = min(rb, ke);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;  // first row
    double b0 = 0.0, b1 = 0.0, b2 = 0.0, b3 = 0.0;  // second row
    if (lane < 30) {
      int k = kb + grp;
      for (; k + 15 < ke; k += 20) {
        const double* s0 = S + (int64_t)k * 36 + comp * 6;
        const double d0 = dot6_sg(s0, zc + lcb[k] * 6);
        const double d1 = dot6_sg(s0 + 5 * 36, zc + lcb[k + 5] * 6);
        const double d2 = dot6_sg(s0 + 10 * 36, zc + lcb[k + 10] * 6);
        const double d3 = dot6_sg(s0 + 15 * 36, zc + lcb[k + 15] * 6);
        if (k < bnd) a0 += d0; else b0 += d0;
        if (k + 5 < bnd) a1 += d1; else b1 += d1;
        if (k + 10 < bnd) a2 += d2; else b2 += d2;
        if (k + 15 < bnd) a3 += d3; else b3 += d3;
      }
      for (; k < ke; k += 5) {
        const double d = dot6_sg(S + (int64_t)k * 36 + comp * 6, zc + lcb[k] * 6);
        if (k < bnd) a0 += d; else b0 += d;
      }
    }
    double acc = (a0 + a1) + (a2 + a3);
    double v1 = __shfl_sync(full, acc, comp + 6);
    double v2 = __shfl_sync(full, acc, comp + 12);
    double v3 = __shfl_sync(full, acc, comp + 18);
    double v4 = __shfl_sync(full, acc, comp + 24);
    if (lane < 6) seg[sidx * 6 + lane] = (((acc + v1) + v2) + v3) + v4;
    if (bnd < ke) {
      acc = (b0 + b1) + (b2 + b3);
      v1 = __shfl_sync(full, acc, comp + 6);
      v2 = __shfl_sync(full, acc, comp + 12);
      v3 = __shfl_sync(full, acc, comp + 18);
      v4 = __shfl_sync(full, acc, comp + 24);
      if (lane < 6) seg[(sidx + 1) * 6 + lane] = (((acc + v1) + v2) + v3) + v4;
    }
    return;
  }
  while (kb < ke) {
    const int re = min(ke, rpl[r + 1]);  // row ends staged in smem: no L2 round trip per segment
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
    if (lane < 30) {
      int k = kb + grp;
      const int rs = min(re, kres);
      for (; k + 15 < rs; k += 20) {
        const double* s0 = Sres + (int64_t)k * 36;
        acc0 += dot6_ss(s0, zc + lcb[k] * 6);
        acc1 += dot6_ss(s0 + 5 * 36, zc + lcb[k + 5] * 6);
        acc2 += dot6_ss(s0 + 10 * 36, zc + lcb[k + 10] * 6);
        acc3 += dot6_ss(s0 + 15 * 36, zc + lcb[k + 15] * 6);
      }
      for (; k < rs; k += 5) acc0 += dot6_ss(Sres + (int64_t)k * 36, zc + lcb[k] * 6);
      for (; k + 15 < re; k += 20) {
        const double* s0 = S + (int64_t)k * 36 + comp * 6;
        acc0 += dot6_sg(s0, zc + lcb[k] * 6);
        acc1 += dot6_sg(s0 + 5 * 36, zc + lcb[k + 5] * 6);
        acc2 += dot6_sg(s0 + 10 * 36, zc + lcb[k + 10] * 6);
        acc3 += dot6_sg(s0 + 15 * 36, zc + lcb[k + 15] * 6);
      }
      for (; k < re; k += 5) acc0 += dot6_sg(S + (int64_t)k * 36 + comp * 6, zc + lcb[k] * 6);
    }
    double acc = (acc0 + acc1) + (acc2 + acc3);
    const double v1 = __shfl_sync(full, acc, comp + 6);
    const double v2 = __shfl_sync(full, acc, comp + 12);
    const double v3 = __shfl_sync(full, acc, comp + 18);
    const double v4 = __shfl_sync(full, acc, comp + 24);
    if (lane < 6) seg[sidx * 6 + lane] = (((acc + v1) + v2) + v3) + v4;
    ++sidx;
    ++r;
    kb = re;
  }
}

// Per-CTA shared-memory image of the CTA's rows: the Krylov vectors of the
// rows it owns never leave the SM (only z is published for the SpMV), and
// the constant operators (block-Jacobi inverse, coarse basis, this
// cluster's rows of A_c^-1) are staged once per solve.
struct PcgSmem {
  double* seg;  // [maxsegs*6]
  double* y;    // [maxrows*kCoarseDim] restriction per row
  double* rc;   // [kCoarseDim*nc]
  double* Ae;   // [kCoarseDim x kCoarseDim*nc]
  double* x;    // [maxrows*6] each
  double* r;
  double* p;
  double* q;
  double* z;
  double* Mi;   // [maxrows*36]
  double* Pc;   // [maxrows*6*kCoarseDim]
  double* Ssm;  // [resblocks*36] resident S blocks
  double* zc;   // [maxdist*6] z cache (distinct columns of the CTA's rows)
  int* lc;      // [maxblk] local column index of each of the CTA's blocks
  int2* rs;     // [maxrows] (first segment, count) of each of the CTA's rows
  int* rp;      // [maxrows+1] row_ptr of the CTA's rows
  int* cc0;     // [nc+1] first CTA of each coarse cluster
};

// z_i = D_i^-1 r_i (+ P_i e) for lanes 0..5 of the warp owning local row i
__device__ __forceinline__ double precond_row(const PcgSmem& m, bool two, int i, double ri, const double* e) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  double rj[6];
#pragma unroll
  for (int j = 0; j < 6; ++j) rj[j] = __shfl_sync(full, ri, j);
  double zi = 0.0;
  if (lane < 6) {
    const double* M = m.Mi + i * 36 + lane * 6;
#pragma unroll
    for (int j = 0; j < 6; ++j) zi = fma(M[j], rj[j], zi);
    if (two) {
      const double* P = m.Pc + i * kT + lane * kCD;
#pragma unroll
      for (int j = 0; j < kCD; ++j) zi = fma(P[j], e[j], zi);
    }
  }
  return zi;
}

// P_i^T v_i for lanes 0..kCoarseDim-1 (coarse component lane)
__device__ __forceinline__ double restrict_row(const PcgSmem& m, int i, double vi) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  double vj[6];
#pragma unroll
  for (int j = 0; j < 6; ++j) vj[j] = __shfl_sync(full, vi, j);
  double y = 0.0;
  if (lane < kCD) {
    const double* P = m.Pc + i * kT;
#pragma unroll
    for (int k = 0; k < 6; ++k) y = fma(P[k * kCD + lane], vj[k], y);
  }
  return y;
}

// Sum of n per-CTA partials by one warp: every lane's loads issued together
// (8 per batch), then added in ascending index order -- the order of a plain
// strided loop, one L2 round trip for n <= 256.
__device__ __forceinline__ double lane_partial_sum(const double* __restrict__ p, int n, int lane) {
  double s = 0.0;
  for (int i0 = lane; i0 < n; i0 += 256) {
    double v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = i0 + 32 * q < n ? __ldcg(p + i0 + 32 * q) : 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += v[q];
  }
  return s;
}

// After a grid barrier: the scalar sum over the G per-CTA partials `part`
// (warp 0, fixed order) and, for the two-level preconditioner, the cluster
// restriction sums (other warps), in one round trip.
//   rc[t] = sum_c rpart (assign) or rc[t] -= scale * sum_c rpart.
__device__ __forceinline__ void gather_after_sync(const Pcg3Args& a, const double* __restrict__ rpart,
                                                  const double* part, double* out, int nsum,
                                                  double* rc, bool two, bool assign, const double* scale_num,
                                                  const double* scale_den, const int* cc0) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < nsum) {
    double s = 0.0;
    s = lane_partial_sum(part + warp * a.G, a.G, lane);
    s = warp_sum(s);
    if (lane == 0) out[warp] = s;
  }
  // up to four restriction entries per thread: the first CTA of each
  // entry's cluster is one independent load (cluster bounds from smem), so
  // the four L2 round trips overlap; clusters of several CTAs add the rest
  // in CTA order
  double qs[4] = {0.0, 0.0, 0.0, 0.0};
  int nq = 0;
  const int t0 = threadIdx.x - 32 * nsum, tstride = kPcgThreads - 32 * nsum;
  if (two && t0 >= 0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int t = t0 + j * tstride;
      if (t < kCD * a.nc) {
        qs[j] = __ldcg(rpart + cc0[t / kCD] * kCD + t % kCD);
        nq = j + 1;
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int t = t0 + j * tstride;
      if (j < nq)
        for (int c = cc0[t / kCD] + 1; c < cc0[t / kCD + 1]; ++c) qs[j] += __ldcg(rpart + c * kCD + t % kCD);
    }
  }
  __syncthreads();
  if (two) {
    const double alpha = assign ? 0.0 : (*scale_num) / (*scale_den);
    int j = 0;
    for (int t = threadIdx.x - 32 * nsum; t < kCD * a.nc && t >= 0 && j < nq; t += kPcgThreads - 32 * nsum, ++j)
      rc[t] = assign ? qs[j] : rc[t] - alpha * qs[j];
    // threads that ran out of register slots finish the tail directly
    for (int t = threadIdx.x - 32 * nsum + 4 * (kPcgThreads - 32 * nsum); t < kCD * a.nc && t >= 0;
         t += kPcgThreads - 32 * nsum) {
      const int k = t / kCD, mm = t % kCD;
      double s = 0.0;
      for (int c = cc0[k]; c < cc0[k + 1]; ++c) s += __ldcg(rpart + c * kCD + mm);
      rc[t] = assign ? s : rc[t] - alpha * s;
    }
  }
  __syncthreads();
}

// The two halves of e[0..5] = A_c^-1[6k.., :] . rc for this CTA's cluster k
// (rows in smem) into tmp[12]; a reader forms e[j] = tmp[2j] + tmp[2j+1]
// (coarse_e).  Warps 0..2*kCoarseDim-1: two warps per output row.
__device__ __forceinline__ void coarse_apply(const Pcg3Args& a, const PcgSmem& m, double* tmp) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = kCD * a.nc, ldA = (n + 1) & ~1;
  static_assert(2 * kCoarseDim <= 16, "two warps per coarse output row (512-thread CTAs have 16)");
  if (warp < 2 * kCD) {
    const int o = warp >> 1, h = warp & 1;
    const double* row = m.Ae + o * ldA;
    const int half = (n + 1) / 2;
    const int j0 = h * half, j1 = min(n, j0 + half);
    double s = 0.0;
    for (int j = j0 + lane; j < j1; j += 32) s = fma(row[j], m.rc[j], s);
    s = warp_sum(s);
    if (lane == 0) tmp[warp] = s;
  }
  __syncthreads();
}

__device__ __forceinline__ void coarse_e(const double* tmp, double e[kCoarseDim]) {
#pragma unroll
  for (int j = 0; j < kCD; ++j) e[j] = tmp[2 * j] + tmp[2 * j + 1];
}

// block_sum2 for a point where `red` is known to be free (right after a
// grid barrier): one CTA barrier instead of two.
__device__ __forceinline__ double2 block_sum2_free(double u, double v, double2* red) {
  u = warp_sum(u);
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = make_double2(u, v);
  __syncthreads();
  double2 r = make_double2(0.0, 0.0);
  if (threadIdx.x == 0)
    for (int w = 0; w < kPcgWarps; ++w) { r.x += red[w].x; r.y += red[w].y; }
  return r;
}

// Deterministic block sum of two values (fixed shuffle tree + warp order).
__device__ __forceinline__ double2 block_sum2(double u, double v, double2* red) {
  u = warp_sum(u);
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = make_double2(u, v);
  __syncthreads();
  double2 r = make_double2(0.0, 0.0);
  if (threadIdx.x == 0)
    for (int w = 0; w < kPcgWarps; ++w) { r.x += red[w].x; r.y += red[w].y; }
  return r;
}

#ifdef SFM_PCG_PHASES  // A/B instrumentation: per-phase cycles on CTA 0, thread 0
#define PH_INIT() long long ph_t = clock64(), ph[11] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}
#define PH(k) do { const long long t_ = clock64(); ph[k] += t_ - ph_t; ph_t = t_; } while (0)
#ifdef SFM_PCG_PHASES_ALL  // every CTA (pipe through tools/pcg_phases.py)
#define PH_DUMP(it) do { if (threadIdx.x == 0 && (it) > 0) \
  printf("PCGCTA %d rows=%d blk=%d it=%d spmv=%lld row1=%lld sync1=%lld gather=%lld coarse=%lld row2=%lld " \
         "sync2=%lld zc=%lld r1loop=%lld r1rpart=%lld r1bsum=%lld\n", blockIdx.x, nrows, nblk, \
         (it), ph[0] / (it), ph[1] / (it), ph[2] / (it), ph[3] / (it), ph[4] / (it), ph[5] / (it), \
         ph[6] / (it), ph[7] / (it), ph[8] / (it), ph[9] / (it), ph[10] / (it)); } while (0)
#else
#define PH_DUMP(it) do { if (blockIdx.x == 0 && threadIdx.x == 0 && (it) > 0) \
  printf("PCGPH it=%d spmv=%lld row1=%lld sync1=%lld gather=%lld coarse=%lld row2=%lld sync2=%lld zc=%lld" \
         " r1loop=%lld r1rpart=%lld r1bsum=%lld\n", \
         (it), ph[0] / (it), ph[1] / (it), ph[2] / (it), ph[3] / (it), ph[4] / (it), ph[5] / (it), \
         ph[6] / (it), ph[7] / (it), ph[8] / (it), ph[9] / (it), ph[10] / (it)); } while (0)
#endif
#else
#define PH_INIT() do {} while (0)
#define PH(k) do {} while (0)
#define PH_DUMP(it) do {} while (0)
#endif

// Barrier across several cooperative launches (one per rank: per-device
// launches of a multi-device context, or per-rank launches sharing a device):
// every CTA of every launch arrives once on a shared counter in rank 0's
// memory (system scope, after fencing its pushes system-wide) and spins until
// all G CTAs of the epoch have arrived -- a one-level grid barrier spanning
// the launches.  A spin that outlives xbar_limit cycles sets the abort flag,
// which releases every later barrier at once (the solve then reports a
// failure instead of hanging the device).
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void xlaunch_barrier(const Pcg3Args& a, unsigned& epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();  // the CTA's pushes (ordered before by the CTA barrier), system-wide
    epoch += 1;
    const unsigned target = epoch * (unsigned)a.G;
    atomicAdd_system(a.xbar, 1u);
    const long long t0 = clock64();
    while (ld_acquire_sys(a.xbar) < target) {
      if (ld_acquire_sys(a.xbar + 1) != 0u) break;
      if (clock64() - t0 > a.xbar_limit) {
        atomicExch_system(a.xbar + 1, 1u);
        break;
      }
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kPcgMaxThreads, 1) k_pcg3(Pcg3Args a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double psm[];
  const int MR = a.maxrows, nco = kCD * a.nc;
  const int ldA = (nco + 1) & ~1;  // even strides keep every array 16-byte aligned
  PcgSmem m;
  m.seg = psm;
  m.y = m.seg + 6 * a.maxsegs;
  m.rc = m.y + ((kCD * MR + 1) & ~1);
  m.Ae = m.rc + ldA;
  m.x = m.Ae + kCD * ldA;
  m.r = m.x + 6 * MR;
  m.p = m.r + 6 * MR;
  m.q = m.p + 6 * MR;
  m.z = m.q + 6 * MR;
  m.Mi = m.z + 6 * MR;
  m.Pc = m.Mi + 36 * MR;
  m.Ssm = m.Pc + kT * MR;
  m.zc = m.Ssm + 36 * a.resblocks;
  m.lc = reinterpret_cast<int*>(m.zc + 6 * a.maxdist);
  m.rs = reinterpret_cast<int2*>(m.lc + ((a.maxblk + 1) & ~1));
  m.rp = reinterpret_cast<int*>(m.rs + a.maxrows);
  m.cc0 = m.rp + a.maxrows + 1;
  __shared__ double2 red[32];
  __shared__ double tmp[16];
  __shared__ double sums[4];
  __shared__ double rr_ck[2];  // stagnation test references (sums_and_zc)
  constexpr int kStagWin = 50;
  if (threadIdx.x == 0) { rr_ck[0] = INFINITY; rr_ck[1] = INFINITY; }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = a.G;                        // CTAs over every launch
  const int cta = a.cta_base + (int)blockIdx.x;
  unsigned xepoch = 0;
  auto gsync = [&]() {
    if (a.xbar) xlaunch_barrier(a, xepoch);
    else grid.sync();
  };
  // this CTA's rank and its buffers; the pushes go to every rank's replica
  int rk = 0;
  while (rk + 1 < a.R && cta >= a.rcta0[rk + 1]) ++rk;
  const PcgRankView& V = a.v[rk];
  const double* __restrict__ Sr = V.S;
  auto push_z = [&](int64_t i, double val) {
    for (int q = 0; q < a.R; ++q) a.v[q].z[i] = val;
  };
  auto push_part = [&](int64_t i, double val) {
    for (int q = 0; q < a.R; ++q) a.v[q].part[i] = val;
  };
  const int row0 = a.cta_row0[cta], row1 = a.cta_row0[cta + 1];
  const int nrows = row1 - row0;
  const int kc0 = __ldg(a.row_ptr + row0);
  const int nblk = __ldg(a.row_ptr + row1) - kc0;
  const int zl0 = a.zl_ptr[cta], ndist = a.zl_ptr[cta + 1] - zl0;
  // z cache fill: 3 double2 per distinct column, straight from L2
  // (threads from `first` on; the first warps are busy with the scalar sums)
  auto fill_zc = [&](int first) {
    for (int t = threadIdx.x - first; t < 3 * ndist && t >= 0; t += kPcgThreads - first) {
      const int c = __ldg(a.zl + zl0 + t / 3);
      reinterpret_cast<double2*>(m.zc)[t] = ldcg2(V.z + c * 6 + 2 * (t % 3));
    }
  };
  // After the r.z / r.r barrier: the scalar sums (warps 0..nsum-1) and the
  // next SpMV's z cache (the other warps) in one L2 round trip.
  // Stagnation test (itn > 0, the loop's r.z / r.r sums): at a nearly
  // converged LM state rtol * |b| can be below what fp64 S x resolves, and CG
  // then wanders at the rounding floor until max_it.  Every kStagWin
  // iterations, if |r|^2 is not below 1/4 of its value kStagWin iterations
  // earlier AND |r| is already within stag_slack of the target (so a slow but
  // progressing solve far from the target is never cut short), sums[2] tells
  // every thread to stop.  One thread owns the test (rr_ck alternates read /
  // write slots), and sums[] is read after the barrier below, so all threads
  // of all CTAs stop at the same iteration.  The stop is reported
  // (PCG_STOP_STAGNATED) so the host can count it.
  double stag_rr = 0.0;  // set once |b| is known
  auto sums_and_zc = [&](const double* part, int nsum, int itn) {
    if (warp < nsum) {
      double sacc = 0.0;
      sacc = lane_partial_sum(part + warp * G, G, lane);
      sacc = warp_sum(sacc);
      if (lane == 0) {
        sums[warp] = sacc;
        if (warp == 1) {
          double stop = 0.0;
          if (itn > 0 && itn % kStagWin == 0) {
            const int slot = (itn / kStagWin) & 1;
            stop = (sacc > 0.25 * rr_ck[slot] && sacc <= stag_rr) ? 1.0 : 0.0;
            rr_ck[slot ^ 1] = sacc;
          }
          sums[2] = stop;
        }
      }
    }
    if (a.fuse_zc) fill_zc(32 * nsum);
    __syncthreads();
    if (!a.fuse_zc) {
      fill_zc(0);
      __syncthreads();
    }
  };
  // partial-sum slots (offsets into every replica of `part`); reads use V.part
  const int part_pq = 0, part_rz = G, part_bb = 3 * G;
  const bool two = a.two != 0;

  // ---- stage the constant operators -----------------------------------------
  for (int t = threadIdx.x; t < 36 * nrows; t += kPcgThreads) m.Mi[t] = V.Minv[(int64_t)row0 * 36 + t];
  if (two) {
    for (int t = threadIdx.x; t < kT * nrows; t += kPcgThreads) m.Pc[t] = V.Pm[(int64_t)row0 * kT + t];
    const int k = a.cta_cluster[cta];
    for (int t = threadIdx.x; t < kCD * nco; t += kPcgThreads)
      m.Ae[(t / nco) * ldA + t % nco] = V.Aci[(int64_t)(kCD * k + t / nco) * a.npad + t % nco];
  }
  for (int t = threadIdx.x; t < nblk; t += kPcgThreads) m.lc[t] = __ldg(a.lcol + kc0 + t);
  for (int t = threadIdx.x; t < nrows; t += kPcgThreads) m.rs[t] = a.rowseg[row0 + t];
  for (int t = threadIdx.x; t <= nrows; t += kPcgThreads) m.rp[t] = __ldg(a.row_ptr + row0 + t);
  for (int t = threadIdx.x; t <= a.nc; t += kPcgThreads) m.cc0[t] = a.cluster_cta0[t];
  const int* rpl = m.rp - row0;  // rpl[r] = row_ptr[r] for the CTA's rows
  // resident S blocks: the head of every warp's chunk (18 double2 per block)
  for (int w = 0; w < kPcgWarps; ++w) {
    const int4 ch = a.wchunk[cta * kPcgWarps + w];
    const int2 wr = a.wres[cta * kPcgWarps + w];
    const double2* src = reinterpret_cast<const double2*>(Sr + (int64_t)ch.x * 36);
    double2* dst = reinterpret_cast<double2*>(m.Ssm + (int64_t)wr.y * 36);
    for (int t = threadIdx.x; t < wr.x * 18; t += kPcgThreads) dst[t] = __ldg(src + t);
  }
  __syncthreads();

  auto write_rpart = [&]() {
    __syncthreads();
    if (threadIdx.x < kCD) {
      double s = 0.0;
      for (int i = 0; i < nrows; ++i) s += m.y[i * kCD + threadIdx.x];
      for (int q = 0; q < a.R; ++q) a.v[q].rpart[cta * kCD + threadIdx.x] = s;
    }
  };

  // ---- warm start: x0 = gamma * (the previous solve's solution, still in
  // a.x), gamma = (x0.b)/(x0.S x0) the energy-optimal multiple, so the
  // starting error is never larger than from x = 0.  Consecutive LM steps
  // are nearly parallel late in a solve, where this removes most of the
  // initial error; the converged solution (to rtol) is the same.
  double gamma = 0.0;
  if (a.warm) {
    for (int i = warp; i < nrows; i += kPcgWarps)
      if (lane < 6) push_z((row0 + i) * 6 + lane, V.x[(row0 + i) * 6 + lane]);
    gsync();
    fill_zc(0);
    __syncthreads();
    spmv_segments(a, cta, Sr, m.zc, m.lc, kc0, m.seg, m.Ssm, rpl);
    __syncthreads();
    double xb = 0.0, xw = 0.0;
    for (int i = warp; i < nrows; i += kPcgWarps)
      if (lane < 6) {
        const int2 rs = m.rs[i];
        double w = 0.0;
        for (int sg = 0; sg < rs.y; ++sg) w += m.seg[(rs.x + sg) * 6 + lane];
        m.q[i * 6 + lane] = w;  // S x0, consumed by the prologue below
        const double x0 = V.x[(row0 + i) * 6 + lane];
        xb += x0 * V.b[(row0 + i) * 6 + lane];
        xw += x0 * w;
      }
    const double2 t = block_sum2(xb, xw, red);
    if (threadIdx.x == 0) { push_part(part_rz + cta, t.x); push_part(part_rz + G + cta, t.y); }
    gsync();
    gather_after_sync(a, V.rpart, V.part + part_rz, sums, 2, m.rc, false, true, nullptr, nullptr, m.cc0);
    const double g = sums[0] / sums[1];
    gamma = (sums[1] > 0.0 && isfinite(g)) ? g : 0.0;
  }

  // ---- prologue: x = gamma x0, r = b - gamma S x0, p = q = 0, rc = P^T r ----
  double bb_l = 0.0;
  for (int i = warp; i < nrows; i += kPcgWarps) {
    double ri = 0.0;
    if (lane < 6) {
      const double bi = V.b[(row0 + i) * 6 + lane];
      const bool ws = gamma != 0.0;
      ri = ws ? bi - gamma * m.q[i * 6 + lane] : bi;
      m.x[i * 6 + lane] = ws ? gamma * V.x[(row0 + i) * 6 + lane] : 0.0;
      m.r[i * 6 + lane] = ri;
      m.p[i * 6 + lane] = 0.0;
      m.q[i * 6 + lane] = 0.0;
      bb_l += bi * bi;  // the stopping test stays relative to |b|
    }
    if (two) {
      const double yv = restrict_row(m, i, ri);
      if (lane < kCD) m.y[i * kCD + lane] = yv;
    }
  }
  if (two) write_rpart();
  double2 sb = block_sum2(bb_l, 0.0, red);
  if (threadIdx.x == 0) push_part(part_bb + cta, sb.x);
  gsync();
  gather_after_sync(a, V.rpart, V.part + part_bb, sums, 1, m.rc, two, true, nullptr, nullptr, m.cc0);
  const double bnorm = sqrt(sums[0]);
  stag_rr = (a.stag_slack * a.rtol * bnorm) * (a.stag_slack * a.rtol * bnorm);
  double ev[kCoarseDim];
#pragma unroll
  for (int j = 0; j < kCD; ++j) ev[j] = 0.0;
  if (two) {
    coarse_apply(a, m, tmp);
    coarse_e(tmp, ev);
  }
  double rz_l = 0.0;
  for (int i = warp; i < nrows; i += kPcgWarps) {
    const double ri = (lane < 6) ? m.r[i * 6 + lane] : 0.0;
    const double zi = precond_row(m, two, i, ri, ev);
    if (lane < 6) {
      m.z[i * 6 + lane] = zi;
      push_z((row0 + i) * 6 + lane, zi);
      rz_l += ri * zi;
    }
  }
  double2 s1 = block_sum2(rz_l, 0.0, red);
  if (threadIdx.x == 0) push_part(part_rz + cta, s1.x);
  gsync();
  sums_and_zc(V.part + part_rz, 1, 0);
  double rz_old = sums[0];
  int it = 0, fail = 0, stop = PCG_STOP_MAX_ITERS;
  double beta = 0.0;
  if (!(bnorm > 0.0) || !isfinite(bnorm)) {
    fail = !isfinite(bnorm);
    stop = PCG_STOP_CONVERGED;  // b = 0: x = 0 is exact
  } else {
    PH_INIT();
    for (it = 0; it < a.max_it;) {
      // ---- phase 1: w = S z; p = z + beta p; q = w + beta q; P^T q --------
      spmv_segments(a, cta, Sr, m.zc, m.lc, kc0, m.seg, m.Ssm, rpl);
      __syncthreads();
      PH(0);
      double pq_l = 0.0;
      for (int i = warp; i < nrows; i += kPcgWarps) {
        double qv = 0.0;
        if (lane < 6) {
          const int2 rs = m.rs[i];
          double w = 0.0;
          for (int sg = 0; sg < rs.y; ++sg) w += m.seg[(rs.x + sg) * 6 + lane];
          const double pv = m.z[i * 6 + lane] + beta * m.p[i * 6 + lane];
          qv = w + beta * m.q[i * 6 + lane];
          m.p[i * 6 + lane] = pv;
          m.q[i * 6 + lane] = qv;
          pq_l += pv * qv;
        }
        if (two) {
          const double yv = restrict_row(m, i, qv);
          if (lane < kCD) m.y[i * kCD + lane] = yv;
        }
      }
      PH(8);
      {  // p.q partial (thread 0) and the restriction partial P^T q (warp 1),
         // one CTA barrier: same sums, same order as block_sum2 / write_rpart
        const double u = warp_sum(pq_l);
        if (lane == 0) red[warp] = make_double2(u, 0.0);
        __syncthreads();
        if (threadIdx.x == 0) {
          double sx = 0.0;
          for (int w = 0; w < kPcgWarps; ++w) sx += red[w].x;
          push_part(part_pq + cta, sx);
        } else if (two && threadIdx.x >= 32 && threadIdx.x < 32 + kCD) {
          const int c = threadIdx.x - 32;
          double sr = 0.0;
          for (int i = 0; i < nrows; ++i) sr += m.y[i * kCD + c];
          for (int q = 0; q < a.R; ++q) a.v[q].rpart[cta * kCD + c] = sr;
        }
      }
      PH(9);
      PH(10);
      PH(1);
      gsync();
      PH(2);
      // ---- phase 2: x += alpha p; r -= alpha q; rc -= alpha P^T q; z = M^-1 r
      gather_after_sync(a, V.rpart, V.part + part_pq, sums, 1, m.rc, two, false, &rz_old, &sums[0], m.cc0);
      const double pq = sums[0];
      if (!(pq > 0.0) || !isfinite(pq)) { fail = 1; break; }
      const double alpha = rz_old / pq;
      PH(3);
      if (two) {
        coarse_apply(a, m, tmp);
        coarse_e(tmp, ev);
      }
      PH(4);
      double rz_n = 0.0, rr_n = 0.0;
      for (int i = warp; i < nrows; i += kPcgWarps) {
        double ri = 0.0;
        if (lane < 6) {
          m.x[i * 6 + lane] += alpha * m.p[i * 6 + lane];
          ri = m.r[i * 6 + lane] - alpha * m.q[i * 6 + lane];
          m.r[i * 6 + lane] = ri;
        }
        const double zi = precond_row(m, two, i, ri, ev);
        if (lane < 6) {
          m.z[i * 6 + lane] = zi;
          push_z((row0 + i) * 6 + lane, zi);
          rz_n += ri * zi;
          rr_n += ri * ri;
        }
      }
      const double2 t = block_sum2_free(rz_n, rr_n, red);  // red last read before the grid barrier
      if (threadIdx.x == 0) { push_part(part_rz + cta, t.x); push_part(part_rz + G + cta, t.y); }
      PH(5);
      gsync();
      PH(6);
      sums_and_zc(V.part + part_rz, 2, it + 1);
      PH(7);
      const double rz_new = sums[0], rr = sums[1];
      ++it;
      if (!isfinite(rr) || !isfinite(rz_new)) { fail = 1; break; }
      if (sqrt(rr) <= a.rtol * bnorm) { stop = PCG_STOP_CONVERGED; break; }
      if (sums[2] != 0.0) { stop = PCG_STOP_STAGNATED; break; }  // at the rounding floor (sums_and_zc)
      beta = rz_new / rz_old;
      rz_old = rz_new;
    }
    PH_DUMP(it);
  }
  for (int i = warp; i < nrows; i += kPcgWarps)
    if (lane < 6) V.x[(row0 + i) * 6 + lane] = m.x[i * 6 + lane];
  if (a.xbar && ld_acquire_sys(a.xbar + 1) != 0u) fail = 1;  // a cross-launch barrier gave up
  if (cta == a.rcta0[rk] && threadIdx.x == 0) {  // every rank's scalars
    V.sc->pcg_iters = it;
    V.sc->pcg_fail = fail;
    V.sc->pcg_stop = fail ? PCG_STOP_FAILED : stop;
    if (fail) V.sc->nonfinite = 1;
  }
}

}  // namespace

void TwoLevelPcg::setup(int nf, int cluster, int refresh, cudaStream_t s) {
  nf_ = nf;
  cluster_ = cluster;
  refresh_ = std::max(1, refresh);
  (void)s;
}

std::vector<int> pcg_rank_rows(const int* rp, int nf, int world) {
  constexpr int64_t kRowCost = 4;
  auto cost_upto = [&](int r) { return (int64_t)rp[r] + kRowCost * r; };
  const int64_t total = cost_upto(nf);
  std::vector<int> out(1, 0);
  for (int r = 1; r < world; ++r) {
    const int64_t target = total * r / world;
    int a0 = out.back() + 1, b0 = nf - (world - r);
    const int lo = a0, hi = b0;
    while (a0 < b0) {
      const int m = (a0 + b0) / 2;
      if (cost_upto(m) < target) a0 = m + 1; else b0 = m;
    }
    out.push_back(std::min(std::max(a0, lo), hi));
  }
  out.push_back(nf);
  return out;
}

void TwoLevelPcg::set_pattern(const int* row_ptr, const int* col, int nnzb, cudaStream_t s) {
  if (nf_ <= 0) return;
  const bool timing = std::getenv("SFM_TIMING") != nullptr;
  auto tp = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!timing) return;
    cudaStreamSynchronize(s);
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[sfm pcg plan] %-24s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(t1 - tp).count());
    tp = t1;
  };
  std::vector<int> rp(nf_ + 1), cl(nnzb);
  SFM_CUDA(cudaMemcpyAsync(rp.data(), row_ptr, sizeof(int) * (nf_ + 1), cudaMemcpyDeviceToHost, s));
  SFM_CUDA(cudaMemcpyAsync(cl.data(), col, sizeof(int) * nnzb, cudaMemcpyDeviceToHost, s));
  SFM_CUDA(cudaStreamSynchronize(s));
  int dev = 0, nsm = 0;
  SFM_CUDA(cudaGetDevice(&dev));
  SFM_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  mark("download pattern");

  // ---- CTA row ranges balanced by (stored blocks + per-row overhead) -------
  const int64_t kRowCost = 4;
  auto cost_upto = [&](int r) { return (int64_t)rp[r] + kRowCost * r; };
  const int64_t total = cost_upto(nf_);
  // CTA size: 512 threads x 1 per SM.  Measured on config 3: 16.2 us per
  // iteration vs 17.7 with 1024 threads, whose 64-register cap spills in
  // the row loops (SFM_PCG_CTA / -DSFM_PCG_MAXT=1024 to compare).
  nt_ = kPcgMaxThreads;
  if (const char* e = std::getenv("SFM_PCG_CTA")) {
    const int v = std::atoi(e);
    if (v >= 512 && v <= 1024 && v % 32 == 0) nt_ = v;
  }
  const int nwarps = nt_ / 32;
  if (const char* e = std::getenv("SFM_COARSE_REFRESH")) refresh_ = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("SFM_COARSE_LAMMAX")) lam_max_ = std::atof(e);
  if (const char* e = std::getenv("SFM_COARSE_DRIFT")) drift_ = std::max(1.0, std::atof(e));
  if (const char* e = std::getenv("SFM_COARSE_LAMFLOOR")) lam_floor_ = std::atof(e);
  lin_count_ = 0;
  have_prev_ = false;
  warm_ = true;
  if (const char* e = std::getenv("SFM_PCG_WARM")) warm_ = std::atoi(e) != 0;
  nt_ = std::min(nt_, kPcgMaxThreads);
  int per_sm = 0;  // co-resident CTAs per SM the register budget allows
  SFM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pcg3, nt_, 0));
  per_sm = std::max(1, std::min(per_sm, 1024 / nt_));
  if (const char* e = std::getenv("SFM_PCG_PERSM")) per_sm = std::max(1, std::min(per_sm, std::atoi(e)));
  int G = std::min(per_sm * nsm, nf_);
  // first row in [lo, hi] whose prefix cost reaches target
  auto row_at = [&](int64_t target, int lo, int hi) {
    int a0 = lo, b0 = hi;
    while (a0 < b0) {
      int m = (a0 + b0) / 2;
      if (cost_upto(m) < target) a0 = m + 1; else b0 = m;
    }
    return std::min(std::max(a0, lo), hi);
  };
  // ranks (row-partitioned solve): contiguous row ranges balanced by cost,
  // then CTAs per rank in proportion, each rank's rows split over its CTAs
  const int R = std::max(1, std::min(world_, G));
  SFM_REQUIRE(R == world_, "row-partitioned PCG: fewer block rows than ranks");
  rank_row0_ = pcg_rank_rows(rp.data(), nf_, R);
  rank_cta0_.assign(1, 0);
  for (int r = 1; r < R; ++r) {
    const int64_t c0 = cost_upto(rank_row0_[r]);
    int cr = (int)((G * c0 + total / 2) / std::max<int64_t>(total, 1));
    cr = std::max(cr, rank_cta0_.back() + 1);
    cr = std::min(cr, rank_row0_[r]);                 // <= rows before it
    cr = std::max(cr, G - (nf_ - rank_row0_[r]));     // >= 1 row per CTA after it
    cr = std::min(cr, G - (R - r));                   // >= 1 CTA per later rank
    rank_cta0_.push_back(cr);
  }
  rank_cta0_.push_back(G);
  rank_blk0_.resize(R + 1);
  for (int r = 0; r <= R; ++r) rank_blk0_[r] = rp[rank_row0_[r]];
  std::vector<int> row0(1, 0);
  for (int r = 0; r < R; ++r) {
    const int ca = rank_cta0_[r], cb = rank_cta0_[r + 1], ra = rank_row0_[r], rb = rank_row0_[r + 1];
    const int64_t ta = cost_upto(ra), tb = cost_upto(rb);
    for (int c = ca + 1; c < cb; ++c)
      row0.push_back(row_at(ta + (tb - ta) * (c - ca) / (cb - ca), row0.back() + 1, rb - (cb - c)));
    row0.push_back(rb);
  }
  mark("partition");
  // ---- per-warp chunks and segments ----------------------------------------
  std::vector<int4> wchunk((size_t)G * nwarps);
  std::vector<int2> rowseg(nf_);
  int maxrows = 1, maxsegs = 1;
  for (int c = 0; c < G; ++c) {
    const int r0 = row0[c], r1 = row0[c + 1];
    const int k0 = rp[r0], k1 = rp[r1];
    maxrows = std::max(maxrows, r1 - r0);
    for (int r = r0; r < r1; ++r) rowseg[r] = make_int2(0, 0);
    const int64_t nb = k1 - k0;
    int sidx = 0;
    int r = r0;
    for (int w = 0; w < nwarps; ++w) {
      const int kb = k0 + (int)(nb * w / nwarps), ke = k0 + (int)(nb * (w + 1) / nwarps);
      while (r + 1 < r1 && rp[r + 1] <= kb) ++r;
      wchunk[(size_t)c * nwarps + w] = make_int4(kb, ke, r, sidx);
      int rr = r, k = kb;
      while (k < ke) {
        const int re = std::min(ke, rp[rr + 1]);
        if (rowseg[rr].y == 0) rowseg[rr].x = sidx;
        rowseg[rr].y += 1;
        ++sidx;
        ++rr;
        k = re;
      }
    }
    maxsegs = std::max(maxsegs, sidx);
  }
  mark("chunks");
  // ---- per-CTA z cache: distinct columns and the local index of each block --
  std::vector<int> zl_ptr(G + 1, 0), zl, lcol(nnzb);
  maxdist_ = 1;
  maxblk_ = 1;
  {
    // distinct columns ascending: flag pass + ordered sweep when the CTA
    // touches a large share of the columns, sort of the few otherwise;
    // local index through a dense position map (no per-block search)
    std::vector<int> mark(nf_, -1), pos(nf_, 0);
    std::vector<int> d;
    for (int c = 0; c < G; ++c) {
      const int k0 = rp[row0[c]], k1 = rp[row0[c + 1]];
      d.clear();
      for (int k = k0; k < k1; ++k)
        if (mark[cl[k]] != c) { mark[cl[k]] = c; d.push_back(cl[k]); }
      if ((int64_t)d.size() * 16 > nf_) {
        d.clear();
        for (int j = 0; j < nf_; ++j)
          if (mark[j] == c) d.push_back(j);
      } else {
        std::sort(d.begin(), d.end());
      }
      for (size_t i = 0; i < d.size(); ++i) pos[d[i]] = (int)i, zl.push_back(d[i]);
      for (int k = k0; k < k1; ++k) lcol[k] = pos[cl[k]];
      zl_ptr[c + 1] = (int)zl.size();
      maxdist_ = std::max(maxdist_, (int)d.size());
      maxblk_ = std::max(maxblk_, k1 - k0);
    }
  }
  mark("z cache");
  // ---- coarse clusters = groups of consecutive CTAs -------------------------
  bool two = cluster_ > 0;
  nc_ = two ? std::min(G, std::max(1, (nf_ + cluster_ - 1) / cluster_)) : 1;
  // clusters never straddle a rank: each rank gets its share of them
  std::vector<int> rank_nc0(1, 0);
  for (int r = 0; r < R; ++r) {
    const int gr = rank_cta0_[r + 1] - rank_cta0_[r];
    int nr = R == 1 ? nc_ : std::max(1, std::min(gr, (int)(((int64_t)nc_ * gr + G / 2) / G)));
    rank_nc0.push_back(rank_nc0.back() + nr);
  }
  nc_ = rank_nc0.back();
  std::vector<int> cta_cluster(G), cluster_cta0(nc_ + 1), frame_cluster(nf_);
  for (int r = 0; r < R; ++r) {
    const int ca = rank_cta0_[r], gr = rank_cta0_[r + 1] - ca, k0 = rank_nc0[r], nr = rank_nc0[r + 1] - k0;
    for (int k = 0; k < nr; ++k) cluster_cta0[k0 + k] = ca + (int)((int64_t)gr * k / nr);
  }
  cluster_cta0[nc_] = G;
  if (two && kCoarseDim > 6) {
    // one frame spans only 6 of a cluster's kCoarseDim columns (A_c would be
    // singular): a cluster of fewer than 2 frames joins the next one of its
    // rank (the last one of a rank joins the previous); a rank of one frame
    // leaves the solve on block-Jacobi
    std::vector<int> cta0, rnc(1, 0);
    for (int r = 0; r < R; ++r) {
      const int kb = rank_nc0[r], ke = rank_nc0[r + 1], rend = cluster_cta0[ke];
      const size_t first = cta0.size();
      int start = cluster_cta0[kb];
      for (int k = kb; k < ke; ++k) {
        const int end = cluster_cta0[k + 1];
        if (row0[end] - row0[start] >= 2) {
          cta0.push_back(start);
          start = end;
        }
      }
      if (start != rend && cta0.size() == first) cta0.push_back(start);  // else: the previous cluster absorbs it
      if (row0[rend] - row0[cluster_cta0[kb]] < 2) two = false;
      rnc.push_back((int)cta0.size());
    }
    cta0.push_back(G);
    nc_ = (int)cta0.size() - 1;
    cluster_cta0 = cta0;
    rank_nc0 = rnc;
    cta_cluster.assign(G, 0);
    frame_cluster.assign(nf_, 0);
  }
  for (int k = 0; k < nc_; ++k)
    for (int c = cluster_cta0[k]; c < cluster_cta0[k + 1]; ++c) {
      cta_cluster[c] = k;
      for (int r = row0[c]; r < row0[c + 1]; ++r) frame_cluster[r] = k;
    }
  // A_c is kCoarseDim*nc square, padded with identity rows to whole 48-row tiles
  npad_ = ((kCoarseDim * nc_ + kNB - 1) / kNB) * kNB;
  ncp_ = npad_ / kCoarseDim;
  grid_ = G;
  maxrows_ = maxrows;
  maxsegs_ = maxsegs;
  {  // the kernel's carve-up (k_pcg3): seg | y | rc | Ae | x r p q z | Mi | Pc
    const size_t ny = ((size_t)kCoarseDim * maxrows + 1) & ~(size_t)1;
    const size_t ldA = ((size_t)kCoarseDim * nc_ + 1) & ~(size_t)1;
    smem_ = sizeof(double) * (6 * (size_t)maxsegs + ny + ldA * (1 + kCoarseDim) +
                              (30 + 36 + 6 * kCoarseDim) * (size_t)maxrows);
  }
  SFM_REQUIRE(smem_ <= 200 * 1024, "PCG partition needs too much shared memory");
  // ---- S blocks kept resident in shared memory for the whole solve ---------
  // (the head of each warp's chunk, the same fraction in every warp)
  int max_smem = 0;
  SFM_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const size_t per_cta_avail = (size_t)max_smem / per_sm - 2048;  // static smem margin
  const size_t zbytes = sizeof(double) * 6 * (size_t)maxdist_ + sizeof(int) * (size_t)(maxblk_ + 1) +
                        sizeof(int2) * maxrows_ + sizeof(int) * (maxrows_ + 1 + nc_ + 1) + 16;
  SFM_REQUIRE(smem_ + zbytes <= per_cta_avail, "PCG z cache does not fit in shared memory");
  // Measured on config 3: keeping S blocks resident costs the L1 capacity
  // the rest of the loop relies on and is slower (20.5 vs 18.2 us/iteration),
  // so it is off unless SFM_PCG_RESIDENT=<blocks> asks for it.
  int resblocks = 0;
  if (const char* e = std::getenv("SFM_PCG_RESIDENT"))
    resblocks = std::min((int)((per_cta_avail - smem_ - zbytes) / 288), std::max(0, std::atoi(e)));
  std::vector<int2> wres((size_t)G * nwarps);
  int maxres = 0;
  for (int c = 0; c < G; ++c) {
    const int64_t nb = rp[row0[c + 1]] - rp[row0[c]];
    const int64_t R = std::min<int64_t>(resblocks, nb);
    int base = 0;
    for (int w = 0; w < nwarps; ++w) {
      const int4 ch = wchunk[(size_t)c * nwarps + w];
      const int len = ch.y - ch.x;
      const int rw = nb > 0 ? (int)((int64_t)len * R / nb) : 0;
      wres[(size_t)c * nwarps + w] = make_int2(rw, base);
      base += rw;
    }
    maxres = std::max(maxres, base);
  }
  resblocks_ = maxres;
  smem_ += sizeof(double) * 36 * (size_t)maxres;
  smem_ += sizeof(double) * 6 * (size_t)maxdist_ + sizeof(int) * (size_t)(maxblk_ + 1) + sizeof(int2) * maxrows_ +
           sizeof(int) * (maxrows_ + 1 + nc_ + 1) + 16;
  SFM_CUDA(cudaFuncSetAttribute(k_pcg3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_));
  int resident = 0;
  SFM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, k_pcg3, nt_, smem_));
  SFM_REQUIRE(resident > 0 && G <= resident * nsm, "PCG grid cannot be made co-resident");
  mark("smem plan + occupancy");
  cta_row0_.upload(row0.data(), row0.size(), s);
  wchunk_.upload(wchunk.data(), wchunk.size(), s);
  wres_.upload(wres.data(), wres.size(), s);
  zl_ptr_.upload(zl_ptr.data(), zl_ptr.size(), s);
  zl_.upload(zl.data(), zl.size(), s);
  lcol_.upload(lcol.data(), lcol.size(), s);
  rowseg_.upload(rowseg.data(), rowseg.size(), s);
  cta_cluster_.upload(cta_cluster.data(), cta_cluster.size(), s);
  cluster_cta0_.upload(cluster_cta0.data(), cluster_cta0.size(), s);
  {  // frames of each cluster (the coarse basis is taken about their centroid)
    std::vector<int> cluster_row0(nc_ + 1);
    for (int k = 0; k <= nc_; ++k) cluster_row0[k] = row0[cluster_cta0[k]];
    cluster_row0_.upload(cluster_row0.data(), cluster_row0.size(), s);
    frame_cluster_.upload(frame_cluster.data(), frame_cluster.size(), s);
    cen_.resize((size_t)3 * nc_);
  }

  mark("uploads");
  Minv_.resize((size_t)nf_ * 36);
  Pm_.resize((size_t)nf_ * 6 * kCoarseDim);
  r_.resize((size_t)nf_ * 6); z_.resize((size_t)nf_ * 6); p_.resize((size_t)nf_ * 6); q_.resize((size_t)nf_ * 6);
  rpart_.resize((size_t)G * kCoarseDim);
  part_.resize(4 * (size_t)G);
  if (two) {
    Ac_[0].resize((size_t)npad_ * npad_);
    Ac_[1].resize((size_t)npad_ * npad_);
    gjpiv_.resize((size_t)2 * kNB * kNB);
    const size_t gsm = sizeof(double) * (4 * kNB * kNB + 4 * kNB);
    SFM_CUDA(cudaFuncSetAttribute(k_gj_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsm));
    int per = 0;
    SFM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_gj_inverse, kGJThreads, gsm));
    const int T = npad_ / kNB;
    gj_grid_ = std::max(1, std::min(T * T, per * nsm));
    // coarse assembly runs (row i, k0, k1) grouped by coarse pair (c(i), d),
    // rows ascending inside a pair (stable sort of the row-ordered runs)
    std::vector<std::array<int, 4>> rr;  // (pair key, i, k0, k1)
    rr.reserve((size_t)nnzb / 4 + 16);
    for (int i = 0; i < nf_; ++i) {
      int k = rp[i];
      while (k < rp[i + 1]) {
        const int d = frame_cluster[cl[k]];
        int k1 = k;
        while (k1 < rp[i + 1] && frame_cluster[cl[k1]] == d) ++k1;
        rr.push_back({frame_cluster[i] * nc_ + d, i, k, k1});
        k = k1;
      }
    }
    {  // stable counting sort by coarse pair key (keys < nc^2)
      std::vector<int> cnt((size_t)nc_ * nc_ + 1, 0);
      for (const auto& e : rr) ++cnt[e[0] + 1];
      for (size_t k = 1; k < cnt.size(); ++k) cnt[k] += cnt[k - 1];
      std::vector<std::array<int, 4>> sorted(rr.size());
      for (const auto& e : rr) sorted[cnt[e[0]]++] = e;
      rr.swap(sorted);
    }
    std::vector<int2> cd;
    std::vector<int> ptr(1, 0);
    std::vector<int4> runs;
    runs.reserve(rr.size());
    for (size_t q = 0; q < rr.size(); ++q) {
      if (q == 0 || rr[q][0] != rr[q - 1][0]) {
        if (q) ptr.push_back((int)runs.size());
        cd.push_back(make_int2(rr[q][0] / nc_, rr[q][0] % nc_));
      }
      runs.push_back(make_int4(rr[q][1], rr[q][2], rr[q][3], 0));
    }
    if (!rr.empty()) ptr.push_back((int)runs.size());
    npairs_ = (int)cd.size();
    rank_pair0_.assign(R + 1, npairs_);
    for (int r = R - 1; r >= 0; --r) {
      int q = 0;
      while (q < npairs_ && cd[q].x < rank_nc0[r]) ++q;
      rank_pair0_[r] = q;
    }
    rank_pair0_[R] = npairs_;
    mark("coarse runs");
    pair_cd_.upload(cd.data(), cd.size(), s);
    pair_ptr_.upload(ptr.data(), ptr.size(), s);
    runs_.upload(runs.data(), runs.size(), s);
  } else {
    Ac_[0].release();
    Ac_[1].release();
    gj_grid_ = 0;
    npairs_ = 0;
  }
  SFM_CUDA(cudaStreamSynchronize(s));
  mark("coarse uploads");
}

void TwoLevelPcg::set_basis(const int* free_frame, const double* q, const double* t, const double* Rt,
                            cudaStream_t s, Profiler* prof) {
  if (nf_ <= 0 || gj_grid_ == 0) return;
  // The coarse operator (basis + A_c^-1) is rebuilt every `refresh_`
  // linearisations; in between PCG keeps the previous one, which is still
  // an SPD preconditioner (only the iteration count depends on it).
  if (lin_count_++ % refresh_ != 0) return;
  coarse_valid_ = false;
  ProfScope ps(*prof, "coarse_basis", 0.0, s);
  k_cluster_centroid<<<grid_for(nc_, 128), 128, 0, s>>>(nc_, cluster_row0_.get(), free_frame, t, Rt, cen_.get());
  k_coarse_basis<<<grid_for(nf_, 128), 128, 0, s>>>(nf_, free_frame, frame_cluster_.get(), cen_.get(), q, t, Rt,
                                                     Pm_.get());
}

void TwoLevelPcg::solve(const PcgProblem& p, int max_it, double rtol, BAScalars* sc, cudaStream_t s,
                        Profiler* prof, PcgCollective* coll) {
  if (nf_ <= 0) return;
  NvtxRange nv("sfm pcg");
  // row-partitioned over the ranks of `coll` (the caller reduce-scattered S
  // and b by rank_rows()); otherwise every row is this rank's
  const bool parted = coll && world_ > 1;
  SFM_REQUIRE(!parted || (coll->world() == world_ && coll->rank() == rank_), "PCG partition / collective mismatch");
  const int my = parted ? rank_ : 0;
  const int r0 = parted ? rank_row0_[my] : 0, r1 = parted ? rank_row0_[my + 1] : nf_;
  {
    ProfScope ps(*prof, "block_jacobi", 0.0, s);
    if (r1 > r0) k_block_jacobi<<<grid_for(r1 - r0, 64), 64, 0, s>>>(r0, r1, p.diag_pos, p.S, Minv_.get(), sc);
  }
  // The coarse operator A_c = P^T S(lam) P depends on the damping: S(lam)
  // has lam*D_c on its diagonal and (V + lam D_p)^-1 in its point term.  An
  // A_c assembled at lam_b and applied at lam >> lam_b over-weights the
  // coarse correction P A_c^-1 P^T by up to lam/lam_b on the coarse
  // directions (and under-weights it for lam << lam_b), which wrecks the
  // conditioning of the preconditioned system -- the rejected-trial tail of
  // an LM solve climbs lam by 10x per trial up to 1e32.  So:
  //   * lam > lam_max_: no coarse level.  There the damping makes S
  //     block-diagonally dominant and block-Jacobi alone converges in a few
  //     iterations;
  //   * otherwise A_c is re-assembled and re-inverted whenever lam has moved
  //     by more than drift_ (either way) from the lam it was built at, or the
  //     basis was refreshed (set_basis).
  //   Below lam_floor_ (1e-5) the damping is negligible next to the coarse
  //   operator's own (coarse-space) spectrum, so dampings under the floor
  //   count as equal.  Config 3, LM iterations 1-14 (bench.py --max-iters 14,
  //   tools/ab_env.sh): floor 1e-6 / 1e-5 / 1e-4 -> 1504 / 1508 / 1548 PCG
  //   iterations and 2.42 / 1.82 / 1.21 ms of coarse inverses, 317 / 323 /
  //   325 LM it/s.
  const bool coarse_on = gj_grid_ > 0 && p.lam <= lam_max_;
  const double lam_eff = std::max(p.lam, lam_floor_);
  bool stale = !coarse_valid_;
  if (coarse_on && !stale) {
    const double ratio = lam_eff / lam_build_;
    stale = ratio > drift_ || ratio * drift_ < 1.0;
  }
  if (coarse_on && stale) {
    lam_build_ = lam_eff;
    {
      ProfScope ps(*prof, "coarse_assemble", 288.0 * p.nnzb, s);
      SFM_CUDA(cudaMemsetAsync(Ac_[0].get(), 0, sizeof(double) * (size_t)npad_ * npad_, s));
      // the coarse blocks (c, d) of this rank's clusters (rows of S it holds)
      const int q0 = parted ? rank_pair0_[my] : 0, q1 = parted ? rank_pair0_[my + 1] : npairs_;
      if (q1 > q0)
        k_coarse_assemble<<<grid_for((int64_t)(q1 - q0) * 32, 128), 128, 0, s>>>(
            q1 - q0, npad_, pair_cd_.get() + q0, pair_ptr_.get() + q0, runs_.get(), p.col, p.S, Pm_.get(),
            Ac_[0].get());
      if (npad_ > kCoarseDim * nc_ && my == 0)
        k_pad_identity<<<1, 256, 0, s>>>(kCoarseDim * nc_, npad_, Ac_[0].get());
      if (parted) coll->sum(Ac_[0].get(), (size_t)npad_ * npad_, s);  // disjoint rows: exact
    }
    double* A0 = Ac_[0].get();
    double* A1 = Ac_[1].get();
    double* pg = gjpiv_.get();
    int n = npad_;
    void* args[] = {&A0, &A1, &n, &pg, &sc};
    const size_t gsm = sizeof(double) * (4 * kNB * kNB + 4 * kNB);
    {
      ProfScope ps(*prof, "coarse_inverse", 0.0, s);
      SFM_CUDA(cudaLaunchCooperativeKernel((void*)k_gj_inverse, gj_grid_, kGJThreads, args, gsm, s));
    }
    Aci_ = Ac_[(npad_ / kNB) & 1].get();
    coarse_valid_ = true;
  }
  Pcg3Args a{};
  a.nf = nf_; a.G = grid_; a.nc = nc_; a.npad = npad_; a.maxrows = maxrows_; a.maxsegs = maxsegs_;
  a.row_ptr = p.row_ptr; a.col = p.col;
  a.two = coarse_on ? 1 : 0;
  a.stag_slack = 100.0;
  a.cta_row0 = cta_row0_.get(); a.wchunk = wchunk_.get();
  a.wres = wres_.get(); a.resblocks = resblocks_;
  a.lcol = lcol_.get(); a.zl_ptr = zl_ptr_.get(); a.zl = zl_.get(); a.maxblk = maxblk_; a.maxdist = maxdist_; a.rowseg = rowseg_.get();
  a.cta_cluster = cta_cluster_.get(); a.cluster_cta0 = cluster_cta0_.get();
  a.max_it = max_it; a.rtol = rtol;
  a.fuse_zc = 1;
  a.warm = have_prev_ && warm_ ? 1 : 0;
  have_prev_ = true;
  if (const char* e = std::getenv("SFM_PCG_FUSEZC")) a.fuse_zc = std::atoi(e);
  PcgRankView mine{};
  mine.S = p.S; mine.b = p.b; mine.x = p.x; mine.Minv = Minv_.get(); mine.Pm = Pm_.get();
  mine.Aci = coarse_on ? Aci_ : nullptr; mine.z = z_.get(); mine.part = part_.get(); mine.rpart = rpart_.get();
  mine.sc = sc;
  mine.xbar = nullptr;
  const bool separate = parted && coll->separate_launches();
  if (separate && my == 0) {
    xbar_.resize(2);
    mine.xbar = xbar_.get();
  }
  ProfScope ps(*prof, "pcg", 0.0, s);
  auto fill = [&](const PcgRankView* views) {
    a.R = parted ? world_ : 1;
    for (int r = 0; r < a.R; ++r) a.v[r] = views[r];
    for (int r = 0; r <= a.R; ++r) a.rcta0[r] = parted ? rank_cta0_[r] : (r ? grid_ : 0);
  };
  if (separate) {
    // one cooperative launch per rank over its CTAs, meeting at the
    // cross-launch barrier (2 s spin budget per barrier, then a reported
    // failure instead of a hang)
    coll->launch_each(mine, s, [&]() { SFM_CUDA(cudaMemsetAsync(xbar_.get(), 0, 2 * sizeof(unsigned), s)); },
                      [&](const PcgRankView* views) {
                        fill(views);
                        a.cta_base = rank_cta0_[my];
                        a.xbar = views[0].xbar;
                        a.xbar_limit = 4000000000ll;
                        void* args[] = {&a};
                        SFM_CUDA(cudaLaunchCooperativeKernel((void*)k_pcg3, rank_cta0_[my + 1] - rank_cta0_[my],
                                                             nt_, args, smem_, s));
                      });
    return;
  }
  auto launch = [&](const PcgRankView* views) {
    fill(views);
    a.cta_base = 0;
    a.xbar = nullptr;
    void* args[] = {&a};
    SFM_CUDA(cudaLaunchCooperativeKernel((void*)k_pcg3, grid_, nt_, args, smem_, s));
  };
  if (parted) coll->launch_all(mine, s, launch);
  else launch(&mine);
}

}  // namespace sfm
