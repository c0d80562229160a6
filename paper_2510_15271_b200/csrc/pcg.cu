// pcg.cu -- two-level preconditioned CG on the reduced camera system
// (see pcg.cuh).  sm_100a, fp64, deterministic.
#include <cooperative_groups.h>

#include <algorithm>
#include <array>
#include <vector>

#include "ba.cuh"
#include "pcg.cuh"
#include "sfm_math.cuh"

namespace cg = cooperative_groups;

namespace sfm {

namespace {

constexpr int kNB = 48;          // Gauss-Jordan tile (8 clusters x 6)
constexpr int kGJThreads = 256;
constexpr int kPcgThreads = 512; // 16 warps
constexpr int kPcgWarps = kPcgThreads / 32;

// Block-Jacobi: inverse of each 6x6 diagonal block of S (Cholesky).
__global__ void k_block_jacobi(int nf, const int* __restrict__ diag_pos, const double* __restrict__ S,
                               double* __restrict__ Minv, BAScalars* sc) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nf) return;
  const double* A = S + (int64_t)diag_pos[j] * 36;
  double L[36];
  for (int i = 0; i < 36; ++i) L[i] = 0.0;
  bool ok = true;
  for (int c = 0; c < 6; ++c) {
    double s = A[c * 6 + c];
    for (int k = 0; k < c; ++k) s -= L[c * 6 + k] * L[c * 6 + k];
    if (!(s > 0.0)) { ok = false; s = 1.0; }
    double d = sqrt(s);
    L[c * 6 + c] = d;
    for (int r = c + 1; r < 6; ++r) {
      double v = A[r * 6 + c];
      for (int k = 0; k < c; ++k) v -= L[r * 6 + k] * L[c * 6 + k];
      L[r * 6 + c] = v / d;
    }
  }
  double Li[36];
  for (int i = 0; i < 36; ++i) Li[i] = 0.0;
  for (int c = 0; c < 6; ++c) {
    Li[c * 6 + c] = 1.0 / L[c * 6 + c];
    for (int r = c + 1; r < 6; ++r) {
      double s = 0.0;
      for (int k = c; k < r; ++k) s += L[r * 6 + k] * Li[k * 6 + c];
      Li[r * 6 + c] = -s / L[r * 6 + r];
    }
  }
  double* M = Minv + (int64_t)j * 36;
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < 6; ++c) {
      double s = 0.0;
      for (int k = max(r, c); k < 6; ++k) s += Li[k * 6 + r] * Li[k * 6 + c];
      M[r * 6 + c] = s;
    }
  if (!ok) atomicOr(&sc->nonfinite, 1);
}

// P_j = Adj(T_j) (se3.py:204-211) of the free frame j's current pose.
__global__ void k_coarse_basis(int nf, const int* __restrict__ free_frame, const double* q, const double* t,
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
  for (int i = 0; i < 36; ++i) Pm[(int64_t)j * 36 + i] = A[i];
}

// A_c = P^T S P, dense [npad x npad] row-major (zeroed beforehand).  Warp
// per nonzero coarse block (c, d); its runs (row i of cluster c, the
// contiguous blocks of row i whose columns fall in cluster d) are visited in
// row order.  Inside a run the lanes take one S block each (T_k = S_k P_j),
// the 36 products are summed over lanes in lane order through shared
// memory, then acc += P_i^T T.
__global__ void __launch_bounds__(128) k_coarse_assemble(int npairs, int npad, const int2* __restrict__ pair_cd,
                                                         const int* __restrict__ pair_run_ptr,
                                                         const int4* __restrict__ runs,
                                                         const int* __restrict__ col,
                                                         const double* __restrict__ S,
                                                         const double* __restrict__ Pm,
                                                         double* __restrict__ Ac) {
  __shared__ double Tsm[4][32][37];
  __shared__ double Tsum[4][36];
  const int pi = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (pi >= npairs) return;
  const int e0 = lane, e1 = lane + 32;
  const int r0 = e0 / 6, cc0 = e0 % 6, r1 = e1 / 6, cc1 = e1 % 6;
  double acc0 = 0.0, acc1 = 0.0;
  for (int q = pair_run_ptr[pi]; q < pair_run_ptr[pi + 1]; ++q) {
    const int4 run = runs[q];  // (row i, k0, k1, -)
    double t0 = 0.0, t1 = 0.0;
    for (int kb = run.y; kb < run.z; kb += 32) {
      const int k = kb + lane;
      const int nv = min(32, run.z - kb);
      if (k < run.z) {
        const double* Sb = S + (int64_t)k * 36;
        const double* Pj = Pm + (int64_t)col[k] * 36;
        double Pc[36];
#pragma unroll
        for (int m = 0; m < 36; ++m) Pc[m] = __ldg(Pj + m);
#pragma unroll
        for (int r = 0; r < 6; ++r) {
          double sr[6];
#pragma unroll
          for (int m = 0; m < 6; ++m) sr[m] = __ldg(Sb + r * 6 + m);
#pragma unroll
          for (int c = 0; c < 6; ++c) {
            double v = 0.0;
#pragma unroll
            for (int m = 0; m < 6; ++m) v += sr[m] * Pc[m * 6 + c];
            Tsm[warp][lane][r * 6 + c] = v;
          }
        }
      }
      __syncwarp();
      for (int l = 0; l < nv; ++l) {
        t0 += Tsm[warp][l][e0];
        if (lane < 4) t1 += Tsm[warp][l][e1];
      }
      __syncwarp();
    }
    Tsum[warp][e0] = t0;
    if (lane < 4) Tsum[warp][e1] = t1;
    __syncwarp();
    const double* Pi = Pm + (int64_t)run.x * 36;
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int m = 0; m < 6; ++m) {
      s0 += __ldg(Pi + m * 6 + r0) * Tsum[warp][m * 6 + cc0];
      if (lane < 4) s1 += __ldg(Pi + m * 6 + r1) * Tsum[warp][m * 6 + cc1];
    }
    acc0 += s0;
    acc1 += s1;
    __syncwarp();
  }
  const int2 cd = pair_cd[pi];
  Ac[(int64_t)(6 * cd.x + r0) * npad + 6 * cd.y + cc0] = acc0;
  if (lane < 4) Ac[(int64_t)(6 * cd.x + r1) * npad + 6 * cd.y + cc1] = acc1;
}

__global__ void k_pad_identity(int first, int npad, double* Ac) {
  int i = first + blockIdx.x * blockDim.x + threadIdx.x;
  if (i < npad) Ac[(int64_t)i * npad + i] = 1.0;
}

// Blocked Gauss-Jordan inversion of the SPD coarse matrix (no pivoting).
// Ping-pongs between two buffers so each block step reads one and writes
// the other: one grid barrier per step.  Result in buf[T & 1].  256
// threads as 16x16, each owning a 3x3 patch of a 48x48 tile: the pivot
// tile is inverted in registers (one barrier per column, double-buffered
// pivot row/column in smem) and the tile updates are register-blocked
// 48x48x48 products.
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

__global__ void __launch_bounds__(kGJThreads) k_gj_inverse(double* A0, double* A1, int n, BAScalars* sc) {
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
  for (int K = 0; K < T; ++K) {
    const double* src = (K & 1) ? A1 : A0;
    double* dst = (K & 1) ? A0 : A1;
    const double* pk_tile = src + (int64_t)(K * kNB) * n + K * kNB;
    double P[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) P[a][b] = __ldcg(pk_tile + (int64_t)(ty * 3 + a) * n + tx * 3 + b);
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
      if (tid == 0 && !(pk > 0.0)) bad = 1;
      const double ip = 1.0 / pk;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const int i = ty * 3 + a;
        const double ci = ck[i];
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          const int j = tx * 3 + b;
          if (i == k) P[a][b] = (j == k) ? ip : rk[j] * ip;
          else P[a][b] = (j == k) ? -ci * ip : P[a][b] - ci * rk[j] * ip;
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
      for (int b = 0; b < 3; ++b) piv[(ty * 3 + a) * kNB + tx * 3 + b] = P[a][b];
    __syncthreads();
    for (int tile = blockIdx.x; tile < T * T; tile += gridDim.x) {
      const int I = tile / T, J = tile % T;
      double* out = dst;
      if (I == K && J == K) {
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b)
            out[(int64_t)(K * kNB + ty * 3 + a) * n + K * kNB + tx * 3 + b] = P[a][b];
        continue;
      }
      double acc[3][3];
      if (I == K || J != K) {  // tM = KKinv * src_KJ
        for (int e = tid; e < kNB * kNB; e += kGJThreads)
          tKJ[e] = __ldcg(src + (int64_t)(K * kNB + e / kNB) * n + J * kNB + e % kNB);
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
      for (int e = tid; e < kNB * kNB; e += kGJThreads)
        tIK[e] = __ldcg(src + (int64_t)(I * kNB + e / kNB) * n + K * kNB + e % kNB);
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
            out[g] = __ldcg(src + g) - acc[a][b];
          }
      }
      __syncthreads();
    }
    grid.sync();
  }
  if (bad && tid == 0) atomicOr(&sc->nonfinite, 1);
}

struct Pcg2Args {
  int nf, C, nc, kc, npad;
  const int* row_ptr;
  const int* col;
  const double* S;
  const double* Minv;
  const double* Pm;
  const double* Aci;   // coarse inverse [npad x npad] (nullptr: one level)
  const double* b;
  double* x;
  double* r;
  double* z;
  double* p;
  double* q;
  double* qc;          // [nc*6]
  double* rc0;         // [nc*6]
  double* part;        // [4*grid]
  BAScalars* sc;
  int max_it;
  double rtol;
};

template <int NT>
__device__ __forceinline__ double block_sum_det(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < NT / 32; ++w) r += red[w];
  return r;
}

// Sum of the per-CTA partials: lane l adds partials l, l+32, ... then a
// fixed shuffle tree (identical in every CTA, every run).
__device__ __forceinline__ double grid_sum_det(const double* part, int G, double* bc) {
  __syncthreads();
  if (threadIdx.x < 32) {
    double s = 0.0;
    for (int i = threadIdx.x; i < G; i += 32) s += __ldcg(part + i);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) *bc = s;
  }
  __syncthreads();
  return *bc;
}

// e[c - c0] = A_c^-1[6c..6c+5, :] . rc  for the CTA's clusters (warp per output)
__device__ __forceinline__ void coarse_apply(const Pcg2Args& a, const double* rc, double* e, int c0, int c1) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nout = 6 * (c1 - c0);
  const int m = 6 * a.nc;
  for (int o = warp; o < nout; o += kPcgWarps) {
    const double* row = a.Aci + (int64_t)(6 * c0 + o) * a.npad;
    double s = 0.0;
    for (int k = lane; k < m; k += 32) s += __ldg(row + k) * rc[k];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
    if (lane == 0) e[o] = s;
  }
}

// z_i = D_i^-1 r_i + P_i e(c(i))   (lanes 0..5 of the warp own row i)
__device__ __forceinline__ double precond_row(const Pcg2Args& a, int row, double ri, const double* e,
                                              int c0) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  double rj[6];
#pragma unroll
  for (int j = 0; j < 6; ++j) rj[j] = __shfl_sync(full, ri, j);
  double zi = 0.0;
  if (lane < 6) {
    const double* M = a.Minv + (int64_t)row * 36 + lane * 6;
#pragma unroll
    for (int j = 0; j < 6; ++j) zi += M[j] * rj[j];
    if (a.Aci) {
      const double* P = a.Pm + (int64_t)row * 36 + lane * 6;
      const double* ec = e + 6 * (row / a.C - c0);
#pragma unroll
      for (int j = 0; j < 6; ++j) zi += P[j] * ec[j];
    }
  }
  return zi;
}

// P_i^T v_i for lanes 0..5 (component lane)
__device__ __forceinline__ double restrict_row(const Pcg2Args& a, int row, double vi) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  double vj[6];
#pragma unroll
  for (int j = 0; j < 6; ++j) vj[j] = __shfl_sync(full, vi, j);
  double y = 0.0;
  if (lane < 6) {
    const double* P = a.Pm + (int64_t)row * 36;
#pragma unroll
    for (int m = 0; m < 6; ++m) y += P[m * 6 + lane] * vj[m];
  }
  return y;
}

__global__ void __launch_bounds__(kPcgThreads) k_pcg2(Pcg2Args a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double psm[];
  double* rc = psm;                        // [6*nc]
  double* e = rc + 6 * a.nc;               // [6*kc]
  double* y = e + 6 * a.kc;                // [kc*C*6]
  __shared__ double red[kPcgWarps];
  __shared__ double bc;
  const unsigned full = 0xffffffffu;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x;
  const int c0 = blockIdx.x * a.kc, c1 = min(c0 + a.kc, a.nc);
  const int row0 = c0 * a.C, row1 = min(c1 * a.C, a.nf);
  double* part_pq = a.part;
  double* part_rz = a.part + G;
  double* part_rr = a.part + 2 * G;
  double* part_bb = a.part + 3 * G;
  const bool two = a.Aci != nullptr;

  // ---- prologue: x = 0, r = b, p = q = 0, rc0 = P^T b ----------------------
  double bb_l = 0.0;
  for (int row = row0 + warp; row < row1; row += kPcgWarps) {
    double bi = 0.0;
    if (lane < 6) {
      bi = a.b[row * 6 + lane];
      a.x[row * 6 + lane] = 0.0;
      a.r[row * 6 + lane] = bi;
      a.p[row * 6 + lane] = 0.0;
      a.q[row * 6 + lane] = 0.0;
      bb_l += bi * bi;
    }
    if (two) {
      double yv = restrict_row(a, row, bi);
      if (lane < 6) y[(row - row0) * 6 + lane] = yv;
    }
  }
  __syncthreads();
  if (two)
    for (int t = threadIdx.x; t < 6 * (c1 - c0); t += kPcgThreads) {
      const int c = c0 + t / 6, k = t % 6;
      double s = 0.0;
      for (int i = c * a.C; i < min((c + 1) * a.C, a.nf); ++i) s += y[(i - row0) * 6 + k];
      a.rc0[c * 6 + k] = s;
    }
  double sb = block_sum_det<kPcgThreads>(bb_l, red);
  if (threadIdx.x == 0) part_bb[blockIdx.x] = sb;
  grid.sync();
  const double bnorm = sqrt(grid_sum_det(part_bb, G, &bc));
  if (two) {
    for (int k = threadIdx.x; k < 6 * a.nc; k += kPcgThreads) rc[k] = __ldcg(a.rc0 + k);
    __syncthreads();
    coarse_apply(a, rc, e, c0, c1);
    __syncthreads();
  }
  double rz_l = 0.0;
  for (int row = row0 + warp; row < row1; row += kPcgWarps) {
    double ri = (lane < 6) ? a.r[row * 6 + lane] : 0.0;
    double zi = precond_row(a, row, ri, e, c0);
    if (lane < 6) {
      a.z[row * 6 + lane] = zi;
      rz_l += ri * zi;
    }
  }
  double s1 = block_sum_det<kPcgThreads>(rz_l, red);
  if (threadIdx.x == 0) part_rz[blockIdx.x] = s1;
  grid.sync();
  double rz_old = grid_sum_det(part_rz, G, &bc);
  int it = 0, fail = 0;
  double beta = 0.0;
  if (!(bnorm > 0.0) || !isfinite(bnorm)) {
    fail = !isfinite(bnorm);
  } else {
    const int grp = lane / 6, comp = lane % 6;
    for (it = 0; it < a.max_it;) {
      // ---- phase 1: w = S z; p = z + beta p; q = w + beta q; P^T q --------
      double pq_l = 0.0;
      for (int row = row0 + warp; row < row1; row += kPcgWarps) {
        double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
        const int k1 = a.row_ptr[row + 1];
        if (lane < 30) {
          int k = a.row_ptr[row] + grp;
          for (; k + 15 < k1; k += 20) {
            const double* s0 = a.S + (int64_t)k * 36 + comp * 6;
            const double* s1p = s0 + 5 * 36;
            const double* s2 = s0 + 10 * 36;
            const double* s3 = s0 + 15 * 36;
            const double* z0 = a.z + a.col[k] * 6;
            const double* z1 = a.z + a.col[k + 5] * 6;
            const double* z2 = a.z + a.col[k + 10] * 6;
            const double* z3 = a.z + a.col[k + 15] * 6;
#pragma unroll
            for (int j = 0; j < 6; ++j) {
              acc0 += __ldg(s0 + j) * __ldcg(z0 + j);
              acc1 += __ldg(s1p + j) * __ldcg(z1 + j);
              acc2 += __ldg(s2 + j) * __ldcg(z2 + j);
              acc3 += __ldg(s3 + j) * __ldcg(z3 + j);
            }
          }
          for (; k < k1; k += 5) {
            const double* s0 = a.S + (int64_t)k * 36 + comp * 6;
            const double* z0 = a.z + a.col[k] * 6;
#pragma unroll
            for (int j = 0; j < 6; ++j) acc0 += __ldg(s0 + j) * __ldcg(z0 + j);
          }
        }
        double acc = (acc0 + acc1) + (acc2 + acc3);
        double v1 = __shfl_sync(full, acc, comp + 6);
        double v2 = __shfl_sync(full, acc, comp + 12);
        double v3 = __shfl_sync(full, acc, comp + 18);
        double v4 = __shfl_sync(full, acc, comp + 24);
        double qv = 0.0;
        if (lane < 6) {
          const double w = (((acc + v1) + v2) + v3) + v4;
          const double pv = a.z[row * 6 + lane] + beta * a.p[row * 6 + lane];
          qv = w + beta * a.q[row * 6 + lane];
          a.p[row * 6 + lane] = pv;
          a.q[row * 6 + lane] = qv;
          pq_l += pv * qv;
        }
        if (two) {
          double yv = restrict_row(a, row, qv);
          if (lane < 6) y[(row - row0) * 6 + lane] = yv;
        }
      }
      __syncthreads();
      if (two)
        for (int t = threadIdx.x; t < 6 * (c1 - c0); t += kPcgThreads) {
          const int c = c0 + t / 6, k = t % 6;
          double s = 0.0;
          for (int i = c * a.C; i < min((c + 1) * a.C, a.nf); ++i) s += y[(i - row0) * 6 + k];
          a.qc[c * 6 + k] = s;
        }
      double s = block_sum_det<kPcgThreads>(pq_l, red);
      if (threadIdx.x == 0) part_pq[blockIdx.x] = s;
      grid.sync();
      const double pq = grid_sum_det(part_pq, G, &bc);
      if (!(pq > 0.0) || !isfinite(pq)) { fail = 1; break; }
      const double alpha = rz_old / pq;
      // ---- phase 2: x += alpha p; r -= alpha q; rc -= alpha qc; z = M^-1 r --
      if (two) {
        for (int k = threadIdx.x; k < 6 * a.nc; k += kPcgThreads) rc[k] -= alpha * __ldcg(a.qc + k);
        __syncthreads();
        coarse_apply(a, rc, e, c0, c1);
        __syncthreads();
      }
      double rz_n = 0.0, rr_n = 0.0;
      for (int row = row0 + warp; row < row1; row += kPcgWarps) {
        double ri = 0.0;
        if (lane < 6) {
          a.x[row * 6 + lane] += alpha * a.p[row * 6 + lane];
          ri = a.r[row * 6 + lane] - alpha * a.q[row * 6 + lane];
          a.r[row * 6 + lane] = ri;
        }
        double zi = precond_row(a, row, ri, e, c0);
        if (lane < 6) {
          a.z[row * 6 + lane] = zi;
          rz_n += ri * zi;
          rr_n += ri * ri;
        }
      }
      double t1 = block_sum_det<kPcgThreads>(rz_n, red);
      double t2 = block_sum_det<kPcgThreads>(rr_n, red);
      if (threadIdx.x == 0) { part_rz[blockIdx.x] = t1; part_rr[blockIdx.x] = t2; }
      grid.sync();
      const double rz_new = grid_sum_det(part_rz, G, &bc);
      const double rr = grid_sum_det(part_rr, G, &bc);
      ++it;
      if (!isfinite(rr) || !isfinite(rz_new)) { fail = 1; break; }
      if (sqrt(rr) <= a.rtol * bnorm) break;
      beta = rz_new / rz_old;
      rz_old = rz_new;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.sc->pcg_iters = it;
    a.sc->pcg_fail = fail;
    if (fail) a.sc->nonfinite = 1;
  }
}

}  // namespace

void TwoLevelPcg::setup(int nf, int cluster, cudaStream_t s) {
  nf_ = nf;
  if (nf <= 0) return;
  int dev = 0, nsm = 0, per_sm = 0;
  SFM_CUDA(cudaGetDevice(&dev));
  SFM_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  C_ = cluster;
  if (C_ > 0) {
    // keep the coarse system small enough for the per-trial inverse
    C_ = std::max(C_, (nf + 191) / 192);
    nc_ = (nf + C_ - 1) / C_;
  } else {
    C_ = 16;
    nc_ = (nf + C_ - 1) / C_;
  }
  ncp_ = ((nc_ + 7) / 8) * 8;
  npad_ = 6 * ncp_;
  // cooperative grid: clusters per CTA so that every CTA is co-resident
  auto smem_for = [&](int kc) { return sizeof(double) * (size_t)(6 * nc_ + 6 * kc + kc * C_ * 6); };
  kc_ = 1;
  for (;;) {
    size_t sm = smem_for(kc_);
    SFM_CUDA(cudaFuncSetAttribute(k_pcg2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    SFM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pcg2, kPcgThreads, sm));
    int grid = (nc_ + kc_ - 1) / kc_;
    if (per_sm > 0 && grid <= per_sm * nsm) { smem_ = sm; grid_ = grid; break; }
    SFM_REQUIRE(kc_ < nc_, "PCG grid cannot be made co-resident");
    ++kc_;
  }
  Minv_.resize((size_t)nf * 36);
  Pm_.resize((size_t)nf * 36);
  r_.resize((size_t)nf * 6); z_.resize((size_t)nf * 6); p_.resize((size_t)nf * 6); q_.resize((size_t)nf * 6);
  qc_.resize((size_t)nc_ * 6);
  rc0_.resize((size_t)nc_ * 6);
  part_.resize(4 * (size_t)grid_);
  if (cluster > 0) {
    Ac_[0].resize((size_t)npad_ * npad_);
    Ac_[1].resize((size_t)npad_ * npad_);
    const size_t gsm = sizeof(double) * (4 * kNB * kNB + 4 * kNB);
    SFM_CUDA(cudaFuncSetAttribute(k_gj_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsm));
    int per = 0;
    SFM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_gj_inverse, kGJThreads, gsm));
    const int T = npad_ / kNB;
    gj_grid_ = std::max(1, std::min(T * T, per * nsm));
  } else {
    Ac_[0].release();
    Ac_[1].release();
    gj_grid_ = 0;
  }
  (void)s;
}

void TwoLevelPcg::set_pattern(const int* row_ptr, const int* col, int nnzb, cudaStream_t s) {
  if (nf_ <= 0 || gj_grid_ == 0) return;
  std::vector<int> rp(nf_ + 1), cl(nnzb);
  SFM_CUDA(cudaMemcpyAsync(rp.data(), row_ptr, sizeof(int) * (nf_ + 1), cudaMemcpyDeviceToHost, s));
  SFM_CUDA(cudaMemcpyAsync(cl.data(), col, sizeof(int) * nnzb, cudaMemcpyDeviceToHost, s));
  SFM_CUDA(cudaStreamSynchronize(s));
  // runs (row i, k0, k1) grouped by coarse pair (c(i), d), rows ascending
  std::vector<std::vector<std::array<int, 3>>> per(nc_ * (size_t)nc_);
  for (int i = 0; i < nf_; ++i) {
    int k = rp[i];
    while (k < rp[i + 1]) {
      const int d = cl[k] / C_;
      int k1 = k;
      while (k1 < rp[i + 1] && cl[k1] / C_ == d) ++k1;
      per[(size_t)(i / C_) * nc_ + d].push_back({i, k, k1});
      k = k1;
    }
  }
  std::vector<int2> cd;
  std::vector<int> ptr(1, 0);
  std::vector<int4> runs;
  for (int c = 0; c < nc_; ++c)
    for (int d = 0; d < nc_; ++d) {
      auto& v = per[(size_t)c * nc_ + d];
      if (v.empty()) continue;
      cd.push_back(make_int2(c, d));
      for (auto& r : v) runs.push_back(make_int4(r[0], r[1], r[2], 0));
      ptr.push_back((int)runs.size());
    }
  npairs_ = (int)cd.size();
  pair_cd_.upload(cd.data(), cd.size(), s);
  pair_ptr_.upload(ptr.data(), ptr.size(), s);
  runs_.upload(runs.data(), runs.size(), s);
  SFM_CUDA(cudaStreamSynchronize(s));
}

void TwoLevelPcg::set_basis(const int* free_frame, const double* q, const double* t, const double* Rt,
                            cudaStream_t s, Profiler* prof) {
  if (nf_ <= 0 || gj_grid_ == 0) return;
  coarse_valid_ = false;
  ProfScope ps(*prof, "coarse_basis", 0.0, s);
  k_coarse_basis<<<grid_for(nf_, 128), 128, 0, s>>>(nf_, free_frame, q, t, Rt, Pm_.get());
}

void TwoLevelPcg::solve(const PcgProblem& p, int max_it, double rtol, BAScalars* sc, cudaStream_t s,
                        Profiler* prof) {
  if (nf_ <= 0) return;
  {
    ProfScope ps(*prof, "block_jacobi", 0.0, s);
    k_block_jacobi<<<grid_for(nf_, 64), 64, 0, s>>>(nf_, p.diag_pos, p.S, Minv_.get(), sc);
  }
  // The coarse operator is rebuilt once per linearisation (first trial);
  // later damping trials reuse it -- any SPD coarse operator is a valid
  // preconditioner, and lambda only rescales the diagonal.
  if (gj_grid_ > 0 && !coarse_valid_) {
    {
      ProfScope ps(*prof, "coarse_assemble", 288.0 * p.nnzb, s);
      SFM_CUDA(cudaMemsetAsync(Ac_[0].get(), 0, sizeof(double) * (size_t)npad_ * npad_, s));
      if (npairs_)
        k_coarse_assemble<<<grid_for((int64_t)npairs_ * 32, 128), 128, 0, s>>>(
            npairs_, npad_, pair_cd_.get(), pair_ptr_.get(), runs_.get(), p.col, p.S, Pm_.get(), Ac_[0].get());
      if (npad_ > 6 * nc_)
        k_pad_identity<<<1, 256, 0, s>>>(6 * nc_, npad_, Ac_[0].get());
    }
    double* A0 = Ac_[0].get();
    double* A1 = Ac_[1].get();
    int n = npad_;
    void* args[] = {&A0, &A1, &n, &sc};
    const size_t gsm = sizeof(double) * (4 * kNB * kNB + 4 * kNB);
    {
      ProfScope ps(*prof, "coarse_inverse", 0.0, s);
      SFM_CUDA(cudaLaunchCooperativeKernel((void*)k_gj_inverse, gj_grid_, kGJThreads, args, gsm, s));
    }
    Aci_ = Ac_[(npad_ / kNB) & 1].get();
    coarse_valid_ = true;
  }
  const double* Aci = gj_grid_ > 0 ? Aci_ : nullptr;
  Pcg2Args a{};
  a.nf = nf_; a.C = C_; a.nc = nc_; a.kc = kc_; a.npad = npad_;
  a.row_ptr = p.row_ptr; a.col = p.col; a.S = p.S; a.Minv = Minv_.get(); a.Pm = Pm_.get(); a.Aci = Aci;
  a.b = p.b; a.x = p.x; a.r = r_.get(); a.z = z_.get(); a.p = p_.get(); a.q = q_.get();
  a.qc = qc_.get(); a.rc0 = rc0_.get(); a.part = part_.get(); a.sc = sc; a.max_it = max_it; a.rtol = rtol;
  void* args[] = {&a};
  ProfScope ps(*prof, "pcg", 0.0, s);
  SFM_CUDA(cudaLaunchCooperativeKernel((void*)k_pcg2, grid_, kPcgThreads, args, smem_, s));
}

}  // namespace sfm
