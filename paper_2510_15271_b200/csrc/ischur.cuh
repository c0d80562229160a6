// ischur.cuh -- matrix-free ("implicit") Schur complement PCG for the
// high-damping LM trials.  Included by ba.cu (uses its helpers).
//
// Every rejected LM trial multiplies lambda by 10 and re-solves the damped
// system with the same linearisation (solver.py:219-245); in the
// `no_decrease` tail of a solve lambda climbs to 1e32 and there
//   S(lam) = U + lam D_c + H_edges - W (V + lam D_p)^-1 W^T
// is so block-diagonally dominant that PCG converges in one or two
// iterations.  Building S explicitly (two Schur kernels over every
// observation pair) then costs several times the solve itself, so those
// trials multiply by S without forming it:
//   S p = (U + lam D_c) p + H_edges p - sum_a W_a s_i,   s_i = V*_i^-1 sum_b W_b^T p_k(b)
// one pass over the points' observations (k_imp_point: t_i, s_i) and one
// over the cameras' observations (k_imp_cam), both with the same weighted
// Jacobians (W = J~c^T J~p rebuilt from the 32-byte linearisation records)
// as the explicit kernels.  The right-hand side b = -g_c + sum_a W_a e_i is
// the same camera pass with e_i.  Preconditioner: block-Jacobi on
// U_jj + lam D_j (the point term is O(1/lam) of the diagonal there).  The
// Krylov update is one single-CTA kernel; every reduction has a fixed order,
// and every kernel returns at once when the device `done` flag is set, so a
// chunk of iterations is launched without a host round trip.

// ImpState (ba.cuh): rz, |b|, iterations, done (1 converged, 2 failed,
// 3 out of iterations).

// t_i = sum_b J~p_b^T (J~c_b p_j(b)) over the free-frame observations of
// point i, s_i = V*_i^-1 t_i.
__global__ void __launch_bounds__(kBlock) k_imp_point(int64_t P, const int64_t* __restrict__ ptr,
                                                      const int* __restrict__ of, const int* __restrict__ free_idx,
                                                      const int* __restrict__ frame_model,
                                                      const sfm_camera_model* __restrict__ models_g, int nmodels,
                                                      const double* __restrict__ Rt, const double* __restrict__ qt,
                                                      const double4* __restrict__ geo,
                                                      const double* __restrict__ pv, const double* __restrict__ pvec,
                                                      double* __restrict__ s, const ImpState* st) {
  __shared__ sfm_camera_model smod[kSmemModels];
  if (st->done) return;
  const sfm_camera_model* models = stage_models(models_g, nmodels, smod);
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
  const int64_t b0 = ptr[p], b1 = ptr[p + 1];
  int f_nx = b0 < b1 ? of[b0] : 0;  // the next observation's frame, one iteration ahead
  for (int64_t o = b0; o < b1; ++o) {
    const int f = f_nx;
    if (o + 1 < b1) f_nx = of[o + 1];
    const int j = free_idx[f];
    if (j < 0) continue;
    Mat3 R; Vec3 t;
    load_cam_q(Rt, qt, f, R, t);
    double Jc[12], Jp[6];
    geo_jacobians(models[frame_model[f]], R, ldg256(geo + o), Jc, Jp);
    double d[6];
    ldg_vec6(pvec + (int64_t)j * 6, d);
    double y0 = 0.0, y1 = 0.0;
#pragma unroll
    for (int k = 0; k < 6; ++k) { y0 += Jc[k] * d[k]; y1 += Jc[6 + k] * d[k]; }
    acc0 += Jp[0] * y0 + Jp[3] * y1;
    acc1 += Jp[1] * y0 + Jp[4] * y1;
    acc2 += Jp[2] * y0 + Jp[5] * y1;
  }
  const double4 pa = ldg256(pv + p * 12), pb = ldg256(pv + p * 12 + 4);
  s[p * 3 + 0] = pa.x * acc0 + pa.y * acc1 + pa.z * acc2;
  s[p * 3 + 1] = pa.y * acc0 + pa.w * acc1 + pb.x * acc2;
  s[p * 3 + 2] = pa.z * acc0 + pb.x * acc1 + pb.y * acc2;
}

struct ImpCamArgs {
  int nf;
  int mode;                    // 0: b = -g_c + sum W e;  1: y = (U + lam D) p + H p - sum W s
  int rank;
  double lam;
  const int* free_frame;
  const int* frame_model;
  const sfm_camera_model* models;
  const double* Rt;
  const int64_t* cm_ptr;
  const int* cm_pt;
  const double4* geo_cm;
  const double* v;             // per point: s (stride 3) or the packed pv record (e at +6, stride 12)
  int vstride, voff;
  const double* U;
  const double* Dc;
  const double* gc;
  const double* pvec;
  const int* term_ptr;         // incident pose terms per free camera (edges: code>>2 < E, side code&3)
  const int* term_list;
  int E;
  const int* edge_ab;
  const int* free_idx;
  const double* edge_H;        // [E*36] J_lo^T J_hi (weighted)
  double* out;
  const ImpState* st;
};

constexpr int kImpWarps = 4;

// CTA per free camera over its camera-major observations: each lane sums
// J~c_a^T (J~p_a v_i) over its strided share, then a fixed-order CTA sum.
__global__ void __launch_bounds__(kImpWarps * 32) k_imp_cam(ImpCamArgs a) {
  __shared__ double red[kImpWarps][6];
  if (a.st && a.st->done) return;
  const int j = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int f = a.free_frame[j];
  Mat3 R; Vec3 t;
  load_cam(a.Rt, f, R, t);
  const sfm_camera_model cm = a.models[a.frame_model[f]];
  const int64_t k0 = a.cm_ptr[j], k1 = a.cm_ptr[j + 1];
  double acc[6] = {0, 0, 0, 0, 0, 0};
  constexpr int kStride = kImpWarps * 32;
  int64_t k = k0 + threadIdx.x;
  int pt_nx = k < k1 ? __ldg(a.cm_pt + k) : 0;  // the next observation's point, one iteration ahead
  for (; k < k1; k += kStride) {
    const int pt = pt_nx;
    if (k + kStride < k1) pt_nx = __ldg(a.cm_pt + k + kStride);
    const double* vi = a.v + (int64_t)pt * a.vstride + a.voff;
    const double v0 = __ldg(vi), v1 = __ldg(vi + 1), v2 = __ldg(vi + 2);
    double Jc[12], Jp[6];
    geo_jacobians(cm, R, ldg256(a.geo_cm + k), Jc, Jp);
    const double u0 = Jp[0] * v0 + Jp[1] * v1 + Jp[2] * v2;
    const double u1 = Jp[3] * v0 + Jp[4] * v1 + Jp[5] * v2;
#pragma unroll
    for (int c = 0; c < 6; ++c) acc[c] += Jc[c] * u0 + Jc[6 + c] * u1;
  }
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    double x = acc[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (lane == 0) red[warp][c] = x;
  }
  __syncthreads();
  if (threadIdx.x >= 6) return;
  const int c = threadIdx.x;
  double sum = 0.0;
#pragma unroll
  for (int w = 0; w < kImpWarps; ++w) sum += red[w][c];
  double y;
  if (a.mode == 0) {
    y = sum - (a.rank == 0 ? a.gc[j * 6 + c] : 0.0);
  } else {
    y = -sum;
    if (a.rank == 0) {
      const double* Uj = a.U + (int64_t)j * 36 + c * 6;
      const double* pj = a.pvec + (int64_t)j * 6;
      double d = 0.0;
#pragma unroll
      for (int m = 0; m < 6; ++m) d += Uj[m] * pj[m];
      d += a.lam * a.Dc[j * 6 + c] * pj[c];
      // lambda_c edge blocks: S_lo,hi = H, S_hi,lo = H^T (H = J_lo^T J_hi)
      for (int q = a.term_ptr[j]; q < a.term_ptr[j + 1]; ++q) {
        const int term = a.term_list[q] >> 2;
        if (term >= a.E) continue;
        const int ja = a.free_idx[a.edge_ab[2 * term]], jb = a.free_idx[a.edge_ab[2 * term + 1]];
        if (ja < 0 || jb < 0 || ja == jb) continue;
        const int other = ja == j ? jb : ja;
        const double* H = a.edge_H + (int64_t)term * 36;
        const double* po = a.pvec + (int64_t)other * 6;
        double h = 0.0;
        if (j < other) {
#pragma unroll
          for (int m = 0; m < 6; ++m) h += H[c * 6 + m] * po[m];
        } else {
#pragma unroll
          for (int m = 0; m < 6; ++m) h += H[m * 6 + c] * po[m];
        }
        d += h;
      }
      y += d;
    }
  }
  a.out[(int64_t)j * 6 + c] = y;
}

// Block-Jacobi factors of U_jj + lam D_j (inverse of each 6x6 block).
__global__ void k_imp_precond(int nf, const double* __restrict__ U, const double* __restrict__ Dc, double lam,
                              double* __restrict__ Minv, ImpState* st) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nf) return;
  double A[36];
#pragma unroll
  for (int i = 0; i < 36; ++i) A[i] = U[(int64_t)j * 36 + i];
#pragma unroll
  for (int i = 0; i < 6; ++i) A[i * 7] += lam * Dc[j * 6 + i];
  if (!spd6_inverse(A, Minv + (int64_t)j * 36)) st->done = 2;
}

__device__ __forceinline__ double imp_block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];  // every thread, same order
  return s;
}

// z = M^-1 r for the 6-vector of camera j owned by thread slots.
__device__ __forceinline__ double imp_precond_entry(const double* Minv, const double* r, int i) {
  const int j = i / 6, c = i % 6;
  const double* M = Minv + (int64_t)j * 36 + c * 6;
  const double* rj = r + (int64_t)j * 6;
  double z = 0.0;
#pragma unroll
  for (int m = 0; m < 6; ++m) z += M[m] * rj[m];
  return z;
}

// x = 0, r = b, z = M^-1 b, p = z, rz = r.z, |b|  (single CTA)
__global__ void __launch_bounds__(1024) k_imp_init(int n, const double* __restrict__ b, const double* __restrict__ Minv,
                                                   double* x, double* r, double* z, double* p, ImpState* st) {
  __shared__ double red[32];
  double rz = 0.0, bb = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double bi = b[i];
    x[i] = 0.0;
    r[i] = bi;
    bb += bi * bi;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double zi = imp_precond_entry(Minv, r, i);
    z[i] = zi;
    p[i] = zi;
    rz += r[i] * zi;
  }
  const double srz = imp_block_sum(rz, red);
  const double sbb = imp_block_sum(bb, red);
  if (threadIdx.x == 0) {
    st->rz = srz;
    st->bnorm = sqrt(sbb);
    st->it = 0;
    if (!(st->bnorm > 0.0)) st->done = isfinite(st->bnorm) ? 1 : 2;  // b = 0: x = 0 is exact
  }
}

// One CG update after q = S p.  (single CTA)
__global__ void __launch_bounds__(1024) k_imp_step(int n, const double* __restrict__ q, const double* __restrict__ Minv,
                                                   double rtol, int max_it, double* x, double* r, double* z,
                                                   double* p, ImpState* st) {
  __shared__ double red[32];
  __shared__ int stop;
  if (st->done) return;
  double pq = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) pq += p[i] * q[i];
  const double spq = imp_block_sum(pq, red);
  const double alpha = st->rz / spq;
  double rr = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    x[i] += alpha * p[i];
    const double ri = r[i] - alpha * q[i];
    r[i] = ri;
    rr += ri * ri;
  }
  const double srr = imp_block_sum(rr, red);
  if (threadIdx.x == 0) {
    stop = 0;
    if (!(spq > 0.0) || !isfinite(spq) || !isfinite(srr)) stop = 2;
    else if (sqrt(srr) <= rtol * st->bnorm) stop = 1;
    else if (st->it + 1 >= max_it) stop = 3;
  }
  __syncthreads();
  if (stop) {
    if (threadIdx.x == 0) { st->it += 1; st->done = stop; }
    return;
  }
  double rz = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double zi = imp_precond_entry(Minv, r, i);
    z[i] = zi;
    rz += r[i] * zi;
  }
  const double srz = imp_block_sum(rz, red);
  const double beta = srz / st->rz;
  for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = z[i] + beta * p[i];
  if (threadIdx.x == 0) {
    st->rz = srz;
    st->it += 1;
  }
}
