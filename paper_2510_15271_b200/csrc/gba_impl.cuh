// gba_impl.cuh -- bundle adjustment with rig-extrinsic and rolling-shutter
// residuals (mapping.py:321-356, :414-439, :464-475): SURVEY.md §8(f) row 2.
// Included at the end of ba.cu (same translation unit: it reuses that file's
// LM building blocks -- pose-term Jacobians, Marquardt point blocks, the
// dense Cholesky, retraction, fixed-order finalisation).
//
// A residual's pose is composed from up to two SE(3) parameter blocks
// ("slots"):
//   GLOBAL   pose = B[s0]                               J_s0 = J_pose
//   RIG      pose = B[e] B[v]    (s0 = v, s1 = e)       J_v = J_pose Ad(E), J_e = J_pose
//   ROLLING  pose = T_a exp(a xi), xi = log(T_a^-1 T_b) J_a = J_pose (I - B), J_b = J_pose B,
//            B = a Ad(T) J_r(a xi) J_l^-1(xi) Ad(T_a^-1)              (_interp_weights)
// so one residual touches two camera-side blocks and the Schur complement
// gains a direct block between them.  Every camera-indexed quantity is a
// fixed-order sum over lists sorted once per solve (no atomics):
//   S_ab = sum_{same residual, slots in a, b} Jc_s^T Jc_t
//        - sum_{same point, slots in a, b} Jc_s^T (Jp V*^-1 Jp^T) Jc_t  (+ pose terms, damping)
// Per-residual weighted Jacobians are stored explicitly (32 doubles).

struct GbaArgs {
  int64_t R, P;
  int nb;
  const int* rpt;
  const int* rmodel;
  const int* rkind;
  const int* rslot;    // [R*2]
  const double* ralpha;
  const double* ruv;   // [R*2]
  const sfm_camera_model* models;
  const double* q;     // block state
  const double* t;
  const double* Rt;
  const double* X;     // point state
  int lk;
  double lp;
};

namespace {


constexpr int kGbaRec = 32;  // r~(2) | Jp~(6) | Jc~ slot0 (12) | Jc~ slot1 (12)

SFM_HD void mat6_mul(const double* A, const double* B, double* C) {
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) {
      double s = 0.0;
      for (int k = 0; k < 6; ++k) s += A[i * 6 + k] * B[k * 6 + j];
      C[i * 6 + j] = s;
    }
}

// se3_left_jacobian (se3.py:238-247): [[J, 0], [Q, J]]
SFM_HD void se3_left_jacobian_fwd(const double xi[6], double out[36]) {
  const Vec3 phi = v3(xi[0], xi[1], xi[2]), rho = v3(xi[3], xi[4], xi[5]);
  const Mat3 J = so3_left_jacobian(phi);
  const Mat3 Q = se3_Q(phi, rho);
  for (int i = 0; i < 36; ++i) out[i] = 0.0;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      out[r * 6 + c] = J.m[r * 3 + c];
      out[(r + 3) * 6 + c] = Q.m[r * 3 + c];
      out[(r + 3) * 6 + c + 3] = J.m[r * 3 + c];
    }
}

__device__ __forceinline__ Pose gba_block(const GbaArgs& a, int b) { return load_pose(a.q, a.t, a.Rt, b); }

// Composed pose of residual i; with chain != nullptr also the two slot
// chain matrices (6x6 each, row-major).
__device__ Pose gba_pose(const GbaArgs& a, int64_t i, double* C0, double* C1) {
  const int kind = a.rkind[i];
  const int s0 = a.rslot[2 * i], s1 = a.rslot[2 * i + 1];
  if (kind == SFM_RES_RIG) {
    const Pose V = gba_block(a, s0), E = gba_block(a, s1);
    if (C0) {
      se3_adjoint(E, C0);
      for (int k = 0; k < 36; ++k) C1[k] = (k % 7 == 0) ? 1.0 : 0.0;
    }
    return compose(E, V);
  }
  if (kind == SFM_RES_ROLLING) {
    const Pose Ta = gba_block(a, s0), Tb = gba_block(a, s1);
    const double al = a.ralpha[i];
    double xi[6];
    se3_log(compose(pose_inverse(Ta), Tb), xi);
    double axi[6];
    for (int k = 0; k < 6; ++k) axi[k] = al * xi[k];
    const Pose T = compose(Ta, se3_exp(axi));
    if (C0) {
      double AdT[36], Jr[36], Jli[36], AdAi[36], nax[6], M1[36], M2[36], B[36];
      se3_adjoint(T, AdT);
      for (int k = 0; k < 6; ++k) nax[k] = -axi[k];
      se3_left_jacobian_fwd(nax, Jr);  // J_r(a xi) = J_l(-a xi)
      se3_left_jacobian_inv(xi, Jli);
      se3_adjoint(pose_inverse(Ta), AdAi);
      mat6_mul(AdT, Jr, M1);
      mat6_mul(M1, Jli, M2);
      mat6_mul(M2, AdAi, B);
      for (int k = 0; k < 36; ++k) {
        B[k] *= al;
        C0[k] = ((k % 7 == 0) ? 1.0 : 0.0) - B[k];
        C1[k] = B[k];
      }
    }
    return T;
  }
  if (C0)
    for (int k = 0; k < 36; ++k) C0[k] = (k % 7 == 0) ? 1.0 : 0.0;
  return gba_block(a, s0);
}

// Linearisation record of every residual (solver.py:164-191): weighted
// residual and Jacobians w.r.t. the point and both slots.
__global__ void k_gba_lin(GbaArgs a, double* __restrict__ rec, BAScalars* sc) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.R) return;
  double C0[36], C1[36];
  const Pose T = gba_pose(a, i, C0, C1);
  const int p = a.rpt[i];
  double u, v, Jc[12], Jp[6];
  double* o = rec + i * kGbaRec;
  const int st = project_with_jacobians(a.models[a.rmodel[i]], T.R, T.t, load_X(a.X, p), u, v, Jc, Jp);
  if (st != PROJ_OK) {
    for (int k = 0; k < kGbaRec; ++k) o[k] = 0.0;
    atomicOr(&sc->nonfinite, 1);
    return;
  }
  double r0 = u - a.ruv[2 * i], r1 = v - a.ruv[2 * i + 1];
  const double w = sqrt(loss_rho_prime(a.lk, a.lp, r0 * r0 + r1 * r1));
  o[0] = w * r0;
  o[1] = w * r1;
  for (int k = 0; k < 6; ++k) o[2 + k] = w * Jp[k];
  const bool two = a.rkind[i] != SFM_RES_GLOBAL;
  for (int rr = 0; rr < 2; ++rr)
    for (int c = 0; c < 6; ++c) {
      double s0 = 0.0, s1 = 0.0;
      for (int k = 0; k < 6; ++k) {
        s0 += Jc[rr * 6 + k] * C0[k * 6 + c];
        if (two) s1 += Jc[rr * 6 + k] * C1[k * 6 + c];
      }
      o[8 + rr * 6 + c] = w * s0;
      o[20 + rr * 6 + c] = w * s1;
    }
}

// V_i = sum Jp^T Jp, g_i = sum Jp^T r over the point's residuals.
__global__ void k_gba_point_lin(int64_t P, const int64_t* __restrict__ pptr, const double* __restrict__ rec,
                                double* __restrict__ V, double* __restrict__ gp, BAScalars* sc) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double gm = 0.0;
  if (p < P) {
    double v[6] = {0, 0, 0, 0, 0, 0}, g[3] = {0, 0, 0};
    for (int64_t i = pptr[p]; i < pptr[p + 1]; ++i) {
      const double* o = rec + i * kGbaRec;
      const double* J = o + 2;
      v[0] += J[0] * J[0] + J[3] * J[3];
      v[1] += J[0] * J[1] + J[3] * J[4];
      v[2] += J[0] * J[2] + J[3] * J[5];
      v[3] += J[1] * J[1] + J[4] * J[4];
      v[4] += J[1] * J[2] + J[4] * J[5];
      v[5] += J[2] * J[2] + J[5] * J[5];
      g[0] += J[0] * o[0] + J[3] * o[1];
      g[1] += J[1] * o[0] + J[4] * o[1];
      g[2] += J[2] * o[0] + J[5] * o[1];
    }
    for (int k = 0; k < 6; ++k) V[p * 6 + k] = v[k];
    for (int k = 0; k < 3; ++k) gp[p * 3 + k] = g[k];
    gm = fmax(fabs(g[0]), fmax(fabs(g[1]), fabs(g[2])));
    if (isnan(g[0]) || isnan(g[1]) || isnan(g[2])) gm = __longlong_as_double(0x7ff8000000000000ll);
  }
  unsigned long long m = warp_max_u64((unsigned long long)__double_as_longlong(gm));
  if ((threadIdx.x & 31) == 0) atomicMax(&sc->gmax, m);
}

// Per free block over its residual-slots (sorted): g_j = sum Jc_s^T r~ and
// the diagonal of the direct block sum Jc_s^T Jc_s (Marquardt D).
__global__ void k_gba_block_grad(int nf, const int* __restrict__ sptr, const int64_t* __restrict__ slist,
                                 const double* __restrict__ rec, double* __restrict__ gc,
                                 double* __restrict__ hdiag) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nf) return;
  double g[6] = {0, 0, 0, 0, 0, 0}, d[6] = {0, 0, 0, 0, 0, 0};
  for (int k = sptr[j]; k < sptr[j + 1]; ++k) {
    const int64_t code = slist[k];
    const double* o = rec + (code >> 1) * kGbaRec;
    const double* J = o + ((code & 1) ? 20 : 8);
    for (int c = 0; c < 6; ++c) {
      g[c] += J[c] * o[0] + J[6 + c] * o[1];
      d[c] += J[c] * J[c] + J[6 + c] * J[6 + c];
    }
  }
  for (int c = 0; c < 6; ++c) {
    gc[j * 6 + c] = g[c];
    hdiag[j * 6 + c] = d[c];
  }
}

// Pose terms per free block in term order: U_term (self block), g_term;
// edge cross blocks per edge (oriented as the upper block).
struct GbaTermArgs {
  int nf, E, A;
  const int* term_ptr;
  const int* term_list;  // term << 2 | side
  const int* ab;
  const int* pb;
  const double* ew;      // per-edge sqrt(lambda)
  const double* pw;      // per-prior sqrt(weight)
  const double* meas_inv;
  const double* init_inv;
  const int* free_idx;
  const double* q;
  const double* t;
  const double* Rt;
  double* Ut;            // [nf*36]
  double* gt;            // [nf*6]
  double* edge_H;        // [E*36]
};

__global__ void k_gba_terms_lin(GbaTermArgs a) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < a.nf) {
    double U[36], g[6];
    for (int k = 0; k < 36; ++k) U[k] = 0.0;
    for (int k = 0; k < 6; ++k) g[k] = 0.0;
    for (int k = a.term_ptr[j]; k < a.term_ptr[j + 1]; ++k) {
      const int code = a.term_list[k];
      const int term = code >> 2, side = code & 3;
      double r[6], J[36];
      if (term < a.E) {
        const Pose Ta = load_pose(a.q, a.t, a.Rt, a.ab[2 * term]);
        const Pose Tb = load_pose(a.q, a.t, a.Rt, a.ab[2 * term + 1]);
        if (side == 0) edge_eval(a.meas_inv + term * 7, Ta, Tb, a.ew[term], r, J, nullptr);
        else edge_eval(a.meas_inv + term * 7, Ta, Tb, a.ew[term], r, nullptr, J);
      } else {
        const int pi = term - a.E;
        prior_eval(a.init_inv + pi * 7, load_pose(a.q, a.t, a.Rt, a.pb[pi]), a.pw[pi], r, J);
      }
      for (int rr = 0; rr < 6; ++rr) {
        for (int cc = 0; cc < 6; ++cc) {
          double s = 0.0;
          for (int m = 0; m < 6; ++m) s += J[m * 6 + rr] * J[m * 6 + cc];
          U[rr * 6 + cc] += s;
        }
        double s = 0.0;
        for (int m = 0; m < 6; ++m) s += J[m * 6 + rr] * r[m];
        g[rr] += s;
      }
    }
    for (int k = 0; k < 36; ++k) a.Ut[(int64_t)j * 36 + k] = U[k];
    for (int k = 0; k < 6; ++k) a.gt[(int64_t)j * 6 + k] = g[k];
  }
  // edge cross blocks (one thread per edge, after the self blocks' threads)
  const int e = j;
  if (e < a.E) {
    const int fa = a.ab[2 * e], fb = a.ab[2 * e + 1];
    const int ja = a.free_idx[fa], jb = a.free_idx[fb];
    if (ja < 0 || jb < 0) return;
    const Pose Ta = load_pose(a.q, a.t, a.Rt, fa), Tb = load_pose(a.q, a.t, a.Rt, fb);
    double r[6], Ja[36], Jb[36];
    edge_eval(a.meas_inv + e * 7, Ta, Tb, a.ew[e], r, Ja, Jb);
    // H_(a,b) = Ja^T Jb, stored as the block (min, max)
    const bool swap = ja > jb;
    for (int rr = 0; rr < 6; ++rr)
      for (int cc = 0; cc < 6; ++cc) {
        double s = 0.0;
        for (int m = 0; m < 6; ++m) s += swap ? Jb[m * 6 + rr] * Ja[m * 6 + cc] : Ja[m * 6 + rr] * Jb[m * 6 + cc];
        a.edge_H[(int64_t)e * 36 + rr * 6 + cc] = s;
      }
  }
}

// S blocks: warp per upper block (a <= b) over its entries (sorted once per
// solve).  Entry = (residual x, slot sx, residual y, slot sy, kind):
//   kind 0 (Schur):  -Jc_x^T (Jp_x V*^-1 Jp_y^T) Jc_y   (same point)
//   kind 1 (direct):  Jc_x^T Jc_y                       (same residual)
// Lane l takes entry l of each 32-entry batch, writes its 6x6 to a shared-
// memory row, lane c sums column c over the rows: fixed order.
struct GbaBlockArgs {
  int n_ub;
  const int2* ub_key;       // (a, b) free-block indices, a <= b
  const int64_t* ent_ptr;   // [n_ub+1]
  const int4* ent;          // (x, y, sx | sy << 1 | kind << 2, point)
  const double* rec;
  const double* pv;         // packed V*^-1 | e per point
  const double* Ut;         // pose-term self blocks
  const double* hdiag;      // direct diag (Marquardt D with Ut)
  const int* ub_edge;       // edge id of block or -1
  const double* edge_H;
  const int* pos_up;
  const int* pos_lo;
  double lam;
  double* S;
};

__global__ void __launch_bounds__(128) k_gba_blocks(GbaBlockArgs a) {
  __shared__ double Tsm[4][32][37];
  const int u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (u >= a.n_ub) return;
  const int2 key = a.ub_key[u];
  double acc0 = 0.0, acc1 = 0.0;
  double* row = &Tsm[warp][lane][0];
  const int64_t k0 = a.ent_ptr[u], k1 = a.ent_ptr[u + 1];
  for (int64_t kb = k0; kb < k1; kb += 32) {
    const int64_t k = kb + lane;
    const int nv = (int)min((int64_t)32, k1 - kb);
    if (k < k1) {
      const int4 e = a.ent[k];
      const double* ox = a.rec + (int64_t)e.x * kGbaRec;
      const double* oy = a.rec + (int64_t)e.y * kGbaRec;
      const double* Jx = ox + ((e.z & 1) ? 20 : 8);
      const double* Jy = oy + ((e.z & 2) ? 20 : 8);
      double m00, m01, m10, m11;
      if (e.z & 4) {
        m00 = 1.0; m01 = 0.0; m10 = 0.0; m11 = 1.0;
      } else {
        const double* pv = a.pv + (int64_t)e.w * 12;
        const double* Px = ox + 2;
        const double* Py = oy + 2;
        double P[6];
        for (int r = 0; r < 2; ++r) {
          P[r * 3 + 0] = pv[0] * Py[r * 3] + pv[1] * Py[r * 3 + 1] + pv[2] * Py[r * 3 + 2];
          P[r * 3 + 1] = pv[1] * Py[r * 3] + pv[3] * Py[r * 3 + 1] + pv[4] * Py[r * 3 + 2];
          P[r * 3 + 2] = pv[2] * Py[r * 3] + pv[4] * Py[r * 3 + 1] + pv[5] * Py[r * 3 + 2];
        }
        m00 = -(Px[0] * P[0] + Px[1] * P[1] + Px[2] * P[2]);
        m01 = -(Px[0] * P[3] + Px[1] * P[4] + Px[2] * P[5]);
        m10 = -(Px[3] * P[0] + Px[4] * P[1] + Px[5] * P[2]);
        m11 = -(Px[3] * P[3] + Px[4] * P[4] + Px[5] * P[5]);
      }
      double MJ[12];
      for (int c = 0; c < 6; ++c) {
        MJ[c] = m00 * Jy[c] + m01 * Jy[6 + c];
        MJ[6 + c] = m10 * Jy[c] + m11 * Jy[6 + c];
      }
      for (int r = 0; r < 6; ++r)
        for (int c = 0; c < 6; ++c) row[r * 6 + c] = Jx[r] * MJ[c] + Jx[6 + r] * MJ[6 + c];
    }
    __syncwarp();
    for (int l = 0; l < nv; ++l) {
      acc0 += Tsm[warp][l][lane];
      if (lane < 4) acc1 += Tsm[warp][l][32 + lane];
    }
    __syncwarp();
  }
  const int e0 = lane, e1 = 32 + lane;
  if (key.x == key.y) {  // pose terms + Marquardt damping (solver.py:217-220)
    const int j = key.x;
    acc0 += a.Ut[(int64_t)j * 36 + e0];
    if (e0 % 7 == 0) acc0 += a.lam * fmax(a.hdiag[j * 6 + e0 / 7] + a.Ut[(int64_t)j * 36 + e0], 1e-12);
    if (lane < 4) {
      acc1 += a.Ut[(int64_t)j * 36 + e1];
      if (e1 % 7 == 0) acc1 += a.lam * fmax(a.hdiag[j * 6 + e1 / 7] + a.Ut[(int64_t)j * 36 + e1], 1e-12);
    }
  } else if (a.ub_edge[u] >= 0) {
    const double* H = a.edge_H + (int64_t)a.ub_edge[u] * 36;
    acc0 += H[e0];
    if (lane < 4) acc1 += H[e1];
  }
  double* up = a.S + (int64_t)a.pos_up[u] * 36;
  up[e0] = acc0;
  if (lane < 4) up[e1] = acc1;
  if (key.x != key.y) {
    double* dn = a.S + (int64_t)a.pos_lo[u] * 36;
    dn[(e0 % 6) * 6 + e0 / 6] = acc0;
    if (lane < 4) dn[(e1 % 6) * 6 + e1 / 6] = acc1;
  }
}

// b_j = -g_j + sum_s Jc_s^T Jp e_p (-> Schur right-hand side), in slot order.
__global__ void k_gba_rhs(int nf, const int* __restrict__ sptr, const int64_t* __restrict__ slist,
                          const int* __restrict__ rpt, const double* __restrict__ rec,
                          const double* __restrict__ pv, const double* __restrict__ gc,
                          const double* __restrict__ gt, double* __restrict__ b) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nf) return;
  double s[6];
  for (int c = 0; c < 6; ++c) s[c] = -(gc[j * 6 + c] + gt[j * 6 + c]);
  for (int k = sptr[j]; k < sptr[j + 1]; ++k) {
    const int64_t code = slist[k];
    const int64_t i = code >> 1;
    const double* o = rec + i * kGbaRec;
    const double* J = o + ((code & 1) ? 20 : 8);
    const double* e = pv + (int64_t)rpt[i] * 12 + 6;
    const double y0 = o[2] * e[0] + o[3] * e[1] + o[4] * e[2];
    const double y1 = o[5] * e[0] + o[6] * e[1] + o[7] * e[2];
    for (int c = 0; c < 6; ++c) s[c] += J[c] * y0 + J[6 + c] * y1;
  }
  for (int c = 0; c < 6; ++c) b[j * 6 + c] = s[c];
}

// delta_p = -e - V*^-1 sum_{residual slots} Jp^T Jc_s dc_blk(s); X' = X + dp.
__global__ void __launch_bounds__(kBlock) k_gba_point_trial(int64_t P, const int64_t* __restrict__ pptr,
                                                            const int* __restrict__ rkind,
                                                            const int* __restrict__ rslot,
                                                            const int* __restrict__ free_idx,
                                                            const double* __restrict__ rec,
                                                            const double* __restrict__ pv,
                                                            const double* __restrict__ dc,
                                                            const double* __restrict__ X,
                                                            double* __restrict__ Xo, double* __restrict__ part,
                                                            BAScalars* sc) {
  __shared__ double red[kBlock / 32];
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double dp2 = 0.0;
  if (p < P) {
    double acc[3] = {0, 0, 0};
    for (int64_t i = pptr[p]; i < pptr[p + 1]; ++i) {
      const double* o = rec + i * kGbaRec;
      const int ns = rkind[i] == SFM_RES_GLOBAL ? 1 : 2;
      for (int sl = 0; sl < ns; ++sl) {
        const int j = free_idx[rslot[2 * i + sl]];
        if (j < 0) continue;
        const double* J = o + (sl ? 20 : 8);
        double y0 = 0.0, y1 = 0.0;
        for (int c = 0; c < 6; ++c) {
          y0 += J[c] * dc[j * 6 + c];
          y1 += J[6 + c] * dc[j * 6 + c];
        }
        acc[0] += o[2] * y0 + o[5] * y1;
        acc[1] += o[3] * y0 + o[6] * y1;
        acc[2] += o[4] * y0 + o[7] * y1;
      }
    }
    const double* v = pv + p * 12;
    const double d0 = -v[6] - (v[0] * acc[0] + v[1] * acc[1] + v[2] * acc[2]);
    const double d1 = -v[7] - (v[1] * acc[0] + v[3] * acc[1] + v[4] * acc[2]);
    const double d2 = -v[8] - (v[2] * acc[0] + v[4] * acc[1] + v[5] * acc[2]);
    if (!(isfinite(d0) && isfinite(d1) && isfinite(d2))) atomicOr(&sc->nonfinite, 1);
    dp2 = d0 * d0 + d1 * d1 + d2 * d2;
    Xo[p * 3] = X[p * 3] + d0;
    Xo[p * 3 + 1] = X[p * 3 + 1] + d1;
    Xo[p * 3 + 2] = X[p * 3 + 2] + d2;
  }
  const double s = block_sum<kBlock>(dp2, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// Problem.evaluate over the residuals (solver.py:132-151): robust cost of
// the state in `a`; the first residual whose projection raises is recorded.
__global__ void __launch_bounds__(kBlock) k_gba_cost(GbaArgs a, int64_t off, double* __restrict__ part,
                                                     BAScalars* sc) {
  __shared__ double red[kBlock / 32];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double c = 0.0;
  unsigned long long bad = ~0ull;
  if (i < a.R) {
    const Pose T = gba_pose(a, i, nullptr, nullptr);
    const Vec3 pc = add(mul(T.R, load_X(a.X, a.rpt[i])), T.t);
    double u, v;
    if (project_point(a.models[a.rmodel[i]], pc, u, v) != PROJ_OK) {
      bad = (unsigned long long)(off + i);
    } else {
      const double r0 = u - a.ruv[2 * i], r1 = v - a.ruv[2 * i + 1];
      c = loss_rho(a.lk, a.lp, r0 * r0 + r1 * r1);
    }
  }
  unsigned long long wb = bad;
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long x = __shfl_down_sync(0xffffffffu, wb, o);
    wb = x < wb ? x : wb;
  }
  if ((threadIdx.x & 31) == 0 && wb != ~0ull) atomicMin(&sc->depth_obs, wb);
  const double s = block_sum<kBlock>(c, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// Pose-term cost with per-term weights (trivial loss, mapping.py:485-509).
__global__ void __launch_bounds__(kBlock) k_gba_terms_cost(int E, int A, const int* __restrict__ ab,
                                                           const int* __restrict__ pb,
                                                           const double* __restrict__ meas_inv,
                                                           const double* __restrict__ init_inv,
                                                           const double* __restrict__ ew,
                                                           const double* __restrict__ pw, const double* q,
                                                           const double* t, const double* Rt,
                                                           double* __restrict__ part) {
  __shared__ double red[kBlock / 32];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double c = 0.0, r[6];
  if (i < E) {
    edge_eval(meas_inv + i * 7, load_pose(q, t, Rt, ab[2 * i]), load_pose(q, t, Rt, ab[2 * i + 1]), ew[i], r,
              nullptr, nullptr);
    for (int k = 0; k < 6; ++k) c += r[k] * r[k];
  } else if (i < E + A) {
    prior_eval(init_inv + (i - E) * 7, load_pose(q, t, Rt, pb[i - E]), pw[i - E], r, nullptr);
    for (int k = 0; k < 6; ++k) c += r[k] * r[k];
  }
  const double s = block_sum<kBlock>(c, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// Probe of one residual's projection failure (message payload).
__global__ void k_gba_probe(GbaArgs a, int64_t i, BAScalars* sc) {
  const Pose T = gba_pose(a, i, nullptr, nullptr);
  const Vec3 pc = add(mul(T.R, load_X(a.X, a.rpt[i])), T.t);
  double u, v;
  sc->proj_code = project_point(a.models[a.rmodel[i]], pc, u, v);
  sc->proj_depth = pc.z;
}

}  // namespace

// ===========================================================================
// host driver
// ===========================================================================

void GBASolver::setup(const sfm_gba_problem& pr, const sfm_ba_options& opt) {
  opt_ = opt;
  cudaStream_t s = stream_;
  SFM_REQUIRE(pr.n_blocks >= 0 && pr.n_points >= 0 && pr.n_res >= 0, "negative sizes");
  SFM_REQUIRE(pr.n_res < (1ll << 30), "too many residuals");
  SFM_REQUIRE(opt.loss_kind >= 0 && opt.loss_kind <= 2, "unknown loss kind");
  nb_ = pr.n_blocks;
  P_ = pr.n_points;
  R_ = pr.n_res;
  E_ = pr.n_edges;
  A_ = pr.n_priors;
  // free blocks (solver.py:154-161: free blocks in insertion order)
  std::vector<int> free_idx(nb_), free_block;
  for (int b = 0; b < nb_; ++b) {
    if (pr.block_fixed[b]) free_idx[b] = -1;
    else { free_idx[b] = (int)free_block.size(); free_block.push_back(b); }
  }
  nf_ = (int)free_block.size();
  n_params_ = (int64_t)nf_ * 6 + P_ * 3;
  // residual validation + point CSR + slot lists
  std::vector<int64_t> pptr(P_ + 1, 0);
  std::vector<std::vector<int64_t>> per_block(nf_);  // residual << 1 | slot
  for (int64_t i = 0; i < R_; ++i) {
    const int p = pr.res_point[i];
    SFM_REQUIRE(p >= 0 && p < P_ && (i == 0 || pr.res_point[i - 1] <= p), "residuals must be sorted by point");
    SFM_REQUIRE(pr.res_model[i] >= 0 && pr.res_model[i] < pr.n_models, "res_model out of range");
    const int kind = pr.res_kind[i];
    SFM_REQUIRE(kind == SFM_RES_GLOBAL || kind == SFM_RES_ROLLING || kind == SFM_RES_RIG, "unknown residual kind");
    const int ns = kind == SFM_RES_GLOBAL ? 1 : 2;
    for (int sl = 0; sl < ns; ++sl) {
      const int b = pr.res_slot[2 * i + sl];
      SFM_REQUIRE(b >= 0 && b < nb_, "residual slot out of range");
      if (free_idx[b] >= 0) per_block[free_idx[b]].push_back(i << 1 | sl);
    }
    ++pptr[p + 1];
  }
  for (int64_t p = 0; p < P_; ++p) pptr[p + 1] += pptr[p];
  std::vector<int> sptr(nf_ + 1, 0);
  std::vector<int64_t> slist;
  for (int j = 0; j < nf_; ++j) {
    slist.insert(slist.end(), per_block[j].begin(), per_block[j].end());
    sptr[j + 1] = (int)slist.size();
  }
  // S entries: per point, ordered pairs of its free residual slots with
  // blk(x) <= blk(y); Schur for all, direct for same-residual pairs.
  struct Ent { int a, b; int64_t p; int x, y, code; };
  std::vector<Ent> ents;
  std::vector<std::pair<int64_t, int>> sl;  // (residual << 1 | slot, free block)
  for (int64_t p = 0; p < P_; ++p) {
    sl.clear();
    for (int64_t i = pptr[p]; i < pptr[p + 1]; ++i) {
      const int ns = pr.res_kind[i] == SFM_RES_GLOBAL ? 1 : 2;
      for (int k = 0; k < ns; ++k) {
        const int j = free_idx[pr.res_slot[2 * i + k]];
        if (j >= 0) sl.push_back({i << 1 | k, j});
      }
    }
    for (auto& X : sl)
      for (auto& Y : sl) {
        if (X.second > Y.second) continue;
        const int x = (int)(X.first >> 1), y = (int)(Y.first >> 1);
        const int sx = (int)(X.first & 1), sy = (int)(Y.first & 1);
        ents.push_back({X.second, Y.second, p, x, y, sx | sy << 1});
        if (x == y) ents.push_back({X.second, Y.second, p, x, y, sx | sy << 1 | 4});
      }
  }
  std::stable_sort(ents.begin(), ents.end(), [](const Ent& u, const Ent& v) {
    return u.a != v.a ? u.a < v.a : u.b < v.b;
  });
  // upper blocks: entry keys + every free diagonal + pose edges
  std::vector<int> ab_h(2 * (size_t)E_);
  if (E_) std::memcpy(ab_h.data(), pr.edge_ab, sizeof(int) * 2 * E_);
  std::vector<std::pair<int, int>> keys;
  for (auto& e : ents) keys.push_back({e.a, e.b});
  for (int j = 0; j < nf_; ++j) keys.push_back({j, j});
  std::vector<int> edge_key(E_, -1);
  for (int e = 0; e < E_; ++e) {
    SFM_REQUIRE(ab_h[2 * e] >= 0 && ab_h[2 * e] < nb_ && ab_h[2 * e + 1] >= 0 && ab_h[2 * e + 1] < nb_ &&
                    ab_h[2 * e] != ab_h[2 * e + 1],
                "edge blocks out of range");
    const int ja = free_idx[ab_h[2 * e]], jb = free_idx[ab_h[2 * e + 1]];
    if (ja >= 0 && jb >= 0) keys.push_back({std::min(ja, jb), std::max(ja, jb)});
  }
  std::sort(keys.begin(), keys.end());
  keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
  n_ub_ = (int)keys.size();
  std::vector<int2> ub_key(n_ub_);
  std::vector<int64_t> ent_ptr(n_ub_ + 1, 0);
  std::vector<int4> ent4(ents.size());
  {
    size_t q = 0;
    for (int u = 0; u < n_ub_; ++u) {
      ub_key[u] = make_int2(keys[u].first, keys[u].second);
      while (q < ents.size() && ents[q].a == keys[u].first && ents[q].b == keys[u].second) {
        ent4[q] = make_int4(ents[q].x, ents[q].y, ents[q].code, (int)ents[q].p);
        ++q;
      }
      ent_ptr[u + 1] = (int64_t)q;
    }
  }
  std::vector<int> ub_edge(n_ub_, -1);
  for (int e = 0; e < E_; ++e) {
    const int ja = free_idx[ab_h[2 * e]], jb = free_idx[ab_h[2 * e + 1]];
    if (ja < 0 || jb < 0) continue;
    const auto kk = std::make_pair(std::min(ja, jb), std::max(ja, jb));
    const int u = (int)(std::lower_bound(keys.begin(), keys.end(), kk) - keys.begin());
    SFM_REQUIRE(ub_edge[u] < 0, "duplicate pose edge between the same blocks");
    ub_edge[u] = e;
  }
  // BSR (both triangles)
  std::vector<std::vector<std::pair<int, int>>> rows(nf_);  // (col, slot-key)
  for (int u = 0; u < n_ub_; ++u) {
    rows[ub_key[u].x].push_back({ub_key[u].y, u});
    if (ub_key[u].x != ub_key[u].y) rows[ub_key[u].y].push_back({ub_key[u].x, -1 - u});
  }
  std::vector<int> row_ptr(nf_ + 1, 0), col;
  std::vector<int> pos_up(n_ub_), pos_lo(n_ub_), diag_pos(nf_);
  for (int r = 0; r < nf_; ++r) {
    std::sort(rows[r].begin(), rows[r].end());
    for (auto& c : rows[r]) {
      const int slot = (int)col.size();
      col.push_back(c.first);
      if (c.second >= 0) pos_up[c.second] = slot;
      else pos_lo[-1 - c.second] = slot;
      if (c.first == r) diag_pos[r] = slot;
    }
    row_ptr[r + 1] = (int)col.size();
  }
  n_full_ = (int)col.size();
  // pose terms per free block (edge side 0 = a, 1 = b; prior 2)
  std::vector<std::vector<int>> tl(nf_);
  std::vector<int> pb_h(A_);
  if (A_) std::memcpy(pb_h.data(), pr.prior_block, sizeof(int) * A_);
  for (int e = 0; e < E_; ++e) {
    const int ja = free_idx[ab_h[2 * e]], jb = free_idx[ab_h[2 * e + 1]];
    if (ja >= 0) tl[ja].push_back(e << 2 | 0);
    if (jb >= 0) tl[jb].push_back(e << 2 | 1);
  }
  for (int k = 0; k < A_; ++k) {
    SFM_REQUIRE(pb_h[k] >= 0 && pb_h[k] < nb_, "prior block out of range");
    if (free_idx[pb_h[k]] >= 0) tl[free_idx[pb_h[k]]].push_back((E_ + k) << 2 | 2);
  }
  std::vector<int> term_ptr(nf_ + 1, 0), term_list;
  for (int j = 0; j < nf_; ++j) {
    term_list.insert(term_list.end(), tl[j].begin(), tl[j].end());
    term_ptr[j + 1] = (int)term_list.size();
  }
  std::vector<double> ew(E_), pw(A_);
  for (int e = 0; e < E_; ++e) ew[e] = std::sqrt(pr.edge_weight[e]);
  for (int k = 0; k < A_; ++k) pw[k] = std::sqrt(pr.prior_weight[k]);

  // ---- uploads ---------------------------------------------------------------
  models_.upload(pr.models, pr.n_models, s);
  for (int k = 0; k < 2; ++k) {
    q_[k].upload(pr.block_q, (size_t)nb_ * 4, s);
    t_[k].upload(pr.block_t, (size_t)nb_ * 3, s);
    Rt_[k].resize((size_t)nb_ * 12);
    if (nb_) k_frames_rt<<<grid_for(nb_, 128), 128, 0, s>>>(nb_, q_[k].get(), t_[k].get(), Rt_[k].get(), nullptr);
    X_[k].upload(pr.points, (size_t)P_ * 3, s);
  }
  cur_ = 0;
  rpt_.upload(pr.res_point, R_, s);
  rmodel_.upload(pr.res_model, R_, s);
  rkind_.upload(pr.res_kind, R_, s);
  rslot_.upload(pr.res_slot, 2 * (size_t)R_, s);
  std::vector<double> alpha(R_, 0.0);
  if (pr.res_alpha) std::memcpy(alpha.data(), pr.res_alpha, sizeof(double) * R_);
  ralpha_.upload(alpha.data(), R_, s);
  ruv_.upload(pr.res_uv, 2 * (size_t)R_, s);
  pptr_.upload(pptr.data(), pptr.size(), s);
  free_idx_.upload(free_idx.data(), nb_, s);
  free_block_.upload(free_block.data(), nf_, s);
  sptr_.upload(sptr.data(), sptr.size(), s);
  slist_.upload(slist.data(), slist.size(), s);
  ub_key_.upload(ub_key.data(), ub_key.size(), s);
  ent_ptr_.upload(ent_ptr.data(), ent_ptr.size(), s);
  ent_.upload(ent4.data(), ent4.size(), s);
  ub_edge_.upload(ub_edge.data(), ub_edge.size(), s);
  pos_up_.upload(pos_up.data(), pos_up.size(), s);
  pos_lo_.upload(pos_lo.data(), pos_lo.size(), s);
  row_ptr_.upload(row_ptr.data(), row_ptr.size(), s);
  col_.upload(col.data(), col.size(), s);
  diag_pos_.upload(diag_pos.data(), diag_pos.size(), s);
  edge_ab_.upload(ab_h.data(), ab_h.size(), s);
  prior_block_.upload(pb_h.data(), pb_h.size(), s);
  ew_.upload(ew.data(), ew.size(), s);
  pw_.upload(pw.data(), pw.size(), s);
  term_ptr_.upload(term_ptr.data(), term_ptr.size(), s);
  term_list_.upload(term_list.data(), term_list.size(), s);
  meas_inv_.resize((size_t)E_ * 7);
  init_inv_.resize((size_t)A_ * 7);
  if (E_ + A_)
    k_terms_init<<<grid_for(E_ + A_, 128), 128, 0, s>>>(E_, A_, edge_ab_.get(), prior_block_.get(), q_[0].get(),
                                                         t_[0].get(), Rt_[0].get(), meas_inv_.get(), init_inv_.get());
  SFM_CHECK_LAUNCH();
  rec_.resize((size_t)R_ * kGbaRec);
  V_.resize((size_t)P_ * 6);
  gp_.resize((size_t)P_ * 3);
  pv_.resize((size_t)P_ * 12);
  gc_.resize((size_t)nf_ * 6);
  hdiag_.resize((size_t)nf_ * 6);
  Ut_.resize((size_t)nf_ * 36);
  gt_.resize((size_t)nf_ * 6);
  edge_H_.resize((size_t)std::max(E_, 1) * 36);
  S_.resize((size_t)n_full_ * 36);
  b_.resize((size_t)nf_ * 6);
  dc_.resize((size_t)nf_ * 6);
  sc_.resize(1);
  SFM_CUDA(cudaMemsetAsync(sc_.get(), 0, sizeof(BAScalars), s));
  part_a_.resize(grid_for(std::max<int64_t>(R_, 1), kBlock));
  part_b_.resize(grid_for(std::max<int64_t>(P_, 1), kBlock));
  part_c_.resize(grid_for(std::max(E_ + A_, 1), kBlock));
  part_d_.resize(grid_for(std::max(nf_, 1), kBlock));
  use_dense_ = 6 * nf_ <= kDenseMax && opt.linear_solver != SFM_LINSOLVE_PCG;
  if (use_dense_ && nf_) {
    const size_t smem = sizeof(double) * (size_t)(6 * nf_) * (6 * nf_ + 1) / 2;
    SFM_CUDA(cudaFuncSetAttribute(k_dense_solve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)std::max<size_t>(smem, 1)));
  } else if (nf_) {
    pcg_.setup(nf_, -1, 1, s);  // block-Jacobi PCG (the rigid-motion coarse space is frame-specific)
    pcg_.set_pattern(row_ptr_.get(), col_.get(), n_full_, s);
  }
  iters_ = 0;
  n_trials_ = 0;
  pcg_total_ = 0;
  term_ = SFM_TERM_MAX_ITERATIONS;
  lam_ = opt_.initial_lambda;
  initial_cost_ = eval_cost(cur_, cur_);
  cost_ = initial_cost_;
  finished_ = false;
  if (n_params_ == 0 || (R_ == 0 && E_ == 0 && A_ == 0)) {
    term_ = SFM_TERM_ALL_FIXED;
    finished_ = true;
  } else if (opt_.max_iters <= 0) {
    finished_ = true;
  }
}

GbaArgs GBASolver::args(int blocks, int points) const {
  GbaArgs a{};
  a.R = R_; a.P = P_; a.nb = nb_;
  a.rpt = rpt_.get(); a.rmodel = rmodel_.get(); a.rkind = rkind_.get(); a.rslot = rslot_.get();
  a.ralpha = ralpha_.get(); a.ruv = ruv_.get(); a.models = models_.get();
  a.q = q_[blocks].get(); a.t = t_[blocks].get(); a.Rt = Rt_[blocks].get(); a.X = X_[points].get();
  a.lk = opt_.loss_kind; a.lp = opt_.loss_param;
  return a;
}

void GBASolver::read() {
  sc_.download(&h_sc_, 1, stream_);
  SFM_CUDA(cudaStreamSynchronize(stream_));
}

void GBASolver::raise_projection(int blocks, int points) {
  const int64_t i = (int64_t)h_sc_.depth_obs;
  k_gba_probe<<<1, 1, 0, stream_>>>(args(blocks, points), i, sc_.get());
  SFM_CHECK_LAUNCH();
  read();
  char msg[160];
  if (h_sc_.proj_code == PROJ_DOMAIN) {
    std::snprintf(msg, sizeof(msg), "incidence angle beyond model domain (observation %lld)", (long long)i);
    throw SfmError(SFM_E_OUT_OF_MODEL_DOMAIN, msg);
  }
  std::snprintf(msg, sizeof(msg), "depth %.3e", h_sc_.proj_depth);
  throw SfmError(SFM_E_NON_POSITIVE_DEPTH, msg);
}

// cost of (blocks state, points state); raises on a projection failure
double GBASolver::eval_cost(int blocks, int points) {
  cudaStream_t s = stream_;
  k_reset_scalars<<<1, 1, 0, s>>>(sc_.get(), 0);
  const unsigned gr = grid_for(std::max<int64_t>(R_, 1), kBlock);
  const unsigned gt = grid_for(std::max(E_ + A_, 1), kBlock);
  k_gba_cost<<<gr, kBlock, 0, s>>>(args(blocks, points), 0, part_a_.get(), sc_.get());
  k_gba_terms_cost<<<gt, kBlock, 0, s>>>(E_, A_, edge_ab_.get(), prior_block_.get(), meas_inv_.get(), init_inv_.get(),
                                        ew_.get(), pw_.get(), q_[blocks].get(), t_[blocks].get(), Rt_[blocks].get(),
                                        part_c_.get());
  k_finalize<<<1, 256, 0, s>>>(part_a_.get(), (int)gr, nullptr, 0, part_c_.get(), (int)gt, nullptr, 0, sc_.get(), 0);
  SFM_CHECK_LAUNCH();
  prof_->launches += 4;
  read();
  if (h_sc_.depth_obs != ~0ull) raise_projection(blocks, points);
  return h_sc_.cost;
}

void GBASolver::linearize() {
  cudaStream_t s = stream_;
  k_reset_scalars<<<1, 1, 0, s>>>(sc_.get(), 0);
  if (R_) k_gba_lin<<<grid_for(R_, 128), 128, 0, s>>>(args(cur_, cur_), rec_.get(), sc_.get());
  if (P_) k_gba_point_lin<<<grid_for(P_, 128), 128, 0, s>>>(P_, pptr_.get(), rec_.get(), V_.get(), gp_.get(), sc_.get());
  if (nf_) {
    k_gba_block_grad<<<grid_for(nf_, 64), 64, 0, s>>>(nf_, sptr_.get(), slist_.get(), rec_.get(), gc_.get(),
                                                      hdiag_.get());
    GbaTermArgs t{};
    t.nf = nf_; t.E = E_; t.A = A_; t.term_ptr = term_ptr_.get(); t.term_list = term_list_.get();
    t.ab = edge_ab_.get(); t.pb = prior_block_.get(); t.ew = ew_.get(); t.pw = pw_.get();
    t.meas_inv = meas_inv_.get(); t.init_inv = init_inv_.get(); t.free_idx = free_idx_.get();
    t.q = q_[cur_].get(); t.t = t_[cur_].get(); t.Rt = Rt_[cur_].get();
    t.Ut = Ut_.get(); t.gt = gt_.get(); t.edge_H = edge_H_.get();
    k_gba_terms_lin<<<grid_for(std::max(nf_, E_), 64), 64, 0, s>>>(t);
  }
  SFM_CHECK_LAUNCH();
  prof_->launches += 4;
  read();
  // gradient max over the camera side (g_c + pose terms), solver.py:211-215
  std::vector<double> g((size_t)nf_ * 6), gt((size_t)nf_ * 6);
  gc_.download(g.data(), g.size(), s);
  gt_.download(gt.data(), gt.size(), s);
  SFM_CUDA(cudaStreamSynchronize(s));
  double gm = __longlong_as_double_host(h_sc_.gmax);
  for (size_t k = 0; k < g.size(); ++k) {
    const double v = g[k] + gt[k];
    gm = std::isnan(v) || std::isnan(gm) ? NAN : std::max(gm, std::fabs(v));
  }
  gmax_ = gm;
}

bool GBASolver::trial(double lam, double* new_cost, double* step_norm) {
  cudaStream_t s = stream_;
  k_reset_scalars<<<1, 1, 0, s>>>(sc_.get(), 1);
  if (P_) k_point_prep<<<grid_for(P_, 256), 256, 0, s>>>(P_, lam, V_.get(), gp_.get(), pv_.get(), sc_.get());
  if (nf_) {
    GbaBlockArgs b{};
    b.n_ub = n_ub_; b.ub_key = ub_key_.get(); b.ent_ptr = ent_ptr_.get(); b.ent = ent_.get(); b.rec = rec_.get();
    b.pv = pv_.get(); b.Ut = Ut_.get(); b.hdiag = hdiag_.get(); b.ub_edge = ub_edge_.get(); b.edge_H = edge_H_.get();
    b.pos_up = pos_up_.get(); b.pos_lo = pos_lo_.get(); b.lam = lam; b.S = S_.get();
    k_gba_blocks<<<grid_for((int64_t)n_ub_ * 32, 128), 128, 0, s>>>(b);
    k_gba_rhs<<<grid_for(nf_, 64), 64, 0, s>>>(nf_, sptr_.get(), slist_.get(), rpt_.get(), rec_.get(), pv_.get(),
                                               gc_.get(), gt_.get(), b_.get());
    if (use_dense_) {
      const size_t smem = sizeof(double) * (size_t)(6 * nf_) * (6 * nf_ + 1) / 2;
      k_dense_solve<<<1, 1024, smem, s>>>(nf_, row_ptr_.get(), col_.get(), S_.get(), b_.get(), dc_.get(), sc_.get());
    } else {
      PcgProblem pp{};
      pp.nf = nf_; pp.row_ptr = row_ptr_.get(); pp.col = col_.get(); pp.S = S_.get(); pp.nnzb = n_full_;
      pp.diag_pos = diag_pos_.get(); pp.b = b_.get(); pp.x = dc_.get(); pp.lam = lam;
      pcg_.solve(pp, opt_.pcg_max_iters > 0 ? opt_.pcg_max_iters : 1000, opt_.pcg_rtol > 0 ? opt_.pcg_rtol : 1e-10,
                 sc_.get(), s, prof_);
    }
  }
  const int o = cur_ ^ 1;
  const unsigned gd = grid_for(std::max(nf_, 1), kBlock);
  // trial state: all blocks copied, free ones retracted; points X + dp
  SFM_CUDA(cudaMemcpyAsync(q_[o].get(), q_[cur_].get(), sizeof(double) * 4 * nb_, cudaMemcpyDeviceToDevice, s));
  SFM_CUDA(cudaMemcpyAsync(t_[o].get(), t_[cur_].get(), sizeof(double) * 3 * nb_, cudaMemcpyDeviceToDevice, s));
  SFM_CUDA(cudaMemcpyAsync(Rt_[o].get(), Rt_[cur_].get(), sizeof(double) * 12 * nb_, cudaMemcpyDeviceToDevice, s));
  if (nf_)
    k_cam_trial<<<gd, kBlock, 0, s>>>(nf_, free_block_.get(), dc_.get(), q_[cur_].get(), t_[cur_].get(),
                                      Rt_[cur_].get(), q_[o].get(), t_[o].get(), Rt_[o].get(), nullptr,
                                      part_d_.get(), sc_.get());
  const unsigned gp = grid_for(std::max<int64_t>(P_, 1), kBlock);
  if (P_)
    k_gba_point_trial<<<gp, kBlock, 0, s>>>(P_, pptr_.get(), rkind_.get(), rslot_.get(), free_idx_.get(), rec_.get(),
                                            pv_.get(), dc_.get(), X_[cur_].get(), X_[o].get(), part_b_.get(),
                                            sc_.get());
  const unsigned gr = grid_for(std::max<int64_t>(R_, 1), kBlock);
  const unsigned gt = grid_for(std::max(E_ + A_, 1), kBlock);
  k_gba_cost<<<gr, kBlock, 0, s>>>(args(o, o), 0, part_a_.get(), sc_.get());
  k_gba_terms_cost<<<gt, kBlock, 0, s>>>(E_, A_, edge_ab_.get(), prior_block_.get(), meas_inv_.get(), init_inv_.get(),
                                        ew_.get(), pw_.get(), q_[o].get(), t_[o].get(), Rt_[o].get(), part_c_.get());
  k_finalize<<<1, 256, 0, s>>>(part_a_.get(), (int)gr, part_b_.get(), P_ ? (int)gp : 0, part_c_.get(), (int)gt,
                               part_d_.get(), nf_ ? (int)gd : 0, sc_.get(), 1);
  SFM_CHECK_LAUNCH();
  prof_->launches += 10;
  read();
  pcg_total_ += use_dense_ ? 0 : h_sc_.pcg_iters;
  if (h_sc_.nonfinite) return false;
  if (h_sc_.depth_obs != ~0ull) raise_projection(o, o);
  *new_cost = h_sc_.cost;
  *step_norm = std::sqrt(h_sc_.dc2 + h_sc_.dp2);
  return true;
}

// solver.py:194-257, the same control flow as BASolver::iterate.
void GBASolver::iterate(int n, sfm_ba_report* rep) {
  int done = 0;
  while (!finished_ && done < n) {
    ++iters_;
    ++done;
    linearize();
    if (gmax_ < opt_.grad_tol) {
      term_ = SFM_TERM_GRADIENT_TOLERANCE;
      --iters_;
      finished_ = true;
      break;
    }
    bool accepted = false;
    double step_norm = 0.0;
    while (lam_ <= opt_.max_lambda) {
      double nc = 0.0, sn = 0.0;
      ++n_trials_;
      if (!trial(lam_, &nc, &sn)) {
        lam_ *= 10.0;
        continue;
      }
      if (std::isfinite(nc) && nc < cost_) {
        cur_ ^= 1;
        cost_ = nc;
        step_norm = sn;
        lam_ = std::max(lam_ * 0.5, 1e-18);
        accepted = true;
        break;
      }
      lam_ *= 10.0;
    }
    if (!accepted) {
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
  if (rep) {
    rep->initial_cost = initial_cost_;
    rep->final_cost = cost_;
    rep->iterations = iters_;
    rep->termination = term_;
    rep->n_trials = n_trials_;
    rep->pcg_iterations = pcg_total_;
    rep->final_lambda = lam_;
    rep->device_ms = 0.0;
    rep->kernel_launches = prof_->launches;
    rep->n_blocks_S = n_full_;
  }
}

void GBASolver::download(double* q, double* t, double* X) {
  if (q) q_[cur_].download(q, (size_t)nb_ * 4, stream_);
  if (t) t_[cur_].download(t, (size_t)nb_ * 3, stream_);
  if (X) X_[cur_].download(X, (size_t)P_ * 3, stream_);
  SFM_CUDA(cudaStreamSynchronize(stream_));
}
