// pcg.cuh -- two-level preconditioned CG on the reduced camera system S.
//
// Replaces the exact sparse solve of the damped normal equations
// (solver.py:220-222, SuperLU on the un-reduced system) for large problems.
// Preconditioner: additive two-level
//     M^-1 r = D^-1 r + P A_c^-1 P^T r
// with D the 6x6 block diagonal of S (block-Jacobi) and P the rigid-motion
// coarse space: cameras are aggregated into clusters of ~C consecutive free
// frames (whole PCG CTA row ranges) and camera j's coarse basis is Adj(T_j) (a world-frame rigid motion
// of the whole cluster, expressed as left perturbations).  A_c = P^T S P is
// assembled on device and inverted by a cooperative blocked Gauss-Jordan.
// The Krylov loop is one persistent cooperative kernel with two grid
// barriers per iteration; every reduction has a fixed order.
#pragma once
#include "common.cuh"

namespace sfm {

struct BAScalars;

// Why a PCG solve stopped (BAScalars::pcg_stop).
enum { PCG_STOP_CONVERGED = 0, PCG_STOP_MAX_ITERS = 1, PCG_STOP_STAGNATED = 2, PCG_STOP_FAILED = 3 };

struct PcgProblem {
  int nf;
  const int* row_ptr;     // BSR (both triangles), [nf+1]
  const int* col;         // [nnzb]
  const double* S;        // [nnzb*36] row-major blocks
  int nnzb;
  const int* diag_pos;    // [nf] BSR slot of the diagonal block
  const double* b;        // [nf*6]
  double* x;              // [nf*6] solution
  double lam;             // Marquardt damping S was assembled at (coarse-level consistency)
};

class TwoLevelPcg {
 public:
  // cluster <= 0 disables the coarse level (plain block-Jacobi).
  void setup(int nf, int cluster, int refresh, cudaStream_t s);
  // Coarse assembly runs from the (fixed) BSR pattern of S.
  void set_pattern(const int* row_ptr, const int* col, int nnzb, cudaStream_t s);
  // Coarse basis P_j = Adj(T_j) from the linearisation-point poses.
  void set_basis(const int* free_frame, const double* q, const double* t, const double* Rt,
                 cudaStream_t s, Profiler* prof);
  // Coarse level only while lam <= lam_max; rebuilt when lam has drifted by
  // more than `drift` (either way) from the lam it was assembled at.
  void set_coarse_policy(double lam_max, double drift) { lam_max_ = lam_max; drift_ = drift; }
  // Solves S x = b; writes iteration count / stop reason / failure into sc.
  void solve(const PcgProblem& p, int max_it, double rtol, BAScalars* sc, cudaStream_t s,
             Profiler* prof);
  int last_grid() const { return grid_; }
  // Forget the coarse operator and the warm-start solution (a new solve).
  void restart() { lin_count_ = 0; coarse_valid_ = false; have_prev_ = false; }

 private:
  int nf_ = 0, cluster_ = 0, nc_ = 0, ncp_ = 0, npad_ = 0, grid_ = 0, gj_grid_ = 0;
  int maxrows_ = 0, maxsegs_ = 0, nt_ = 512, refresh_ = 1, lin_count_ = 0, resblocks_ = 0, maxdist_ = 1, maxblk_ = 1;
  size_t smem_ = 0;
  int npairs_ = 0;
  bool coarse_valid_ = false;
  double lam_build_ = 0.0, lam_max_ = 1e-2, drift_ = 4.0;
  double lam_floor_ = 1e-5;   // dampings below this count as equal (coarse rebuild rule)
  bool have_prev_ = false, warm_ = true;  // warm start from the previous solution
  const double* Aci_ = nullptr;
  DevBuf<double> Minv_, Pm_, Ac_[2], gjpiv_, r_, z_, p_, q_, rpart_, part_;
  DevBuf<int2> pair_cd_, rowseg_, wres_;
  DevBuf<int> pair_ptr_, cta_row0_, cta_cluster_, cluster_cta0_, zl_ptr_, zl_, lcol_;
  DevBuf<int4> runs_, wchunk_;
};

}  // namespace sfm
