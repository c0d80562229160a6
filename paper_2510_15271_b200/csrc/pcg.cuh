// pcg.cuh -- two-level preconditioned CG on the reduced camera system S.
//
// Replaces the exact sparse solve of the damped normal equations
// (solver.py:220-222, SuperLU on the un-reduced system) for large problems.
// Preconditioner: additive two-level
//     M^-1 r = D^-1 r + P A_c^-1 P^T r
// with D the 6x6 block diagonal of S (block-Jacobi) and P the similarity
// coarse space: cameras are aggregated into clusters of ~C consecutive free
// frames (whole PCG CTA row ranges) and camera j's coarse basis is
// [Adj(T_j) K_c | (0, t_j + R_j c)] -- a world-frame rigid motion of the
// whole cluster about its camera centroid c and its scaling about c,
// expressed as left perturbations (kCoarseDim = 7 columns).  A_c = P^T S P
// is assembled on device and inverted by a cooperative blocked Gauss-Jordan.
// The Krylov loop is one persistent cooperative kernel with two grid
// barriers per iteration; every reduction has a fixed order.
#pragma once
#include <functional>
#include <vector>

#include "common.cuh"

namespace sfm {

struct BAScalars;

// ---- row-partitioned PCG over R ranks (north-star variant)
// Rank r owns the block rows [row0[r], row0[r+1]) of S (reduce-scattered by
// the caller) and the CTAs of those rows.  Inside the persistent kernel a CTA
// reads S, b, x, M^-1 and A_c^-1 from its own rank's buffers and PUSHES what
// the other ranks need -- its rows of z and its partial sums -- into every
// rank's replica before each grid barrier (the allgather of z and the
// allreduce of the dot products, fused into the Krylov loop), so every read
// after a barrier is rank-local.
constexpr int kPcgMaxRanks = 16;

// Coarse dimensions per cluster: the 6 rigid motions of the cluster plus its
// scale (world scaling t_j -> (1+s) t_j, the similarity gauge's weak
// direction that rigid motions do not span).  tools/precond_study.py, PCG
// iterations to 1e-8 on S at the initial state: configs[2] 77 -> 26,
// configs[1] 146 -> 25.
constexpr int kCoarseDim = 7;

struct PcgRankView {       // one rank's buffers for one solve
  const double* S;         // [nnzb*36]  valid in the rank's rows
  const double* b;         // [nf*6]     valid in the rank's rows
  double* x;               // [nf*6]     written in the rank's rows (warm start read there)
  const double* Minv;      // [nf*36]    block-Jacobi inverses of the rank's rows
  const double* Pm;        // [nf*6*kCoarseDim] coarse basis (all rows), row-major 6 x kCoarseDim
  const double* Aci;       // [npad^2]   coarse inverse (replicated), null = one level
  double* z;               // [nf*6]     replica of z (every CTA pushes its rows here)
  double* part;            // [4G]       replica of the per-CTA scalar partials
  double* rpart;           // [6G]       replica of the per-CTA restriction partials
  BAScalars* sc;           // the rank's scalars (iterations, stop reason, failure)
  unsigned* xbar;          // rank 0: the cross-launch barrier counter | abort flag
};

// How a rank's TwoLevelPcg meets the others (implemented over Comm in ba.cu).
class PcgCollective {
 public:
  virtual ~PcgCollective() = default;
  virtual int rank() const = 0;
  virtual int world() const = 0;
  // sum over ranks, result on every rank (the coarse operator A_c)
  virtual void sum(double* d, size_t n, cudaStream_t s) = 0;
  // every rank hands in its view; `launch` runs once with all R views
  // (shard emulation: rank 0 launches one cooperative kernel covering every
  // rank's CTAs on the shared device)
  virtual void launch_all(const PcgRankView& mine, cudaStream_t s,
                          const std::function<void(const PcgRankView*)>& launch) = 0;
  // true: every rank launches its own cooperative kernel over its CTAs and
  // the launches meet at a cross-launch barrier (separate devices in one
  // process with peer access, or -- pcg_partition 2 -- ranks sharing a device)
  virtual bool separate_launches() const = 0;
  // every rank hands in its view and gets all of them; rank 0 runs
  // `root_prep` first (barrier reset); then every rank runs `launch` on its
  // own stream and waits for it
  virtual void launch_each(const PcgRankView& mine, cudaStream_t s, const std::function<void()>& root_prep,
                           const std::function<void(const PcgRankView*)>& launch) = 0;
};

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

// Rank row ranges of the row-partitioned PCG: block rows split into `world`
// contiguous ranges balanced by stored blocks + 4 per row (the same cost the
// CTA partition balances).  Host-only; row_ptr has nf+1 entries.
std::vector<int> pcg_rank_rows(const int* row_ptr, int nf, int world);

class TwoLevelPcg {
 public:
  // cluster <= 0 disables the coarse level (plain block-Jacobi).
  void setup(int nf, int cluster, int refresh, cudaStream_t s);
  // Row-partitioned solve over `world` ranks (call before set_pattern):
  // the CTA partition and the coarse clusters are cut at the rank row
  // boundaries, which rank_rows() / rank_blocks() then report.
  void set_partition(int world, int rank) { world_ = std::max(1, world); rank_ = rank; }
  int world() const { return world_; }
  const std::vector<int>& rank_rows() const { return rank_row0_; }    // [world+1]
  const std::vector<int>& rank_blocks() const { return rank_blk0_; }  // [world+1]
  // Coarse assembly runs from the (fixed) BSR pattern of S.
  void set_pattern(const int* row_ptr, const int* col, int nnzb, cudaStream_t s);
  // Coarse basis P_j (rigid motions + scale about the cluster centroid) from
  // the linearisation-point poses.
  void set_basis(const int* free_frame, const double* q, const double* t, const double* Rt,
                 cudaStream_t s, Profiler* prof);
  // Coarse level only while lam <= lam_max; rebuilt when lam has drifted by
  // more than `drift` (either way) from the lam it was assembled at.
  void set_coarse_policy(double lam_max, double drift) { lam_max_ = lam_max; drift_ = drift; }
  // Solves S x = b; writes iteration count / stop reason / failure into sc.
  void solve(const PcgProblem& p, int max_it, double rtol, BAScalars* sc, cudaStream_t s,
             Profiler* prof, PcgCollective* coll = nullptr);
  int last_grid() const { return grid_; }
  // Forget the coarse operator and the warm-start solution (a new solve).
  void restart() { lin_count_ = 0; coarse_valid_ = false; have_prev_ = false; }

 private:
  int nf_ = 0, cluster_ = 0, nc_ = 0, ncp_ = 0, npad_ = 0, grid_ = 0, gj_grid_ = 0;
  int maxrows_ = 0, maxsegs_ = 0, nt_ = 512, refresh_ = 1, lin_count_ = 0, resblocks_ = 0, maxdist_ = 1, maxblk_ = 1;
  size_t smem_ = 0;
  int npairs_ = 0;
  int world_ = 1, rank_ = 0;
  std::vector<int> rank_row0_, rank_blk0_, rank_cta0_, rank_pair0_;
  DevBuf<unsigned> xbar_;                 // cross-launch barrier (rank 0)
  bool coarse_valid_ = false;
  double lam_build_ = 0.0, lam_max_ = 1e-2, drift_ = 4.0;
  double lam_floor_ = 1e-5;   // dampings below this count as equal (coarse rebuild rule)
  bool have_prev_ = false, warm_ = true;  // warm start from the previous solution
  const double* Aci_ = nullptr;
  DevBuf<double> Minv_, Pm_, Ac_[2], gjpiv_, r_, z_, p_, q_, rpart_, part_;
  DevBuf<int2> pair_cd_, rowseg_, wres_;
  DevBuf<int> pair_ptr_, cta_row0_, cta_cluster_, cluster_cta0_, zl_ptr_, zl_, lcol_;
  DevBuf<int> cluster_row0_, frame_cluster_;  // frames of each coarse cluster, cluster of each frame
  DevBuf<double> cen_;                        // [nc*3] cluster centroids (coarse basis origin)
  DevBuf<int4> runs_, wchunk_;
};

}  // namespace sfm
