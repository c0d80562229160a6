// ba.cuh -- device-resident Levenberg-Marquardt bundle adjustment.
//
// Replaces solver.solve (solver.py:194-257) as driven by bundle_adjust
// (mapping.py:390-527): same residual set, robust IRLS weighting, Marquardt
// damping D = max(diag H, 1e-12), lambda schedule and termination rules, but
// the normal equations are reduced onto the cameras (Schur complement) and
// solved on device (dense Cholesky when small, block-Jacobi PCG otherwise).
// See DESIGN.md for the data layout and the kernel/roofline inventory.
#pragma once
#include <memory>
#include "comm.cuh"
#include "common.cuh"
#include "pcg.cuh"

namespace sfm {

struct BlkArgs;

inline double __longlong_as_double_host(unsigned long long b) {
  double d;
  std::memcpy(&d, &b, sizeof(d));
  return d;
}

// Device scalars read back once per LM trial (one small D2H).
struct BAScalars {
  double cost;               // robust cost of the evaluated state (local part)
  double dp2;                // sum |delta_p|^2 (local points)
  double dc2;                // sum |delta_c|^2 (replicated cameras)
  double bnorm2;             // |b_S|^2 (PCG)
  unsigned long long gmax;   // bit pattern of max|g| (non-negative doubles)
  unsigned long long depth_obs;  // min global obs index whose projection raised
  int nonfinite;             // delta or Schur factor not finite / not PD
  int pcg_iters;
  int pcg_fail;
  int pcg_stop;              // PCG_STOP_* of the last solve
  int proj_code;             // PROJ_* code of depth_obs (filled on demand)
  double proj_depth;         // p_cam.z of depth_obs
};

// Device state of the matrix-free Schur PCG (csrc/ischur.cuh).
struct ImpState {
  double rz;       // r.z
  double bnorm;    // |b|
  int it;          // iterations done
  int done;        // 0 running, 1 converged, 2 failed, 3 out of iterations
};

class BASolver {
 public:
  BASolver(cudaStream_t s, Profiler* p, Comm* c) : stream_(s), prof_(p), comm_(c) {}
  ~BASolver();
  BASolver(const BASolver&) = delete;
  BASolver& operator=(const BASolver&) = delete;
  void setup(const sfm_ba_problem& prob, const sfm_ba_options& opt);
  // Runs up to n LM iterations continuing the current solve.
  void iterate(int n, sfm_ba_report* rep);
  // Stepwise sessions: keep a device copy of the entry state (after setup)
  // and restart the solve from it -- a fresh bundle_adjust over the same
  // device-resident problem and structure (bench.py's per-step solves).
  void save_entry();
  void restart();
  void download(double* q, double* t, double* X);
  // Parity/debug evaluation of the reprojection residuals.
  static void eval(cudaStream_t s, Profiler* p, const sfm_ba_problem& prob, int loss_kind,
                   double loss_param, double* cost, double* res, double* jc, double* jp);
  bool finished() const { return finished_; }

 private:
  // --- host-side control (solver.py:194-257) ---
  double eval_cost_current();
  void linearize();
  bool trial(double lam, double* new_cost, double* step_norm);
  void point_prep(double lam);
  void build_schur(double lam);
  bool solve_reduced(double lam);
  // Matrix-free Schur PCG (high-damping trials); false if it did not converge.
  bool solve_implicit(double lam);
  void raise_projection_error(bool trial_state);
  void read_scalars();
  BlkArgs blk_args(double lam) const;

  cudaStream_t stream_;
  cudaStream_t side_ = nullptr;          // setup: bulk H2D copies overlapped with the structure build
  cudaEvent_t side_ready_ = nullptr, side_done_ = nullptr;
  cudaStream_t plan_stream_ = nullptr;   // setup: the PCG plan's copies, on its own host thread
  cudaEvent_t plan_ev_ = nullptr;
  Profiler* prof_;
  Comm* comm_;
  sfm_ba_options opt_{};
  int rank_ = 0;

  // dims
  int F_ = 0, nfree_ = 0, nmodels_ = 0;
  int64_t P_ = 0, N_ = 0;
  int64_t obs_offset_ = 0;
  int64_t n_params_ = 0;
  int n_edges_ = 0, n_priors_ = 0;
  double edge_w_ = 0.0, prior_w_ = 0.0;
  bool has_residuals_ = false;

  // LM state
  bool finished_ = true;
  double initial_cost_ = 0.0, cost_ = 0.0, lam_ = 0.0;
  int iters_ = 0, term_ = SFM_TERM_MAX_ITERATIONS, n_trials_ = 0, pcg_total_ = 0;
  int pcg_stagnated_ = 0, pcg_max_hit_ = 0;
  int use_dense_ = 0;
  bool trace_ = std::getenv("SFM_TRACE") != nullptr;

  // frames / models
  DevBuf<sfm_camera_model> models_;
  DevBuf<int> frame_model_, free_idx_, free_frame_;
  DevBuf<double> q_[2], t_[2], Rt_[2];  // [F*4], [F*3], [F*12]; index cur_
  DevBuf<double> qt_[2];                // [F*8] q | t | 0 (the point passes' camera record)
  DevBuf<double> X_[2];                 // [P*3]
  DevBuf<double> q0_, t0_, X0_;         // entry state (save_entry / restart)
  int cur_ = 0;

  // observations (point-major)
  DevBuf<int> obs_frame_, obs_point_;
  DevBuf<double> obs_uv_;   // [N*2]
  DevBuf<int64_t> pt_ptr_;  // [P+1]
  DevBuf<double4> geo_;     // [N] linearisation records (x, y, 1/Z, w)

  // pair structure (sorted by S block, then point)
  int64_t n_pairs_ = 0;
  int n_pb_ = 0, n_ub_ = 0, n_full_ = 0;
  DevBuf<unsigned long long> pairs_;     // (obs_lo << 32) | obs_hi
  DevBuf<int64_t> pb_pair_ptr_;          // [n_pb+1] pair range per pair block
  DevBuf<int> work_;                     // [n_off] off-diagonal S blocks (row-major)
  DevBuf<int4> offrec_;                  // [2*n_off] packed work headers (k_off_records)
  DevBuf<longlong2> offk_;               // [n_off] pair range per off-diagonal block
  DevBuf<int> pair_pt_;                  // [n_pairs] point of each pair
  int n_off_ = 0;
  int64_t n_cm_ = 0;                     // observations in free cameras
  DevBuf<int64_t> cm_ptr_, cm_obs_;      // camera-major observation streams
  DevBuf<int> cm_pt_, cm_pos_;
  DevBuf<double> cm_uv_;
  DevBuf<double4> geo_cm_;
  DevBuf<unsigned long long> ub_key_;    // [n_ub] upper block keys lo*nfree+hi
  DevBuf<int> ub_pb_;                    // [n_ub] pair block or -1
  DevBuf<int> ub_edge_;                  // [n_ub] edge or -1
  DevBuf<int> ub_pos_up_, ub_pos_lo_;    // [n_ub] BSR slots (lo = -1 on diagonal)
  DevBuf<int> row_ptr_, col_idx_;        // BSR full pattern

  // pose terms
  DevBuf<int> edge_ab_, prior_frame_;
  DevBuf<double> edge_meas_inv_;         // [E*7] q(4) t(3) of meas^-1
  DevBuf<double> prior_init_inv_;        // [A*7]
  DevBuf<int> term_ptr_, term_list_;     // per free camera incident terms
  DevBuf<BAScalars> sc_pre_;             // flags of the point prep done inside k_point_lin
  bool prep_ready_ = false;              // pv holds V*^-1 at prep_lam_ for the next trial
  double prep_lam_ = 0.0;
  double prep_done_lam_ = -1.0;          // pv holds this trial's V*^-1 (point_prep ran)
  bool prep_folded_ = false;             // ... prepared inside k_point_lin (flags in sc_pre_)
  DevBuf<double> term_contrib_;          // [2E+A][42] per-term J^T J | J^T r (k_terms_lin)
  DevBuf<double> edge_H_;                // [E*36] J_a^T J_b (weighted)

  // linearization
  DevBuf<double> V_, gp_;                // [P*6], [P*3]
  DevBuf<double> U_, gc_, Dc_;           // [nf*36], [nf*6], [nf*6]
  // trial
  DevBuf<double> pv_;                    // [P*12] V*^-1 (6) | e (3) | pad
  DevBuf<double> S_, b_;                 // [n_full*36], [nf*6]
  DevBuf<double> dc_;                    // [nf*6]
  // matrix-free Schur PCG (ischur.cuh)
  bool imp_enabled_ = std::getenv("SFM_IMPLICIT") == nullptr || std::atoi(std::getenv("SFM_IMPLICIT")) != 0;
  int last_pcg_ = -1;                    // PCG iterations of the previous trial of this linearisation
  int imp_iters_ = 0;
  int imp_trials_ = 0;
  DevBuf<double> imp_s_, imp_r_, imp_z_, imp_p_, imp_q_, imp_b_, imp_M_;
  DevBuf<ImpState> imp_st_;
  TwoLevelPcg pcg_;
  // row-partitioned PCG over point-sharded ranks sharing a device
  // (sfm_ba_options.pcg_partition): S / b reduce-scattered by block rows
  bool partitioned_ = false;
  std::vector<int64_t> s_off_, b_off_;    // element offsets of each rank's rows in S / b
  std::unique_ptr<PcgCollective> coll_;

  // reductions
  DevBuf<double> part_a_, part_b_, part_c_, part_d_;
  DevBuf<int> diag_ub_, diag_pos_;      // per free camera: upper index, BSR slot
  std::vector<int> diag_ub_host_;
  DevBuf<BAScalars> sc_;
  BAScalars h_sc_{};
  BAScalars* h_pin_ = nullptr;          // pinned staging of the per-trial scalar read-back
};

struct GbaArgs;

// Bundle adjustment with rig-extrinsic / rolling-shutter residuals (two SE(3)
// slots per residual): csrc/gba_impl.cuh.
class GBASolver {
 public:
  GBASolver(cudaStream_t s, Profiler* p) : stream_(s), prof_(p) {}
  void setup(const sfm_gba_problem& prob, const sfm_ba_options& opt);
  void iterate(int n, sfm_ba_report* rep);
  void download(double* q, double* t, double* X);

 private:
  GbaArgs args(int blocks, int points) const;
  double eval_cost(int blocks, int points);
  void linearize();
  bool trial(double lam, double* new_cost, double* step_norm);
  void read();
  void raise_projection(int blocks, int points);

  cudaStream_t stream_;
  Profiler* prof_;
  sfm_ba_options opt_{};
  int nb_ = 0, nf_ = 0, E_ = 0, A_ = 0, n_ub_ = 0, n_full_ = 0;
  int64_t P_ = 0, R_ = 0, n_params_ = 0;
  bool use_dense_ = true, finished_ = true;
  double initial_cost_ = 0.0, cost_ = 0.0, lam_ = 0.0, gmax_ = 0.0;
  int iters_ = 0, n_trials_ = 0, pcg_total_ = 0, term_ = 0, cur_ = 0;
  BAScalars h_sc_{};
  DevBuf<sfm_camera_model> models_;
  DevBuf<double> q_[2], t_[2], Rt_[2], X_[2];
  DevBuf<int> rpt_, rmodel_, rkind_, rslot_, free_idx_, free_block_, sptr_, ub_edge_, pos_up_, pos_lo_,
      row_ptr_, col_, diag_pos_, edge_ab_, prior_block_, term_ptr_, term_list_;
  DevBuf<double> ralpha_, ruv_, ew_, pw_, meas_inv_, init_inv_, rec_, V_, gp_, pv_, gc_, hdiag_, Ut_, gt_,
      edge_H_, S_, b_, dc_, part_a_, part_b_, part_c_, part_d_;
  DevBuf<int64_t> pptr_, slist_, ent_ptr_;
  DevBuf<int2> ub_key_;
  DevBuf<int4> ent_;
  DevBuf<BAScalars> sc_;
  TwoLevelPcg pcg_;
};

}  // namespace sfm
