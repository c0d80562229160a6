/*
 * sfm_b200.h -- C-ABI of the B200-native LM bundle-adjustment / triangulation
 * core (libsfm_b200.so).  Plain pointers and sizes only; every array is
 * host memory owned by the caller (C-contiguous, fp64 / int32 / int64 / u8),
 * copied to context-owned device memory inside the call.  No pointer is
 * retained after a call returns.
 *
 * Each entry point replaces one function of the reference Python package
 * (`sfmkit`, /root/reference/pkg/src/sfmkit); the citation above each
 * declaration names the reference interface it stands in for.  The Python
 * drop-in layer (paper_2510_15271_b200/mapping.py) flattens the reference's
 * object model into the arrays below and maps the return codes back onto the
 * reference's exception classes (errors.py).
 *
 * Return codes: 0 = OK, negative = error (see SFM_E_*); a human-readable
 * message with the payload the reference puts in its exception text is
 * available from sfm_last_error(ctx).
 */
#ifndef SFM_B200_H
#define SFM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SFM_ABI_VERSION 7

/* ---- error codes (mapped to sfmkit.errors classes by the Python layer) --- */
#define SFM_OK 0
#define SFM_E_INVALID (-1)            /* ValueError: malformed arguments      */
#define SFM_E_NON_POSITIVE_DEPTH (-2) /* NonPositiveDepth   cameras.py:132-133 */
#define SFM_E_OUT_OF_MODEL_DOMAIN (-3)/* OutOfModelDomain   cameras.py:68-69   */
#define SFM_E_SOLVER_DIVERGED (-4)    /* SolverDiverged     solver.py:247-248  */
#define SFM_E_UNDISTORT_DIVERGED (-5) /* UndistortDiverged  cameras.py:119-125 */
#define SFM_E_NO_GAUGE (-6)           /* NoGauge            mapping.py:408-409 (iterative_map's BA) */
#define SFM_E_CUDA (-10)              /* CUDA runtime failure                  */
#define SFM_E_NCCL (-11)              /* NCCL failure                          */
#define SFM_E_OOM (-12)               /* device allocation failure             */

/* ---- per-track triangulation status codes (sfm_tri_output.status) ------- */
#define SFM_TRI_OK 0
#define SFM_TRI_INSUFFICIENT_PARALLAX 1 /* InsufficientParallax mapping.py:205-207, :217-218 */
#define SFM_TRI_CHEIRALITY 2            /* CheiralityViolation  mapping.py:186-191 */
#define SFM_TRI_PARALLEL_RAYS 3         /* ParallelRays         mapping.py:236-237 */
#define SFM_TRI_TOO_FEW_OBS 4           /* ValueError           mapping.py:202-203 */
#define SFM_TRI_CAMERA_ERROR 5          /* unproject raised UndistortDiverged cameras.py:119-125 */
#define SFM_TRI_FAILED 6                /* ransac: track.status = FAILED mapping.py:286-303 */
#define SFM_TRI_SKIPPED 7               /* track not active (not PENDING)       */
#define SFM_TRI_CAMERA_DOMAIN 8         /* unproject raised OutOfModelDomain cameras.py:106-108 */

/* ---- camera models: cameras.py:35-54 -------------------------------------- */
#define SFM_CAM_PINHOLE 0
#define SFM_CAM_PINHOLE_RADIAL 1
#define SFM_CAM_EQUIDISTANT_FISHEYE 2

typedef struct {
  int32_t kind;     /* SFM_CAM_*                                   */
  int32_t width;
  int32_t height;
  int32_t _pad;
  double fx, fy, cx, cy;
  double k1, k2;    /* radial distortion (PINHOLE_RADIAL only)     */
} sfm_camera_model;

/* ---- robust losses: solver.py:25-51 -------------------------------------- */
#define SFM_LOSS_TRIVIAL 0
#define SFM_LOSS_HUBER 1
#define SFM_LOSS_CAUCHY 2

/* ---- linear solver for the reduced camera system ------------------------ */
#define SFM_LINSOLVE_AUTO 0   /* dense Cholesky when small, PCG otherwise */
#define SFM_LINSOLVE_DENSE 1  /* on-device dense Cholesky of S            */
#define SFM_LINSOLVE_PCG 2    /* block-Jacobi PCG on S                    */

/* ---- termination codes: solver.py:194-257 (SolverReport.termination) ---- */
#define SFM_TERM_MAX_ITERATIONS 0
#define SFM_TERM_GRADIENT_TOLERANCE 1
#define SFM_TERM_NO_DECREASE 2
#define SFM_TERM_PARAMETER_TOLERANCE 3
#define SFM_TERM_COST_ZERO 4
#define SFM_TERM_ALL_FIXED 5

typedef struct sfm_ctx sfm_ctx;

/*
 * Flattened bundle-adjustment problem: the array layout mapping.py:390-509
 * builds as closures.  Frames are `sorted(keyframes)`; points are the
 * TRIANGULATED landmarks in map order; observations are every inlier
 * observation, landmark-major in track order (the reference residual order,
 * mapping.py:452-475), so `obs_point` is non-decreasing.
 * Pose terms: lambda_c sequential edges (frame index pairs, measurement taken
 * from the entry poses on device, mapping.py:477-498) and lambda_a absolute
 * priors (frame indices, anchored at the entry poses, mapping.py:500-509).
 * Under point-sharding each rank passes only its points/observations and
 * rank 0 alone passes the pose terms.
 */
typedef struct {
  int32_t n_frames;
  int32_t n_models;
  const double* cam_q;          /* [n_frames,4] unit quaternion (w,x,y,z)  */
  const double* cam_t;          /* [n_frames,3] cam_from_world translation */
  const int32_t* frame_model;   /* [n_frames] index into models            */
  const uint8_t* frame_fixed;   /* [n_frames] 1 = fixed block              */
  const sfm_camera_model* models;
  int64_t n_points;
  const double* points;         /* [n_points,3]                            */
  int64_t n_obs;
  const int32_t* obs_frame;     /* [n_obs]                                 */
  const int32_t* obs_point;     /* [n_obs] non-decreasing                  */
  const double* obs_uv;         /* [n_obs,2] measured pixel                */
  int32_t n_edges;
  int32_t n_priors;
  const int32_t* edge_ab;       /* [n_edges,2] frame indices (a, b)        */
  const int32_t* prior_frame;   /* [n_priors]                              */
  double edge_weight;           /* lambda_c  (information = lambda_c * I)  */
  double prior_weight;          /* lambda_a                                */
  int64_t obs_offset;           /* global index of obs 0 (sharding)        */
  int64_t n_params_global;      /* 6*free frames + 3*all points (0 = local) */
} sfm_ba_problem;

/* SolverOptions (solver.py:81-87) + the robust loss + B200 solver knobs. */
typedef struct {
  int32_t loss_kind;
  int32_t max_iters;
  double loss_param;
  double grad_tol;
  double param_tol;
  double initial_lambda;
  double max_lambda;
  int32_t linear_solver;      /* SFM_LINSOLVE_*                           */
  int32_t pcg_max_iters;
  double pcg_rtol;            /* relative residual tolerance of PCG       */
  int32_t dense_max_dim;      /* AUTO: dense Cholesky when 6*free <= this */
  int32_t coarse_cluster;     /* PCG coarse level: frames per cluster (0 =
                                 default 8, < 0 = block-Jacobi only)       */
  int32_t coarse_refresh;     /* rebuild the coarse operator every this many
                                 linearisations (0 = default 8)            */
  double coarse_max_lambda;   /* coarse level only while lambda <= this
                                 (0 = default 1e-2; above it block-Jacobi)  */
  double coarse_drift;        /* re-assemble A_c when lambda moved by more
                                 than this factor since (0 = default 4)    */
  int32_t pcg_partition;      /* point-sharded ranks: 0 = replicated PCG on
                                 the all-reduced S; 1 = row-partitioned PCG
                                 (S / b reduce-scattered by block rows, z and
                                 the dot products pushed between ranks inside
                                 the Krylov kernel): ranks sharing a device
                                 run one launch over all their CTAs, the
                                 devices of a multi-device context (peer
                                 access) one launch each meeting at a
                                 cross-launch barrier; 2 = per-rank launches
                                 also for ranks sharing a device (the test of
                                 that barrier).  Ranks in separate processes
                                 always use 0.                              */
  int32_t _pad0;
} sfm_ba_options;

/* SolverReport (solver.py:90-95) + device-side statistics. */
typedef struct {
  double initial_cost;
  double final_cost;
  int32_t iterations;
  int32_t termination;        /* SFM_TERM_*                                */
  int32_t n_trials;           /* linear solves (accepted + rejected)       */
  int32_t pcg_iterations;     /* summed over trials                        */
  double final_lambda;
  double device_ms;           /* CUDA-event time of the LM loop            */
  int64_t kernel_launches;    /* kernels launched during the call          */
  int64_t n_blocks_S;         /* stored 6x6 blocks of S (both triangles)   */
  int32_t pcg_stagnated;      /* PCG solves stopped at the rounding floor
                                 (within 100x of the tolerance, no progress) */
  int32_t pcg_max_hit;        /* PCG solves that ran into pcg_max_iters    */
} sfm_ba_report;

/* ---- context ------------------------------------------------------------ */
int sfm_abi_version(void);
/* 128-byte NCCL unique id for rank 0 to broadcast (torch.distributed). */
int sfm_nccl_unique_id(uint8_t out[128]);
/* world == 1: nccl_id may be NULL.  device = CUDA ordinal used by this rank. */
int sfm_ctx_create(int32_t device, int32_t rank, int32_t world,
                   const uint8_t* nccl_id, sfm_ctx** out);
/* Single-process multi-GPU context (one context owning
 * n_gpus devices).  sfm_ba_solve on it shards the points by observation
 * count (8(e)), one host thread per device drives its shard, and the
 * camera-indexed sums / scalars are all-reduced over NCCL communicators
 * created in-process with ncclCommInitAll (NVLink / NVSwitch).
 * sfm_iterative_map keeps its track state on devices[0] and runs every
 * bundle adjustment sharded over the devices.  A repeated device id makes
 * the ranks on it run as shard emulation (no NCCL): the test path on one
 * GPU.  Replaces nothing in the reference (sfmkit is single-process,
 * single-threaded); it is how bundle_adjust / iterative_map
 * (mapping.py:390, :569) scale without a process launcher. */
int sfm_ctx_create_multi(int32_t n_devices, const int32_t* devices, sfm_ctx** out);
/* devices of the context (1 unless multi) and whether NCCL carries the sums */
int sfm_ctx_devices(const sfm_ctx* ctx, int32_t* out_n, int32_t* out_nccl);
/* cudaGetDeviceCount (0 without a GPU / driver) */
int sfm_device_count(int32_t* out);
void sfm_ctx_destroy(sfm_ctx* ctx);
const char* sfm_last_error(const sfm_ctx* ctx);
/* Per-kernel CUDA-event timing (bench / roofline).  Off by default. */
/* The CUDA stream (cudaStream_t) every call on ctx launches on, so a caller
 * can bracket calls with its own CUDA events (bench.py's device timing). */
int sfm_ctx_stream(const sfm_ctx* ctx, void** out);
int sfm_set_profiling(sfm_ctx* ctx, int32_t enabled);
int sfm_prof_count(const sfm_ctx* ctx);
int sfm_prof_get(const sfm_ctx* ctx, int32_t i, const char** name,
                 int64_t* launches, double* total_ms, double* bytes);
int sfm_prof_reset(sfm_ctx* ctx);

/* ---- bundle adjustment -------------------------------------------------- */
/*
 * Replaces solver.solve (solver.py:194-257) as driven by
 * mapping.bundle_adjust (mapping.py:390-527).  Reads the initial state from
 * `prob`, runs LM on device, writes the final poses/points into
 * out_cam_q/out_cam_t/out_points (same shapes as the inputs; fixed frames are
 * copied bit-identically) and fills `report`.  On SFM_E_NON_POSITIVE_DEPTH the
 * outputs are left untouched (the reference raises before writing back).
 * Ends any stepwise (sfm_ba_setup/iterate) session on the context.
 */
int sfm_ba_solve(sfm_ctx* ctx, const sfm_ba_problem* prob,
                 const sfm_ba_options* opt, double* out_cam_q,
                 double* out_cam_t, double* out_points, sfm_ba_report* report);

/* Stepwise form of sfm_ba_solve for device-resident benchmarking:
 * setup uploads + builds structure and evaluates the initial cost;
 * iterate runs up to n LM iterations continuing the same solve;
 * restart begins a new solve from the entry state (poses, points, lambda_0,
 * counters, initial cost) on the same device-resident problem and structure;
 * download copies the current state out. */
int sfm_ba_setup(sfm_ctx* ctx, const sfm_ba_problem* prob,
                 const sfm_ba_options* opt);
int sfm_ba_iterate(sfm_ctx* ctx, int32_t n_iters, sfm_ba_report* report);
int sfm_ba_restart(sfm_ctx* ctx);
int sfm_ba_download(sfm_ctx* ctx, double* out_cam_q, double* out_cam_t,
                    double* out_points);

/*
 * Test path for the point-sharded multi-GPU solve on ONE
 * device: n_shards logical ranks (host threads, one stream each) run the
 * exact per-rank control flow of the NCCL path on their shard
 * (shards[r] = what rank r would pass to sfm_ba_solve: its contiguous
 * points and their observations, obs_offset, n_params_global; pose terms on
 * shard 0 only), with every collective executed as a fixed-rank-order
 * device reduction.  Writes the (replicated) poses and each shard's points
 * into out_points[r].
 */
int sfm_ba_solve_emulated(sfm_ctx* ctx, int32_t n_shards, const sfm_ba_problem* shards,
                          const sfm_ba_options* opt, double* out_cam_q, double* out_cam_t,
                          double* const* out_points, sfm_ba_report* report);

/*
 * Parity/debug: Problem.evaluate (solver.py:132-142) + _assemble
 * (solver.py:164-191) restricted to the reprojection residuals: robust cost
 * per observation, weighted residual r~ [n_obs,2], weighted pose Jacobian
 * J~_c [n_obs,2,6] and point Jacobian J~_p [n_obs,2,3] (any output may be
 * NULL).  Fixed frames still get their J~_c here.
 */
int sfm_ba_eval(sfm_ctx* ctx, const sfm_ba_problem* prob, int32_t loss_kind,
                double loss_param, double* out_cost_per_obs, double* out_res,
                double* out_jc, double* out_jp);

/* ---- rig-extrinsic / rolling-shutter bundle adjustment ------------------- */
/* Residual kinds (mapping.py:310-356): the pose a residual projects through
 * is composed from one or two SE(3) parameter blocks ("slots"). */
#define SFM_RES_GLOBAL 0   /* pose = B[s0]                                 */
#define SFM_RES_ROLLING 1  /* pose = B[s0] exp(alpha log(B[s0]^-1 B[s1]))  */
#define SFM_RES_RIG 2      /* pose = B[s1] B[s0]  (extrinsic s1, vehicle s0) */

/*
 * The problem bundle_adjust builds when keyframes are rolling-shutter or in
 * rig_extrinsic mode (mapping.py:414-509): pose blocks (frames; or vehicle
 * instants + per-camera extrinsics), TRIANGULATED points, residuals in the
 * reference residual order (landmark-major, so res_point is non-decreasing)
 * with their kind, slots and scanline fraction, and the pose terms with
 * per-term weights (lambda_c edges; lambda_a or extrinsic priors).
 */
typedef struct {
  int32_t n_blocks;
  int32_t n_models;
  const double* block_q;        /* [n_blocks,4]                             */
  const double* block_t;        /* [n_blocks,3]                             */
  const uint8_t* block_fixed;   /* [n_blocks]                               */
  const sfm_camera_model* models;
  int64_t n_points;
  const double* points;         /* [n_points,3]                             */
  int64_t n_res;
  const int32_t* res_point;     /* [n_res] non-decreasing                   */
  const int32_t* res_model;     /* [n_res]                                  */
  const int32_t* res_kind;      /* [n_res] SFM_RES_*                        */
  const int32_t* res_slot;      /* [n_res,2] (second = -1 for GLOBAL)       */
  const double* res_alpha;      /* [n_res] ROLLING scanline fraction or NULL */
  const double* res_uv;         /* [n_res,2]                                */
  int32_t n_edges;
  int32_t n_priors;
  const int32_t* edge_ab;       /* [n_edges,2] blocks (a, b)                */
  const double* edge_weight;    /* [n_edges] information weight            */
  const int32_t* prior_block;   /* [n_priors]                               */
  const double* prior_weight;   /* [n_priors]                               */
} sfm_gba_problem;

/*
 * solver.solve (solver.py:194-257) on that problem: same LM rules and
 * report as sfm_ba_solve; final block poses and points written out.
 */
int sfm_gba_solve(sfm_ctx* ctx, const sfm_gba_problem* prob, const sfm_ba_options* opt,
                  double* out_block_q, double* out_block_t, double* out_points,
                  sfm_ba_report* report);

/* ---- triangulation / gating --------------------------------------------- */
/*
 * Tracks as CSR: observations of track i are [track_ptr[i], track_ptr[i+1]),
 * in track order; obs_frame indexes the frame arrays (cam_q/cam_t/
 * frame_model).  `active` (may be NULL = all) selects the tracks to process
 * (PENDING tracks in iterative_map, mapping.py:600-602).
 */
typedef struct {
  int32_t n_frames;
  int32_t n_models;
  const double* cam_q;
  const double* cam_t;
  const int32_t* frame_model;
  const sfm_camera_model* models;
  int64_t n_tracks;
  int64_t n_obs;
  const int64_t* track_ptr;     /* [n_tracks+1]                             */
  const int32_t* obs_frame;     /* [n_obs]                                  */
  const double* obs_uv;         /* [n_obs,2]                                */
  const uint8_t* active;        /* [n_tracks] or NULL                       */
} sfm_tracks;

#define SFM_TRI_DLT 0
#define SFM_TRI_MIDPOINT 1

/*
 * Replaces ransac_triangulate (mapping.py:255-305) for every active track:
 * exhaustive i<j pair hypotheses, strict `<` inlier test, lexicographic
 * (count, -sum err) score with first-best, refine on inliers, final mask.
 * Outputs: out_X [n_tracks,3], out_mask [n_obs] (u8), out_status [n_tracks]
 * (SFM_TRI_OK or SFM_TRI_FAILED; SFM_TRI_SKIPPED for inactive tracks).
 */
int sfm_ransac_triangulate(sfm_ctx* ctx, const sfm_tracks* tracks,
                           double threshold_px, double min_angle,
                           int32_t method, double* out_X, uint8_t* out_mask,
                           int8_t* out_status);

/*
 * Replaces triangulate_dlt (mapping.py:194-221) / triangulate_midpoint
 * (mapping.py:224-240) over all observations of each track (batched):
 * out_status carries the exception the reference would raise per track.
 */
int sfm_triangulate(sfm_ctx* ctx, const sfm_tracks* tracks, double min_angle,
                    int32_t method, double* out_X, int8_t* out_status);

/*
 * Replaces remove_outliers (mapping.py:544-566) for the landmarks given as
 * tracks (one track per TRIANGULATED landmark, all of its observations):
 * an inlier observation with reprojection error > threshold (strict) is
 * cleared in mask_inout; out_inliers[i] = surviving inlier count of landmark
 * i (< 2 means demote to PENDING); *out_removed = cleared count.
 */
int sfm_gate(sfm_ctx* ctx, const sfm_tracks* tracks, const double* points,
             double threshold_px, uint8_t* mask_inout, int32_t* out_inliers,
             int64_t* out_removed);

/*
 * reprojection_error (mapping.py:243-252) for every observation of every
 * track against points [n_tracks,3] (inf where projection raises).
 */
int sfm_reprojection_errors(sfm_ctx* ctx, const sfm_tracks* tracks,
                            const double* points, double* out_err);

/* ---- track formation (host-native, no context) ------------------------- */
/*
 * Replaces build_tracks (mapping.py:113-161): connected components of the
 * feature-match graph with the reference's conflict rule (a merge that would
 * put two features of one frame into a track is skipped).  Pairs
 * pair_frames [n_pairs,2] = (frame_a, frame_b) with their matches
 * match_index [pair_ptr[p] .. pair_ptr[p+1]) as (index_a, index_b); any
 * order (merges run in the reference's sorted order).  Outputs sized by the
 * caller for the worst case (2 * matches observations, matches + 1 track
 * pointers): tracks as CSR (out_track_ptr, out_obs_frame, out_obs_feature),
 * in the reference's track and observation order.  Needs no GPU.
 */
/* Host-only helpers of the multi-GPU partition (no context, no GPU):
 * the point shards -- contiguous point ranges balanced by observation
 * count, out_bounds[world+1] -- and the rank row ranges
 * of the row-partitioned PCG over a BSR pattern, out_row0[world+1]. */
int sfm_shard_points(int64_t n_obs, const int32_t* obs_point, int64_t n_points, int32_t world,
                     int64_t* out_bounds);
int sfm_pcg_rank_rows(int32_t n_rows, const int32_t* row_ptr, int32_t world, int32_t* out_row0);

int sfm_build_tracks(int64_t n_pairs, const int32_t* pair_frames, const int64_t* pair_ptr,
                     const int32_t* match_index, int64_t* out_track_ptr, int32_t* out_obs_frame,
                     int32_t* out_obs_feature, int64_t* out_n_tracks, int64_t* out_n_obs);

/* ---- device-resident iterative mapping ---------------------------------- */
/* Track status (Track.status, mapping.py:48-52): in/out of sfm_iterative_map */
#define SFM_TRACK_PENDING 0
#define SFM_TRACK_TRIANGULATED 1
#define SFM_TRACK_FAILED 2

/*
 * The inputs of iterative_map (mapping.py:569-571) flattened: frames (sorted
 * keyframe ids) with the fixed set already resolved (anchor frame,
 * mapping.py:583-593), the pose terms every bundle_adjust call of the loop
 * builds (lambda_c consecutive-frame edges, lambda_a priors; mapping.py:477-
 * 509), and the tracks as CSR in track order.
 */
typedef struct {
  int32_t n_frames;
  int32_t n_models;
  const double* cam_q;          /* [n_frames,4] initial poses              */
  const double* cam_t;          /* [n_frames,3]                            */
  const int32_t* frame_model;   /* [n_frames]                              */
  const uint8_t* frame_fixed;   /* [n_frames]                              */
  const sfm_camera_model* models;
  int64_t n_tracks;
  int64_t n_obs;
  const int64_t* track_ptr;     /* [n_tracks+1]                            */
  const int32_t* obs_frame;     /* [n_obs]                                 */
  const double* obs_uv;         /* [n_obs,2]                               */
  const int8_t* track_status;   /* [n_tracks] SFM_TRACK_* (NULL = pending) */
  int32_t n_edges;
  int32_t n_priors;
  const int32_t* edge_ab;       /* [n_edges,2]                             */
  const int32_t* prior_frame;   /* [n_priors]                              */
  double edge_weight;           /* lambda_c                                */
  double prior_weight;          /* lambda_a                                */
} sfm_map_problem;

/* MappingConfig (mapping.py:84-108) + the B200 solver knobs of each BA. */
typedef struct {
  int32_t max_outer_iters;
  int32_t max_solver_iters;
  int32_t stage1_loss_kind;
  int32_t stage2_loss_kind;
  double stage1_loss_param;
  double stage2_loss_param;
  double stage1_outlier_px;
  double stage2_outlier_px;
  double min_angle;             /* min_triangulation_angle (radians)       */
  int32_t method;               /* SFM_TRI_DLT / SFM_TRI_MIDPOINT          */
  int32_t _pad;
  sfm_ba_options solver;        /* loss / max_iters fields ignored         */
} sfm_map_options;

typedef struct {
  int32_t round;                /* -1 = the final stage-2 pass             */
  int32_t _pad;
  int64_t added;
  int64_t removed;
  int64_t landmarks;
} sfm_round_stat;

/*
 * Replaces iterative_map (mapping.py:569-624) with the whole loop on the
 * device: rounds of {RANSAC-triangulate PENDING tracks -> stage-1 BA over
 * the landmarks -> stage-1 outlier gate (demoted tracks back to PENDING)}
 * until a round neither adds nor removes (cap max_outer_iters), then stage-2
 * BA + gate.  Tracks, masks, landmark positions and the landmark order stay
 * on the device between rounds.  Outputs: final poses, per-track position
 * ([n_tracks,3], NaN if not a landmark), per-observation inlier mask, per-
 * track status, the landmarks as track ids in map order (out_lm_track
 * [n_tracks], *out_n_landmarks of them) and the round statistics
 * (out_stats [max_outer_iters+1], *out_n_stats).
 */
int sfm_iterative_map(sfm_ctx* ctx, const sfm_map_problem* prob, const sfm_map_options* opt,
                      double* out_cam_q, double* out_cam_t, double* out_X, uint8_t* out_mask,
                      int8_t* out_status, int64_t* out_lm_track, int64_t* out_n_landmarks,
                      sfm_round_stat* out_stats, int32_t* out_n_stats);

#ifdef __cplusplus
}
#endif
#endif /* SFM_B200_H */
