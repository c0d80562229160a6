// capi.cu -- the extern "C" boundary (include/sfm_b200.h).
//
// Every entry point catches the driver's SfmError and returns its code; the
// message (with the payload the reference puts in its exception text) is kept
// on the context for sfm_last_error().
#include <memory>
#include <string>

#include "ba.cuh"
#include "comm.cuh"
#include "emu.cuh"
#include "tracks.cuh"
#include "imap.cuh"
#include "tri.cuh"

struct sfm_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  sfm::Profiler prof;
  sfm::Comm comm;
  sfm::DeviceGroup group;  // multi-device context (sfm_ctx_create_multi): devices + in-process NCCL comms
  std::string err;
  std::unique_ptr<sfm::BASolver> ba;
  bool multi() const { return group.size() > 1; }
};

namespace {

template <typename F>
int guarded(sfm_ctx* ctx, F&& body) {
  if (!ctx) return SFM_E_INVALID;
  try {
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e != cudaSuccess) throw sfm::SfmError(SFM_E_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    ctx->err.clear();
    sfm::alloc_stream() = ctx->stream;
    body();
    return SFM_OK;
  } catch (const sfm::SfmError& e) {
    ctx->err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    ctx->err = e.what();
    return SFM_E_CUDA;
  }
}

}  // namespace

extern "C" {

int sfm_abi_version(void) { return SFM_ABI_VERSION; }

int sfm_nccl_unique_id(uint8_t out[128]) {
  if (!out) return SFM_E_INVALID;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return SFM_E_NCCL;
  static_assert(sizeof(id) == 128, "NCCL unique id must be 128 bytes");
  std::memcpy(out, &id, sizeof(id));
  return SFM_OK;
}

int sfm_ctx_create(int32_t device, int32_t rank, int32_t world, const uint8_t* nccl_id, sfm_ctx** out) {
  if (!out || world < 1 || rank < 0 || rank >= world) return SFM_E_INVALID;
  *out = nullptr;
  auto* ctx = new sfm_ctx();
  ctx->device = device;
  int rc = guarded(ctx, [&] {
    SFM_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    sfm::alloc_stream() = ctx->stream;
    // keep freed device blocks cached in the default pool (stream-ordered
    // allocation, see DevBuf)
    cudaMemPool_t pool;
    SFM_CUDA(cudaDeviceGetDefaultMemPool(&pool, ctx->device));
    uint64_t thr = UINT64_MAX;
    SFM_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    ctx->comm.init(rank, world, nccl_id);
  });
  if (rc != SFM_OK) {
    std::fprintf(stderr, "sfm_ctx_create: %s\n", ctx->err.c_str());
    delete ctx;
    return rc;
  }
  *out = ctx;
  return SFM_OK;
}

int sfm_device_count(int32_t* out) {
  if (!out) return SFM_E_INVALID;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) n = 0;
  *out = n;
  return SFM_OK;
}

int sfm_ctx_create_multi(int32_t n_devices, const int32_t* devices, sfm_ctx** out) {
  if (!out || n_devices < 1 || n_devices > 16 || !devices) return SFM_E_INVALID;
  *out = nullptr;
  auto* ctx = new sfm_ctx();
  ctx->device = devices[0];
  int rc = guarded(ctx, [&] {
    SFM_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    sfm::alloc_stream() = ctx->stream;
    ctx->group.devices.assign(devices, devices + n_devices);
    bool distinct = true;
    for (int i = 0; i < n_devices; ++i) {
      cudaMemPool_t pool;
      SFM_CUDA(cudaDeviceGetDefaultMemPool(&pool, devices[i]));
      uint64_t thr = UINT64_MAX;
      SFM_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
      for (int j = 0; j < i; ++j) distinct &= devices[j] != devices[i];
    }
    // distinct devices: one NCCL communicator per device, created in this
    // process (NVLink / NVSwitch); a repeated device: shard emulation
    if (n_devices > 1 && distinct) {
      ctx->group.comms.resize(n_devices);
      SFM_NCCL(ncclCommInitAll(ctx->group.comms.data(), n_devices, ctx->group.devices.data()));
      // peer access between every pair: the row-partitioned PCG pushes z and
      // its partial sums straight into the other devices' replicas
      bool peer = true;
      for (int i = 0; i < n_devices && peer; ++i)
        for (int j = 0; j < n_devices && peer; ++j) {
          if (i == j) continue;
          int ok = 0;
          SFM_CUDA(cudaDeviceCanAccessPeer(&ok, devices[i], devices[j]));
          if (!ok) { peer = false; break; }
          SFM_CUDA(cudaSetDevice(devices[i]));
          const cudaError_t e = cudaDeviceEnablePeerAccess(devices[j], 0);
          if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
          else if (e != cudaSuccess) { cudaGetLastError(); peer = false; }
        }
      ctx->group.peer = peer;
    }
    SFM_CUDA(cudaSetDevice(ctx->device));
  });
  if (rc != SFM_OK) {
    std::fprintf(stderr, "sfm_ctx_create_multi: %s\n", ctx->err.c_str());
    for (auto c : ctx->group.comms)
      if (c) ncclCommDestroy(c);
    delete ctx;
    return rc;
  }
  *out = ctx;
  return SFM_OK;
}

int sfm_ctx_devices(const sfm_ctx* ctx, int32_t* out_n, int32_t* out_nccl) {
  if (!ctx || !out_n) return SFM_E_INVALID;
  *out_n = ctx->multi() ? ctx->group.size() : 1;
  if (out_nccl) *out_nccl = ctx->multi() ? (int32_t)!ctx->group.comms.empty() : (ctx->comm.world > 1);
  return SFM_OK;
}

void sfm_ctx_destroy(sfm_ctx* ctx) {
  if (!ctx) return;
  for (auto c : ctx->group.comms)
    if (c) ncclCommDestroy(c);
  cudaSetDevice(ctx->device);
  sfm::alloc_stream() = ctx->stream;
  ctx->ba.reset();
  if (ctx->stream) {
    cudaStreamSynchronize(ctx->stream);
    cudaStreamDestroy(ctx->stream);
  }
  sfm::alloc_stream() = nullptr;
  delete ctx;
}

const char* sfm_last_error(const sfm_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int sfm_ctx_stream(const sfm_ctx* ctx, void** out) {
  if (!ctx || !out) return SFM_E_INVALID;
  *out = (void*)ctx->stream;
  return SFM_OK;
}

int sfm_set_profiling(sfm_ctx* ctx, int32_t enabled) {
  return guarded(ctx, [&] { ctx->prof.enabled = enabled != 0; });
}

int sfm_prof_count(const sfm_ctx* ctx) { return ctx ? (int)ctx->prof.entries.size() : 0; }

int sfm_prof_get(const sfm_ctx* ctx, int32_t i, const char** name, int64_t* launches, double* total_ms,
                 double* bytes) {
  if (!ctx || i < 0 || i >= (int)ctx->prof.entries.size()) return SFM_E_INVALID;
  const auto& e = ctx->prof.entries[i];
  if (name) *name = e.name.c_str();
  if (launches) *launches = e.launches;
  if (total_ms) *total_ms = e.ms;
  if (bytes) *bytes = e.bytes;
  return SFM_OK;
}

int sfm_prof_reset(sfm_ctx* ctx) {
  return guarded(ctx, [&] { ctx->prof.reset(); });
}

int sfm_ba_setup(sfm_ctx* ctx, const sfm_ba_problem* prob, const sfm_ba_options* opt) {
  return guarded(ctx, [&] {
    SFM_REQUIRE(prob && opt, "null problem/options");
    ctx->ba.reset();  // back to the pool before the new solver allocates
    ctx->ba.reset(new sfm::BASolver(ctx->stream, &ctx->prof, &ctx->comm));
    try {
      ctx->ba->setup(*prob, *opt);
      ctx->ba->save_entry();
    } catch (...) {
      ctx->ba.reset();
      throw;
    }
  });
}

int sfm_ba_iterate(sfm_ctx* ctx, int32_t n_iters, sfm_ba_report* report) {
  return guarded(ctx, [&] {
    SFM_REQUIRE(ctx->ba != nullptr, "sfm_ba_iterate before sfm_ba_setup");
    ctx->ba->iterate(n_iters, report);
  });
}

int sfm_ba_restart(sfm_ctx* ctx) {
  return guarded(ctx, [&] {
    SFM_REQUIRE(ctx->ba != nullptr, "sfm_ba_restart before sfm_ba_setup");
    ctx->ba->restart();
  });
}

int sfm_ba_download(sfm_ctx* ctx, double* out_cam_q, double* out_cam_t, double* out_points) {
  return guarded(ctx, [&] {
    SFM_REQUIRE(ctx->ba != nullptr, "sfm_ba_download before sfm_ba_setup");
    ctx->ba->download(out_cam_q, out_cam_t, out_points);
  });
}

int sfm_ba_solve(sfm_ctx* ctx, const sfm_ba_problem* prob, const sfm_ba_options* opt, double* out_cam_q,
                 double* out_cam_t, double* out_points, sfm_ba_report* report) {
  return guarded(ctx, [&] {
    SFM_REQUIRE(prob && opt, "null problem/options");
    // a full solve ends any stepwise session: its device memory goes back
    // to the pool first, so the solve reuses it instead of growing the pool
    ctx->ba.reset();
    if (ctx->multi()) {  // point-sharded over the context's devices
      sfm::ba_solve_multi(ctx->group, *prob, *opt, out_cam_q, out_cam_t, out_points, report);
      return;
    }
    sfm::BASolver solver(ctx->stream, &ctx->prof, &ctx->comm);
    solver.setup(*prob, *opt);
    solver.iterate(opt->max_iters > 0 ? opt->max_iters : 0, report);
    solver.download(out_cam_q, out_cam_t, out_points);
  });
}

int sfm_ba_solve_emulated(sfm_ctx* ctx, int32_t n_shards, const sfm_ba_problem* shards,
                          const sfm_ba_options* opt, double* out_cam_q, double* out_cam_t,
                          double* const* out_points, sfm_ba_report* report) {
  return guarded(ctx, [&] {
    SFM_REQUIRE(shards && opt && out_cam_q && out_cam_t && out_points, "null argument");
    ctx->ba.reset();
    sfm::ba_solve_emulated(ctx->device, n_shards, shards, *opt, out_cam_q, out_cam_t, out_points, report);
  });
}

int sfm_gba_solve(sfm_ctx* ctx, const sfm_gba_problem* prob, const sfm_ba_options* opt, double* out_block_q,
                  double* out_block_t, double* out_points, sfm_ba_report* report) {
  return guarded(ctx, [&] {
    SFM_REQUIRE(prob && opt, "null problem/options");
    ctx->ba.reset();
    sfm::GBASolver solver(ctx->stream, &ctx->prof);
    solver.setup(*prob, *opt);
    solver.iterate(opt->max_iters > 0 ? opt->max_iters : 0, report);
    solver.download(out_block_q, out_block_t, out_points);
  });
}

int sfm_ba_eval(sfm_ctx* ctx, const sfm_ba_problem* prob, int32_t loss_kind, double loss_param,
                double* out_cost_per_obs, double* out_res, double* out_jc, double* out_jp) {
  return guarded(ctx, [&] {
    SFM_REQUIRE(prob != nullptr, "null problem");
    sfm::BASolver::eval(ctx->stream, &ctx->prof, *prob, loss_kind, loss_param, out_cost_per_obs, out_res,
                        out_jc, out_jp);
  });
}

int sfm_iterative_map(sfm_ctx* ctx, const sfm_map_problem* prob, const sfm_map_options* opt,
                      double* out_cam_q, double* out_cam_t, double* out_X, uint8_t* out_mask,
                      int8_t* out_status, int64_t* out_lm_track, int64_t* out_n_landmarks,
                      sfm_round_stat* out_stats, int32_t* out_n_stats) {
  return guarded(ctx, [&] {
    SFM_REQUIRE(prob && opt && out_cam_q && out_cam_t && out_X && out_mask && out_status && out_lm_track &&
                    out_n_landmarks && out_stats && out_n_stats,
                "null argument");
    ctx->ba.reset();  // device memory back to the pool
    sfm::iterative_map(ctx->stream, &ctx->prof, *prob, *opt, out_cam_q, out_cam_t, out_X, out_mask, out_status,
                       out_lm_track, out_n_landmarks, out_stats, out_n_stats,
                       ctx->multi() ? &ctx->group : nullptr);
  });
}

int sfm_shard_points(int64_t n_obs, const int32_t* obs_point, int64_t n_points, int32_t world,
                     int64_t* out_bounds) {
  // host-only: no context
  try {
    if (n_obs < 0 || n_points < 0 || world < 1 || !out_bounds || (n_obs && !obs_point)) return SFM_E_INVALID;
    const auto b = sfm::shard_bounds(obs_point, n_obs, n_points, world);
    for (int r = 0; r <= world; ++r) out_bounds[r] = b[r];
    return SFM_OK;
  } catch (...) {
    return SFM_E_INVALID;
  }
}

int sfm_pcg_rank_rows(int32_t n_rows, const int32_t* row_ptr, int32_t world, int32_t* out_row0) {
  // host-only: no context
  try {
    if (n_rows < 1 || world < 1 || world > n_rows || !row_ptr || !out_row0) return SFM_E_INVALID;
    const auto r = sfm::pcg_rank_rows(row_ptr, n_rows, world);
    for (int q = 0; q <= world; ++q) out_row0[q] = r[q];
    return SFM_OK;
  } catch (...) {
    return SFM_E_INVALID;
  }
}

int sfm_build_tracks(int64_t n_pairs, const int32_t* pair_frames, const int64_t* pair_ptr,
                     const int32_t* match_index, int64_t* out_track_ptr, int32_t* out_obs_frame,
                     int32_t* out_obs_feature, int64_t* out_n_tracks, int64_t* out_n_obs) {
  // host-only: no context (runs without a GPU)
  try {
    if (n_pairs < 0 || (n_pairs && (!pair_frames || !pair_ptr)) || !out_track_ptr || !out_n_tracks ||
        !out_n_obs)
      return SFM_E_INVALID;
    sfm::build_tracks(n_pairs, pair_frames, pair_ptr, match_index, out_track_ptr, out_obs_frame, out_obs_feature,
                      out_n_tracks, out_n_obs);
    return SFM_OK;
  } catch (const sfm::SfmError& e) {
    return e.code;
  } catch (...) {
    return SFM_E_INVALID;
  }
}

int sfm_ransac_triangulate(sfm_ctx* ctx, const sfm_tracks* tracks, double threshold_px, double min_angle,
                           int32_t method, double* out_X, uint8_t* out_mask, int8_t* out_status) {
  return guarded(ctx, [&] {
    SFM_REQUIRE(tracks != nullptr, "null tracks");
    sfm::tri_ransac(ctx->stream, &ctx->prof, *tracks, threshold_px, min_angle, method, out_X, out_mask,
                    out_status);
  });
}

int sfm_triangulate(sfm_ctx* ctx, const sfm_tracks* tracks, double min_angle, int32_t method, double* out_X,
                    int8_t* out_status) {
  return guarded(ctx, [&] {
    SFM_REQUIRE(tracks != nullptr, "null tracks");
    sfm::tri_direct(ctx->stream, &ctx->prof, *tracks, min_angle, method, out_X, out_status);
  });
}

int sfm_gate(sfm_ctx* ctx, const sfm_tracks* tracks, const double* points, double threshold_px,
             uint8_t* mask_inout, int32_t* out_inliers, int64_t* out_removed) {
  return guarded(ctx, [&] {
    SFM_REQUIRE(tracks && points && mask_inout, "null arguments");
    sfm::tri_gate(ctx->stream, &ctx->prof, *tracks, points, threshold_px, mask_inout, out_inliers,
                  out_removed);
  });
}

int sfm_reprojection_errors(sfm_ctx* ctx, const sfm_tracks* tracks, const double* points, double* out_err) {
  return guarded(ctx, [&] {
    SFM_REQUIRE(tracks && points && out_err, "null arguments");
    sfm::tri_reproj_errors(ctx->stream, &ctx->prof, *tracks, points, out_err);
  });
}

}  // extern "C"
