// imap.cu -- device-resident iterative_map (mapping.py:569-624).
//
// The reference loop re-flattens its object model for every call it makes
// (ransac_triangulate per track, bundle_adjust, remove_outliers).  Here the
// tracks (CSR), their status, inlier masks, landmark positions and the
// landmark order (the map's `landmarks` list, whose order is the BA residual
// order, mapping.py:452-475) stay on the device for the whole loop:
//
//   round r:  RANSAC on the PENDING tracks (tri_ransac_device)
//             -> new landmarks appended in track order (mapping.py:600-609)
//             -> stage-1 BA over the landmarks' inlier observations
//             -> stage-1 gate; landmarks left with < 2 inliers go back to
//                PENDING and leave the list, order kept (mapping.py:544-566)
//             stop when a round neither adds nor removes (mapping.py:616)
//   final:    stage-2 BA + stage-2 gate (mapping.py:618-622)
//
// Every list edit is a stable device compaction (CUB select), so the
// landmark order matches the reference's list operations exactly.
#include <cub/cub.cuh>

#include <cmath>
#include <vector>

#include "ba.cuh"
#include "emu.cuh"
#include "imap.cuh"
#include "tri.cuh"

namespace sfm {

namespace {

__global__ void k_map_active(int64_t T, const int8_t* __restrict__ status, uint8_t* __restrict__ active) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < T) active[t] = status[t] == SFM_TRACK_PENDING;
}

// RANSAC results -> map state for the tracks that were PENDING.
__global__ void k_map_merge(int64_t T, const int64_t* __restrict__ ptr, const uint8_t* __restrict__ active,
                            const int8_t* __restrict__ rst, const double* __restrict__ Xr,
                            const uint8_t* __restrict__ maskr, int8_t* __restrict__ status,
                            double* __restrict__ X, uint8_t* __restrict__ mask, uint8_t* __restrict__ newflag) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  uint8_t nf = 0;
  if (active[t]) {
    if (rst[t] == SFM_TRI_OK) {
      status[t] = SFM_TRACK_TRIANGULATED;
      X[t * 3] = Xr[t * 3];
      X[t * 3 + 1] = Xr[t * 3 + 1];
      X[t * 3 + 2] = Xr[t * 3 + 2];
      for (int64_t o = ptr[t]; o < ptr[t + 1]; ++o) mask[o] = maskr[o];
      nf = 1;
    } else {
      status[t] = SFM_TRACK_FAILED;  // failed tracks are never retried
    }
  }
  newflag[t] = nf;
}

__global__ void k_iota(int64_t n, int* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (int)i;
}

// inlier observations per landmark (BA residuals of landmark i)
__global__ void k_lm_count(int64_t L, const int* __restrict__ lm, const int64_t* __restrict__ ptr,
                           const uint8_t* __restrict__ mask, int64_t* __restrict__ cnt) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > L) return;
  int64_t c = 0;
  if (i < L) {
    const int t = lm[i];
    for (int64_t o = ptr[t]; o < ptr[t + 1]; ++o) c += mask[o];
  }
  cnt[i] = c;
}

// BA arrays in landmark order: points, inlier observations in track order
// (mapping.py:452-475)
__global__ void k_lm_fill(int64_t L, const int* __restrict__ lm, const int64_t* __restrict__ ptr,
                          const uint8_t* __restrict__ mask, const int* __restrict__ of,
                          const double* __restrict__ uv, const double* __restrict__ X,
                          const int64_t* __restrict__ off, int* __restrict__ ba_of, int* __restrict__ ba_op,
                          double* __restrict__ ba_uv, double* __restrict__ ba_X) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= L) return;
  const int t = lm[i];
  ba_X[i * 3] = X[(int64_t)t * 3];
  ba_X[i * 3 + 1] = X[(int64_t)t * 3 + 1];
  ba_X[i * 3 + 2] = X[(int64_t)t * 3 + 2];
  int64_t w = off[i];
  for (int64_t o = ptr[t]; o < ptr[t + 1]; ++o) {
    if (!mask[o]) continue;
    ba_of[w] = of[o];
    ba_op[w] = (int)i;
    ba_uv[w * 2] = uv[o * 2];
    ba_uv[w * 2 + 1] = uv[o * 2 + 1];
    ++w;
  }
}

__global__ void k_lm_scatter(int64_t L, const int* __restrict__ lm, const double* __restrict__ ba_X,
                             double* __restrict__ X) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= L) return;
  const int64_t t = lm[i];
  X[t * 3] = ba_X[i * 3];
  X[t * 3 + 1] = ba_X[i * 3 + 1];
  X[t * 3 + 2] = ba_X[i * 3 + 2];
}

// remove_outliers' demotion: < 2 inliers -> PENDING, dropped from the list
__global__ void k_lm_demote(int64_t L, const int* __restrict__ lm, const int* __restrict__ inl,
                            const int64_t* __restrict__ ptr, int8_t* __restrict__ status,
                            uint8_t* __restrict__ mask, double* __restrict__ X, uint8_t* __restrict__ keep) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= L) return;
  const int t = lm[i];
  if (inl[t] < 2) {
    status[t] = SFM_TRACK_PENDING;
    for (int64_t o = ptr[t]; o < ptr[t + 1]; ++o) mask[o] = 0;
    X[(int64_t)t * 3] = X[(int64_t)t * 3 + 1] = X[(int64_t)t * 3 + 2] = NAN;
    keep[i] = 0;
  } else {
    keep[i] = 1;
  }
}

__global__ void k_fill_nan(int64_t n, double* p) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = NAN;
}

struct CubScratch {
  DevBuf<char> buf;
  void* get(size_t bytes) { return buf.resize(bytes); }
};

}  // namespace

void iterative_map(cudaStream_t s, Profiler* prof, const sfm_map_problem& pr, const sfm_map_options& op,
                   double* out_q, double* out_t, double* out_X, uint8_t* out_mask, int8_t* out_status,
                   int64_t* out_lm, int64_t* out_nlm, sfm_round_stat* out_stats, int32_t* out_nstats,
                   const DeviceGroup* group) {
  SFM_REQUIRE(pr.n_frames >= 0 && pr.n_tracks >= 0 && pr.n_obs >= 0, "negative sizes");
  SFM_REQUIRE(pr.n_tracks < (1ll << 31), "n_tracks must fit in 31 bits");
  SFM_REQUIRE(op.max_outer_iters >= 0, "max_outer_iters < 0");
  for (int f = 0; f < pr.n_frames; ++f)
    SFM_REQUIRE(pr.frame_model[f] >= 0 && pr.frame_model[f] < pr.n_models, "frame_model out of range");
  SFM_REQUIRE(pr.track_ptr[0] == 0 && pr.track_ptr[pr.n_tracks] == pr.n_obs, "track_ptr must span obs");
  const int F = pr.n_frames;
  const int64_t T = pr.n_tracks, N = pr.n_obs;

  // ---- device state ----------------------------------------------------------
  DevBuf<double> q, t, Rt, uv, ray, X, Xr, baX, baUV;
  DevBuf<int> fm, of, rst_ray, lm, lm2, ids, inl, ba_of, ba_op;
  DevBuf<int64_t> ptr, cnt, off;
  DevBuf<int8_t> status, rst;
  DevBuf<uint8_t> active, mask, maskr, newflag, keep;
  DevBuf<sfm_camera_model> models;
  DevBuf<unsigned long long> removed;
  DevBuf<int> nsel;
  q.upload(pr.cam_q, (size_t)F * 4, s);
  t.upload(pr.cam_t, (size_t)F * 3, s);
  Rt.resize((size_t)F * 12);
  fm.upload(pr.frame_model, F, s);
  models.upload(pr.models, pr.n_models, s);
  ptr.upload(pr.track_ptr, T + 1, s);
  of.upload(pr.obs_frame, N, s);
  uv.upload(pr.obs_uv, (size_t)N * 2, s);
  status.resize(T);
  if (pr.track_status) status.upload(pr.track_status, T, s);
  else status.zero(s);
  X.resize((size_t)T * 3);
  if (T) k_fill_nan<<<grid_for(T * 3, 256), 256, 0, s>>>(T * 3, X.get());
  mask.resize(N);
  mask.zero(s);
  Xr.resize((size_t)T * 3);
  maskr.resize(N);
  rst.resize(T);
  active.resize(T);
  newflag.resize(T);
  ids.resize(T);
  if (T) k_iota<<<grid_for(T, 256), 256, 0, s>>>(T, ids.get());
  lm.resize(T);
  lm2.resize(T);
  keep.resize(T);
  inl.resize(T);
  removed.resize(1);
  nsel.resize(1);
  ray.resize((size_t)N * 3);
  rst_ray.resize(N);
  SFM_CHECK_LAUNCH();

  TriDeviceTracks tr{};
  tr.n_frames = F; tr.Rt = Rt.get(); tr.frame_model = fm.get(); tr.models = models.get();
  tr.n_tracks = T; tr.n_obs = N; tr.ptr = ptr.get(); tr.obs_frame = of.get(); tr.obs_uv = uv.get();
  tr.ray = ray.get(); tr.ray_st = rst_ray.get();
  tri_rt_device(s, F, q.get(), t.get(), Rt.get());
  tri_rays_device(s, prof, tr, ray.get(), rst_ray.get());

  // host copies of the pose-term arrays for every BA call (BASolver reads
  // frame_model / frame_fixed / edges / priors on the host)
  std::vector<int> h_fm(pr.frame_model, pr.frame_model + F);
  CubScratch tmp;
  int64_t nlm = 0;
  std::vector<sfm_round_stat> stats;

  auto select = [&](const int* in, const uint8_t* flags, int* out, int64_t n) -> int64_t {
    if (n == 0) return 0;
    size_t tb = 0;
    SFM_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, in, flags, out, nsel.get(), (int)n, s));
    SFM_CUDA(cub::DeviceSelect::Flagged(tmp.get(tb), tb, in, flags, out, nsel.get(), (int)n, s));
    int h = 0;
    nsel.download(&h, 1, s);
    SFM_CUDA(cudaStreamSynchronize(s));
    return h;
  };

  // bundle_adjust's gauge check (mapping.py:408-409): it runs only once
  // there are landmarks, so an empty map never raises
  bool gauge = pr.n_priors > 0 && pr.prior_weight > 0.0;
  for (int f = 0; f < F && !gauge; ++f) gauge = pr.frame_fixed[f] != 0;
  auto run_ba = [&](int loss_kind, double loss_param) {
    if (nlm == 0) return;
    if (!gauge) throw SfmError(SFM_E_NO_GAUGE, "no fixed pose and no absolute prior");
    cnt.resize(nlm + 1);
    off.resize(nlm + 1);
    k_lm_count<<<grid_for(nlm + 1, 256), 256, 0, s>>>(nlm, lm.get(), ptr.get(), mask.get(), cnt.get());
    SFM_CHECK_LAUNCH();
    size_t tb = 0;
    SFM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.get(), off.get(), nlm + 1, s));
    SFM_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(tb), tb, cnt.get(), off.get(), nlm + 1, s));
    int64_t nba = 0;
    SFM_CUDA(cudaMemcpyAsync(&nba, off.get() + nlm, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SFM_CUDA(cudaStreamSynchronize(s));
    ba_of.resize(nba);
    ba_op.resize(nba);
    baUV.resize((size_t)nba * 2);
    baX.resize((size_t)nlm * 3);
    k_lm_fill<<<grid_for(nlm, 128), 128, 0, s>>>(nlm, lm.get(), ptr.get(), mask.get(), of.get(), uv.get(),
                                                  X.get(), off.get(), ba_of.get(), ba_op.get(), baUV.get(),
                                                  baX.get());
    SFM_CHECK_LAUNCH();
    sfm_ba_problem bp{};
    bp.n_frames = F; bp.n_models = pr.n_models;
    bp.cam_q = q.get(); bp.cam_t = t.get();                       // device
    bp.frame_model = h_fm.data(); bp.frame_fixed = pr.frame_fixed;  // host
    bp.models = pr.models;
    bp.n_points = nlm; bp.points = baX.get();                      // device
    bp.n_obs = nba; bp.obs_frame = ba_of.get(); bp.obs_point = ba_op.get(); bp.obs_uv = baUV.get();
    bp.n_edges = pr.n_edges; bp.n_priors = pr.n_priors;
    bp.edge_ab = pr.edge_ab; bp.prior_frame = pr.prior_frame;      // host
    bp.edge_weight = pr.edge_weight; bp.prior_weight = pr.prior_weight;
    sfm_ba_options bo = op.solver;
    bo.loss_kind = loss_kind;
    bo.loss_param = loss_param;
    bo.max_iters = op.max_solver_iters;
    if (group && group->size() > 1) {
      // point-sharded over the context's devices; the shards read this
      // device's arrays and write the solution back into them
      SFM_CUDA(cudaStreamSynchronize(s));
      ba_solve_multi(*group, bp, bo, q.get(), t.get(), baX.get(), nullptr);
      alloc_stream() = s;
    } else {
      BASolver solver(s, prof, nullptr);
      solver.setup(bp, bo);
      solver.iterate(bo.max_iters > 0 ? bo.max_iters : 0, nullptr);
      solver.download(q.get(), t.get(), baX.get());
    }
    k_lm_scatter<<<grid_for(nlm, 256), 256, 0, s>>>(nlm, lm.get(), baX.get(), X.get());
    SFM_CHECK_LAUNCH();
    tri_rt_device(s, F, q.get(), t.get(), Rt.get());
  };

  auto gate = [&](double thr) -> int64_t {
    removed.zero(s);
    tri_gate_device(s, prof, tr, X.get(), thr, mask.get(), inl.get(), removed.get());
    unsigned long long h = 0;
    if (nlm) {
      k_lm_demote<<<grid_for(nlm, 256), 256, 0, s>>>(nlm, lm.get(), inl.get(), ptr.get(), status.get(),
                                                       mask.get(), X.get(), keep.get());
      SFM_CHECK_LAUNCH();
      const int64_t kept = select(lm.get(), keep.get(), lm2.get(), nlm);
      std::swap(lm.ptr, lm2.ptr);
      std::swap(lm.cap, lm2.cap);
      std::swap(lm.n, lm2.n);
      nlm = kept;
    }
    removed.download(&h, 1, s);
    SFM_CUDA(cudaStreamSynchronize(s));
    return (int64_t)h;
  };

  for (int round = 0; round < op.max_outer_iters; ++round) {
    NvtxRange nv("sfm imap round");
    // 1. RANSAC on the pending tracks (mapping.py:600-609)
    int64_t added = 0;
    if (T) {
      k_map_active<<<grid_for(T, 256), 256, 0, s>>>(T, status.get(), active.get());
      SFM_CHECK_LAUNCH();
      tri_ransac_device(s, prof, tr, active.get(), op.stage1_outlier_px, op.min_angle, op.method, Xr.get(),
                        maskr.get(), rst.get());
      k_map_merge<<<grid_for(T, 128), 128, 0, s>>>(T, ptr.get(), active.get(), rst.get(), Xr.get(), maskr.get(),
                                                    status.get(), X.get(), mask.get(), newflag.get());
      SFM_CHECK_LAUNCH();
      added = select(ids.get(), newflag.get(), lm.get() + nlm, T);  // appended in track order
      nlm += added;
    }
    // 2. stage-1 BA, 3. stage-1 gate (mapping.py:611-612)
    run_ba(op.stage1_loss_kind, op.stage1_loss_param);
    const int64_t rm = gate(op.stage1_outlier_px);
    stats.push_back(sfm_round_stat{round, 0, added, rm, nlm});
    if (added == 0 && rm == 0) break;
  }
  if (nlm) {  // mapping.py:618-622
    NvtxRange nv("sfm imap final");
    run_ba(op.stage2_loss_kind, op.stage2_loss_param);
    const int64_t rm = gate(op.stage2_outlier_px);
    stats.push_back(sfm_round_stat{-1, 0, 0, rm, nlm});
  }

  q.download(out_q, (size_t)F * 4, s);
  t.download(out_t, (size_t)F * 3, s);
  X.download(out_X, (size_t)T * 3, s);
  mask.download(out_mask, N, s);
  status.download(out_status, T, s);
  std::vector<int> h_lm(nlm);
  lm.download(h_lm.data(), nlm, s);
  SFM_CUDA(cudaStreamSynchronize(s));
  for (int64_t i = 0; i < nlm; ++i) out_lm[i] = h_lm[i];
  *out_nlm = nlm;
  for (size_t i = 0; i < stats.size(); ++i) out_stats[i] = stats[i];
  *out_nstats = (int32_t)stats.size();
}

}  // namespace sfm
