// emu.cu -- shard emulation of the point-sharded multi-GPU BA on one device
// (see EmuGroup in comm.cuh): the collectives as fixed-rank-order device
// reductions over the R logical ranks' buffers, and the R-thread driver
// behind sfm_ba_solve_emulated.
#include <algorithm>
#include <string>
#include <thread>
#include <vector>

#include "ba.cuh"
#include "comm.cuh"
#include "emu.cuh"

namespace sfm {

namespace {

constexpr int kEmuMaxRanks = 16;

template <typename T>
struct PtrPack {
  T* d[kEmuMaxRanks];
};

// v = d_0 (op) d_1 (op) ... in rank order, written back to every rank
template <typename T>
__global__ void k_emu_reduce(PtrPack<T> p, int world, size_t n, int op) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    T v = p.d[0][i];
    for (int r = 1; r < world; ++r) {
      const T w = p.d[r][i];
      v = op == 0 ? v + w : (op == 1 ? (w > v ? w : v) : (w < v ? w : v));
    }
    for (int r = 0; r < world; ++r) p.d[r][i] = v;
  }
}

// v = d_0 + d_1 + ... (rank order) over [lo, hi), written to d_dst only
__global__ void k_emu_reduce_to(PtrPack<double> p, int world, int64_t lo, int64_t hi, int dst) {
  for (int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += (int64_t)gridDim.x * blockDim.x) {
    double v = p.d[0][i];
    for (int r = 1; r < world; ++r) v += p.d[r][i];
    p.d[dst][i] = v;
  }
}

}  // namespace

void EmuGroup::reduce_ranges(int rank, double* d, const std::vector<int64_t>& off, cudaStream_t s) {
  SFM_CUDA(cudaStreamSynchronize(s));
  ptr_a[rank] = d;
  barrier();
  if (rank == 0) {
    PtrPack<double> pk{};
    for (int r = 0; r < world; ++r) pk.d[r] = static_cast<double*>(ptr_a[r]);
    for (int q = 0; q < world; ++q) {
      const int64_t n = off[q + 1] - off[q];
      if (n <= 0) continue;
      k_emu_reduce_to<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, s>>>(pk, world, off[q],
                                                                                          off[q + 1], q);
      SFM_CHECK_LAUNCH();
    }
    SFM_CUDA(cudaStreamSynchronize(s));
  }
  barrier();
}

void EmuGroup::allgather_ranges(int rank, double* d, const std::vector<int64_t>& off, cudaStream_t s) {
  SFM_CUDA(cudaStreamSynchronize(s));
  ptr_a[rank] = d;
  barrier();
  if (rank == 0) {
    for (int q = 0; q < world; ++q)
      for (int r = 0; r < world; ++r)
        if (r != q && off[q + 1] > off[q])
          SFM_CUDA(cudaMemcpyAsync(static_cast<double*>(ptr_a[r]) + off[q], static_cast<double*>(ptr_a[q]) + off[q],
                                   sizeof(double) * (size_t)(off[q + 1] - off[q]), cudaMemcpyDeviceToDevice, s));
    SFM_CUDA(cudaStreamSynchronize(s));
  }
  barrier();
}

void EmuGroup::run_root(int rank, const void* mine, cudaStream_t s,
                        const std::function<void(const void* const*)>& fn) {
  SFM_CUDA(cudaStreamSynchronize(s));
  ptr_a[rank] = const_cast<void*>(mine);
  barrier();
  if (rank == 0) {
    try {
      fn(ptr_a.data());
      SFM_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
      abort();
      throw;
    }
  }
  barrier();
}

void EmuGroup::run_each(int rank, const void* mine, cudaStream_t s, const std::function<void()>& root_prep,
                        const std::function<void(const void* const*)>& fn) {
  SFM_CUDA(cudaStreamSynchronize(s));
  ptr_a[rank] = const_cast<void*>(mine);
  barrier();
  std::vector<const void*> all(ptr_a.begin(), ptr_a.end());
  if (rank == 0) {
    try {
      root_prep();
      SFM_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
      abort();
      throw;
    }
  }
  barrier();
  try {
    fn(all.data());
    SFM_CUDA(cudaStreamSynchronize(s));
  } catch (...) {
    abort();
    throw;
  }
  barrier();
}

template <typename T>
void EmuGroup::reduce(int rank, T* d, size_t n, cudaStream_t s, int op) {
  SFM_CUDA(cudaStreamSynchronize(s));
  ptr_a[rank] = d;
  barrier();
  if (rank == 0) {
    PtrPack<T> pk{};
    for (int r = 0; r < world; ++r) pk.d[r] = static_cast<T*>(ptr_a[r]);
    k_emu_reduce<T><<<(unsigned)std::min<size_t>((n + 255) / 256, 4096), 256, 0, s>>>(pk, world, n, op);
    SFM_CHECK_LAUNCH();
    SFM_CUDA(cudaStreamSynchronize(s));
  }
  barrier();
}

template void EmuGroup::reduce<double>(int, double*, size_t, cudaStream_t, int);
template void EmuGroup::reduce<unsigned long long>(int, unsigned long long*, size_t, cudaStream_t, int);
template void EmuGroup::reduce<int>(int, int*, size_t, cudaStream_t, int);

void EmuGroup::allgather_u64(int rank, const unsigned long long* send, unsigned long long* recv, size_t n,
                             cudaStream_t s) {
  SFM_CUDA(cudaStreamSynchronize(s));
  ptr_a[rank] = const_cast<unsigned long long*>(send);
  ptr_b[rank] = recv;
  barrier();
  if (rank == 0) {
    for (int r = 0; r < world; ++r)
      for (int q = 0; q < world; ++q)
        if (n)
          SFM_CUDA(cudaMemcpyAsync(static_cast<unsigned long long*>(ptr_b[r]) + (size_t)q * n, ptr_a[q],
                                   n * sizeof(unsigned long long), cudaMemcpyDeviceToDevice, s));
    SFM_CUDA(cudaStreamSynchronize(s));
  }
  barrier();
}

std::vector<int64_t> shard_bounds(const int* op, int64_t N, int64_t P, int world) {
  // first observation of every point (obs_point is non-decreasing)
  auto first_obs = [&](int64_t p) { return (int64_t)(std::lower_bound(op, op + N, (int)p) - op); };
  std::vector<int64_t> bounds(1, 0);
  for (int r = 1; r < world; ++r) {
    // first point whose observations start at or after r*N/world (the point
    // straddling the target stays whole on the lower rank)
    const int64_t target = N * r / world;
    int64_t p = P;
    if (target < N) {
      const int64_t q = op[target];
      p = first_obs(q) >= target ? q : q + 1;
    }
    bounds.push_back(std::max(bounds.back(), std::min(p, P)));
  }
  bounds.push_back(P);
  return bounds;
}

ShardSet shard_problem(const sfm_ba_problem& full, int world) {
  SFM_REQUIRE(world >= 1, "world must be >= 1");
  const int64_t N = full.n_obs, P = full.n_points;
  std::vector<int> op((size_t)N);
  if (N) SFM_CUDA(cudaMemcpy(op.data(), full.obs_point, sizeof(int) * N, cudaMemcpyDefault));
  auto first_obs = [&](int64_t p) {
    return (int64_t)(std::lower_bound(op.begin(), op.end(), (int)p) - op.begin());
  };
  int n_free = 0;
  {
    std::vector<uint8_t> fx((size_t)full.n_frames);
    if (full.n_frames)
      SFM_CUDA(cudaMemcpy(fx.data(), full.frame_fixed, full.n_frames, cudaMemcpyDefault));
    for (uint8_t v : fx) n_free += v == 0;
  }
  ShardSet ss;
  const std::vector<int64_t> bounds = shard_bounds(op.data(), N, P, world);
  ss.shards.resize(world);
  ss.local_op.resize(world);
  ss.p0.resize(world);
  for (int r = 0; r < world; ++r) {
    const int64_t p0 = bounds[r], p1 = bounds[r + 1];
    const int64_t o0 = first_obs(p0), o1 = first_obs(p1);
    auto& lop = ss.local_op[r];
    lop.resize((size_t)(o1 - o0));
    for (int64_t o = o0; o < o1; ++o) lop[(size_t)(o - o0)] = op[(size_t)o] - (int)p0;
    sfm_ba_problem sh = full;
    sh.n_points = p1 - p0;
    sh.points = full.points + 3 * p0;
    sh.n_obs = o1 - o0;
    sh.obs_frame = full.obs_frame + o0;
    sh.obs_point = lop.data();
    sh.obs_uv = full.obs_uv + 2 * o0;
    if (r != 0) {
      sh.n_edges = 0;
      sh.n_priors = 0;
    }
    sh.obs_offset = full.obs_offset + o0;
    sh.n_params_global = 6 * (int64_t)n_free + 3 * P;
    ss.shards[r] = sh;
    ss.p0[r] = p0;
  }
  return ss;
}

void ba_solve_group(const DeviceGroup& g, const sfm_ba_problem* shards, const sfm_ba_options& opt,
                    double* out_q, double* out_t, double* const* out_points, sfm_ba_report* report) {
  const int n = g.size();
  SFM_REQUIRE(n >= 1 && n <= kEmuMaxRanks, "group size must be in [1, 16]");
  SFM_REQUIRE(g.comms.empty() || (int)g.comms.size() == n, "one communicator per rank");
  EmuGroup grp(n);
  std::vector<int> codes(n, SFM_OK);
  std::vector<std::string> msgs(n);
  std::vector<std::thread> th;
  for (int r = 0; r < n; ++r) {
    th.emplace_back([&, r] {
      cudaStream_t s = nullptr;
      try {
        SFM_CUDA(cudaSetDevice(g.devices[r]));
        SFM_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        alloc_stream() = s;
        Profiler prof;
        Comm comm;
        comm.rank = r;
        comm.world = n;
        if (!g.comms.empty()) {
          comm.comm = g.comms[r];
          comm.owned = false;
          comm.peer = g.peer;
        } else {
          comm.emu = &grp;
        }
        comm.host = &grp;
        {
          BASolver solver(s, &prof, &comm);
          solver.setup(shards[r], opt);
          sfm_ba_report rep{};
          solver.iterate(opt.max_iters > 0 ? opt.max_iters : 0, &rep);
          solver.download(r == 0 ? out_q : nullptr, r == 0 ? out_t : nullptr, out_points[r]);
          if (r == 0 && report) *report = rep;
        }
        SFM_CUDA(cudaStreamSynchronize(s));
      } catch (const SfmError& e) {
        codes[r] = e.code;
        msgs[r] = e.what();
        grp.abort();
      } catch (const std::exception& e) {
        codes[r] = SFM_E_CUDA;
        msgs[r] = e.what();
        grp.abort();
      }
      if (s) cudaStreamDestroy(s);
      alloc_stream() = nullptr;
    });
  }
  for (auto& t : th) t.join();
  // the root cause: the lowest rank whose failure is not the abort echo
  for (int r = 0; r < n; ++r)
    if (codes[r] != SFM_OK && msgs[r].find("aborted by another rank") == std::string::npos)
      throw SfmError(codes[r], msgs[r]);
  for (int r = 0; r < n; ++r)
    if (codes[r] != SFM_OK) throw SfmError(codes[r], msgs[r]);
}

void ba_solve_emulated(int device, int n_shards, const sfm_ba_problem* shards, const sfm_ba_options& opt,
                       double* out_q, double* out_t, double* const* out_points, sfm_ba_report* report) {
  SFM_REQUIRE(n_shards >= 1 && n_shards <= kEmuMaxRanks, "n_shards must be in [1, 16]");
  DeviceGroup g;
  g.devices.assign(n_shards, device);
  ba_solve_group(g, shards, opt, out_q, out_t, out_points, report);
}

void ba_solve_multi(const DeviceGroup& g, const sfm_ba_problem& full, const sfm_ba_options& opt,
                    double* out_q, double* out_t, double* out_points, sfm_ba_report* report) {
  ShardSet ss = shard_problem(full, g.size());
  std::vector<double*> outs(g.size());
  for (int r = 0; r < g.size(); ++r) outs[r] = out_points ? out_points + 3 * ss.p0[r] : nullptr;
  ba_solve_group(g, ss.shards.data(), opt, out_q, out_t, outs.data(), report);
}

}  // namespace sfm
