// emu.cu -- shard emulation of the point-sharded multi-GPU BA on one device
// (see EmuGroup in comm.cuh): the collectives as fixed-rank-order device
// reductions over the R logical ranks' buffers, and the R-thread driver
// behind sfm_ba_solve_emulated.
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

}  // namespace

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

void ba_solve_emulated(int device, int n_shards, const sfm_ba_problem* shards, const sfm_ba_options& opt,
                       double* out_q, double* out_t, double* const* out_points, sfm_ba_report* report) {
  SFM_REQUIRE(n_shards >= 1 && n_shards <= kEmuMaxRanks, "n_shards must be in [1, 16]");
  EmuGroup grp(n_shards);
  std::vector<int> codes(n_shards, SFM_OK);
  std::vector<std::string> msgs(n_shards);
  std::vector<std::thread> th;
  for (int r = 0; r < n_shards; ++r) {
    th.emplace_back([&, r] {
      cudaStream_t s = nullptr;
      try {
        SFM_CUDA(cudaSetDevice(device));
        SFM_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        alloc_stream() = s;
        Profiler prof;
        Comm comm;
        comm.rank = r;
        comm.world = n_shards;
        comm.emu = &grp;
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
  for (int r = 0; r < n_shards; ++r)
    if (codes[r] != SFM_OK && msgs[r].find("aborted by another rank") == std::string::npos)
      throw SfmError(codes[r], msgs[r]);
  for (int r = 0; r < n_shards; ++r)
    if (codes[r] != SFM_OK) throw SfmError(codes[r], msgs[r]);
}

}  // namespace sfm
