// comm.cuh -- rank-to-rank reductions for point-sharded BA.
//
// One process per GPU.  world == 1 makes every call a no-op; otherwise the
// camera-indexed sums (U, g_c, S, b_S) and the scalars (cost, step norm,
// depth flag) are all-reduced with NCCL over NVLink on the context stream.
// NCCL's ring/tree results are identical on every rank, so the replicated
// PCG on S takes identical decisions everywhere.
#pragma once
#include <nccl.h>

#include <condition_variable>
#include <functional>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace sfm {

#define SFM_NCCL(call)                                                              \
  do {                                                                              \
    ncclResult_t r_ = (call);                                                       \
    if (r_ != ncclSuccess)                                                          \
      throw ::sfm::SfmError(SFM_E_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
  } while (0)

// Shard emulation (test path): R logical ranks as R host
// threads on ONE device, each driving its own BASolver on its own stream.
// The collectives are the same calls the NCCL path makes (same points in
// the LM control flow, same buffers), executed as a fixed-rank-order
// reduction kernel over the ranks' device buffers plus host barriers, so
// the partitioned math (point shards, partial Schur complements, replicated
// PCG, scalar reductions) runs exactly as across GPUs.  NCCL itself rejects
// a communicator with the same device twice, hence this path.
struct EmuGroup {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long gen = 0;
  bool aborted = false;
  std::vector<void*> ptr_a, ptr_b;
  explicit EmuGroup(int w) : world(w), ptr_a(w), ptr_b(w) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) throw SfmError(SFM_E_INVALID, "shard emulation aborted by another rank");
    const unsigned long long g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g || aborted; });
      if (aborted) throw SfmError(SFM_E_INVALID, "shard emulation aborted by another rank");
    }
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    aborted = true;
    cv.notify_all();
  }
  // op: 0 sum, 1 max, 2 min
  template <typename T>
  void reduce(int rank, T* d, size_t n, cudaStream_t s, int op);
  void allgather_u64(int rank, const unsigned long long* send, unsigned long long* recv, size_t n,
                     cudaStream_t s);
  // rank q's range [off[q], off[q+1]) of every rank's d, summed in rank
  // order, lands in rank q's d only (reduce-scatter with variable counts)
  void reduce_ranges(int rank, double* d, const std::vector<int64_t>& off, cudaStream_t s);
  // rank q's range of its d is copied into every rank's d (allgatherv)
  void allgather_ranges(int rank, double* d, const std::vector<int64_t>& off, cudaStream_t s);
  // every rank hands in `mine`; rank 0 runs fn(all ranks' pointers) on its
  // stream, then everyone continues (one launch covering every rank)
  void run_root(int rank, const void* mine, cudaStream_t s, const std::function<void(const void* const*)>& fn);
  // every rank hands in `mine` and gets everyone's; rank 0 runs root_prep;
  // then every rank runs fn on its own stream and waits for it
  void run_each(int rank, const void* mine, cudaStream_t s, const std::function<void()>& root_prep,
                const std::function<void(const void* const*)>& fn);
};

struct Comm {
  int rank = 0;
  int world = 1;
  ncclComm_t comm = nullptr;
  bool owned = true;        // false: a communicator of a multi-device context (sfm_ctx_create_multi)
  EmuGroup* emu = nullptr;  // ranks sharing a device: every collective through this host group
  EmuGroup* host = nullptr; // ranks of one process (multi-device context): host-side exchanges / barriers
  bool peer = false;        // every device pair of the process has peer access
  int pcg_partition = 0;    // sfm_ba_options.pcg_partition (set by the solver)

  void init(int r, int w, const uint8_t* id_bytes) {
    rank = r;
    world = w;
    if (w <= 1) return;
    SFM_REQUIRE(id_bytes != nullptr, "world > 1 needs an NCCL unique id");
    ncclUniqueId id;
    std::memcpy(&id, id_bytes, sizeof(id));
    SFM_NCCL(ncclCommInitRank(&comm, w, id, r));
  }
  ~Comm() {
    if (comm && owned) ncclCommDestroy(comm);
  }
  bool active() const { return world > 1; }
  void sum(double* d, size_t n, cudaStream_t s) {
    if (world <= 1 || n == 0) return;
    if (emu) return emu->reduce(rank, d, n, s, 0);
    SFM_NCCL(ncclAllReduce(d, d, n, ncclFloat64, ncclSum, comm, s));
  }
  void max_u64(unsigned long long* d, size_t n, cudaStream_t s) {
    if (world <= 1 || n == 0) return;
    if (emu) return emu->reduce(rank, d, n, s, 1);
    SFM_NCCL(ncclAllReduce(d, d, n, ncclUint64, ncclMax, comm, s));
  }
  void min_u64(unsigned long long* d, size_t n, cudaStream_t s) {
    if (world <= 1 || n == 0) return;
    if (emu) return emu->reduce(rank, d, n, s, 2);
    SFM_NCCL(ncclAllReduce(d, d, n, ncclUint64, ncclMin, comm, s));
  }
  void max_i32(int* d, size_t n, cudaStream_t s) {
    if (world <= 1 || n == 0) return;
    if (emu) return emu->reduce(rank, d, n, s, 1);
    SFM_NCCL(ncclAllReduce(d, d, n, ncclInt32, ncclMax, comm, s));
  }
  void allgather_u64(const unsigned long long* send, unsigned long long* recv, size_t n_per_rank,
                     cudaStream_t s) {
    if (world <= 1) return;
    if (emu) return emu->allgather_u64(rank, send, recv, n_per_rank, s);
    SFM_NCCL(ncclAllGather(send, recv, n_per_rank, ncclUint64, comm, s));
  }
  // Reduce-scatter with variable counts: rank r ends with the sum over ranks
  // of d[off[r] .. off[r+1]) (the block rows of S it owns); NCCL: one
  // ncclReduce per range, rooted at its owner, in a group.
  void reduce_ranges(double* d, const std::vector<int64_t>& off, cudaStream_t s) {
    if (world <= 1) return;
    if (emu) return emu->reduce_ranges(rank, d, off, s);
    SFM_NCCL(ncclGroupStart());
    for (int r = 0; r < world; ++r) {
      const size_t n = (size_t)(off[r + 1] - off[r]);
      if (n) SFM_NCCL(ncclReduce(d + off[r], d + off[r], n, ncclFloat64, ncclSum, r, comm, s));
    }
    SFM_NCCL(ncclGroupEnd());
  }
  // Allgather with variable counts: every rank receives rank r's
  // d[off[r] .. off[r+1]) (the PCG solution rows); NCCL: one ncclBroadcast
  // per range from its owner, in a group.
  void allgather_ranges(double* d, const std::vector<int64_t>& off, cudaStream_t s) {
    if (world <= 1) return;
    if (emu) return emu->allgather_ranges(rank, d, off, s);
    SFM_NCCL(ncclGroupStart());
    for (int r = 0; r < world; ++r) {
      const size_t n = (size_t)(off[r + 1] - off[r]);
      if (n) SFM_NCCL(ncclBroadcast(d + off[r], d + off[r], n, ncclFloat64, r, comm, s));
    }
    SFM_NCCL(ncclGroupEnd());
  }
};

}  // namespace sfm
