// comm.cuh -- rank-to-rank reductions for point-sharded BA.
//
// One process per GPU.  world == 1 makes every call a no-op; otherwise the
// camera-indexed sums (U, g_c, S, b_S) and the scalars (cost, step norm,
// depth flag) are all-reduced with NCCL over NVLink on the context stream.
// NCCL's ring/tree results are identical on every rank, so the replicated
// PCG on S takes identical decisions everywhere.
#pragma once
#include <nccl.h>

#include "common.cuh"

namespace sfm {

#define SFM_NCCL(call)                                                              \
  do {                                                                              \
    ncclResult_t r_ = (call);                                                       \
    if (r_ != ncclSuccess)                                                          \
      throw ::sfm::SfmError(SFM_E_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
  } while (0)

struct Comm {
  int rank = 0;
  int world = 1;
  ncclComm_t comm = nullptr;

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
    if (comm) ncclCommDestroy(comm);
  }
  bool active() const { return world > 1; }
  void sum(double* d, size_t n, cudaStream_t s) {
    if (world <= 1 || n == 0) return;
    SFM_NCCL(ncclAllReduce(d, d, n, ncclFloat64, ncclSum, comm, s));
  }
  void max_u64(unsigned long long* d, size_t n, cudaStream_t s) {
    if (world <= 1 || n == 0) return;
    SFM_NCCL(ncclAllReduce(d, d, n, ncclUint64, ncclMax, comm, s));
  }
  void min_u64(unsigned long long* d, size_t n, cudaStream_t s) {
    if (world <= 1 || n == 0) return;
    SFM_NCCL(ncclAllReduce(d, d, n, ncclUint64, ncclMin, comm, s));
  }
  void max_i32(int* d, size_t n, cudaStream_t s) {
    if (world <= 1 || n == 0) return;
    SFM_NCCL(ncclAllReduce(d, d, n, ncclInt32, ncclMax, comm, s));
  }
  void allgather_u64(const unsigned long long* send, unsigned long long* recv, size_t n_per_rank,
                     cudaStream_t s) {
    if (world <= 1) return;
    SFM_NCCL(ncclAllGather(send, recv, n_per_rank, ncclUint64, comm, s));
  }
};

}  // namespace sfm
