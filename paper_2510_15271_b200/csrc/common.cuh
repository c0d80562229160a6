// common.cuh -- error plumbing, device buffers, profiling hooks shared by the
// BA / triangulation drivers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/sfm_b200.h"

namespace sfm {

// Error carried from deep inside the driver up to the C-ABI boundary.
struct SfmError : public std::runtime_error {
  int code;
  SfmError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define SFM_CUDA(call)                                                          \
  do {                                                                          \
    cudaError_t e_ = (call);                                                    \
    if (e_ != cudaSuccess) {                                                    \
      int c_ = (e_ == cudaErrorMemoryAllocation) ? SFM_E_OOM : SFM_E_CUDA;     \
      throw ::sfm::SfmError(c_, std::string(#call) + ": " + cudaGetErrorString(e_) + \
                                    " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")"); \
    }                                                                           \
  } while (0)

#define SFM_CHECK_LAUNCH() SFM_CUDA(cudaGetLastError())

#define SFM_REQUIRE(cond, msg)                                                  \
  do {                                                                          \
    if (!(cond)) throw ::sfm::SfmError(SFM_E_INVALID, msg);                    \
  } while (0)

// Stream on which device buffers are allocated and freed (stream-ordered
// allocation from the device's default memory pool, whose release threshold
// is raised at context creation so freed blocks stay cached across calls:
// repeated bundle_adjust / triangulation calls do not pay cudaMalloc).  Set
// by the C-ABI guard to the context stream for the duration of a call.
inline cudaStream_t& alloc_stream() {
  static thread_local cudaStream_t s = nullptr;
  return s;
}

// Owning device buffer (grow-only).
template <typename T>
struct DevBuf {
  T* ptr = nullptr;
  size_t cap = 0;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (ptr) cudaFreeAsync(ptr, alloc_stream());
    ptr = nullptr;
    cap = n = 0;
  }
  T* resize(size_t count) {
    if (count > cap) {
      if (ptr) cudaFreeAsync(ptr, alloc_stream());
      ptr = nullptr;
      size_t bytes = (count ? count : 1) * sizeof(T);
      SFM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ptr), bytes, alloc_stream()));
      cap = count;
    }
    n = count;
    return ptr;
  }
  T* get() const { return ptr; }
  size_t bytes() const { return n * sizeof(T); }
  // `src` / `dst` may be host or device memory (unified addressing): the
  // C-ABI passes host arrays, the device-resident mapping loop device arrays.
  void upload(const T* src, size_t count, cudaStream_t s) {
    resize(count);
    if (count) SFM_CUDA(cudaMemcpyAsync(ptr, src, count * sizeof(T), cudaMemcpyDefault, s));
  }
  void download(T* dst, size_t count, cudaStream_t s) const {
    if (count) SFM_CUDA(cudaMemcpyAsync(dst, ptr, count * sizeof(T), cudaMemcpyDefault, s));
  }
  void zero(cudaStream_t s) {
    if (n) SFM_CUDA(cudaMemsetAsync(ptr, 0, n * sizeof(T), s));
  }
};

// NVTX range for Nsight timelines (setup, linearisation, trials, PCG,
// iterative_map rounds); a no-op unless a tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Per-kernel CUDA-event timing.  Events are recorded on the launching
// stream; resolution happens at flush() after a stream sync.
struct Profiler {
  bool enabled = false;
  struct Entry {
    std::string name;
    int64_t launches = 0;
    double ms = 0.0;
    double bytes = 0.0;
  };
  std::vector<Entry> entries;
  struct Pending {
    int idx;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> pool;
  int64_t launches = 0;  // every kernel launched by the library

  ~Profiler() {
    for (auto& p : pending) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); }
    for (auto e : pool) cudaEventDestroy(e);
  }
  int index(const char* name) {
    for (size_t i = 0; i < entries.size(); ++i)
      if (entries[i].name == name) return (int)i;
    entries.push_back(Entry{name});
    return (int)entries.size() - 1;
  }
  cudaEvent_t take() {
    if (!pool.empty()) { cudaEvent_t e = pool.back(); pool.pop_back(); return e; }
    cudaEvent_t e;
    SFM_CUDA(cudaEventCreate(&e));
    return e;
  }
  // Returns an index into `pending` or -1.
  int begin(const char* name, double bytes, cudaStream_t s) {
    ++launches;
    if (!enabled) return -1;
    int idx = index(name);
    entries[idx].launches += 1;
    entries[idx].bytes += bytes;
    Pending p{idx, take(), take()};
    SFM_CUDA(cudaEventRecord(p.a, s));
    pending.push_back(p);
    return (int)pending.size() - 1;
  }
  void end(int h, cudaStream_t s) {
    if (h < 0) return;
    SFM_CUDA(cudaEventRecord(pending[h].b, s));
  }
  void flush() {
    for (auto& p : pending) {
      float ms = 0.f;
      SFM_CUDA(cudaEventSynchronize(p.b));
      SFM_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
      entries[p.idx].ms += ms;
      pool.push_back(p.a);
      pool.push_back(p.b);
    }
    pending.clear();
  }
  void reset() {
    flush();
    entries.clear();
  }
  // Adds algorithmic bytes known only after a launch (e.g. PCG iterations).
  void add_bytes(const char* name, double bytes) {
    if (!enabled) return;
    entries[index(name)].bytes += bytes;
  }
};

// RAII launch bracket: `PROF(prof, "name", bytes, stream) kernel<<<...>>>(...);`
struct ProfScope {
  Profiler& p;
  int h;
  cudaStream_t s;
  ProfScope(Profiler& prof, const char* name, double bytes, cudaStream_t st)
      : p(prof), h(prof.begin(name, bytes, st)), s(st) {}
  ~ProfScope() noexcept(false) {
    if (std::uncaught_exceptions() > 0) return;
    SFM_CHECK_LAUNCH();
    p.end(h, s);
  }
};

inline unsigned grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace sfm
