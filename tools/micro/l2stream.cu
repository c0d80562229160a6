// Microbenchmark: how fast can 148 CTAs (one per SM) re-stream an
// L2-resident 82.6 MB matrix (the PCG's S at config 3), each CTA its own
// contiguous ~560 KB slice, per pass?  (a) LDG.128 loads, 8-deep unroll;
// (b) TMA 1-D bulk copies (cp.async.bulk) into a 4-stage shared-memory ring
// with mbarriers, consumers summing from shared memory.
#include <cuda.h>
#include <cstdio>
#include <cstdint>

__global__ void __launch_bounds__(1024, 1) k_ldg(const double2* __restrict__ S, int64_t per_cta, int passes, double* out) {
  const double2* p = S + (int64_t)blockIdx.x * per_cta;
  double acc = 0;
  for (int it = 0; it < passes; ++it) {
    for (int64_t i = threadIdx.x; i < per_cta; i += 8 * 1024) {
      double2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = (i + u * 1024 < per_cta) ? __ldg(p + i + u * 1024) : make_double2(0, 0);
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += v[u].x * v[u].y;
    }
    __syncthreads();
  }
  if (acc == 12345.0) out[0] = acc;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n LAB_WAIT:\n"
      " mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n"
      " @!p bra LAB_WAIT;\n}\n" :: "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(parity));
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"((unsigned)__cvta_generic_to_shared(smem)), "l"(gmem), "r"(bytes),
                  "r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}

constexpr int kStages = 4;
constexpr int kStageBytes = 48 * 1024;
__global__ void __launch_bounds__(1024, 1) k_tma(const char* __restrict__ S, int64_t bytes_per_cta, int passes, double* out) {
  extern __shared__ __align__(128) char ring[];
  __shared__ uint64_t full[kStages];
  const char* base = S + (int64_t)blockIdx.x * bytes_per_cta;
  const int nst = (int)((bytes_per_cta + kStageBytes - 1) / kStageBytes);
  if (threadIdx.x == 0) for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
  __syncthreads();
  const int total = nst * passes;
  auto issue = [&](int k) {
    const int s = k % kStages, c = k % nst;
    const int64_t off = (int64_t)c * kStageBytes;
    const unsigned b = (unsigned)(int64_t)(kStageBytes < bytes_per_cta - off ? kStageBytes : bytes_per_cta - off);
    mbar_expect_tx(&full[s], b);
    bulk_g2s(ring + s * kStageBytes, base + off, b, &full[s]);
  };
  if (threadIdx.x == 0) for (int k = 0; k < kStages && k < total; ++k) issue(k);
  double acc = 0;
  for (int k = 0; k < total; ++k) {
    const int s = k % kStages;
    mbar_wait(&full[s], (k / kStages) & 1);
    const int c = k % nst;
    const int64_t off = (int64_t)c * kStageBytes;
    const int b = (int)(int64_t)(kStageBytes < bytes_per_cta - off ? kStageBytes : bytes_per_cta - off);
    const double2* v = reinterpret_cast<const double2*>(ring + s * kStageBytes);
    for (int i = threadIdx.x; i < b / 16; i += 1024) acc += v[i].x * v[i].y;
    __syncthreads();
    if (threadIdx.x == 0 && k + kStages < total) issue(k + kStages);
  }
  if (acc == 12345.0) out[0] = acc;
}

int main() {
  int nsm = 0; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int64_t total = 82600000;  // bytes of S at config 3
  const int64_t per = (total / nsm) / 256 * 256;
  char* S; cudaMalloc(&S, per * nsm); cudaMemset(S, 0, per * nsm);
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int passes = 200;
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    k_ldg<<<nsm, 1024>>>((const double2*)S, per / 16, passes, out);
    cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    if (rep) printf("LDG.128 x8 unroll : %.2f us/pass  %.2f TB/s\n", 1000 * ms / passes, per * nsm * passes / (ms * 1e-3) / 1e12);
    const int smem = kStages * kStageBytes;
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEventRecord(a);
    k_tma<<<nsm, 1024, smem>>>(S, per, passes, out);
    cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    if (rep) printf("TMA bulk 4x48KB   : %.2f us/pass  %.2f TB/s\n", 1000 * ms / passes, per * nsm * passes / (ms * 1e-3) / 1e12);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
