// Microbenchmark: fp64 peak of the B200 for the compute-leaning Schur
// kernels' roofline -- DFMA (vector pipe) and DMMA.8x8x4 (mma.sync f64,
// the tensor path k_offdiag_blocks / k_cam_blocks use).  Many independent
// accumulator chains per thread, all SMs, timed with CUDA events.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64peak.cu -o fp64peak
#include <cstdio>

constexpr int kChains = 8;

__global__ void k_dfma(int iters, double* out) {
  double a[kChains], b = 1.0000001, c = 1e-9;
#pragma unroll
  for (int k = 0; k < kChains; ++k) a[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < kChains; ++k) a[k] = fma(a[k], b, c);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < kChains; ++k) s += a[k];
  if (s == 12345.678) out[0] = s;  // keep the chains live
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void k_dmma(int iters, double* out) {
  double d[kChains][2];
#pragma unroll
  for (int k = 0; k < kChains; ++k) d[k][0] = d[k][1] = 0.0;
  const double a = 1e-3 * (threadIdx.x & 31), b = 1.0 + 1e-4 * (threadIdx.x & 31);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < kChains; ++k) dmma(d[k][0], d[k][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < kChains; ++k) s += d[k][0] + d[k][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000, threads = 256, blocks = nsm * 8;
  for (int rep = 0; rep < 2; ++rep) {
    k_dfma<<<blocks, threads>>>(iters, out);
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * kChains * (double)iters * threads * blocks;
    if (rep) printf("{\"dfma_tflops\": %.2f, ", flops / (ms * 1e-3) / 1e12);
    k_dmma<<<blocks, threads>>>(iters, out);
    cudaEventRecord(e0);
    k_dmma<<<blocks, threads>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    // one m8n8k4 = 8*8*4 FMA per warp
    const double mflops = 2.0 * 256.0 * kChains * (double)iters * (threads / 32) * blocks;
    if (rep) printf("\"dmma_tflops\": %.2f, \"sms\": %d, \"clock_mhz_attr\": %d}\n",
                    mflops / (ms * 1e-3) / 1e12, nsm, clk / 1000);
  }
  return cudaGetLastError() != cudaSuccess;
}
