// Microbenchmark: cost of cooperative-groups grid.sync() and of a
// hand-rolled monotonic-counter barrier on the PCG grid shape (one
// 1024-thread CTA per SM).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 gridsync.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int n, double* out) {
  cg::grid_group g = cg::this_grid();
  double acc = 0;
  for (int i = 0; i < n; ++i) { acc += i; g.sync(); }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = acc;
}

__device__ unsigned int g_count;
__global__ void k_mono(int n, double* out) {
  double acc = 0;
  for (int i = 0; i < n; ++i) {
    acc += i;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(&g_count, 1u);
      const unsigned target = (unsigned)(i + 1) * gridDim.x;
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&g_count) : "memory");
      } while ((int)(v - target) < 0);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = acc;
}


// two-level arrival tree: CTAs arrive on one of 8 group counters; the last
// arrival of a group arrives on the top counter; the last of those bumps the
// generation word every CTA spins on (monotonic counts, no resets)
__device__ unsigned int g_grp[8 * 32];  // one counter per 128 B line
__device__ unsigned int g_top;
__device__ unsigned int g_gen;
__global__ void k_tree(int n, double* out) {
  double acc = 0;
  const int G = gridDim.x, g = blockIdx.x & 7;
  const unsigned gsize = (unsigned)((G - g + 7) / 8);  // CTAs with blockIdx % 8 == g
  for (int i = 0; i < n; ++i) {
    acc += i;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      const unsigned old = atomicAdd(&g_grp[g * 32], 1u);
      if (old == (unsigned)(i + 1) * gsize - 1) {
        const unsigned o2 = atomicAdd(&g_top, 1u);
        if (o2 == (unsigned)(i + 1) * 8 - 1) {
          __threadfence();
          atomicExch(&g_gen, (unsigned)(i + 1));
        }
      }
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&g_gen) : "memory");
      } while ((int)(v - (unsigned)(i + 1)) < 0);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = acc;
}

int main() {
  int dev = 0, nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int nt : {256, 512, 1024}) {
    int n = 2000;
    void* args[] = {&n, &out};
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k_cg, nsm, nt, args, 0, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("cg grid.sync   grid=%d x %d: %.3f us/sync\n", nsm, nt, 1000.0 * ms / n);
      unsigned z = 0; cudaMemcpyToSymbol(g_count, &z, 4);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k_mono, nsm, nt, args, 0, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("monotonic ctr  grid=%d x %d: %.3f us/sync\n", nsm, nt, 1000.0 * ms / n);
      {
        unsigned zz[8 * 32] = {0};
        cudaMemcpyToSymbol(g_grp, zz, sizeof(zz)); cudaMemcpyToSymbol(g_top, &z, 4); cudaMemcpyToSymbol(g_gen, &z, 4);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k_tree, nsm, nt, args, 0, 0);
        cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        if (rep) printf("8-group tree   grid=%d x %d: %.3f us/sync\n", nsm, nt, 1000.0 * ms / n);
      }
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
