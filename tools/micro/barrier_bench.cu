// Microbenchmark: cost of a grid-wide barrier on B200 (cooperative groups vs
// a hand-rolled generation barrier), for the coarse-tail kernel design.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void cg_bar(int iters, long long* out) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cg::this_grid().sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}

__device__ unsigned g_count = 0;
__device__ volatile unsigned g_gen = 0;
__device__ __forceinline__ void my_bar(unsigned nb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned g = g_gen;
    __threadfence();
    if (atomicAdd(&g_count, 1u) == nb - 1) {
      g_count = 0;
      __threadfence();
      g_gen = g + 1;
    } else {
      while (g_gen == g) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}
__global__ void my_barrier(int iters, long long* out) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) my_bar(gridDim.x);
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}
__global__ void cta_bar(int iters, long long* out) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  if (threadIdx.x == 0) *out = clock64() - t0;
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  long long h;
  int iters = 2000;
  for (int nb : {1, 16, 32, 64, 148}) {
    void* args[] = {&iters, &d};
    cudaLaunchCooperativeKernel((void*)cg_bar, nb, 512, args, 0, 0);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    double cg_c = (double)h / iters;
    cudaLaunchCooperativeKernel((void*)my_barrier, nb, 512, args, 0, 0);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("blocks %3d: cg grid.sync %8.0f cycles, custom barrier %8.0f cycles (%s)\n", nb, cg_c,
           (double)h / iters, cudaGetErrorString(cudaGetLastError()));
  }
  cta_bar<<<1, 512>>>(iters, d);
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("__syncthreads (512 thr): %.0f cycles\n", (double)h / iters);
  return 0;
}
