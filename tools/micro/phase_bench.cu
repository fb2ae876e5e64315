// Microbenchmark: cost of one coloured Gauss-Seidel phase of the K-column
// cluster tail (tail.cu nm_gs) on a small synthetic level, by variant.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o phase_bench phase_bench.cu
// Each phase: every active thread updates one (row, 4-column group): 8 x
// 256-bit gathers of x, fold, divide, 256-bit store; then a cluster barrier.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
namespace cg = cooperative_groups;

constexpr int K = 32, T = K / 4, E = 8;
struct d4 {
  double x, y, z, w;
};
__device__ __forceinline__ d4 ld4(const double* p) {
  d4 r;
  asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void st4(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}
template <int BAR>
__device__ __forceinline__ void bar() {
  if (BAR == 0) cg::this_cluster().sync();
  if (BAR == 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;\n barrier.cluster.wait.aligned;" ::: "memory");
  if (BAR == 2) __syncthreads();
}

// VAR bit 0: divide (else multiply by a precomputed inverse); bit 1: cp.async
// gathers into shared memory (else ld4 into registers)
template <int VAR, int BAR>
__global__ void phases(const int* __restrict__ col, const double* __restrict__ val, const double* __restrict__ diag,
                       const double* __restrict__ b, double* x, int rows_per_colour, int ncol, int iters,
                       long long* out) {
  __shared__ __align__(32) double sg[(VAR & 2) ? 256 * E * 4 / 2 : 8];
  const int gt = (BAR == 2 ? 0 : blockIdx.x) * blockDim.x + threadIdx.x;
  const int slot = gt / T, k0 = (gt % T) * 4;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
    for (int cc = 0; cc < ncol; ++cc) {
      if (slot < rows_per_colour) {
        const int u = cc * rows_per_colour + slot;
        double s[4];
        const d4 bv = ld4(b + (long)u * K + k0);
        s[0] = bv.x, s[1] = bv.y, s[2] = bv.z, s[3] = bv.w;
        int c[E];
        double v[E];
#pragma unroll
        for (int j = 0; j < E; ++j) {
          c[j] = __ldg(col + u * E + j);
          v[j] = __ldg(val + u * E + j);
        }
        if (VAR & 2) {
          double* g = sg + (threadIdx.x % 128) * E * 4;
#pragma unroll
          for (int j = 0; j < E; ++j) {
            const double* src = x + (long)c[j] * K + k0;
            unsigned dst = (unsigned)__cvta_generic_to_shared(g + j * 4);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16), "l"(src + 2) : "memory");
          }
          asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
          for (int j = 0; j < E; ++j) {
            s[0] = s[0] - v[j] * g[j * 4 + 0];
            s[1] = s[1] - v[j] * g[j * 4 + 1];
            s[2] = s[2] - v[j] * g[j * 4 + 2];
            s[3] = s[3] - v[j] * g[j * 4 + 3];
          }
        } else {
          d4 xv[E];
#pragma unroll
          for (int j = 0; j < E; ++j) xv[j] = ld4(x + (long)c[j] * K + k0);
#pragma unroll
          for (int j = 0; j < E; ++j) {
            s[0] = s[0] - v[j] * xv[j].x;
            s[1] = s[1] - v[j] * xv[j].y;
            s[2] = s[2] - v[j] * xv[j].z;
            s[3] = s[3] - v[j] * xv[j].w;
          }
        }
        const double d = __ldg(diag + u);
        if (VAR & 1) st4(x + (long)u * K + k0, s[0] / d, s[1] / d, s[2] / d, s[3] / d);
        else st4(x + (long)u * K + k0, s[0] * d, s[1] * d, s[2] * d, s[3] * d);
      }
      bar<BAR>();
    }
  if (gt == 0) *out = clock64() - t0;
}

template <int VAR, int BAR>
void run(const char* name, int ctas, int* col, double* val, double* diag, double* b, double* x, int rpc, int ncol,
         long long* d_out) {
  const int iters = 200;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(BAR == 2 ? 1 : ctas);
  cfg.blockDim = dim3(256);
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = BAR == 2 ? 1 : ctas;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  cudaFuncSetAttribute(phases<VAR, BAR>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int w = 0; w < 2; ++w) {
    cudaLaunchKernelEx(&cfg, phases<VAR, BAR>, (const int*)col, (const double*)val, (const double*)diag,
                       (const double*)b, x, rpc, ncol, iters, d_out);
  }
  cudaError_t e = cudaDeviceSynchronize();
  long long cyc = 0;
  cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
  printf("%-34s ctas %2d rows/colour %4d: %7.0f cycles/phase %s\n", name, BAR == 2 ? 1 : ctas, rpc,
         (double)cyc / (iters * ncol), e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  const int ncol = 12;
  for (int rpc : {28, 256}) {
    const int n = rpc * ncol;
    std::vector<int> col(n * E);
    std::vector<double> val(n * E, -0.1), diag(n, 1.0), bb((size_t)n * K, 1.0);
    srand(1);
    for (int i = 0; i < n * E; ++i) col[i] = rand() % n;
    int* dc;
    double *dv, *dd, *db, *dx;
    long long* dout;
    cudaMalloc(&dc, n * E * 4);
    cudaMalloc(&dv, n * E * 8);
    cudaMalloc(&dd, n * 8);
    cudaMalloc(&db, (size_t)n * K * 8);
    cudaMalloc(&dx, (size_t)n * K * 8);
    cudaMalloc(&dout, 8);
    cudaMemcpy(dc, col.data(), n * E * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dv, val.data(), n * E * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dd, diag.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(db, bb.data(), (size_t)n * K * 8, cudaMemcpyHostToDevice);
    cudaMemset(dx, 0, (size_t)n * K * 8);
    run<1, 0>("div, ld4, cg cluster sync", 16, dc, dv, dd, db, dx, rpc, ncol, dout);
    run<0, 0>("mul, ld4, cg cluster sync", 16, dc, dv, dd, db, dx, rpc, ncol, dout);
    run<3, 0>("div, cp.async, cg cluster sync", 16, dc, dv, dd, db, dx, rpc, ncol, dout);
    run<1, 1>("div, ld4, relaxed cluster barrier", 16, dc, dv, dd, db, dx, rpc, ncol, dout);
    run<1, 0>("div, ld4, cg cluster sync", 8, dc, dv, dd, db, dx, rpc, ncol, dout);
    run<1, 0>("div, ld4, cg cluster sync", 2, dc, dv, dd, db, dx, rpc, ncol, dout);
    run<1, 2>("div, ld4, one CTA __syncthreads", 1, dc, dv, dd, db, dx, rpc, ncol, dout);
    run<3, 2>("div, cp.async, one CTA", 1, dc, dv, dd, db, dx, rpc, ncol, dout);
    cudaFree(dc);
    cudaFree(dv);
    cudaFree(dd);
    cudaFree(db);
    cudaFree(dx);
    cudaFree(dout);
  }
  return 0;
}
