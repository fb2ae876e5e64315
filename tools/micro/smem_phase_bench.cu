// Microbenchmark: cost of one coloured Gauss-Seidel colour phase executed by a
// single CTA on a shared-memory-resident coarse level (the tail kernel's
// CTA-0 path). Random graph, n rows, ~deg entries per row, greedy colouring.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

template <int G, int VAR>
__global__ void phases(const int32_t* g_rp, const int32_t* g_c, const double* g_v, const double* g_d,
                       const double* g_b, const int32_t* g_cp, int n, int nnz, int ncol, int reps,
                       long long* out, double* xout) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* s_x = (double*)smem;
  double* s_b = s_x + n;
  double* s_d = s_b + n;
  double* s_v = s_d + n;
  int32_t* s_c = (int32_t*)(s_v + nnz);
  int32_t* s_rp = s_c + nnz;
  int32_t* s_cp = s_rp + n + 1;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    s_x[i] = 0.0; s_b[i] = g_b[i]; s_d[i] = VAR == 1 ? 1.0 / g_d[i] : g_d[i]; s_rp[i] = g_rp[i];
  }
  if (threadIdx.x == 0) s_rp[n] = g_rp[n];
  for (int k = threadIdx.x; k < nnz; k += blockDim.x) { s_c[k] = g_c[k]; s_v[k] = g_v[k]; }
  for (int i = threadIdx.x; i <= ncol; i += blockDim.x) s_cp[i] = g_cp[i];
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r)
    for (int cc = 0; cc < ncol; ++cc) {
      const int i0 = s_cp[cc], i1 = s_cp[cc + 1];
      const int span = ((i1 - i0) * G + 31) / 32 * 32;
      for (int t = threadIdx.x; t < span; t += blockDim.x) {
        const int i = i0 + t / G;
        const bool ok = i < i1;
        const int lane = t & (G - 1);
        double p = 0.0;
        if (ok) {
          const int e = s_rp[i + 1];
          if (VAR == 2) {
            int k = s_rp[i] + lane;
            double pv[4]; int pc[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) { bool o = k + j * G < e; pc[j] = o ? s_c[k + j * G] : 0; pv[j] = o ? s_v[k + j * G] : 0.0; }
#pragma unroll
            for (int j = 0; j < 4; ++j) p += pv[j] * s_x[pc[j]];
            for (k += 4 * G; k < e; k += G) p += s_v[k] * s_x[s_c[k]];
          } else {
            for (int k = s_rp[i] + lane; k < e; k += G) p += s_v[k] * s_x[s_c[k]];
          }
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o, G);
        if (ok && lane == 0) s_x[i] = VAR == 1 ? (s_b[i] - p) * s_d[i] : (s_b[i] - p) / s_d[i];
      }
      __syncthreads();
    }
  long long t1 = clock64();
  if (threadIdx.x == 0) *out = t1 - t0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) xout[i] = s_x[i];
}

int main(int argc, char** argv) {
  int n = argc > 1 ? atoi(argv[1]) : 700, deg = argc > 2 ? atoi(argv[2]) : 14;
  srand(1);
  std::vector<std::vector<int>> adj(n);
  for (int u = 0; u < n; ++u)
    while ((int)adj[u].size() < deg / 2) { int v = rand() % n; if (v != u) { adj[u].push_back(v); adj[v].push_back(u); } }
  std::vector<int> color(n, -1);
  int ncol = 0;
  for (int u = 0; u < n; ++u) { std::vector<bool> used(256, false); for (int v : adj[u]) if (color[v] >= 0) used[color[v]] = true; int c = 0; while (used[c]) ++c; color[u] = c; ncol = std::max(ncol, c + 1); }
  std::vector<int> order(n); for (int i = 0; i < n; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return color[a] < color[b]; });
  std::vector<int> cp(ncol + 1, 0); for (int u = 0; u < n; ++u) cp[color[u] + 1]++; for (int c = 0; c < ncol; ++c) cp[c + 1] += cp[c];
  // rows stored in colour order, columns refer to stored positions
  std::vector<int> pos(n); for (int i = 0; i < n; ++i) pos[order[i]] = i;
  std::vector<int> rp(1, 0), ci; std::vector<double> vv, dd(n), bb(n);
  for (int i = 0; i < n; ++i) { int u = order[i]; for (int v : adj[u]) { ci.push_back(pos[v]); vv.push_back(-1.0); } rp.push_back(ci.size()); dd[i] = adj[u].size() + 0.5; bb[i] = (i % 7) - 3; }
  int nnz = ci.size();
  int32_t *d_rp, *d_c, *d_cp; double *d_v, *d_d, *d_b, *d_x; long long* d_o;
  cudaMalloc(&d_rp, 4 * (n + 1)); cudaMalloc(&d_c, 4 * nnz); cudaMalloc(&d_cp, 4 * (ncol + 1));
  cudaMalloc(&d_v, 8 * nnz); cudaMalloc(&d_d, 8 * n); cudaMalloc(&d_b, 8 * n); cudaMalloc(&d_x, 8 * n); cudaMalloc(&d_o, 8);
  cudaMemcpy(d_rp, rp.data(), 4 * (n + 1), cudaMemcpyHostToDevice); cudaMemcpy(d_c, ci.data(), 4 * nnz, cudaMemcpyHostToDevice);
  cudaMemcpy(d_cp, cp.data(), 4 * (ncol + 1), cudaMemcpyHostToDevice); cudaMemcpy(d_v, vv.data(), 8 * nnz, cudaMemcpyHostToDevice);
  cudaMemcpy(d_d, dd.data(), 8 * n, cudaMemcpyHostToDevice); cudaMemcpy(d_b, bb.data(), 8 * n, cudaMemcpyHostToDevice);
  size_t sm = (size_t)n * 24 + (size_t)nnz * 12 + 4 * (n + 1) + 4 * (ncol + 1) + 64;
  int reps = 200;
  auto run = [&](auto kern, const char* name, int threads) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    kern<<<1, threads, sm>>>(d_rp, d_c, d_v, d_d, d_b, d_cp, n, nnz, ncol, reps, d_o, d_x);
    long long h; cudaMemcpy(&h, d_o, 8, cudaMemcpyDeviceToHost);
    printf("%-22s threads %4d: %7.0f cycles/phase (%s)\n", name, threads, (double)h / (reps * ncol), cudaGetErrorString(cudaGetLastError()));
  };
  printf("n %d nnz %d colours %d smem %zu\n", n, nnz, ncol, sm);
  run(phases<4, 0>, "G4 div", 512); run(phases<4, 1>, "G4 mul-rcp", 512); run(phases<4, 2>, "G4 batched", 512);
  run(phases<8, 0>, "G8 div", 512); run(phases<2, 0>, "G2 div", 512); run(phases<1, 0>, "G1 div", 512);
  run(phases<4, 0>, "G4 div", 256); run(phases<4, 0>, "G4 div", 1024); run(phases<8, 2>, "G8 batched", 1024);
  return 0;
}
