// batch.cu -- THROUGHPUT-mode kernels over a node-major block of K
// right-hand sides (see batch.cuh). Each (row, column) pair is one thread of
// a K-lane group: the row's entries are loaded once per group (same address
// in every lane: one transaction), the x gathers of the K columns are one
// coalesced K*8-byte segment, and lane k folds its column in entry order.
#include <algorithm>
#include <vector>

#include "batch.cuh"

namespace lamgb {

namespace {

constexpr int kBT = 256;  // threads per block of the batched kernels

inline int bblocks(int64_t threads) { return (int)std::max<int64_t>(1, (threads + kBT - 1) / kBT); }

// V = 4 columns per thread (two 16-byte loads per gather), K/V threads per
// row: the row's entries are loaded once per K/V threads instead of once per
// lane, so the instruction count per row drops ~V-fold; each column is still
// folded in entry order (same arithmetic as one thread per column).
constexpr int kV = 4;
template <int K, bool SUB>
__device__ __forceinline__ void fold4(double (&s)[kV], const int32_t* __restrict__ col,
                                      const double* __restrict__ val, const double* X, int64_t b, int64_t e, int k0) {
  constexpr int U = 8;  // a 7-point row in one round: every gather in flight together
  for (int64_t e0 = b; e0 < e; e0 += U) {
    int32_t c[U];
    double v[U];
    double2 x01[U], x23[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const bool ok = e0 + j < e;
      c[j] = ok ? __ldg(col + e0 + j) : 0;
      v[j] = ok ? __ldg(val + e0 + j) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const double2* px = reinterpret_cast<const double2*>(X + (int64_t)c[j] * K + k0);
      const bool ok = e0 + j < e;
      x01[j] = ok ? px[0] : make_double2(0.0, 0.0);
      x23[j] = ok ? px[1] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (e0 + j < e) {
        if (SUB) {
          s[0] = s[0] - v[j] * x01[j].x;
          s[1] = s[1] - v[j] * x01[j].y;
          s[2] = s[2] - v[j] * x23[j].x;
          s[3] = s[3] - v[j] * x23[j].y;
        } else {
          s[0] = s[0] + v[j] * x01[j].x;
          s[1] = s[1] + v[j] * x01[j].y;
          s[2] = s[2] + v[j] * x23[j].x;
          s[3] = s[3] + v[j] * x23[j].y;
        }
      }
  }
}

// one colour of the permuted operator; heavy rows go to bgs_heavy_kernel
template <int K>
__global__ void __launch_bounds__(kBT) bgs_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                  const double* __restrict__ val, const double* __restrict__ diag,
                                                  const int32_t* __restrict__ row_ids, int32_t i0, int32_t i1,
                                                  const double* __restrict__ B, double* X, const int32_t* done) {
  constexpr int T = K / kV;  // threads per row
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t i = i0 + t / T;
  const int k0 = (int)(t % T) * kV;
  if (i >= i1) return;
  const int64_t b = __ldg(rp + i), e = __ldg(rp + i + 1);
  if (e - b > kHeavyRow) return;
  const int32_t u = __ldg(row_ids + i);
  const double2* pb = reinterpret_cast<const double2*>(B + (int64_t)u * K + k0);
  const double2 b01 = pb[0], b23 = pb[1];
  double s[kV] = {b01.x, b01.y, b23.x, b23.y};
  fold4<K, true>(s, col, val, X, b, e, k0);
  const double d = __ldg(diag + i);
  double* px = X + (int64_t)u * K + k0;
  if (done) {
#pragma unroll
    for (int q = 0; q < kV; ++q)
      if (!done[k0 + q]) px[q] = s[q] / d;
  } else {
    reinterpret_cast<double2*>(px)[0] = make_double2(s[0] / d, s[1] / d);
    reinterpret_cast<double2*>(px)[1] = make_double2(s[2] / d, s[3] / d);
  }
}

// heavy (hub) row: 8 strided slices per column (independent of K, so a
// column's sum is the same in every batch), slice partials folded in order
constexpr int kHS = 8;
template <int K>
__device__ __forceinline__ double heavy_dot(const int32_t* __restrict__ col, const double* __restrict__ val,
                                            const double* X, int64_t b, int64_t e) {
  __shared__ double sh[kHS * 32];
  for (int pr = threadIdx.x; pr < kHS * K; pr += blockDim.x) {
    const int sl = pr / K, k = pr % K;
    double p = 0.0;
    for (int64_t j = b + sl; j < e; j += kHS) p += __ldg(val + j) * X[(int64_t)__ldg(col + j) * K + k];
    sh[sl * K + k] = p;
  }
  __syncthreads();
  double t = 0.0;
  if ((int)threadIdx.x < K)
    for (int q = 0; q < kHS; ++q) t += sh[q * K + threadIdx.x];
  return t;  // valid in threads [0, K)
}

template <int K>
__global__ void __launch_bounds__(kBT) bgs_heavy_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                        const double* __restrict__ val, const double* __restrict__ diag,
                                                        const int32_t* __restrict__ row_ids,
                                                        const int32_t* __restrict__ heavy, const double* __restrict__ B,
                                                        double* X, const int32_t* done) {
  const int32_t i = heavy[blockIdx.x];
  const double dot = heavy_dot<K>(col, val, X, rp[i], rp[i + 1]);
  const int k = threadIdx.x;
  if (k < K && !(done && done[k])) {
    const int32_t u = row_ids[i];
    X[(int64_t)u * K + k] = (B[(int64_t)u * K + k] - dot) / diag[i];
  }
}

template <int K>
__global__ void __launch_bounds__(kBT) bres_kernel(CSRv a, const double* __restrict__ B, const double* __restrict__ X,
                                                   double* __restrict__ R, bool skip_heavy) {
  constexpr int T = K / kV;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t u = t / T;
  const int k0 = (int)(t % T) * kV;
  if (u >= a.n) return;
  const int64_t b = __ldg(a.rp + u), e = __ldg(a.rp + u + 1);
  if (skip_heavy && e - b > kHeavyRow) return;
  const double d = __ldg(a.diag + u);
  const double2* pxu = reinterpret_cast<const double2*>(X + u * K + k0);
  const double2 x01 = pxu[0], x23 = pxu[1];
  double s[kV] = {d * x01.x, d * x01.y, d * x23.x, d * x23.y};
  fold4<K, false>(s, a.col, a.val, X, b, e, k0);
  const double2* pb = reinterpret_cast<const double2*>(B + u * K + k0);
  const double2 b01 = pb[0], b23 = pb[1];
  double2* pr = reinterpret_cast<double2*>(R + u * K + k0);
  pr[0] = make_double2(b01.x - s[0], b01.y - s[1]);
  pr[1] = make_double2(b23.x - s[2], b23.y - s[3]);
}

template <int K>
__global__ void __launch_bounds__(kBT) bres_heavy_kernel(CSRv a, const int32_t* __restrict__ heavy,
                                                         const double* __restrict__ B, const double* X, double* R) {
  const int32_t u = heavy[blockIdx.x];
  const double dot = heavy_dot<K>(a.col, a.val, X, a.rp[u], a.rp[u + 1]);
  const int k = threadIdx.x;
  if (k < K) R[(int64_t)u * K + k] = B[(int64_t)u * K + k] - (a.diag[u] * X[(int64_t)u * K + k] + dot);
}

template <int K>
__global__ void brestrict_kernel(int32_t cn, const int64_t* __restrict__ mem_ptr, const int32_t* __restrict__ mem,
                                 const double* __restrict__ R, double mu, double* __restrict__ Bc,
                                 double* __restrict__ Xc) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t g = t / K;
  const int k = (int)(t % K);
  if (g >= cn) return;
  double s = 0.0;
  for (int64_t j = mem_ptr[g]; j < mem_ptr[g + 1]; ++j) s = s + R[(int64_t)mem[j] * K + k];
  Bc[g * K + k] = mu != 1.0 ? s * mu : s;
  Xc[g * K + k] = 0.0;
}

template <int K>
__global__ void binterp_kernel(int32_t n, const int32_t* __restrict__ agg, const double* __restrict__ Xc,
                               double* __restrict__ X) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t u = t / K;
  const int k = (int)(t % K);
  if (u < n) X[t] = X[t] + Xc[(int64_t)agg[u] * K + k];
}

template <int K>
__global__ void bcoarsen_kernel(StageV s, const double* __restrict__ B, double* __restrict__ Bc) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t q = t / K;
  const int k = (int)(t % K);
  if (q >= s.coarse_n) return;
  double v = B[(int64_t)s.poc[q] * K + k];
  for (int64_t j = s.t_ptr[q]; j < s.t_ptr[q + 1]; ++j) {
    const int64_t p = s.t_p[j];
    const int32_t i = s.f_of_p[p];
    v = v - s.f_val[p] * (B[(int64_t)s.f_nodes[i] * K + k] / s.f_diag[i]);
  }
  Bc[t] = v;
}

template <int K>
__global__ void binject_kernel(StageV s, const double* __restrict__ X, double* __restrict__ Xc) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t q = t / K;
  if (q < s.coarse_n) Xc[t] = X[(int64_t)s.poc[q] * K + (t % K)];
}

template <int K>
__global__ void bscatter_kernel(StageV s, const double* __restrict__ Xc, double* __restrict__ X) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t q = t / K;
  if (q < s.coarse_n) X[(int64_t)s.poc[q] * K + (t % K)] = Xc[t];
}

template <int K>
__global__ void bbacksub_f_kernel(StageV s, const double* __restrict__ B, double* X) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t i = t / K;
  const int k = (int)(t % K);
  if (i >= s.nf) return;
  const int32_t f = s.f_nodes[i];
  double sum = B[(int64_t)f * K + k];
  for (int64_t p = s.f_ptr[i]; p < s.f_ptr[i + 1]; ++p) sum = sum - s.f_val[p] * X[(int64_t)s.f_nbr[p] * K + k];
  X[(int64_t)f * K + k] = sum / s.f_diag[i];
}

// X = Minv[:n,:n] B per component (throughput inverse)
template <int K>
__global__ void bdirect_kernel(const int32_t* comp_start, int32_t ncomp, const int32_t* nodes,
                               const int64_t* inv_off, const double* inv, bool whole, const double* B, double* X) {
  for (int32_t ci = 0; ci < ncomp; ++ci) {
    const int32_t s0 = comp_start[ci], cn = comp_start[ci + 1] - s0;
    const double* Mi = inv + inv_off[ci];
    for (int64_t t = threadIdx.x; t < (int64_t)cn * K; t += blockDim.x) {
      const int32_t i = (int32_t)(t / K);
      const int k = (int)(t % K);
      double s = 0.0;
      for (int32_t j = 0; j < cn; ++j) s += Mi[(int64_t)i * cn + j] * B[(int64_t)(whole ? j : nodes[s0 + j]) * K + k];
      X[(int64_t)(whole ? i : nodes[s0 + i]) * K + k] = s;
    }
    __syncthreads();
  }
}

// per-column sums in an order that does not depend on K: chunk p of R rows
// is folded sequentially by one thread per column (coalesced across the K
// lanes), then each column's P chunk sums by one block: 256 sequential
// strips and a fixed tree. A column's result is the same in any batch.
template <int K, bool SQ>
__global__ void __launch_bounds__(kBT) bcolchunk_kernel(const double* __restrict__ X, int64_t n, int64_t R, int P,
                                                        double* part) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t p = t / K;
  const int k = (int)(t % K);
  if (p >= P) return;
  const int64_t u1 = (p + 1) * R < n ? (p + 1) * R : n;
  double s = 0.0;
  for (int64_t u = p * R; u < u1; ++u) {
    const double v = X[u * K + k];
    s += SQ ? v * v : v;
  }
  part[(int64_t)k * P + p] = s;
}
__global__ void __launch_bounds__(kBT) bcolfinal_kernel(const double* part, int P, double* out) {
  __shared__ double sh[kBT];
  const double* q = part + (int64_t)blockIdx.x * P;
  double s = 0.0;
  for (int i = threadIdx.x; i < P; i += kBT) s += q[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = kBT / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = sh[0];
}

template <int K>
__global__ void bsubmean_kernel(double* X, int64_t n, const double* sums, const int32_t* done) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n * K && !(done && done[t % K])) X[t] = X[t] - sums[t % K] / (double)n;
}

// per-column max |x| (exact: max is order-free); one atomic per column per block
__global__ void bcolabsmax_kernel(const double* X, int64_t n, int K, unsigned long long* out) {
  __shared__ double sh[kBT];
  double m = 0.0;  // blockDim.x and the grid stride are multiples of K: fixed column per thread
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * K; t += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs(X[t]));
  sh[threadIdx.x] = m;
  __syncthreads();
  if ((int)threadIdx.x < K) {
    for (int j = threadIdx.x + K; j < kBT; j += K) m = fmax(m, sh[j]);
    atomicMax(out + threadIdx.x, (unsigned long long)__double_as_longlong(m));
  }
}

__global__ void to_node_major_kernel(const double* __restrict__ src, int64_t n, int nrhs, int K, double* dst) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n * K) return;
  const int64_t u = t / K;
  const int k = (int)(t % K);
  dst[t] = k < nrhs ? src[(int64_t)k * n + u] : 0.0;
}
__global__ void column_out_kernel(const double* __restrict__ X, int64_t n, int K, int k, const double* sums,
                                  double* dst) {
  const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u < n) dst[u] = sums ? X[u * K + k] - sums[k] / (double)n : X[u * K + k];
}

template <class F>
void dispatch_k(int K, F&& f) {
  switch (K) {
    case 4: f(std::integral_constant<int, 4>{}); break;
    case 8: f(std::integral_constant<int, 8>{}); break;
    case 16: f(std::integral_constant<int, 16>{}); break;
    case 32: f(std::integral_constant<int, 32>{}); break;
    default: throw LamgError(LAMG_E_ARGUMENT, "batch width must be 4, 8, 16 or 32");
  }
}

}  // namespace

void bgs_colored(Ctx& c, const DColor& cl, int32_t n, const double* B, double* X, int sweeps, int K,
                 const int32_t* done) {
  if (n == 0 || sweeps <= 0) return;
  dispatch_k(K, [&](auto kc) {
    constexpr int KK = decltype(kc)::value;
    for (int sw = 0; sw < sweeps; ++sw)
      for (int32_t cc = 0; cc < cl.ncolors; ++cc) {
        const int32_t i0 = cl.cptr_h[cc], i1 = cl.cptr_h[cc + 1];
        if (i1 <= i0) continue;
        const int32_t nh = cl.hptr_h.empty() ? 0 : cl.hptr_h[cc + 1] - cl.hptr_h[cc];
        if (nh)
          count_launch(), bgs_heavy_kernel<KK><<<nh, kBT, 0, c.s>>>(cl.rp.p, cl.col.p, cl.val.p, cl.diag.p,
                                                                   cl.row_ids.p, cl.heavy.p + cl.hptr_h[cc], B, X,
                                                                   done);
        count_launch(), bgs_kernel<KK><<<bblocks((int64_t)(i1 - i0) * (KK / kV)), kBT, 0, c.s>>>(
            cl.rp.p, cl.col.p, cl.val.p, cl.diag.p, cl.row_ids.p, i0, i1, B, X, done);
      }
  });
  CK_LAUNCH();
}

void bresidual(Ctx& c, const CSRv& a, const DColor* cl, const double* B, const double* X, double* R, int K) {
  if (a.n == 0) return;
  const int32_t nh = cl ? cl->nheavy_nat : 0;
  dispatch_k(K, [&](auto kc) {
    constexpr int KK = decltype(kc)::value;
    count_launch(), bres_kernel<KK><<<bblocks((int64_t)a.n * (KK / kV)), kBT, 0, c.s>>>(a, B, X, R, nh > 0);
    if (nh) count_launch(), bres_heavy_kernel<KK><<<nh, kBT, 0, c.s>>>(a, cl->heavy_nat.p, B, X, R);
  });
  CK_LAUNCH();
}

void brestrict(Ctx& c, int32_t coarse_n, const int64_t* mem_ptr, const int32_t* mem, const double* R, double mu,
               double* Bc, double* Xc, int K) {
  if (coarse_n == 0) return;
  dispatch_k(K, [&](auto kc) {
    constexpr int KK = decltype(kc)::value;
    count_launch(), brestrict_kernel<KK><<<bblocks((int64_t)coarse_n * KK), kBT, 0, c.s>>>(coarse_n, mem_ptr, mem, R,
                                                                                         mu, Bc, Xc);
  });
  CK_LAUNCH();
}

void binterpolate(Ctx& c, int32_t fine_n, const int32_t* agg, const double* Xc, double* X, int K) {
  if (fine_n == 0) return;
  dispatch_k(K, [&](auto kc) {
    constexpr int KK = decltype(kc)::value;
    count_launch(), binterp_kernel<KK><<<bblocks((int64_t)fine_n * KK), kBT, 0, c.s>>>(fine_n, agg, Xc, X);
  });
  CK_LAUNCH();
}

void bcoarsen_rhs(Ctx& c, const StageV& s, const double* B, double* Bc, int K) {
  if (s.coarse_n == 0) return;
  dispatch_k(K, [&](auto kc) {
    constexpr int KK = decltype(kc)::value;
    count_launch(), bcoarsen_kernel<KK><<<bblocks((int64_t)s.coarse_n * KK), kBT, 0, c.s>>>(s, B, Bc);
  });
  CK_LAUNCH();
}

void binject(Ctx& c, const StageV& s, const double* X, double* Xc, int K) {
  if (s.coarse_n == 0) return;
  dispatch_k(K, [&](auto kc) {
    constexpr int KK = decltype(kc)::value;
    count_launch(), binject_kernel<KK><<<bblocks((int64_t)s.coarse_n * KK), kBT, 0, c.s>>>(s, X, Xc);
  });
  CK_LAUNCH();
}

void bbacksub(Ctx& c, const StageV& s, const double* Xc, const double* B, double* X, int K) {
  dispatch_k(K, [&](auto kc) {
    constexpr int KK = decltype(kc)::value;
    if (s.coarse_n) count_launch(), bscatter_kernel<KK><<<bblocks((int64_t)s.coarse_n * KK), kBT, 0, c.s>>>(s, Xc, X);
    if (s.nf) count_launch(), bbacksub_f_kernel<KK><<<bblocks((int64_t)s.nf * KK), kBT, 0, c.s>>>(s, B, X);
  });
  CK_LAUNCH();
}

void bdirect(Ctx& c, const DDirect& d, const double* B, double* X, int K) {
  if (d.inv.n == 0) throw LamgError(LAMG_E_ERROR, "batched direct solve needs the throughput inverse");
  dispatch_k(K, [&](auto kc) {
    constexpr int KK = decltype(kc)::value;
    count_launch(), bdirect_kernel<KK><<<1, 1024, 0, c.s>>>(d.comp_start.p, d.ncomp, d.nodes.p, d.inv_off.p, d.inv.p,
                                                           d.ncomp == 1, B, X);
  });
  CK_LAUNCH();
  c.work += (double)d.m;
}

void bcolsum(Ctx& c, const double* X, int64_t n, int K, bool sq, double* out) {
  const int64_t R = std::max<int64_t>(1, (n + kColChunks - 1) / kColChunks);
  const int P = (int)std::max<int64_t>(1, (n + R - 1) / R);
  double* part = c.dbpart;  // [K][P], P <= kColChunks
  dispatch_k(K, [&](auto kc) {
    constexpr int KK = decltype(kc)::value;
    if (sq) count_launch(), bcolchunk_kernel<KK, true><<<bblocks((int64_t)P * KK), kBT, 0, c.s>>>(X, n, R, P, part);
    else count_launch(), bcolchunk_kernel<KK, false><<<bblocks((int64_t)P * KK), kBT, 0, c.s>>>(X, n, R, P, part);
  });
  count_launch(), bcolfinal_kernel<<<K, kBT, 0, c.s>>>(part, P, out);
  CK_LAUNCH();
}

void bsub_mean(Ctx& c, double* X, int64_t n, int K, const double* sums, const int32_t* done) {
  dispatch_k(K, [&](auto kc) {
    constexpr int KK = decltype(kc)::value;
    count_launch(), bsubmean_kernel<KK><<<bblocks(n * KK), kBT, 0, c.s>>>(X, n, sums, done);
  });
  CK_LAUNCH();
}

void bcolabsmax(Ctx& c, const double* X, int64_t n, int K, unsigned long long* out) {
  CK(cudaMemsetAsync(out, 0, sizeof(unsigned long long) * K, c.s));
  count_launch(), bcolabsmax_kernel<<<std::min(bblocks(n * K), 1024), kBT, 0, c.s>>>(X, n, K, out);
  CK_LAUNCH();
}

void to_node_major(Ctx& c, const double* src, int64_t n, int nrhs, int K, double* dst) {
  count_launch(), to_node_major_kernel<<<bblocks(n * K), kBT, 0, c.s>>>(src, n, nrhs, K, dst);
  CK_LAUNCH();
}

void column_out(Ctx& c, const double* X, int64_t n, int K, int k, double* dst, const double* sums) {
  count_launch(), column_out_kernel<<<bblocks(n), kBT, 0, c.s>>>(X, n, K, k, sums, dst);
  CK_LAUNCH();
}

void brelax(Ctx& c, const CSRv& a, const DColor& cl, const double* B, double* X, double* R, int K,
            std::vector<int>& sweeps) {
  sweeps.assign(K, 0);
  int32_t* done = c.dbdone;
  double* nrm = c.dbscal;          // [K]
  double* sums = c.dbscal + 64;    // [K]
  std::vector<double> r0(K), rn(K);
  std::vector<int32_t> hdone(K, 0);
  bresidual(c, a, &cl, B, X, R, K);
  c.work += (double)a.m;
  bcolsum(c, R, a.n, K, true, nrm);
  CK(cudaMemcpyAsync(rn.data(), nrm, K * sizeof(double), cudaMemcpyDeviceToHost, c.s));
  c.sync();
  int active = 0;
  for (int k = 0; k < K; ++k) {
    r0[k] = std::sqrt(rn[k]);
    hdone[k] = r0[k] == 0.0;
    active += !hdone[k];
  }
  CK(cudaMemcpyAsync(done, hdone.data(), K * sizeof(int32_t), cudaMemcpyHostToDevice, c.s));
  for (int sweep = 0; sweep < 400 && active; ++sweep) {
    bgs_colored(c, cl, a.n, B, X, 1, K, done);
    c.work += (double)a.m;
    bcolsum(c, X, a.n, K, false, sums);
    bsub_mean(c, X, a.n, K, sums, done);
    bresidual(c, a, &cl, B, X, R, K);
    c.work += (double)a.m;
    bcolsum(c, R, a.n, K, true, nrm);
    CK(cudaMemcpyAsync(rn.data(), nrm, K * sizeof(double), cudaMemcpyDeviceToHost, c.s));
    c.sync();
    for (int k = 0; k < K; ++k) {
      if (hdone[k]) continue;
      ++sweeps[k];
      if (std::sqrt(rn[k]) <= 1e-12 * r0[k]) {
        hdone[k] = 1;
        --active;
      }
    }
    CK(cudaMemcpyAsync(done, hdone.data(), K * sizeof(int32_t), cudaMemcpyHostToDevice, c.s));
  }
  c.sync();
}

}  // namespace lamgb
