// batch.cu -- THROUGHPUT-mode kernels over a node-major block of K
// right-hand sides (see batch.cuh). Each (row, column) pair is one thread of
// a K-lane group: the row's entries are loaded once per group (same address
// in every lane: one transaction), the x gathers of the K columns are one
// coalesced K*8-byte segment, and lane k folds its column in entry order.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "batch.cuh"

namespace lamgb {

namespace {

constexpr int kBT = 256;  // threads per block of the batched kernels

inline int bblocks(int64_t threads) { return (int)std::max<int64_t>(1, (threads + kBT - 1) / kBT); }

template <int K, bool SUB>
__device__ __forceinline__ void fold4(double (&s)[kV], const int32_t* __restrict__ col,
                                      const double* __restrict__ val, const double* X, int64_t b, int64_t e, int k0) {
  constexpr int U = 8;  // a 7-point row in one round: every gather in flight together
  for (int64_t e0 = b; e0 < e; e0 += U) {
    int32_t c[U];
    double v[U];
    d4 xv[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const bool ok = e0 + j < e;
      c[j] = ok ? __ldg(col + e0 + j) : 0;
      v[j] = ok ? __ldg(val + e0 + j) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const bool ok = e0 + j < e;
      xv[j] = ok ? ld4(X + (int64_t)c[j] * K + k0) : d4{0.0, 0.0, 0.0, 0.0};
    }
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (e0 + j < e) {
        if (SUB) {
          s[0] = s[0] - v[j] * xv[j].x;
          s[1] = s[1] - v[j] * xv[j].y;
          s[2] = s[2] - v[j] * xv[j].z;
          s[3] = s[3] - v[j] * xv[j].w;
        } else {
          s[0] = s[0] + v[j] * xv[j].x;
          s[1] = s[1] + v[j] * xv[j].y;
          s[2] = s[2] + v[j] * xv[j].z;
          s[3] = s[3] + v[j] * xv[j].w;
        }
      }
  }
}

// one colour of the permuted operator; rows longer than kLongRow go to the long-row kernels
// 6 CTAs/SM (40 registers): the occupancy/in-flight-gathers optimum on the
// cfg2 finest level (per colour: 1 CTA/SM bound -> 101 registers 464 us,
// 6 -> 246 us, 8 -> spills 433 us)
template <int K, int MINB = 6>
__global__ void __launch_bounds__(kBT, MINB) bgs_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                  const double* __restrict__ val, const double* __restrict__ diag,
                                                  const int32_t* __restrict__ row_ids, int32_t i0, int32_t i1,
                                                  const double* __restrict__ B, double* X, const int32_t* done) {
  constexpr int T = K / kV;  // threads per row
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t i = i0 + t / T;
  const int k0 = (int)(t % T) * kV;
  if (i >= i1) return;
  const int64_t b = __ldg(rp + i), e = __ldg(rp + i + 1);
  if (e - b > kLongRow) return;  // bgs_long_kernel / blong_*_kernel
  const int32_t u = __ldg(row_ids + i);
  const d4 bv = ld4(B + (int64_t)u * K + k0);
  double s[kV] = {bv.x, bv.y, bv.z, bv.w};
  fold4<K, true>(s, col, val, X, b, e, k0);
  const double d = __ldg(diag + i);
  double* px = X + (int64_t)u * K + k0;
  if (done) {
#pragma unroll
    for (int q = 0; q < kV; ++q)
      if (!done[k0 + q]) px[q] = s[q] / d;
  } else {
    st4(px, s[0] / d, s[1] / d, s[2] / d, s[3] / d);
  }
}

// The same colour launch with programmatic dependent launch (sm_90+): on the
// coarser host-driven levels a colour is ONE wave of CTAs whose life is three
// dependent round trips (row extent -> entries -> x gathers) after ~2 us of
// launch latency. Launched with cudaLaunchAttributeProgrammaticStreamSerialization
// the grid starts while the previous colour is still running, loads everything
// that no earlier launch writes (row extent, row id, diagonal, the first eight
// entries), waits for the previous grid to complete and flush
// (griddepcontrol.wait), lets the next colour start its own prologue
// (griddepcontrol.launch_dependents) and only then reads b, gathers x, folds
// in entry order (the arithmetic of bgs_kernel) and stores.
template <int K>
__global__ void __launch_bounds__(kBT, 4) bgs_pdl_kernel(const int64_t* __restrict__ rp,
                                                         const int32_t* __restrict__ col,
                                                         const double* __restrict__ val,
                                                         const double* __restrict__ diag,
                                                         const int32_t* __restrict__ row_ids, int32_t i0, int32_t i1,
                                                         const double* B, double* X, const int32_t* done) {
  constexpr int T = K / kV;
  constexpr int U = 8;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t i = i0 + t / T;
  const int k0 = (int)(t % T) * kV;
  const bool act = i < i1;
  int64_t b = 0, e = 0;
  int32_t u = 0;
  double d = 1.0;
  int32_t c[U];
  double v[U];
  if (act) {
    b = __ldg(rp + i);
    e = __ldg(rp + i + 1);
    u = __ldg(row_ids + i);
    d = __ldg(diag + i);
  }
  const bool mine = act && e - b <= kLongRow;  // long rows: bgs_long_kernel / blong_*_kernel
#pragma unroll
  for (int j = 0; j < U; ++j) {
    const bool ok = mine && b + j < e;
    c[j] = ok ? __ldg(col + b + j) : 0;
    v[j] = ok ? __ldg(val + b + j) : 0.0;
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (!mine) return;
  const d4 bv = ld4(B + (int64_t)u * K + k0);
  d4 xv[U];
#pragma unroll
  for (int j = 0; j < U; ++j) xv[j] = b + j < e ? ld4(X + (int64_t)c[j] * K + k0) : d4{0.0, 0.0, 0.0, 0.0};
  double s[kV] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
  for (int j = 0; j < U; ++j)
    if (b + j < e) {
      s[0] = s[0] - v[j] * xv[j].x;
      s[1] = s[1] - v[j] * xv[j].y;
      s[2] = s[2] - v[j] * xv[j].z;
      s[3] = s[3] - v[j] * xv[j].w;
    }
  if (e - b > U) fold4<K, true>(s, col, val, X, b + U, e, k0);
  double* px = X + (int64_t)u * K + k0;
  if (done) {
#pragma unroll
    for (int q = 0; q < kV; ++q)
      if (!done[k0 + q]) px[q] = s[q] / d;
  } else {
    st4(px, s[0] / d, s[1] / d, s[2] / d, s[3] / d);
  }
}

// ---------------------------------------------- exact-order block sweep
// gauss_seidel_sweep (smoothing.cpp:29-40) in the reference's row order for
// K columns at once, without a grid barrier: the level's wavefronts (rows
// whose lower neighbours all lie in earlier fronts) are cut into items of at
// most kExactItemRows rows (ExactItems). A persistent grid claims items by a
// ticket in front order; an item of front g waits (ld.acquire) until every
// item of front g-1 has released its done counter, so front g-1 complete
// implies every earlier front complete, and every row reads exactly the
// values the sequential sweep reads. Tickets are handed out in order and an
// item only waits on smaller tickets held by running CTAs: no co-residency
// requirement, so concurrent lanes share the SMs. Each column's fold is
// s = b; s -= a_uv x_v in the row's column order; x_u = s / d_u --
// bit-identical per column to the one-column exact sweep.
__device__ __forceinline__ int ld_acquire_i32(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// One item per CTA pass: kExactItemRows rows x K/4 threads per row. Before
// waiting on front g-1 the CTA loads everything that does not depend on it:
// the rows, their extents, the first kXU entries (columns and values), b, the
// diagonal and -- once the previous sweep is complete -- x of the upper
// neighbours (col > u: rows of later fronts, not written before this item).
// After the acquire only the lower neighbours' x (just written, L2 hits) are
// gathered, then the fold in column order and the store.
constexpr int kXU = 8;
template <int K, bool PRE>
__global__ void __launch_bounds__(kBT, PRE ? 2 : 3) bgs_exact_kernel(
    CSRv a, const int32_t* __restrict__ rows, const int32_t* __restrict__ item_front,
    const int32_t* __restrict__ item_r0, const int32_t* __restrict__ item_r1, const int32_t* __restrict__ front_items,
    int32_t nfronts, int32_t nitems, int sweeps, const double* __restrict__ B, double* X, int32_t* ctl) {
  constexpr int T = K / kV;  // threads per row
  __shared__ int32_t s_t, s_up;
  int32_t* done = ctl + 1;  // [sweeps * nfronts]
  const int32_t total = nitems * sweeps;
  const int k0 = (int)(threadIdx.x % T) * kV;
  for (;;) {
    if (threadIdx.x == 0) {
      const int32_t t = atomicAdd(ctl, 1);
      s_t = t;
      int up = 1;  // upper neighbours hold their final previous-sweep values
      if (PRE && t < total) {
        const int32_t sw = t / nitems;
        if (sw > 0) up = ld_acquire_i32(done + sw * nfronts - 1) >= __ldg(front_items + nfronts - 1);
      }
      s_up = up;
    }
    __syncthreads();
    const int32_t t = s_t;
    if (t >= total) break;
    const int32_t sw = t / nitems, it = t - sw * nitems;
    const int32_t f = __ldg(item_front + it);
    const int32_t g = sw * nfronts + f;
    const int32_t r0 = __ldg(item_r0 + it), r1 = __ldg(item_r1 + it);
    const int32_t i = r0 + (int32_t)(threadIdx.x / T);
    const bool act = i < r1;
    int32_t u = 0;
    int64_t e0 = 0, e1 = 0;
    double d = 1.0;
    d4 bv{0.0, 0.0, 0.0, 0.0};
    int32_t c[kXU];
    double v[kXU];
    d4 xv[kXU];
    if (act) {
      u = __ldg(rows + i);
      e0 = __ldg(a.rp + u);
      e1 = __ldg(a.rp + u + 1);
      d = __ldg(a.diag + u);
      bv = ld4(B + (int64_t)u * K + k0);
    }
#pragma unroll
    for (int j = 0; j < kXU; ++j) {
      const bool ok = e0 + j < e1;
      c[j] = ok ? __ldg(a.col + e0 + j) : 0;
      v[j] = ok ? __ldg(a.val + e0 + j) : 0.0;
    }
    const bool up = PRE && s_up;
#pragma unroll
    for (int j = 0; j < kXU; ++j)
      xv[j] = (up && e0 + j < e1 && c[j] > u) ? ld4_cg(X + (int64_t)c[j] * K + k0) : d4{0.0, 0.0, 0.0, 0.0};
    if (threadIdx.x == 0 && g > 0) {
      const int32_t need = __ldg(front_items + (g - 1) % nfronts);
      while (ld_acquire_i32(done + g - 1) < need) __nanosleep(20);
    }
    __syncthreads();
    if (act) {
#pragma unroll
      for (int j = 0; j < kXU; ++j)
        if (e0 + j < e1 && !(up && c[j] > u)) xv[j] = ld4_cg(X + (int64_t)c[j] * K + k0);
      double s0 = bv.x, s1 = bv.y, s2 = bv.z, s3 = bv.w;
#pragma unroll
      for (int j = 0; j < kXU; ++j)
        if (e0 + j < e1) {
          s0 = s0 - v[j] * xv[j].x;
          s1 = s1 - v[j] * xv[j].y;
          s2 = s2 - v[j] * xv[j].z;
          s3 = s3 - v[j] * xv[j].w;
        }
      for (int64_t e = e0 + kXU; e < e1; ++e) {  // long rows: the rest in column order
        const d4 q = ld4_cg(X + (int64_t)__ldg(a.col + e) * K + k0);
        const double w = __ldg(a.val + e);
        s0 = s0 - w * q.x;
        s1 = s1 - w * q.y;
        s2 = s2 - w * q.z;
        s3 = s3 - w * q.w;
      }
      if (d != 0.0) st4(X + (int64_t)u * K + k0, s0 / d, s1 / d, s2 / d, s3 / d);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(done + g, 1);
  }
}

// Long rows (more than kLongRow entries): one CTA per row -- or per chunk of
// L.chunk entries for the longest -- folds 32 strided slices of the entries
// for all K columns; slice partials combine in slice order, chunk sums in
// chunk order. The order depends on the row only, never on K.
constexpr int kSL = 32;
template <int K>
__device__ __forceinline__ void fold4_strided(double (&s)[kV], const int32_t* __restrict__ col,
                                              const double* __restrict__ val, const double* X, int64_t j0,
                                              int64_t e, int k0) {
  constexpr int U = 8;
  for (int64_t base = j0; base < e; base += (int64_t)U * kSL) {
    int32_t c[U];
    double v[U];
    d4 xv[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int64_t j = base + (int64_t)q * kSL;
      const bool ok = j < e;
      c[q] = ok ? __ldg(col + j) : 0;
      v[q] = ok ? __ldg(val + j) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const bool ok = base + (int64_t)q * kSL < e;
      xv[q] = ok ? ld4(X + (int64_t)c[q] * K + k0) : d4{0.0, 0.0, 0.0, 0.0};
    }
#pragma unroll
    for (int q = 0; q < U; ++q)
      if (base + (int64_t)q * kSL < e) {
        s[0] = s[0] + v[q] * xv[q].x;
        s[1] = s[1] + v[q] * xv[q].y;
        s[2] = s[2] + v[q] * xv[q].z;
        s[3] = s[3] + v[q] * xv[q].w;
      }
  }
}
// sum over entries [cb, ce) for this CTA's K columns; valid in threads [0, K)
template <int K>
__device__ __forceinline__ double long_chunk_dot(const int32_t* __restrict__ col, const double* __restrict__ val,
                                                 const double* X, int64_t cb, int64_t ce) {
  __shared__ double sh[kSL * K];
  constexpr int Q = K / kV;
  for (int pr = threadIdx.x; pr < kSL * Q; pr += blockDim.x) {
    const int sl = pr / Q, k0 = (pr % Q) * kV;
    double s[kV] = {0.0, 0.0, 0.0, 0.0};
    fold4_strided<K>(s, col, val, X, cb + sl, ce, k0);
#pragma unroll
    for (int q = 0; q < kV; ++q) sh[sl * K + k0 + q] = s[q];
  }
  __syncthreads();
  double t = 0.0;
  if ((int)threadIdx.x < K)
    for (int sl = 0; sl < kSL; ++sl) t += sh[sl * K + threadIdx.x];
  return t;
}

template <int K>
__global__ void __launch_bounds__(kBT) bgs_long_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                       const double* __restrict__ val, const double* __restrict__ diag,
                                                       const int32_t* __restrict__ row_ids,
                                                       const int32_t* __restrict__ rows, const double* __restrict__ B,
                                                       double* X, const int32_t* done) {
  const int32_t i = rows[blockIdx.x];
  const double t = long_chunk_dot<K>(col, val, X, rp[i], rp[i + 1]);
  const int k = threadIdx.x;
  if (k < K && !(done && done[k])) {
    const int64_t u = row_ids[i];
    X[u * K + k] = (B[u * K + k] - t) / diag[i];
  }
}
// one CTA per (super-long row, chunk) work item: chunk sums to scratch
template <int K>
__global__ void __launch_bounds__(kBT) blong_part_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                         const double* __restrict__ val,
                                                         const int32_t* __restrict__ item_row,
                                                         const int32_t* __restrict__ item_chunk, int32_t it0,
                                                         int64_t chunk, const double* X, double* scratch) {
  const int32_t it = it0 + blockIdx.x;
  const int32_t i = item_row[it];
  const int64_t cb = rp[i] + (int64_t)item_chunk[it] * chunk;
  const int64_t ce = cb + chunk < rp[i + 1] ? cb + chunk : rp[i + 1];
  const double t = long_chunk_dot<K>(col, val, X, cb, ce);
  if ((int)threadIdx.x < K) scratch[(int64_t)it * K + threadIdx.x] = t;
}
// chunk sums in chunk order -> the row's update (GS: stored rows; residual:
// natural rows, row_ids == nullptr)
template <int K, bool RES>
__global__ void blong_fin_kernel(const int32_t* __restrict__ srows, const int32_t* __restrict__ sitem0, int32_t s0,
                                 int32_t ns, const double* __restrict__ scratch, const int32_t* __restrict__ row_ids,
                                 const double* __restrict__ diag, const double* __restrict__ B, double* X, double* R,
                                 const int32_t* done) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)ns * K) return;
  const int32_t s = s0 + (int32_t)(t / K);
  const int k = (int)(t % K);
  double tot = 0.0;
  for (int32_t it = sitem0[s]; it < sitem0[s + 1]; ++it) tot += scratch[(int64_t)it * K + k];
  const int32_t i = srows[s];
  if (RES) {
    const int64_t q = (int64_t)i * K + k;
    R[q] = B[q] - (diag[i] * X[q] + tot);
  } else if (!(done && done[k])) {
    const int64_t u = row_ids[i];
    X[u * K + k] = (B[u * K + k] - tot) / diag[i];
  }
}

template <int K, int MINB = 6>
__global__ void __launch_bounds__(kBT, MINB) bres_kernel(CSRv a, const double* __restrict__ B, const double* __restrict__ X,
                                                   double* __restrict__ R) {
  constexpr int T = K / kV;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t u = t / T;
  const int k0 = (int)(t % T) * kV;
  if (u >= a.n) return;
  const int64_t b = __ldg(a.rp + u), e = __ldg(a.rp + u + 1);
  if (e - b > kLongRow) return;  // bres_long_kernel / blong_*_kernel
  const double d = __ldg(a.diag + u);
  const d4 xu = ld4(X + u * K + k0);
  double s[kV] = {d * xu.x, d * xu.y, d * xu.z, d * xu.w};
  fold4<K, false>(s, a.col, a.val, X, b, e, k0);
  const d4 bv = ld4(B + u * K + k0);
  st4(R + u * K + k0, bv.x - s[0], bv.y - s[1], bv.z - s[2], bv.w - s[3]);
}

template <int K>
__global__ void __launch_bounds__(kBT) bres_long_kernel(CSRv a, const int32_t* __restrict__ rows,
                                                        const double* __restrict__ B, const double* X, double* R) {
  const int32_t u = rows[blockIdx.x];
  const double t = long_chunk_dot<K>(a.col, a.val, X, a.rp[u], a.rp[u + 1]);
  const int k = threadIdx.x;
  if (k < K) {
    const int64_t q = (int64_t)u * K + k;
    R[q] = B[q] - (a.diag[u] * X[q] + t);
  }
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

// r = b - A x and restrict_residual fused (cycle.cpp:180-186, aggregation.cpp:333-337):
// a thread owns four columns of one aggregate, forms each member row's
// residual exactly as bres_kernel does and folds them in member order
// exactly as brestrict_kernel does -- the same bits, without writing and
// re-reading R (16 n K bytes per visit). Levels without long rows only.
template <int K, int MINB = 4>
__global__ void __launch_bounds__(kBT, MINB) bres_restrict_kernel(CSRv a, int32_t cn,
                                                                 const int64_t* __restrict__ mem_ptr,
                                                                 const int32_t* __restrict__ mem,
                                                                 const double* __restrict__ B,
                                                                 const double* __restrict__ X, double mu,
                                                                 double* __restrict__ Bc, double* __restrict__ Xc) {
  constexpr int T = K / kV;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t g = t / T;
  const int k0 = (int)(t % T) * kV;
  if (g >= cn) return;
  double acc[kV] = {0.0, 0.0, 0.0, 0.0};
  const int64_t j1 = __ldg(mem_ptr + g + 1);
  for (int64_t j = __ldg(mem_ptr + g); j < j1; ++j) {
    const int64_t u = __ldg(mem + j);
    const int64_t b = __ldg(a.rp + u), e = __ldg(a.rp + u + 1);
    const double d = __ldg(a.diag + u);
    const d4 xu = ld4(X + u * K + k0);
    double s[kV] = {d * xu.x, d * xu.y, d * xu.z, d * xu.w};
    fold4<K, false>(s, a.col, a.val, X, b, e, k0);
    const d4 bv = ld4(B + u * K + k0);
    acc[0] = acc[0] + (bv.x - s[0]);
    acc[1] = acc[1] + (bv.y - s[1]);
    acc[2] = acc[2] + (bv.z - s[2]);
    acc[3] = acc[3] + (bv.w - s[3]);
  }
  if (mu != 1.0) st4(Bc + g * K + k0, acc[0] * mu, acc[1] * mu, acc[2] * mu, acc[3] * mu);
  else st4(Bc + g * K + k0, acc[0], acc[1], acc[2], acc[3]);
  st4(Xc + g * K + k0, 0.0, 0.0, 0.0, 0.0);
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
  if (s.ntlong && s.t_ptr[q + 1] - s.t_ptr[q] > kLongT) return;  // bcoarsen_long_kernel
  double v = B[(int64_t)s.poc[q] * K + k];
  for (int64_t j = s.t_ptr[q]; j < s.t_ptr[q + 1]; ++j) {
    const int64_t p = s.t_p[j];
    const int32_t i = s.f_of_p[p];
    v = v - s.f_val[p] * (B[(int64_t)s.f_nodes[i] * K + k] / s.f_diag[i]);
  }
  Bc[t] = v;
}

// a coarse node with a long contribution list, K columns: 32 strided slices
// (fixed, so a column's sum does not depend on K), summed in slice order
template <int K>
__global__ void __launch_bounds__(kBT) bcoarsen_long_kernel(StageV s, const double* __restrict__ B,
                                                            double* __restrict__ Bc) {
  __shared__ double sh[kSL * K];
  const int32_t q = s.tlong[blockIdx.x];
  const int64_t j0 = s.t_ptr[q], j1 = s.t_ptr[q + 1];
  for (int pr = threadIdx.x; pr < kSL * K; pr += blockDim.x) {
    const int sl = pr / K, k = pr % K;
    double acc = 0.0;
    for (int64_t j = j0 + sl; j < j1; j += kSL) {
      const int64_t p = s.t_p[j];
      const int32_t i = s.f_of_p[p];
      acc += s.f_val[p] * (B[(int64_t)s.f_nodes[i] * K + k] / s.f_diag[i]);
    }
    sh[sl * K + k] = acc;
  }
  __syncthreads();
  if ((int)threadIdx.x < K) {
    double t = 0.0;
    for (int sl = 0; sl < kSL; ++sl) t += sh[sl * K + threadIdx.x];
    Bc[(int64_t)q * K + threadIdx.x] = B[(int64_t)s.poc[q] * K + threadIdx.x] - t;
  }
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
    case 64: f(std::integral_constant<int, 64>{}); break;
    case 128: f(std::integral_constant<int, 128>{}); break;
    default: throw LamgError(LAMG_E_ARGUMENT, "batch width must be 4, 8, 16, 32, 64 or 128");
  }
}

}  // namespace

static double* long_scratch(Ctx& c, const LongRows& L, int K) {
  const int64_t need = std::max<int64_t>((int64_t)L.iptr_h.back() * K, 1);
  if (c.bscratch.n < need) c.bscratch.alloc(need, c.s);
  return c.bscratch.p;
}

void bgs_colored(Ctx& c, const DColor& cl, int32_t n, const double* B, double* X, int sweeps, int K,
                 const int32_t* done) {
  if (n == 0 || sweeps <= 0) return;
  const LongRows& L = cl.blong;
  double* scratch = long_scratch(c, L, K);
  // LAMG_PDL_THREADS=t: colour launches of at most t threads (about one wave: 148 SMs x
  // 1024 = 160000) go through programmatic dependent launch
  static const int64_t pdl_threads = [] {
    const char* e = getenv("LAMG_PDL_THREADS");
    return e ? atoll(e) : (int64_t)0;  // off by default: measured 74.6 -> 72.4 ms per block cycle for one
                                        // lane on config 2, no gain with 8 lanes in flight (LAMG_PDL_THREADS=160000)
  }();
  dispatch_k(K, [&](auto kc) {
    constexpr int KK = decltype(kc)::value;
    for (int sw = 0; sw < sweeps; ++sw)
      for (int32_t cc = 0; cc < cl.ncolors; ++cc) {
        const int32_t i0 = cl.cptr_h[cc], i1 = cl.cptr_h[cc + 1];
        if (i1 <= i0) continue;
        const int64_t nthreads = (int64_t)(i1 - i0) * (KK / kV);
        if (pdl_threads > 0 && nthreads <= pdl_threads) {
          // one-wave colours: programmatic dependent launch (see bgs_pdl_kernel)
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3((unsigned)bblocks(nthreads));
          cfg.blockDim = dim3(kBT);
          cfg.stream = c.s;
          cudaLaunchAttribute at;
          at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at.val.programmaticStreamSerializationAllowed = 1;
          cfg.attrs = &at;
          cfg.numAttrs = 1;
          count_launch();
          CK(cudaLaunchKernelEx(&cfg, bgs_pdl_kernel<KK>, (const int64_t*)cl.rp.p, (const int32_t*)cl.col.p,
                                (const double*)cl.val.p, (const double*)cl.diag.p, (const int32_t*)cl.row_ids.p, i0,
                                i1, B, X, done));
        } else {
          count_launch(), bgs_kernel<KK><<<bblocks(nthreads), kBT, 0, c.s>>>(
              cl.rp.p, cl.col.p, cl.val.p, cl.diag.p, cl.row_ids.p, i0, i1, B, X, done);
        }
        const int32_t nl = L.ptr_h[cc + 1] - L.ptr_h[cc];
        if (nl)
          count_launch(), bgs_long_kernel<KK><<<nl, kBT, 0, c.s>>>(cl.rp.p, cl.col.p, cl.val.p, cl.diag.p,
                                                                  cl.row_ids.p, L.rows.p + L.ptr_h[cc], B, X, done);
        const int32_t ni = L.iptr_h[cc + 1] - L.iptr_h[cc];
        if (ni) {
          count_launch(), blong_part_kernel<KK><<<ni, kBT, 0, c.s>>>(cl.rp.p, cl.col.p, cl.val.p, L.item_row.p,
                                                                    L.item_chunk.p, L.iptr_h[cc], L.chunk, X, scratch);
          const int32_t ns = L.sptr_h[cc + 1] - L.sptr_h[cc];
          count_launch(), blong_fin_kernel<KK, false><<<bblocks((int64_t)ns * KK), kBT, 0, c.s>>>(
              L.srows.p, L.sitem0.p, L.sptr_h[cc], ns, scratch, cl.row_ids.p, cl.diag.p, B, X, nullptr, done);
        }
      }
  });
  CK_LAUNCH();
}

void bgs_exact(Ctx& c, const CSRv& a, const Schedule& sch, const ExactItems& it, const double* B, double* X,
               int sweeps, int K, int32_t* ctl) {
  if (a.n == 0 || sweeps <= 0 || it.nitems == 0) return;
  if (it.rows * std::max(1, K / kV) > kBT) throw LamgError(LAMG_E_ERROR, "exact sweep items too large for the block width");
  static const int env_ctas = [] {
    const char* e = getenv("LAMG_XB_CTAS");
    return e ? std::max(1, atoi(e)) : 0;
  }();
  static const bool pre = [] {
    const char* e = getenv("LAMG_XB_PRE");
    return !(e && atoi(e) == 0);
  }();
  for (int s0 = 0; s0 < sweeps; s0 += kMaxExactSweeps) {
    const int ns = std::min(kMaxExactSweeps, sweeps - s0);
    const int64_t total = (int64_t)it.nitems * ns;
    // a persistent grid of two CTAs per SM: an average cfg2 front (5.5k rows,
    // ~170 items) in one pass
    const int ctas = (int)std::min<int64_t>(total, env_ctas ? env_ctas : 2 * c.sms);
    CK(cudaMemsetAsync(ctl, 0, sizeof(int32_t) * (1 + (size_t)ns * it.nfronts), c.s));
    dispatch_k(K, [&](auto kc) {
      constexpr int KK = decltype(kc)::value;
      if (pre)
        count_launch(), bgs_exact_kernel<KK, true><<<ctas, kBT, 0, c.s>>>(
            a, sch.rows.p, it.front.p, it.r0.p, it.r1.p, it.count.p, it.nfronts, it.nitems, ns, B, X, ctl);
      else
        count_launch(), bgs_exact_kernel<KK, false><<<ctas, kBT, 0, c.s>>>(
            a, sch.rows.p, it.front.p, it.r0.p, it.r1.p, it.count.p, it.nfronts, it.nitems, ns, B, X, ctl);
    });
    CK_LAUNCH();
  }
}

void bresidual(Ctx& c, const CSRv& a, const LongRows& L, const double* B, const double* X, double* R, int K) {
  if (a.n == 0) return;
  if (L.ptr_h.empty()) throw LamgError(LAMG_E_ERROR, "batched residual needs the level's throughput data");
  double* scratch = long_scratch(c, L, K);
  dispatch_k(K, [&](auto kc) {
    constexpr int KK = decltype(kc)::value;
    count_launch(), bres_kernel<KK><<<bblocks((int64_t)a.n * (KK / kV)), kBT, 0, c.s>>>(a, B, X, R);
    const int32_t nl = L.ptr_h[1];
    if (nl) count_launch(), bres_long_kernel<KK><<<nl, kBT, 0, c.s>>>(a, L.rows.p, B, X, R);
    const int32_t ni = L.iptr_h[1];
    if (ni) {
      count_launch(), blong_part_kernel<KK><<<ni, kBT, 0, c.s>>>(a.rp, a.col, a.val, L.item_row.p, L.item_chunk.p, 0,
                                                                L.chunk, X, scratch);
      const int32_t ns = L.sptr_h[1];
      count_launch(), blong_fin_kernel<KK, true><<<bblocks((int64_t)ns * KK), kBT, 0, c.s>>>(
          L.srows.p, L.sitem0.p, 0, ns, scratch, nullptr, a.diag, B, const_cast<double*>(X), R, nullptr);
    }
  });
  CK_LAUNCH();
}

bool bresidual_restrict(Ctx& c, const CSRv& a, const LongRows& L, int32_t coarse_n, const int64_t* mem_ptr,
                        const int32_t* mem, const double* B, const double* X, double mu, double* Bc, double* Xc,
                        int K) {
  static const bool off = [] {
    const char* e = getenv("LAMG_NO_FUSED_RESTRICT");
    return e && atoi(e) == 1;
  }();
  if (off || a.n == 0 || coarse_n == 0 || L.ptr_h.empty() || L.ptr_h[1] || L.iptr_h[1]) return false;
  dispatch_k(K, [&](auto kc) {
    constexpr int KK = decltype(kc)::value;
    count_launch(), bres_restrict_kernel<KK><<<bblocks((int64_t)coarse_n * (KK / kV)), kBT, 0, c.s>>>(
        a, coarse_n, mem_ptr, mem, B, X, mu, Bc, Xc);
  });
  CK_LAUNCH();
  return true;
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
    if (s.ntlong) count_launch(), bcoarsen_long_kernel<KK><<<s.ntlong, kBT, 0, c.s>>>(s, B, Bc);
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

void brelax(Ctx& c, const CSRv& a, const DColor& cl, const LongRows& nat, const double* B, double* X, double* R,
            int K, std::vector<int>& sweeps) {
  sweeps.assign(K, 0);
  int32_t* done = c.dbdone;
  double* nrm = c.dbscal;                  // [K]
  double* sums = c.dbscal + kMaxBlock;     // [K]
  std::vector<double> r0(K), rn(K);
  std::vector<int32_t> hdone(K, 0);
  bresidual(c, a, nat, B, X, R, K);
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
    bresidual(c, a, nat, B, X, R, K);
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
