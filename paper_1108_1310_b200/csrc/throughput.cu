// throughput.cu -- THROUGHPUT-mode smoother: greedy colouring, colour-
// permuted operator copies, coloured Gauss-Seidel, and the coarsest inverse.
//
// The hierarchy (every integer artefact and coarse value) is the bit-exact
// VALIDATE-mode one; only the solve's smoother order and its reductions
// change.
#include <algorithm>

#include "hier.cuh"

namespace lamgb {

// First-fit colour in index order: u takes the smallest colour unused by its
// lower neighbours. Lower neighbours sit in earlier wavefronts, so walking
// the exact-order fronts reproduces the sequential greedy colouring. Rows of
// one front are independent: short rows take a thread, medium rows a warp
// and hub rows a whole CTA (power-law levels have hubs with 10^5-10^6 lower
// neighbours; one thread per hub serialised the colouring for minutes).
constexpr int64_t kColorWarpRow = 32, kColorBlockRow = 4096;

__device__ __forceinline__ unsigned long long color_window(const CSRv& a, int32_t u, int64_t k0, int64_t step,
                                                           int32_t base, const int32_t* color) {
  unsigned long long used = 0ull;
  for (int64_t k = a.rp[u] + k0; k < a.rp[u + 1]; k += step) {
    const int32_t v = a.col[k];
    if (v >= u) break;  // rows are sorted: lower neighbours first
    const int32_t cv = ((volatile const int32_t*)color)[v] - base;
    if (cv >= 0 && cv < 64) used |= 1ull << cv;
  }
  return used;
}

__device__ __forceinline__ unsigned long long warp_or64(unsigned long long v) {
  const unsigned lo = __reduce_or_sync(0xffffffffu, (unsigned)v);
  const unsigned hi = __reduce_or_sync(0xffffffffu, (unsigned)(v >> 32));
  return ((unsigned long long)hi << 32) | lo;
}

__global__ void color_fronts_kernel(CSRv a, const int32_t* __restrict__ front_ptr,
                                    const int32_t* __restrict__ rows, int32_t nfronts, int32_t* color) {
  __shared__ unsigned long long sh_used;
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  const int64_t gwarp = gtid >> 5, nwarps = gstride >> 5;
  const int lane = threadIdx.x & 31;
  for (int32_t f = 0; f < nfronts; ++f) {
    const int32_t lo = front_ptr[f], hi = front_ptr[f + 1];
    for (int64_t i = lo + gtid; i < hi; i += gstride) {
      const int32_t u = rows[i];
      if (a.rp[u + 1] - a.rp[u] > kColorWarpRow) continue;
      for (int32_t base = 0;; base += 64) {
        const unsigned long long used = color_window(a, u, 0, 1, base, color);
        if (~used) {
          color[u] = base + __ffsll((long long)~used) - 1;
          break;
        }
      }
    }
    for (int64_t i = lo + gwarp; i < hi; i += nwarps) {
      const int32_t u = rows[i];
      const int64_t len = a.rp[u + 1] - a.rp[u];
      if (len <= kColorWarpRow || len > kColorBlockRow) continue;
      for (int32_t base = 0;; base += 64) {
        const unsigned long long used = warp_or64(color_window(a, u, lane, 32, base, color));
        if (~used) {
          if (lane == 0) color[u] = base + __ffsll((long long)~used) - 1;
          break;
        }
      }
    }
    for (int64_t i = lo + blockIdx.x; i < hi; i += gridDim.x) {
      const int32_t u = rows[i];
      if (a.rp[u + 1] - a.rp[u] <= kColorBlockRow) continue;
      for (int32_t base = 0;; base += 64) {
        if (threadIdx.x == 0) sh_used = 0ull;
        __syncthreads();
        const unsigned long long used = warp_or64(color_window(a, u, threadIdx.x, blockDim.x, base, color));
        if (lane == 0 && used) atomicOr(&sh_used, used);
        __syncthreads();
        const unsigned long long all = sh_used;
        __syncthreads();
        if (~all) {
          if (threadIdx.x == 0) color[u] = base + __ffsll((long long)~all) - 1;
          break;
        }
      }
    }
    grid_barrier();
  }
}

__global__ void iota32_kernel(int32_t* x, int32_t n) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = i;
}
__global__ void color_bounds_kernel(const uint32_t* sorted, int32_t n, int32_t ncol, int32_t* cptr) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > n) return;
  int32_t lo = i == 0 ? 0 : (int32_t)sorted[i - 1] + 1;
  int32_t hi = i == n ? ncol : (int32_t)sorted[i];
  for (int32_t k = lo; k <= hi && k <= ncol; ++k) cptr[k] = i;
}
__global__ void perm_deg_kernel(CSRv a, const int32_t* row_ids, int64_t* deg) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  int32_t u = row_ids[i];
  deg[i] = a.rp[u + 1] - a.rp[u];
}
// one warp per stored row (hub rows hold up to 10^6 entries)
__global__ void perm_fill_kernel(CSRv a, const int32_t* row_ids, const int64_t* prp, int32_t* pcol,
                                 double* pval, double* pdiag) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= a.n) return;
  const int32_t u = row_ids[w];
  const int64_t o = prp[w] - a.rp[u];
  for (int64_t k = a.rp[u] + lane; k < a.rp[u + 1]; k += 32) {
    pcol[o + k] = a.col[k];
    pval[o + k] = a.val[k];
  }
  if (lane == 0) pdiag[w] = a.diag[u];
}

__global__ void heavy_flags_kernel(const int64_t* rp, int32_t n, uint8_t* f) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) f[i] = rp[i + 1] - rp[i] > kHeavyRow;
}

void build_coloring(Ctx& c, const CSRv& a, const Schedule& sch, DColor& out) {
  const int32_t n = a.n;
  DVec<int32_t> color(n, c.s);
  color.fill_bytes(0xff);  // -1: not yet coloured
  const int threads = 256;
  int blocks = (int)std::min<int64_t>(c.max_coop_blocks((const void*)color_fronts_kernel, threads),
                                      std::max<int64_t>(1, (sch.max_width + threads - 1) / threads));
  if (sch.max_width <= 2 * threads) blocks = 1;
  CSRv av = a;
  const int32_t* fp = sch.front_ptr.p;
  const int32_t* rw = sch.rows.p;
  int32_t nf = sch.nfronts;
  void* args[] = {&av, (void*)&fp, (void*)&rw, &nf, &color.p};
  coop_launch(c, (const void*)color_fronts_kernel, blocks, threads, args);
  const int32_t ncol = reduce_max_i32(c, color.p, n) + 1;
  DVec<int32_t> ids(n, c.s);
  DVec<uint32_t> ks(n, c.s);
  count_launch(), iota32_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(ids.p, n);
  CK_LAUNCH();
  out.row_ids.alloc(n, c.s);
  int bits = 1;
  while ((1 << bits) <= ncol && bits < 31) ++bits;
  sort_pairs_u32_i32(c, (const uint32_t*)color.p, ks.p, ids.p, out.row_ids.p, n, bits);
  DVec<int32_t> cptr(ncol + 1, c.s);
  count_launch(), color_bounds_kernel<<<blocks_for(n + 1), kThreads, 0, c.s>>>(ks.p, n, ncol, cptr.p);
  CK_LAUNCH();
  out.ncolors = ncol;
  out.group = row_group_for(a.n, a.m);
  out.cptr_h = cptr.to_host();
  DVec<int64_t> deg(n + 1, c.s);
  count_launch(), perm_deg_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(a, out.row_ids.p, deg.p);
  CK_LAUNCH();
  CK(cudaMemsetAsync(deg.p + n, 0, sizeof(int64_t), c.s));
  out.rp.alloc(n + 1, c.s);
  exclusive_scan_i64(c, deg.p, out.rp.p, n + 1);
  out.col.alloc(std::max<int64_t>(2 * a.m, 1), c.s);
  out.val.alloc(std::max<int64_t>(2 * a.m, 1), c.s);
  out.diag.alloc(n, c.s);
  count_launch(), perm_fill_kernel<<<blocks_for((int64_t)n * 32), kThreads, 0, c.s>>>(a, out.row_ids.p, out.rp.p, out.col.p,
                                                                     out.val.p, out.diag.p);
  CK_LAUNCH();
  // heavy rows: per colour (stored positions) and in natural order
  DVec<uint8_t> hf(n, c.s);
  count_launch(), heavy_flags_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(out.rp.p, n, hf.p);
  CK_LAUNCH();
  out.heavy.alloc(n, c.s);
  const int64_t nh = select_flagged_index(c, hf.p, out.heavy.p, n);
  out.hptr_h.assign(ncol + 1, 0);
  if (nh) {
    std::vector<int32_t> hv((size_t)nh);
    out.heavy.download(hv.data(), nh);
    c.sync();
    for (int32_t cc = 0; cc <= ncol; ++cc)
      out.hptr_h[cc] = (int32_t)(std::lower_bound(hv.begin(), hv.end(), out.cptr_h[cc]) - hv.begin());
    out.group = 8;
  }
  out.hptr.alloc(ncol + 1, c.s);
  out.hptr.upload(out.hptr_h.data(), ncol + 1);
  count_launch(), heavy_flags_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(a.rp, n, hf.p);
  CK_LAUNCH();
  out.heavy_nat.alloc(n, c.s);
  out.nheavy_nat = (int32_t)select_flagged_index(c, hf.p, out.heavy_nat.p, n);
  c.sync();
  // long-row lists for the K-column kernels (batch.cu)
  std::vector<int64_t> prp((size_t)n + 1);
  out.rp.download(prp.data(), n + 1);
  c.sync();
  build_long_rows(c, prp, out.cptr_h, out.blong);
  c.sync();
}

void build_long_rows(Ctx& c, const std::vector<int64_t>& rp, const std::vector<int32_t>& bounds, LongRows& L) {
  std::vector<int32_t> rows, irow, ichunk, srows, sitem0;
  const size_t nb = bounds.size() - 1;
  L.ptr_h.assign(nb + 1, 0);
  L.iptr_h.assign(nb + 1, 0);
  L.sptr_h.assign(nb + 1, 0);
  for (size_t g = 0; g < nb; ++g) {
    L.ptr_h[g] = (int32_t)rows.size();
    L.iptr_h[g] = (int32_t)irow.size();
    L.sptr_h[g] = (int32_t)srows.size();
    for (int32_t i = bounds[g]; i < bounds[g + 1]; ++i) {
      const int64_t len = rp[i + 1] - rp[i];
      if (len <= kLongRow) continue;
      if (len <= kChunk) {
        rows.push_back(i);
      } else {
        srows.push_back(i);
        sitem0.push_back((int32_t)irow.size());
        for (int64_t q = 0; q * kChunk < len; ++q) {
          irow.push_back(i);
          ichunk.push_back((int32_t)q);
        }
      }
    }
  }
  L.ptr_h[nb] = (int32_t)rows.size();
  L.iptr_h[nb] = (int32_t)irow.size();
  L.sptr_h[nb] = (int32_t)srows.size();
  sitem0.push_back((int32_t)irow.size());
  auto up = [&](DVec<int32_t>& d, const std::vector<int32_t>& h) {
    d.alloc(std::max<size_t>(h.size(), 1), c.s);
    if (!h.empty()) d.upload(h.data(), (int64_t)h.size());
  };
  up(L.rows, rows);
  up(L.item_row, irow);
  up(L.item_chunk, ichunk);
  up(L.srows, srows);
  up(L.sitem0, sitem0);
  c.sync();
}

// One colour: rows [i0, i1) of the permuted operator update in parallel.
__global__ void gs_color_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                const double* __restrict__ val, const double* __restrict__ diag,
                                const int32_t* __restrict__ row_ids, const double* __restrict__ b,
                                double* x, int32_t i0, int32_t i1) {
  int32_t i = i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= i1) return;
  const int32_t u = row_ids[i];
  double s = row_fold<8, true, true>(b[u], col, val, x, rp[i], rp[i + 1]);
  x[u] = s / diag[i];
}

// One colour with G lanes per row (coarse levels: rows of ~10-40 entries
// would otherwise serialise their loads in one thread).
template <int G>
__global__ void gs_color_group_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                      const double* __restrict__ val, const double* __restrict__ diag,
                                      const int32_t* __restrict__ row_ids, const double* __restrict__ b,
                                      double* x, int32_t i0, int32_t i1) {
  const int64_t gid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
  const int64_t i = i0 + gid;
  const bool ok = i < i1 && rp[i + 1] - rp[i] <= kHeavyRow;
  const double dot = group_dot<G>(col, val, x, ok ? rp[i] : 0, ok ? rp[i + 1] : 0);
  if (ok && (threadIdx.x & (G - 1)) == 0) {
    const int32_t u = row_ids[i];
    x[u] = (b[u] - dot) / diag[i];
  }
}

template <int G>
__global__ void residual_group_kernel(CSRv a, const double* __restrict__ b, const double* __restrict__ x,
                                      double* __restrict__ r) {
  const int64_t u = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
  const bool ok = u < a.n && a.rp[u + 1] - a.rp[u] <= kHeavyRow;
  const double dot = group_dot<G>(a.col, a.val, x, ok ? a.rp[u] : 0, ok ? a.rp[u + 1] : 0);
  if (ok && (threadIdx.x & (G - 1)) == 0) r[u] = b[u] - (a.diag[u] * x[u] + dot);
}

// one CTA per heavy row (stored position list) of one colour
__global__ void gs_heavy_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                const double* __restrict__ val, const double* __restrict__ diag,
                                const int32_t* __restrict__ row_ids, const int32_t* __restrict__ heavy,
                                const double* __restrict__ b, double* x) {
  const int32_t i = heavy[blockIdx.x];
  const double dot = block_dot(col, val, x, rp[i], rp[i + 1]);
  if (threadIdx.x == 0) {
    const int32_t u = row_ids[i];
    x[u] = (b[u] - dot) / diag[i];
  }
}
__global__ void residual_heavy_kernel(CSRv a, const int32_t* __restrict__ heavy, const double* __restrict__ b,
                                      const double* x, double* r) {
  const int32_t u = heavy[blockIdx.x];
  const double dot = block_dot(a.col, a.val, x, a.rp[u], a.rp[u + 1]);
  if (threadIdx.x == 0) r[u] = b[u] - (a.diag[u] * x[u] + dot);
}

void residual_tp(Ctx& c, const CSRv& a, const double* b, const double* x, double* r, const DColor& cl) {
  const int group = cl.group;
  if (a.n == 0) return;
  if (cl.nheavy_nat)
    count_launch(), residual_heavy_kernel<<<cl.nheavy_nat, 256, 0, c.s>>>(a, cl.heavy_nat.p, b, x, r);
  if (group == 1) {
    residual_exact(c, a, b, x, r);
    return;
  }
  const int64_t threads = (int64_t)a.n * group;
  if (group == 4) count_launch(), residual_group_kernel<4><<<blocks_for(threads), kThreads, 0, c.s>>>(a, b, x, r);
  else count_launch(), residual_group_kernel<8><<<blocks_for(threads), kThreads, 0, c.s>>>(a, b, x, r);
  CK_LAUNCH();
}

// All colours and sweeps of a small level in one CTA (no launch per colour).
__global__ void gs_color_cta_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                    const double* __restrict__ val, const double* __restrict__ diag,
                                    const int32_t* __restrict__ row_ids, const int32_t* __restrict__ cptr,
                                    int32_t ncolors, const double* __restrict__ b, double* x, int sweeps) {
  for (int sw = 0; sw < sweeps; ++sw)
    for (int32_t cc = 0; cc < ncolors; ++cc) {
      for (int32_t i = cptr[cc] + threadIdx.x; i < cptr[cc + 1]; i += blockDim.x) {
        const int32_t u = row_ids[i];
        double s = row_fold<8, true>(b[u], col, val, x, rp[i], rp[i + 1]);
        x[u] = s / diag[i];
      }
      __syncthreads();
    }
}

void gs_colored(Ctx& c, const DColor& cl, int32_t n, const double* b, double* x, int sweeps) {
  if (n == 0 || sweeps <= 0) return;
  if (n <= 16384) {
    // device copy of the colour pointers lives right after the permuted rp
    static_assert(sizeof(int64_t) >= sizeof(int32_t), "");
    count_launch(), gs_color_cta_kernel<<<1, 1024, 0, c.s>>>(cl.rp.p, cl.col.p, cl.val.p, cl.diag.p, cl.row_ids.p,
                                                           (const int32_t*)(cl.rp.p + n + 1), cl.ncolors, b, x,
                                                           sweeps);
    CK_LAUNCH();
    return;
  }
  for (int sw = 0; sw < sweeps; ++sw)
    for (int32_t cc = 0; cc < cl.ncolors; ++cc) {
      int32_t i0 = cl.cptr_h[cc], i1 = cl.cptr_h[cc + 1];
      if (i1 <= i0) continue;
      const int64_t rows = i1 - i0;
      const int32_t nh = cl.hptr_h.empty() ? 0 : cl.hptr_h[cc + 1] - cl.hptr_h[cc];
      if (nh)
        count_launch(), gs_heavy_kernel<<<nh, 256, 0, c.s>>>(cl.rp.p, cl.col.p, cl.val.p, cl.diag.p, cl.row_ids.p,
                                                             cl.heavy.p + cl.hptr_h[cc], b, x);
      if (cl.group == 1)
        count_launch(), gs_color_kernel<<<blocks_for(rows), kThreads, 0, c.s>>>(cl.rp.p, cl.col.p, cl.val.p, cl.diag.p,
                                                                             cl.row_ids.p, b, x, i0, i1);
      else if (cl.group == 4)
        count_launch(), gs_color_group_kernel<4><<<blocks_for(rows * 4), kThreads, 0, c.s>>>(
            cl.rp.p, cl.col.p, cl.val.p, cl.diag.p, cl.row_ids.p, b, x, i0, i1);
      else
        count_launch(), gs_color_group_kernel<8><<<blocks_for(rows * 8), kThreads, 0, c.s>>>(
            cl.rp.p, cl.col.p, cl.val.p, cl.diag.p, cl.row_ids.p, b, x, i0, i1);
    }
  CK_LAUNCH();
}

// RelaxationSolver::solve (coarse_solver.cpp:82-93) for THROUGHPUT mode in
// ONE cooperative launch: coloured sweeps separated by grid barriers, fixed-
// order tree reductions (block partials summed in block order by every
// thread), the convergence test on the device. Power-law hierarchies end in a
// multi-million-row relaxation coarsest with hundreds of colours; host-driven
// that is a launch per colour plus a host round trip per sweep.
template <int G>
__device__ inline void coop_residual(const CSRv& a, const double* __restrict__ b, const double* x, double* r,
                                     const int32_t* heavy_nat, int32_t nheavy) {
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  for (int32_t h = blockIdx.x; h < nheavy; h += gridDim.x) {
    const int32_t u = heavy_nat[h];
    const double dot = block_dot(a.col, a.val, x, a.rp[u], a.rp[u + 1]);
    if (threadIdx.x == 0) r[u] = b[u] - (a.diag[u] * x[u] + dot);
  }
  const int64_t span = ((int64_t)a.n * G + 31) / 32 * 32;
  for (int64_t t = gtid; t < span; t += gstride) {
    const int64_t u = t / G;
    const bool ok = u < a.n && a.rp[u + 1] - a.rp[u] <= kHeavyRow;
    const double dot = group_dot<G, true>(a.col, a.val, x, ok ? a.rp[u] : 0, ok ? a.rp[u + 1] : 0);
    if (ok && (threadIdx.x & (G - 1)) == 0) r[u] = b[u] - (a.diag[u] * x[u] + dot);
  }
}

__device__ inline double coop_sum(double v, double* part) {
  __shared__ double sh[33];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
    part[blockIdx.x] = t;
  }
  cg::this_grid().sync();
  double t = 0.0;
  for (unsigned g = 0; g < gridDim.x; ++g) t += ((volatile double*)part)[g];
  cg::this_grid().sync();
  return t;
}

template <int G>
__global__ void relax_coop_kernel(CSRv a, const int64_t* __restrict__ prp, const int32_t* __restrict__ pcol,
                                  const double* __restrict__ pval, const double* __restrict__ pdiag,
                                  const int32_t* __restrict__ row_ids, const int32_t* __restrict__ cptr,
                                  int32_t ncolors, const int32_t* __restrict__ heavy,
                                  const int32_t* __restrict__ hptr, const int32_t* __restrict__ heavy_nat,
                                  int32_t nheavy_nat, const double* __restrict__ b, double* x, double* r,
                                  double* part, int* sweeps_out) {
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  coop_residual<G>(a, b, x, r, heavy_nat, nheavy_nat);
  cg::this_grid().sync();
  double loc = 0.0;
  for (int64_t u = gtid; u < a.n; u += gstride) loc += r[u] * r[u];
  const double r0 = sqrt(coop_sum(loc, part));
  int sweeps = 0;
  if (r0 != 0.0) {
    const double target = 1e-12 * r0;
    for (int sweep = 0; sweep < 400; ++sweep) {
      for (int32_t cc = 0; cc < ncolors; ++cc) {
        const int32_t i0 = cptr[cc], i1 = cptr[cc + 1];
        for (int32_t hh = hptr[cc] + blockIdx.x; hh < hptr[cc + 1]; hh += gridDim.x) {
          const int32_t i = heavy[hh];
          const double dot = block_dot(pcol, pval, x, prp[i], prp[i + 1]);
          if (threadIdx.x == 0) {
            const int32_t u = row_ids[i];
            x[u] = (b[u] - dot) / pdiag[i];
          }
        }
        const int64_t span = ((int64_t)(i1 - i0) * G + 31) / 32 * 32;
        for (int64_t t = gtid; t < span; t += gstride) {
          const int64_t i = i0 + t / G;
          const bool ok = i < i1 && prp[i + 1] - prp[i] <= kHeavyRow;
          const double dot = group_dot<G, true>(pcol, pval, x, ok ? prp[i] : 0, ok ? prp[i + 1] : 0);
          if (ok && (threadIdx.x & (G - 1)) == 0) {
            const int32_t u = row_ids[i];
            x[u] = (b[u] - dot) / pdiag[i];
          }
        }
        cg::this_grid().sync();
      }
      loc = 0.0;
      for (int64_t u = gtid; u < a.n; u += gstride) loc += x[u];
      const double mean = coop_sum(loc, part) / (double)a.n;
      for (int64_t u = gtid; u < a.n; u += gstride) x[u] = x[u] - mean;
      cg::this_grid().sync();
      coop_residual<G>(a, b, x, r, heavy_nat, nheavy_nat);
      cg::this_grid().sync();
      loc = 0.0;
      for (int64_t u = gtid; u < a.n; u += gstride) loc += r[u] * r[u];
      ++sweeps;
      if (sqrt(coop_sum(loc, part)) <= target) break;
    }
  }
  if (gtid == 0) *sweeps_out = sweeps;
}

int relax_colored_coop(Ctx& c, const CSRv& a, const DColor& cl, const double* b, double* x, double* r) {
  const int threads = 256;
  const void* k = cl.group == 8 ? (const void*)relax_coop_kernel<8> : (const void*)relax_coop_kernel<1>;
  const int blocks = c.max_coop_blocks(k, threads);
  static thread_local DVec<double> part;
  if (part.n < blocks || part.s != c.s) part.alloc(blocks, c.s);
  int* sw = c.dflag + 30;
  CSRv av = a;
  const int64_t* prp = cl.rp.p;
  const int32_t* pcol = cl.col.p;
  const double* pval = cl.val.p;
  const double* pdiag = cl.diag.p;
  const int32_t* rid = cl.row_ids.p;
  const int32_t* cptr = (const int32_t*)(cl.rp.p + a.n + 1);
  int32_t nc = cl.ncolors;
  double* pp = part.p;
  const int32_t* hv = cl.heavy.p;
  const int32_t* hp = cl.hptr.p;
  const int32_t* hn = cl.heavy_nat.p;
  int32_t nhn = cl.nheavy_nat;
  void* args[] = {&av, (void*)&prp, (void*)&pcol, (void*)&pval, (void*)&pdiag, (void*)&rid, (void*)&cptr, &nc,
                  (void*)&hv, (void*)&hp, (void*)&hn, &nhn, (void*)&b, &x, &r, &pp, &sw};
  coop_launch(c, k, blocks, threads, args);
  return read_i32(c, sw);
}

// Rows [0, cn) of the inverse of each bordered LU factor: x = Minv[:cn,:cn] b
// (rhs[cn] = 0). One thread per unit right-hand side.
__global__ void lu_inverse_kernel(const double* M, const int32_t* perm, int32_t N, double* inv, double* work) {
  int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  const int32_t cn = N - 1;
  if (j >= cn) return;
  double* y = work + (int64_t)j * N;
  for (int32_t i = 0; i < N; ++i) {
    double s = perm[i] == j ? 1.0 : 0.0;
    for (int32_t k = 0; k < i; ++k) s -= M[(int64_t)i * N + k] * y[k];
    y[i] = s;
  }
  for (int32_t i = N; i-- > 0;) {
    double s = y[i];
    for (int32_t k = i + 1; k < N; ++k) s -= M[(int64_t)i * N + k] * y[k];
    y[i] = s / M[(int64_t)i * N + i];
  }
  for (int32_t i = 0; i < cn; ++i) inv[(int64_t)i * cn + j] = y[i];
}

void build_direct_inverse(Ctx& c, DDirect& d) {
  if (d.inv.n) return;
  std::vector<int64_t> off = d.lu_off.to_host();
  std::vector<int32_t> start = d.comp_start.to_host();
  int64_t total = 0;
  std::vector<int64_t> ioff(d.ncomp);
  for (int32_t ci = 0; ci < d.ncomp; ++ci) {
    ioff[ci] = total;
    total += (int64_t)d.comp_size[ci] * d.comp_size[ci];
  }
  d.inv.alloc(std::max<int64_t>(total, 1), c.s);
  DVec<double> work((int64_t)d.maxN * d.maxN + 1, c.s);
  for (int32_t ci = 0; ci < d.ncomp; ++ci) {
    const int32_t N = d.comp_size[ci] + 1;
    count_launch(), lu_inverse_kernel<<<blocks_for(N, 128), 128, 0, c.s>>>(d.lu.p + off[ci], d.perm.p + start[ci] + ci, N,
                                                                   d.inv.p + ioff[ci], work.p);
    CK_LAUNCH();
    c.sync();
  }
  // the inverse kernel indexes per component through lu_off: store inverse
  // offsets in place of the LU offsets for the throughput solve
  d.inv_off.alloc(d.ncomp, c.s);
  d.inv_off.upload(ioff.data(), d.ncomp);
  c.sync();
}

void prepare_throughput(Ctx& c, DHier& h) {
  for (size_t l = 0; l < h.levels.size(); ++l) {
    DLevel& L = *h.levels[l];
    const bool smooths = (L.coarsest == CM_RELAX) ||
                         (L.coarsest == CM_NONE && l + 1 < h.levels.size() && h.levels[l + 1]->kind == KIND_AGG);
    if (smooths && !L.color) {
      auto col = std::make_unique<DColor>();
      build_coloring(c, L.op.view(), L.sched, *col);
      // append the colour pointers after rp for the single-CTA kernel
      DVec<int64_t> rp2(L.op.n + 1 + (col->ncolors + 2) / 2 + 1, c.s);
      CK(cudaMemcpyAsync(rp2.p, col->rp.p, sizeof(int64_t) * (L.op.n + 1), cudaMemcpyDeviceToDevice, c.s));
      CK(cudaMemcpyAsync(rp2.p + L.op.n + 1, col->cptr_h.data(), sizeof(int32_t) * (col->ncolors + 1),
                         cudaMemcpyHostToDevice, c.s));
      col->rp = std::move(rp2);
      L.color = std::move(col);
    }
    if (L.direct) build_direct_inverse(c, *L.direct);
    std::vector<int64_t> nrp((size_t)L.op.n + 1);
    L.op.rp.download(nrp.data(), L.op.n + 1);
    c.sync();
    build_long_rows(c, nrp, std::vector<int32_t>{0, L.op.n}, L.blong_nat);
  }
  c.sync();
}

}  // namespace lamgb
