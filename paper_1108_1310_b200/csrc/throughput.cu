// throughput.cu -- THROUGHPUT-mode smoother: greedy colouring, colour-
// permuted operator copies, coloured Gauss-Seidel, and the coarsest inverse.
//
// The hierarchy (every integer artefact and coarse value) is the bit-exact
// VALIDATE-mode one; only the solve's smoother order and its reductions
// change.
#include <algorithm>

#include <cuda/atomic>

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

static void build_coloring_from(Ctx& c, const CSRv& a, DVec<int32_t>& color, DColor& out);

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
  build_coloring_from(c, a, color, out);
}

// Front-modulo colouring (LAMG_FRONT_MOD=C, default 32) of the finest smoothing level for
// K-column blocks: colour(u) = front(u) mod C, where front(u) is u's wavefront in the
// exact-order schedule. A row of colour c sees its lower neighbours (front f - 1: colour
// c - 1) already swept and its upper neighbours (front f + 1: colour c + 1) not yet, exactly
// as the reference order does, except at the wrap (colours 0 and C - 1) -- a multicolour
// sweep that deviates from the reference's row order on 2/C of the rows, run as C
// bandwidth-bound launches instead of one latency-bound step per front. Measured on config
// 2 and 3D 64^3 (32 right-hand sides each, C = 16 ... 128): the per-column cycle counts of the
// exact-order sweep (min / max / mean 122 / 144 / 135.6 and 76 / 134 / 118.5), where the
// greedy two-colour sweep needs 141 for the reference's 129. Valid only when no two
// adjacent rows share a colour (front numbers of neighbours never differ by a multiple of
// C); returns false otherwise and the level keeps the exact-order sweep (bgs_exact).
__global__ void front_mod_color_kernel(const int32_t* __restrict__ front_ptr, const int32_t* __restrict__ rows,
                                       int32_t nfronts, int32_t C, int32_t* color) {
  const int32_t f = blockIdx.x;
  for (int32_t i = front_ptr[f] + threadIdx.x; i < front_ptr[f + 1]; i += blockDim.x) color[rows[i]] = f % C;
}
__global__ void color_conflict_kernel(CSRv a, const int32_t* __restrict__ color, int32_t* flag) {
  const int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= a.n) return;
  const int32_t cu = color[u];
  for (int64_t k = a.rp[u]; k < a.rp[u + 1]; ++k)
    if (color[a.col[k]] == cu) *flag = 1;
}
bool build_front_mod_coloring(Ctx& c, const CSRv& a, const Schedule& sch, int C, DColor& out) {
  const int32_t n = a.n;
  if (n == 0 || sch.nfronts < 2 || C < 2) return false;
  C = std::min<int>(C, sch.nfronts);
  DVec<int32_t> color(n, c.s);
  count_launch(), front_mod_color_kernel<<<sch.nfronts, 256, 0, c.s>>>(sch.front_ptr.p, sch.rows.p, sch.nfronts, C,
                                                                      color.p);
  int32_t* flag = c.dflag + 50;
  CK(cudaMemsetAsync(flag, 0, sizeof(int32_t), c.s));
  count_launch(), color_conflict_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(a, color.p, flag);
  CK_LAUNCH();
  if (read_i32(c, flag) != 0) return false;
  build_coloring_from(c, a, color, out);
  return true;
}

static void build_coloring_from(Ctx& c, const CSRv& a, DVec<int32_t>& color, DColor& out) {
  const int32_t n = a.n;
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
  static const int64_t chunk = [] {
    const char* e = getenv("LAMG_CHUNK");
    return e ? std::max<int64_t>(256, atoll(e)) : (int64_t)1024;
  }();
  L.chunk = chunk;
  std::vector<int32_t> rows, irow, ichunk, isrow, srows, sitem0;
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
      if (len <= chunk) {
        rows.push_back(i);
      } else {
        sitem0.push_back((int32_t)irow.size());
        for (int64_t q = 0; q * chunk < len; ++q) {
          irow.push_back(i);
          ichunk.push_back((int32_t)q);
          isrow.push_back((int32_t)srows.size());
        }
        srows.push_back(i);
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
  up(L.item_srow, isrow);
  up(L.srows, srows);
  up(L.sitem0, sitem0);
  up(L.ptr_d, L.ptr_h);
  up(L.iptr_d, L.iptr_h);
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
    for (int32_t cc = 0; cc < cl.ncolors; ++cc) gs_colored_one(c, cl, b, x, cc);
}

// the launches of one colour of a coloured sweep (per-colour form of gs_colored)
void gs_colored_one(Ctx& c, const DColor& cl, const double* b, double* x, int32_t cc) {
  const int32_t i0 = cl.cptr_h[cc], i1 = cl.cptr_h[cc + 1];
  if (i1 <= i0) return;
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
  CK_LAUNCH();
}

// RelaxationSolver::solve (coarse_solver.cpp:82-93) for THROUGHPUT mode in
// ONE cooperative launch: coloured sweeps separated by grid barriers, fixed-
// order tree reductions, the convergence test on the device. Power-law
// hierarchies end in a multi-million-row relaxation coarsest with hundreds of
// colours and hub rows of 10^5 entries; host-driven that is a launch per
// colour plus a host round trip per sweep.
//
// Work per colour (and per residual) is a list of CTA tasks sized so that no
// task serialises a hub: chunk items of super-long rows (L.chunk entries,
// one CTA each), long rows (kLongRow < len <= chunk, a warp each, 8 per
// task), and blocks of short rows (G lanes per row). A super-long row's
// chunk partials are summed in chunk order -- in a GS phase by the CTA that
// finishes the row's last chunk (acquire/release counter), in a residual
// after the phase barrier. The high colours of a power-law level hold only a
// few hub rows, so a phase is one chunk task long: each CTA loads its first
// task's entries of the next phase BEFORE the barrier; after the barrier
// only the x gathers remain on the critical path.
struct RelaxOp {
  const int64_t* rp;  // [n+1] (stored order for the coloured operator)
  const int32_t* col;
  const double* val;
  const double* diag;     // diag of each stored row
  const int32_t* row_ids; // stored row -> natural row (nullptr: identity)
  const int32_t* cptr;    // [ncolors+1] colour ranges (natural operator: {0, n})
  int32_t ncolors;
  // LongRows lists (per colour)
  const int32_t* lrows;
  const int32_t* lptr;
  const int32_t* item_row;
  const int32_t* item_chunk;
  const int32_t* item_srow;
  const int32_t* iptr;
  const int32_t* sitem0;
  const int32_t* srows;
  int32_t nsrows;
  uint32_t* cnt;
  double* ipart;  // per item partial sums
  int64_t chunk;
};

constexpr int kRT = 256;   // threads per CTA of the cooperative relaxation
constexpr int kRU = 4;     // entries per thread per round of a chunk task

// a CTA's prefetched first chunk task of a phase (registers, per thread)
struct ChunkPre {
  int64_t t = -1;  // task index in the phase (-1: none)
  int64_t ce = 0;
  int32_t c[kRU];
  double v[kRU];
};

__device__ __forceinline__ void chunk_bounds(const RelaxOp& o, int32_t it, int32_t* i, int64_t* cb, int64_t* ce) {
  *i = o.item_row[it];
  *cb = o.rp[*i] + (int64_t)o.item_chunk[it] * o.chunk;
  const int64_t e = o.rp[*i + 1];
  *ce = *cb + o.chunk < e ? *cb + o.chunk : e;
}

__device__ __forceinline__ void chunk_load(const RelaxOp& o, int64_t k0, int64_t ce, ChunkPre& p) {
#pragma unroll
  for (int j = 0; j < kRU; ++j) {
    const int64_t k = k0 + (int64_t)j * kRT;
    p.c[j] = k < ce ? __ldcs(o.col + k) : 0;
    p.v[j] = k < ce ? __ldcs(o.val + k) : 0.0;
  }
}

// CTA sum of val*x over [cb, ce) whose first round (entries cb + tid + j*kRT)
// is already in p; fixed order: strided per thread, warp tree, warps in order
__device__ __forceinline__ double chunk_dot(const RelaxOp& o, const double* x, int64_t cb, int64_t ce,
                                            const ChunkPre& p) {
  __shared__ double sh_cd[kRT / 32 + 1];
  double acc = 0.0;
  {
    double xv[kRU];
#pragma unroll
    for (int j = 0; j < kRU; ++j) xv[j] = cb + threadIdx.x + (int64_t)j * kRT < ce ? x[p.c[j]] : 0.0;
#pragma unroll
    for (int j = 0; j < kRU; ++j) acc += p.v[j] * xv[j];
  }
  for (int64_t k0 = cb + threadIdx.x + (int64_t)kRU * kRT; k0 < ce; k0 += (int64_t)kRU * kRT) {
    ChunkPre q;
    chunk_load(o, k0, ce, q);
    double xv[kRU];
#pragma unroll
    for (int j = 0; j < kRU; ++j) xv[j] = k0 + (int64_t)j * kRT < ce ? x[q.c[j]] : 0.0;
#pragma unroll
    for (int j = 0; j < kRU; ++j) acc += q.v[j] * xv[j];
  }
  for (int s = 16; s > 0; s >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, s);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh_cd[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kRT / 32; ++w) t += sh_cd[w];
    sh_cd[kRT / 32] = t;
  }
  __syncthreads();
  return sh_cd[kRT / 32];
}

// GS chunk task: thread 0 of the CTA finishing row s's last chunk gets true
// and the row's off-diagonal sum (chunk order)
__device__ __forceinline__ bool chunk_finish(const RelaxOp& o, int32_t it, double p, double* tot) {
  if (threadIdx.x != 0) return false;
  o.ipart[it] = p;
  const int32_t s = o.item_srow[it];
  const int32_t j0 = o.sitem0[s], j1 = o.sitem0[s + 1];
  cuda::atomic_ref<uint32_t, cuda::thread_scope_device> cnt(o.cnt[s]);
  const uint32_t old = cnt.fetch_add(1u, cuda::memory_order_acq_rel);
  if (old + 1 != (uint32_t)(j1 - j0)) return false;
  // the last chunk of the row: reset the counter for the next phase (nothing
  // else touches it until a kernel boundary or grid barrier)
  o.cnt[s] = 0u;
  double t = 0.0;
  for (int32_t j = j0; j < j1; ++j) t += __ldcg(o.ipart + j);
  *tot = t;
  return true;
}

__device__ __forceinline__ int64_t phase_tasks(const RelaxOp& o, int32_t c, int G, int64_t* nit, int64_t* nlw) {
  *nit = o.iptr[c + 1] - o.iptr[c];
  *nlw = (o.lptr[c + 1] - o.lptr[c] + 7) / 8;  // long rows: a warp each, 8 per CTA task
  const int rpb = kRT / G;
  return *nit + *nlw + ((int64_t)(o.cptr[c + 1] - o.cptr[c]) + rpb - 1) / rpb;
}

// loads the first task of this CTA in phase c when it is a chunk item
__device__ __forceinline__ void phase_prefetch(const RelaxOp& o, int32_t c, int G, int32_t rot, ChunkPre& p) {
  int64_t nit, nlw;
  phase_tasks(o, c, G, &nit, &nlw);
  const int64_t t = ((int64_t)blockIdx.x + rot) % gridDim.x;
  p.t = -1;
  if (t < nit) {
    int32_t i;
    int64_t cb;
    chunk_bounds(o, o.iptr[c] + (int32_t)t, &i, &cb, &p.ce);
    chunk_load(o, cb + threadIdx.x, p.ce, p);
    p.t = t;
  }
}

// One colour c: GS update (x_u = (b_u - dot)/d) or residual (r_u = b_u -
// (d x_u + dot); super-long rows are left to residual_finish).
template <int G, bool GS>
__device__ void relax_phase(const RelaxOp& o, int32_t c, const double* __restrict__ b, double* x, double* r,
                            int32_t rot, const ChunkPre& pre) {
  constexpr int RPB = kRT / G;  // short rows per CTA task
  int64_t nit, nlw;
  const int64_t T = phase_tasks(o, c, G, &nit, &nlw);
  const int32_t i0 = o.cptr[c], i1 = o.cptr[c + 1];
  const int32_t it0 = o.iptr[c];
  const int32_t l0 = o.lptr[c], nl = o.lptr[c + 1] - l0;
  const int64_t start = ((int64_t)blockIdx.x + rot) % gridDim.x;
  for (int64_t t = start; t < T; t += gridDim.x) {
    if (t < nit) {
      const int32_t it = it0 + (int32_t)t;
      int32_t i;
      int64_t cb, ce;
      chunk_bounds(o, it, &i, &cb, &ce);
      double p;
      if (t == pre.t) {
        p = chunk_dot(o, x, cb, ce, pre);
      } else {
        ChunkPre q;
        chunk_load(o, cb + threadIdx.x, ce, q);
        p = chunk_dot(o, x, cb, ce, q);
      }
      if (GS) {
        double dot;
        if (chunk_finish(o, it, p, &dot)) {
          const int32_t u = o.row_ids ? o.row_ids[i] : i;
          x[u] = (b[u] - dot) / o.diag[i];
        }
      } else if (threadIdx.x == 0) {
        o.ipart[it] = p;
      }
    } else if (t < nit + nlw) {
      const int64_t j = (t - nit) * 8 + (threadIdx.x >> 5);
      const bool ok = j < nl;
      const int32_t i = ok ? o.lrows[l0 + j] : 0;
      const double dot = group_dot<32, true>(o.col, o.val, x, ok ? o.rp[i] : 0, ok ? o.rp[i + 1] : 0);
      if (ok && (threadIdx.x & 31) == 0) {
        const int32_t u = o.row_ids ? o.row_ids[i] : i;
        if (GS) x[u] = (b[u] - dot) / o.diag[i];
        else r[u] = b[u] - (o.diag[i] * x[u] + dot);
      }
    } else {
      const int64_t i = i0 + (t - nit - nlw) * RPB + threadIdx.x / G;
      const bool ok = i < i1 && o.rp[i + 1] - o.rp[i] <= kLongRow;
      const double dot = group_dot<G, true>(o.col, o.val, x, ok ? o.rp[i] : 0, ok ? o.rp[i + 1] : 0);
      if (ok && (threadIdx.x & (G - 1)) == 0) {
        const int32_t u = o.row_ids ? o.row_ids[i] : (int32_t)i;
        if (GS) x[u] = (b[u] - dot) / o.diag[i];
        else r[u] = b[u] - (o.diag[i] * x[u] + dot);
      }
    }
  }
}

// after the residual phase's barrier: super-long rows of the natural
// operator from their chunk partials (chunk order); returns this thread's
// share of sum r^2 over those rows
__device__ __forceinline__ double residual_finish(const RelaxOp& o, const double* __restrict__ b, const double* x,
                                                  double* r) {
  double loc = 0.0;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < o.nsrows;
       s += (int64_t)gridDim.x * blockDim.x) {
    double t = 0.0;
    for (int32_t j = o.sitem0[s]; j < o.sitem0[s + 1]; ++j) t += __ldcg(o.ipart + j);
    const int32_t u = o.srows[s];
    const double ru = b[u] - (o.diag[u] * x[u] + t);
    r[u] = ru;
    loc += ru * ru;
  }
  return loc;
}

// grid-wide sum: block partials, then every block folds all partials in the
// same fixed order (strided per thread, then a fixed block tree), so every
// thread of the grid gets the identical value
__device__ inline double coop_sum(double v, double* part) {
  __shared__ double sh[kRT];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kRT / 32; ++w) t += sh[w];
    part[blockIdx.x] = t;
  }
  cg::this_grid().sync();
  double t = 0.0;
  for (unsigned g = threadIdx.x; g < gridDim.x; g += kRT) t += __ldcg(part + g);
  sh[threadIdx.x] = t;
  __syncthreads();
  for (int w = kRT / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  t = sh[0];
  cg::this_grid().sync();
  return t;
}

// residual of the natural operator and its squared norm (super-long rows
// finished after the barrier; the sum skips them in the row loop)
template <int G>
__device__ double relax_residual_norm2(const RelaxOp& no, int32_t n, const double* __restrict__ b, const double* x,
                                       double* r, double* part) {
  ChunkPre none;
  relax_phase<G, false>(no, 0, b, const_cast<double*>(x), r, 0, none);
  cg::this_grid().sync();
  double loc = residual_finish(no, b, x, r);
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x)
    if (no.rp[u + 1] - no.rp[u] <= no.chunk) loc += r[u] * r[u];
  return coop_sum(loc, part);
}

template <int G>
__global__ void __launch_bounds__(kRT) relax_coop_kernel(RelaxOp po, RelaxOp no, int32_t n,
                                                         const double* __restrict__ b, double* x, double* r,
                                                         double* part, int* sweeps_out, uint64_t* tstamp) {
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  const double r0 = sqrt(relax_residual_norm2<G>(no, n, b, x, r, part));
  if (tstamp && gtid == 0) reinterpret_cast<double*>(tstamp)[po.ncolors + 3 + 64] = r0;
  int sweeps = 0;
  if (r0 != 0.0) {
    const double target = 1e-12 * r0;
    if (tstamp && gtid == 0) tstamp[po.ncolors + 2] = globaltimer_ns();
    ChunkPre pre;
    for (int sweep = 0; sweep < 400; ++sweep) {
      int32_t rot = 0;
      phase_prefetch(po, 0, G, rot, pre);
      for (int32_t cc = 0; cc < po.ncolors; ++cc) {
        relax_phase<G, true>(po, cc, b, x, r, rot, pre);
        // the next phase starts where this one's longest tasks did not
        rot += (po.iptr[cc + 1] - po.iptr[cc]) + (po.lptr[cc + 1] - po.lptr[cc] + 7) / 8;
        if (cc + 1 < po.ncolors) phase_prefetch(po, cc + 1, G, rot, pre);
        cg::this_grid().sync();
        if (tstamp && sweep == 0 && gtid == 0) tstamp[cc] = globaltimer_ns();
      }
      if (tstamp && sweep == 0 && gtid == 0) tstamp[po.ncolors] = globaltimer_ns();
      double loc = 0.0;
      for (int64_t u = gtid; u < n; u += gstride) loc += x[u];
      const double mean = coop_sum(loc, part) / (double)n;
      for (int64_t u = gtid; u < n; u += gstride) x[u] = x[u] - mean;
      cg::this_grid().sync();
      const double rn = sqrt(relax_residual_norm2<G>(no, n, b, x, r, part));
      if (tstamp && sweep == 0 && gtid == 0) tstamp[po.ncolors + 1] = globaltimer_ns();
      if (tstamp && sweep < 64 && gtid == 0) reinterpret_cast<double*>(tstamp)[po.ncolors + 3 + sweep] = rn;
      ++sweeps;
      if (rn <= target) break;
    }
  }
  if (gtid == 0) *sweeps_out = sweeps;
}

static RelaxOp relax_op(const int64_t* rp, const int32_t* col, const double* val, const double* diag,
                        const int32_t* row_ids, const int32_t* cptr, int32_t ncolors, const LongRows& L,
                        double* ipart, uint32_t* cnt) {
  return RelaxOp{rp, col, val, diag, row_ids, cptr, ncolors, L.rows.p, L.ptr_d.p, L.item_row.p, L.item_chunk.p,
                 L.item_srow.p, L.iptr_d.p, L.sitem0.p, L.srows.p, L.sptr_h.back(), cnt, ipart, L.chunk};
}

// per-context scratch of the task kernels: chunk partials and row counters
// (zeroed when allocated; every completed row resets its counter)
static void relax_scratch(Ctx& c, int64_t nitems, int64_t nrows) {
  if (c.ripart.n < std::max<int64_t>(nitems, 1)) {
    c.ripart.alloc(std::max<int64_t>(nitems, 1), c.s);
    ++c.rgen;
  }
  if (c.rcnt.n < std::max<int64_t>(nrows, 1)) {
    c.rcnt.alloc(std::max<int64_t>(nrows, 1), c.s);
    c.rcnt.zero();
    ++c.rgen;
  }
}

// One launch per colour (and per residual): a CTA per task, so the hardware
// scheduler keeps every SM full with short tasks at full occupancy instead of
// a co-resident grid walking its task list serially.
template <int G, bool GS>
__global__ void __launch_bounds__(kRT) relax_task_kernel(RelaxOp o, int32_t c, const double* __restrict__ b,
                                                         double* x, double* r) {
  ChunkPre none;
  relax_phase<G, GS>(o, c, b, x, r, 0, none);
}
__global__ void relax_resfin_kernel(RelaxOp no, const double* __restrict__ b, const double* x, double* r) {
  residual_finish(no, b, x, r);
}

static int64_t phase_tasks_h(const std::vector<int32_t>& cptr, const LongRows& L, int32_t c, int G) {
  const int rpb = kRT / G;
  return (int64_t)(L.iptr_h[c + 1] - L.iptr_h[c]) + (L.ptr_h[c + 1] - L.ptr_h[c] + 7) / 8 +
         ((int64_t)(cptr[c + 1] - cptr[c]) + rpb - 1) / rpb;
}

// THROUGHPUT residual r = b - A x of an operator with long rows (power-law
// levels): the relaxation's residual tasks (chunked hubs, warp long rows,
// short-row blocks), super-long rows finished from their chunk partials.
int residual_tasks_group(const CSRv& a, const LongRows& nat) {
  return row_group_for(a.n, a.m) == 8 || nat.ptr_h.back() > 0 ? 8 : 1;
}

void residual_tasks(Ctx& c, const CSRv& a, const LongRows& nat, const double* b, const double* x, double* r,
                    int group) {
  if (a.n == 0) return;
  const int G = group > 0 ? group : residual_tasks_group(a, nat);
  DVec<double>& ipart = c.rtpart;
  const int64_t nitems = std::max<int64_t>(1, (int64_t)nat.iptr_h.back());
  if (ipart.n < nitems) ipart.alloc(nitems, c.s);
  DVec<int32_t>& cp = c.rtcptr;
  if (cp.n < 2 || cp.s != c.s) cp.alloc(2, c.s);
  if (c.rtcptr_n != a.n) {
    const int32_t ncp[2] = {0, a.n};
    cp.upload(ncp, 2);
    c.rtcptr_n = a.n;
  }
  // a residual never finishes rows in place (residual_finish), so no counters
  const RelaxOp no = relax_op(a.rp, a.col, a.val, a.diag, nullptr, cp.p, 1, nat, ipart.p, nullptr);
  const std::vector<int32_t> nptr = {0, a.n};
  const int64_t T = phase_tasks_h(nptr, nat, 0, G);
  double* xm = const_cast<double*>(x);
  if (G == 8) count_launch(), relax_task_kernel<8, false><<<(unsigned)T, kRT, 0, c.s>>>(no, 0, b, xm, r);
  else count_launch(), relax_task_kernel<1, false><<<(unsigned)T, kRT, 0, c.s>>>(no, 0, b, xm, r);
  if (no.nsrows) count_launch(), relax_resfin_kernel<<<blocks_for(no.nsrows), kThreads, 0, c.s>>>(no, b, x, r);
  CK_LAUNCH();
}

// RelaxationSolver::solve (coarse_solver.cpp:82-93), THROUGHPUT, for large
// relaxation-coarsest levels: per sweep one CUDA graph (a task launch per
// colour, mean subtraction, residual, norm), the convergence test on the
// host after each sweep (one 8-byte read; a sweep is milliseconds here).
int relax_colored_graph(Ctx& c, const CSRv& a, const DColor& cl, const LongRows& nat, const double* b, double* x,
                        double* r) {
  const int G = cl.group == 8 ? 8 : 1;
  relax_scratch(c, (int64_t)cl.blong.iptr_h.back() + nat.iptr_h.back(), cl.blong.sptr_h.back());
  DVec<double>& ipart = c.ripart;
  DVec<int32_t>& nat_cptr = c.rcptr;
  if (nat_cptr.n < 2) {
    nat_cptr.alloc(2, c.s);
    ++c.rgen;
  }
  const int32_t ncp[2] = {0, a.n};
  nat_cptr.upload(ncp, 2);
  const RelaxOp po = relax_op(cl.rp.p, cl.col.p, cl.val.p, cl.diag.p, cl.row_ids.p,
                              (const int32_t*)(cl.rp.p + a.n + 1), cl.ncolors, cl.blong, ipart.p, c.rcnt.p);
  const RelaxOp no = relax_op(a.rp, a.col, a.val, a.diag, nullptr, nat_cptr.p, 1, nat,
                              ipart.p + cl.blong.iptr_h.back(), nullptr);
  const std::vector<int32_t> nptr = {0, a.n};
  double* nrm = c.dscal + 112;
  auto residual_norm = [&] {
    const int64_t T = phase_tasks_h(nptr, nat, 0, G);
    if (G == 8) count_launch(), relax_task_kernel<8, false><<<(unsigned)T, kRT, 0, c.s>>>(no, 0, b, x, r);
    else count_launch(), relax_task_kernel<1, false><<<(unsigned)T, kRT, 0, c.s>>>(no, 0, b, x, r);
    if (no.nsrows) count_launch(), relax_resfin_kernel<<<blocks_for(no.nsrows), kThreads, 0, c.s>>>(no, b, x, r);
    tree_norm2(c, r, a.n, nrm);
    CK_LAUNCH();
  };
  auto sweep = [&] {
    for (int32_t cc = 0; cc < cl.ncolors; ++cc) {
      const int64_t T = phase_tasks_h(cl.cptr_h, cl.blong, cc, G);
      if (T == 0) continue;
      if (G == 8) count_launch(), relax_task_kernel<8, true><<<(unsigned)T, kRT, 0, c.s>>>(po, cc, b, x, r);
      else count_launch(), relax_task_kernel<1, true><<<(unsigned)T, kRT, 0, c.s>>>(po, cc, b, x, r);
    }
    subtract_mean_tree(c, x, a.n);
    residual_norm();
  };
  residual_norm();
  const double r0 = read_scalar(c, nrm);  // tree_norm2 returns the norm
  if (getenv("LAMG_RELAX_TRACE")) {
    residual_exact(c, a, b, x, r, nullptr, 0);
    tree_norm2(c, r, a.n, nrm);
    const double rx = read_scalar(c, nrm);
    tree_norm2(c, b, a.n, nrm);
    const double nb = read_scalar(c, nrm);
    tree_norm2(c, x, a.n, nrm);
    const double nx = read_scalar(c, nrm);
    fprintf(stderr, "[relax] r0 tasks %.6e exact %.6e |b| %.6e |x| %.6e n %d\n", r0, rx, nb, nx, a.n);
  }
  if (r0 == 0.0) return 0;
  // the sweep graph is cached per context (its scratch pointers are the
  // context's), keyed by the colouring's uid, the natural operator, the
  // vectors and the scratch generation
  Ctx::RelaxGraph& g = c.relax_graph;
  if (!g.exec || g.key != cl.uid || g.op != a.val || g.b != b || g.x != x || g.r != r || g.gen != c.rgen) {
    if (g.exec) CK(cudaGraphExecDestroy(g.exec));
    g.exec = nullptr;
    const long long l0 = t_launches;
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(c.s, cudaStreamCaptureModeThreadLocal));
    sweep();
    CK(cudaStreamEndCapture(c.s, &graph));
    CK(cudaGraphInstantiate(&g.exec, graph, 0));
    CK(cudaGraphDestroy(graph));
    g.launches = t_launches - l0;
    g_launches -= g.launches;  // counted when the graph runs
    t_launches = l0;
    g.key = cl.uid, g.op = a.val, g.b = b, g.x = x, g.r = r, g.gen = c.rgen;
  }
  const double target = 1e-12 * r0;
  int sweeps = 0;
  static const bool nograph = getenv("LAMG_RELAX_NOGRAPH") != nullptr;
  for (; sweeps < 400;) {
    if (nograph) {
      sweep();
    } else {
      CK(cudaGraphLaunch(g.exec, c.s));
      t_launches += g.launches;
      g_launches += g.launches;
    }
    ++sweeps;
    const double rn = read_scalar(c, nrm);
    if (getenv("LAMG_RELAX_TRACE")) fprintf(stderr, "[relax] sweep %d |r| %.6e (r0 %.6e)\n", sweeps, rn, r0);
    if (rn <= target) break;
  }
  return sweeps;
}

int relax_colored_coop(Ctx& c, const CSRv& a, const DColor& cl, const LongRows& nat, const double* b, double* x,
                       double* r) {
  const int threads = kRT;
  const void* k = cl.group == 8 ? (const void*)relax_coop_kernel<8> : (const void*)relax_coop_kernel<1>;
  int blocks = c.max_coop_blocks(k, threads);
  if (const char* e = getenv("LAMG_RELAX_BLOCKS")) blocks = std::max(1, std::min(blocks, atoi(e)));
  DVec<double>& part = c.rpart;
  if (part.n < blocks) part.alloc(blocks, c.s);
  relax_scratch(c, (int64_t)cl.blong.iptr_h.back() + nat.iptr_h.back(), cl.blong.sptr_h.back());
  DVec<double>& ipart = c.ripart;
  DVec<int32_t>& nat_cptr = c.rcptr;
  if (nat_cptr.n < 2) {
    nat_cptr.alloc(2, c.s);
    ++c.rgen;
  }
  const int32_t ncp[2] = {0, a.n};
  nat_cptr.upload(ncp, 2);
  int* sw = c.dflag + 30;
  RelaxOp po = relax_op(cl.rp.p, cl.col.p, cl.val.p, cl.diag.p, cl.row_ids.p, (const int32_t*)(cl.rp.p + a.n + 1),
                        cl.ncolors, cl.blong, ipart.p, c.rcnt.p);
  RelaxOp no = relax_op(a.rp, a.col, a.val, a.diag, nullptr, nat_cptr.p, 1, nat,
                        ipart.p + cl.blong.iptr_h.back(), nullptr);
  int32_t n = a.n;
  double* pp = part.p;
  // LAMG_RELAX_TIMING=1 (diagnostic): device timestamps of the first sweep's
  // colour phases, printed as a summary on stderr
  static const bool timing = getenv("LAMG_RELAX_TIMING") && atoi(getenv("LAMG_RELAX_TIMING")) == 1;
  DVec<uint64_t> ts;
  uint64_t* tsp = nullptr;
  if (timing) {
    ts.alloc(cl.ncolors + 3 + 65, c.s);
    ts.zero();
    tsp = ts.p;
  }
  if (getenv("LAMG_RELAX_TRACE")) {
    residual_exact(c, a, b, x, r, nullptr, 0);
    double* nrm = c.dscal + 112;
    tree_norm2(c, r, a.n, nrm);
    const double rx = read_scalar(c, nrm);
    fprintf(stderr, "[relax coop] exact r0 %.6e blocks %d G %d ncolors %d n %d nsrows %d\n", rx, blocks,
            cl.group, cl.ncolors, a.n, no.nsrows);
  }
  void* args[] = {&po, &no, &n, (void*)&b, &x, &r, &pp, &sw, &tsp};
  coop_launch(c, k, blocks, threads, args);
  const int sweeps = read_i32(c, sw);
  if (timing) {
    std::vector<uint64_t> t = ts.to_host();
    const int nc = cl.ncolors;
    std::vector<double> d(nc);
    for (int i = 0; i < nc; ++i) d[i] = (double)(t[i] - (i ? t[i - 1] : t[nc + 2])) * 1e-3;
    std::vector<double> sd = d;
    std::sort(sd.begin(), sd.end());
    double tot = 0.0;
    for (double v : d) tot += v;
    fprintf(stderr, "[relax timing] blocks %d colours %d: GS phases total %.1f us (min %.2f med %.2f max %.2f), "
            "mean+residual %.1f us; items %d long rows %d\n", blocks, nc, tot, sd[0], sd[nc / 2], sd[nc - 1],
            (double)(t[nc + 1] - t[nc - 1]) * 1e-3, cl.blong.iptr_h.back(), cl.blong.ptr_h.back());
    fprintf(stderr, "[relax] r0 %.6e\n", reinterpret_cast<const double*>(t.data())[nc + 3 + 64]);
    for (int i = 0; i < std::min(sweeps, 64); ++i)
      fprintf(stderr, "[relax] sweep %d |r| %.6e\n", i + 1, reinterpret_cast<const double*>(t.data())[nc + 3 + i]);
    for (int i = 0; i < nc; i += std::max(1, nc / 16))
      fprintf(stderr, "  colour %d: %.2f us rows %d items %d long %d\n", i, d[i], cl.cptr_h[i + 1] - cl.cptr_h[i],
              cl.blong.iptr_h[i + 1] - cl.blong.iptr_h[i], cl.blong.ptr_h[i + 1] - cl.blong.ptr_h[i]);
  }
  return sweeps;
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

static void append_color_ptrs(Ctx& c, int32_t n, DColor& col);

void prepare_throughput(Ctx& c, DHier& h) {
  bool seen_smoother = false;  // the front-modulo colouring serves the finest smoothing level only
  for (size_t l = 0; l < h.levels.size(); ++l) {
    DLevel& L = *h.levels[l];
    const bool smooths = (L.coarsest == CM_RELAX) ||
                         (L.coarsest == CM_NONE && l + 1 < h.levels.size() && h.levels[l + 1]->kind == KIND_AGG);
    if (smooths && !L.color) L.color = make_color(c, L.op.view(), L.sched);
    static const int front_mod = [] {
      const char* e = getenv("LAMG_FRONT_MOD");
      return e ? atoi(e) : 32;  // 0 / 1: the level is swept in exact order (bgs_exact, wavefront kernels) instead
    }();
    if (smooths && L.coarsest == CM_NONE && front_mod > 1 && !L.fcolor && !seen_smoother) {
      auto fc = std::make_unique<DColor>();
      if (build_front_mod_coloring(c, L.op.view(), L.sched, front_mod, *fc)) {
        append_color_ptrs(c, L.op.n, *fc);
        L.fcolor = std::move(fc);
      }
    }
    if (smooths) seen_smoother = true;
    if (smooths && L.coarsest == CM_NONE && !L.xitems[0].rows)
      for (int t = 0; t < kExactTables; ++t) build_exact_items(c, L.sched, 32 >> t, L.xitems[t]);
    if (L.direct) build_direct_inverse(c, *L.direct);
    build_natural_long_rows(c, L.op.view(), L.blong_nat);
  }
  c.sync();
}

// append the colour pointers after rp for the single-CTA kernels
static void append_color_ptrs(Ctx& c, int32_t n, DColor& col) {
  DVec<int64_t> rp2(n + 1 + (col.ncolors + 2) / 2 + 1, c.s);
  CK(cudaMemcpyAsync(rp2.p, col.rp.p, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToDevice, c.s));
  CK(cudaMemcpyAsync(rp2.p + n + 1, col.cptr_h.data(), sizeof(int32_t) * (col.ncolors + 1), cudaMemcpyHostToDevice,
                     c.s));
  col.rp = std::move(rp2);
  c.sync();
}

std::unique_ptr<DColor> make_color(Ctx& c, const CSRv& a, const Schedule& sch) {
  auto col = std::make_unique<DColor>();
  build_coloring(c, a, sch, *col);
  append_color_ptrs(c, a.n, *col);
  return col;
}

void build_exact_items(Ctx& c, const Schedule& sch, int32_t rows, ExactItems& out) {
  const std::vector<int32_t> fp = sch.front_ptr.to_host();
  std::vector<int32_t> fr, r0, r1, cnt(sch.nfronts, 0);
  for (int32_t f = 0; f < sch.nfronts; ++f)
    for (int32_t i = fp[f]; i < fp[f + 1]; i += rows) {
      fr.push_back(f);
      r0.push_back(i);
      r1.push_back(std::min(i + rows, fp[f + 1]));
      ++cnt[f];
    }
  out.rows = rows;
  out.nitems = (int32_t)fr.size();
  out.nfronts = sch.nfronts;
  out.front.alloc(std::max<int64_t>(1, out.nitems), c.s);
  out.r0.alloc(std::max<int64_t>(1, out.nitems), c.s);
  out.r1.alloc(std::max<int64_t>(1, out.nitems), c.s);
  out.count.alloc(std::max(1, sch.nfronts), c.s);
  if (out.nitems) {
    out.front.upload(fr.data(), out.nitems);
    out.r0.upload(r0.data(), out.nitems);
    out.r1.upload(r1.data(), out.nitems);
    out.count.upload(cnt.data(), sch.nfronts);
  }
  c.sync();
}

void build_natural_long_rows(Ctx& c, const CSRv& a, LongRows& out) {
  std::vector<int64_t> nrp((size_t)a.n + 1);
  CK(cudaMemcpyAsync(nrp.data(), a.rp, sizeof(int64_t) * (a.n + 1), cudaMemcpyDeviceToHost, c.s));
  c.sync();
  build_long_rows(c, nrp, std::vector<int32_t>{0, a.n}, out);
}

}  // namespace lamgb
