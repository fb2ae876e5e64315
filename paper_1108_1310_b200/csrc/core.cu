// core.cu -- CSR residual, exact-order Gauss-Seidel, transfers, validation.
//
// Arithmetic follows the reference op-for-op (no FMA, left-to-right folds in
// the reference's order) so every kernel here is bit-identical to it.
#include <algorithm>
#include <cmath>

#include "core.cuh"

namespace lamgb {

// ------------------------------------------------------------- residual
// thread per row; the row fold runs in column order (sparse_laplacian.cpp:156-160)
__global__ void residual_exact_kernel(CSRv a, const double* __restrict__ b,
                                      const double* __restrict__ x, double* __restrict__ r, bool skip_heavy) {
  int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= a.n) return;
  if (skip_heavy && a.rp[u + 1] - a.rp[u] > kHeavyRowExact) return;
  double s = a.diag[u] * x[u];
  s = row_fold<8, false, true>(s, a.col, a.val, x, a.rp[u], a.rp[u + 1]);
  r[u] = b ? b[u] - s : s;
}

__global__ void residual_heavy_exact_kernel(CSRv a, const int32_t* heavy, const double* __restrict__ b,
                                            const double* __restrict__ x, double* __restrict__ r) {
  const int32_t u = heavy[blockIdx.x];
  const double s = block_seq_fold<false>(a.diag[u] * x[u], a.col, a.val, x, a.rp[u], a.rp[u + 1]);
  if (threadIdx.x == 0) r[u] = b ? b[u] - s : s;
}

__global__ void heavy_flag_rows_kernel(CSRv a, uint8_t* f) {
  int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u < a.n) f[u] = a.rp[u + 1] - a.rp[u] > kHeavyRowExact;
}

int32_t heavy_rows(Ctx& c, const CSRv& a, DVec<int32_t>& out) {
  out.alloc(std::max(a.n, 1), c.s);
  if (a.n == 0) return 0;
  DVec<uint8_t> f(a.n, c.s);
  count_launch(), heavy_flag_rows_kernel<<<blocks_for(a.n), kThreads, 0, c.s>>>(a, f.p);
  CK_LAUNCH();
  return (int32_t)select_flagged_index(c, f.p, out.p, a.n);
}

void residual_exact(Ctx& c, const CSRv& a, const double* b, const double* x, double* r, const int32_t* heavy,
                    int32_t nheavy) {
  if (a.n == 0) return;
  count_launch(), residual_exact_kernel<<<blocks_for(a.n), kThreads, 0, c.s>>>(a, b, x, r, nheavy > 0);
  if (nheavy) count_launch(), residual_heavy_exact_kernel<<<nheavy, 256, 0, c.s>>>(a, heavy, b, x, r);
  CK_LAUNCH();
}

// ------------------------------------------------------ GS wavefronts
__global__ void deps_kernel(CSRv a, bool backward, int32_t* cnt) {
  int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= a.n) return;
  // rows are sorted: the lower neighbours are the prefix below u
  int64_t lo = a.rp[u], hi = a.rp[u + 1];
  while (lo < hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (a.col[mid] < u) lo = mid + 1;
    else hi = mid;
  }
  const int64_t lower = lo - a.rp[u];
  cnt[u] = (int32_t)(backward ? (a.rp[u + 1] - a.rp[u]) - lower : lower);
}

__global__ void zero_dep_flags_kernel(const int32_t* cnt, int32_t n, uint8_t* flag) {
  int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u < n) flag[u] = cnt[u] == 0;
}

// Kahn's algorithm, one grid barrier per front: finishing a row releases its
// later neighbours; a row joins the next front when its last earlier
// neighbour finishes.
__global__ void kahn_kernel(CSRv a, bool backward, int32_t* cnt, int32_t* level, int32_t* queue,
                            int32_t* ctl /* [0]=tail, [1]=nfronts */, int32_t first_count) {
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  // one warp per finished row: hubs release their many later neighbours
  // with 32 lanes instead of one thread
  const int64_t gwarp = gtid >> 5, nwarps = gstride >> 5;
  const int lane = threadIdx.x & 31;
  int32_t fs = 0, fe = first_count, r = 0;
  while (fs < fe) {
    // hubs (over kHeavyRowExact entries) release their neighbours with a whole CTA
    for (int64_t i = fs + blockIdx.x; i < fe; i += gridDim.x) {
      const int32_t u = queue[i];
      if (a.rp[u + 1] - a.rp[u] <= kHeavyRowExact) continue;
      if (threadIdx.x == 0) level[u] = r;
      for (int64_t k = a.rp[u] + threadIdx.x; k < a.rp[u + 1]; k += blockDim.x) {
        const int32_t v = a.col[k];
        const bool later = backward ? (v < u) : (v > u);
        if (later && atomicSub(&cnt[v], 1) == 1) queue[atomicAdd(&ctl[0], 1)] = v;
      }
    }
    for (int64_t i = fs + gwarp; i < fe; i += nwarps) {
      int32_t u = queue[i];
      if (a.rp[u + 1] - a.rp[u] > kHeavyRowExact) continue;
      if (lane == 0) level[u] = r;
      for (int64_t k = a.rp[u] + lane; k < a.rp[u + 1]; k += 32) {
        int32_t v = a.col[k];
        bool later = backward ? (v < u) : (v > u);
        if (later && atomicSub(&cnt[v], 1) == 1) queue[atomicAdd(&ctl[0], 1)] = v;
      }
    }
    grid_barrier();
    fs = fe;
    fe = *(volatile int32_t*)&ctl[0];
    ++r;
    grid_barrier();
  }
  if (gtid == 0) ctl[1] = r;
}

__global__ void front_bounds_kernel(const uint32_t* lvl_sorted, int32_t n, int32_t* front_ptr,
                                    int32_t nfronts) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (i == 0 || lvl_sorted[i] != lvl_sorted[i - 1]) front_ptr[lvl_sorted[i]] = i;
  if (i == 0) front_ptr[nfronts] = n;
}

__global__ void heavy_pos_kernel(CSRv a, const int32_t* rows, int32_t n, uint8_t* f) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) f[i] = a.rp[rows[i] + 1] - a.rp[rows[i]] > kHeavyRowExact;
}

__global__ void iota_kernel(int32_t* x, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) x[i] = (int32_t)i;
}

void build_schedule(Ctx& c, const CSRv& a, bool backward, Schedule& out) {
  const int32_t n = a.n;
  out.nfronts = 0;
  out.max_width = 0;
  if (n == 0) return;
  DVec<int32_t> cnt(n, c.s), level(n, c.s), queue(n, c.s);
  DVec<uint8_t> flag(n, c.s);
  count_launch(), deps_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(a, backward, cnt.p);
  count_launch(), zero_dep_flags_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(cnt.p, n, flag.p);
  CK_LAUNCH();
  int32_t first = (int32_t)select_flagged_index(c, flag.p, queue.p, n);
  int32_t* ctl = c.dflag + 8;
  int32_t init[2] = {first, 0};
  CK(cudaMemcpyAsync(ctl, init, sizeof init, cudaMemcpyHostToDevice, c.s));
  const int threads = 256;
  int blocks = std::min(c.max_coop_blocks((const void*)kahn_kernel, threads), blocks_for(n, threads));
  if (n < 4096) blocks = 1;
  CSRv av = a;
  bool bw = backward;
  void* args[] = {&av, &bw, &cnt.p, &level.p, &queue.p, &ctl, &first};
  coop_launch(c, (const void*)kahn_kernel, blocks, threads, args);
  int32_t nf = read_i32(c, ctl + 1);
  // rows sorted by (front, row): stable radix sort of the identity by front
  DVec<uint32_t> keys_out(n, c.s);
  DVec<int32_t> ids(n, c.s);
  count_launch(), iota_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(ids.p, n);
  CK_LAUNCH();
  out.rows.alloc(n, c.s);
  int bits = 1;
  while ((1u << bits) <= (uint32_t)nf && bits < 32) ++bits;
  sort_pairs_u32_i32(c, (const uint32_t*)level.p, keys_out.p, ids.p, out.rows.p, n, bits);
  out.front_ptr.alloc(nf + 1, c.s);
  count_launch(), front_bounds_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(keys_out.p, n, out.front_ptr.p, nf);
  CK_LAUNCH();
  out.nfronts = nf;
  std::vector<int32_t> fp = out.front_ptr.to_host();
  int32_t w = 0;
  for (int32_t f = 0; f < nf; ++f) w = std::max(w, fp[f + 1] - fp[f]);
  out.max_width = w;
  {
    std::vector<int64_t> rph((size_t)n + 1);
    CK(cudaMemcpyAsync(rph.data(), a.rp, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost, c.s));
    c.sync();
    int64_t ml = 0;
    for (int32_t u = 0; u < n; ++u) ml = std::max(ml, rph[u + 1] - rph[u]);
    out.max_len = ml;
  }
  // heavy rows in sweep order, grouped by front
  DVec<uint8_t> hf(n, c.s);
  count_launch(), heavy_pos_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(a, out.rows.p, n, hf.p);
  CK_LAUNCH();
  out.heavy.alloc(n, c.s);
  out.nheavy = (int32_t)select_flagged_index(c, hf.p, out.heavy.p, n);
  std::vector<int32_t> hp(nf + 1, 0);
  if (out.nheavy) {
    std::vector<int32_t> hv(out.nheavy);
    out.heavy.download(hv.data(), out.nheavy);
    c.sync();
    for (int32_t f = 0; f <= nf; ++f) hp[f] = (int32_t)(std::lower_bound(hv.begin(), hv.end(), fp[f]) - hv.begin());
  }
  out.heavy_ptr.alloc(nf + 1, c.s);
  out.heavy_ptr.upload(hp.data(), nf + 1);
  out.nheavy_nat = heavy_rows(c, a, out.heavy_nat);
  c.sync();
}

// One persistent launch per sweep set: rows of a front update in parallel,
// a grid barrier separates fronts. K-wide rows reuse the row's column and
// value loads for all K vectors.
__global__ void gs_fronts_kernel(CSRv a, const double* __restrict__ b, double* x, int K,
                                 const int32_t* __restrict__ front_ptr, const int32_t* __restrict__ rows,
                                 int32_t nfronts, int sweeps, int backward, DevErr* err,
                                 const int32_t* __restrict__ heavy, const int32_t* __restrict__ heavy_ptr) {
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  for (int sw = 0; sw < sweeps; ++sw) {
    for (int32_t f = 0; f < nfronts; ++f) {
      const int32_t fs = front_ptr[f], fe = front_ptr[f + 1];
      // heavy rows of this front: one CTA each, bit-exact sequential fold
      for (int32_t h = heavy_ptr[f] + blockIdx.x; h < heavy_ptr[f + 1]; h += gridDim.x) {
        const int32_t u = rows[heavy[h]];
        const double d = a.diag[u];
        for (int kk = 0; kk < K; ++kk) {
          const double s = block_seq_fold<true>(b ? b[(int64_t)u * K + kk] : 0.0, a.col, a.val, x, a.rp[u],
                                                a.rp[u + 1], K, kk);
          if (threadIdx.x == 0) {
            if (d != 0.0) x[(int64_t)u * K + kk] = s / d;
            else
              dev_report(err, backward ? (unsigned long long)(a.n - 1 - u) : (unsigned long long)u,
                         DE_GS_SINGULAR, u, 0);
          }
        }
      }
      // long rows of this front: a warp each (exact chain over shuffled products);
      // blockDim is a multiple of K, so only its full warps take part
      const int nfw = blockDim.x >> 5;
      const int64_t gw = (int64_t)blockIdx.x * nfw + (threadIdx.x >> 5);
      const bool full_warp = (int)(threadIdx.x >> 5) < nfw;
      for (int64_t i = fs + gw; full_warp && i < fe; i += (int64_t)gridDim.x * nfw) {
        const int32_t u = rows[i];
        const int64_t len = a.rp[u + 1] - a.rp[u];
        if (len <= kWarpRowExact || len > kHeavyRowExact) continue;
        const double d = a.diag[u];
        for (int kk = 0; kk < K; ++kk) {
          const double s = warp_seq_fold<true>(b ? b[(int64_t)u * K + kk] : 0.0, a.col, a.val, x, a.rp[u],
                                               a.rp[u + 1], K, kk);
          if ((threadIdx.x & 31) == 0) {
            if (d != 0.0) x[(int64_t)u * K + kk] = s / d;
            else
              dev_report(err, backward ? (unsigned long long)(a.n - 1 - u) : (unsigned long long)u,
                         DE_GS_SINGULAR, u, 0);
          }
        }
      }
      for (int64_t i = fs + gtid / K; i < fe; i += gstride / K) {
        const int kk = (int)(gtid % K);
        const int32_t u = rows[i];
        if (a.rp[u + 1] - a.rp[u] > kWarpRowExact) continue;
        double s = b ? b[(int64_t)u * K + kk] : 0.0;
        const int64_t e = a.rp[u + 1];
        if (K == 1) s = row_fold<8, true>(s, a.col, a.val, x, a.rp[u], e);
        else
          for (int64_t k = a.rp[u]; k < e; ++k) s = s - a.val[k] * x[(int64_t)a.col[k] * K + kk];
        const double d = a.diag[u];
        if (d == 0.0) {
          if (e != a.rp[u])
            dev_report(err, backward ? (unsigned long long)(a.n - 1 - u) : (unsigned long long)u,
                       DE_GS_SINGULAR, u, 0);
          continue;
        }
        x[(int64_t)u * K + kk] = s / d;
      }
      grid_barrier();
    }
  }
}

// Exact-order sweep of a level whose rows all fit one 8-entry round (grids:
// 7 entries), one column: each thread loads its row of the NEXT front (row
// id, bounds, the 8 column/value pairs, b, diag) before the grid barrier, so
// after it only the x gathers and the fold remain on the critical path.
constexpr int kLightRow = 8;
struct FrontRow {
  int32_t u;
  int32_t len;
  double bu, d;
  int32_t c[kLightRow];
  double v[kLightRow];
};
__device__ __forceinline__ void front_row_load(const CSRv& a, const double* b, const int32_t* rows, int64_t i,
                                               FrontRow& r) {
  r.u = rows[i];
  const int64_t k0 = a.rp[r.u];
  r.len = (int32_t)(a.rp[r.u + 1] - k0);
  r.bu = b ? b[r.u] : 0.0;
  r.d = a.diag[r.u];
#pragma unroll
  for (int j = 0; j < kLightRow; ++j) {
    const bool ok = j < r.len;
    r.c[j] = ok ? a.col[k0 + j] : 0;
    r.v[j] = ok ? a.val[k0 + j] : 0.0;
  }
}
__global__ void gs_fronts_light_kernel(CSRv a, const double* __restrict__ b, double* x,
                                       const int32_t* __restrict__ front_ptr, const int32_t* __restrict__ rows,
                                       int32_t nfronts, int sweeps, int backward, DevErr* err) {
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  FrontRow pre;
  bool have = false;
  auto prefetch = [&](int32_t f) {
    const int64_t i = front_ptr[f] + gtid;
    have = i < front_ptr[f + 1];
    if (have) front_row_load(a, b, rows, i, pre);
  };
  auto finish = [&](const FrontRow& r) {
    double xv[kLightRow];
#pragma unroll
    for (int j = 0; j < kLightRow; ++j) xv[j] = j < r.len ? x[r.c[j]] : 0.0;
    double s = r.bu;
#pragma unroll
    for (int j = 0; j < kLightRow; ++j)
      if (j < r.len) s = s - r.v[j] * xv[j];
    if (r.d == 0.0) {
      if (r.len)
        dev_report(err, backward ? (unsigned long long)(a.n - 1 - r.u) : (unsigned long long)r.u, DE_GS_SINGULAR,
                   r.u, 0);
      return;
    }
    x[r.u] = s / r.d;
  };
  if (nfronts > 0) prefetch(0);
  for (int sw = 0; sw < sweeps; ++sw) {
    for (int32_t f = 0; f < nfronts; ++f) {
      const int32_t fe = front_ptr[f + 1];
      if (have) finish(pre);
      for (int64_t i = front_ptr[f] + gtid + gstride; i < fe; i += gstride) {  // wide fronts
        FrontRow r;
        front_row_load(a, b, rows, i, r);
        finish(r);
      }
      if (f + 1 < nfronts) prefetch(f + 1);
      else if (sw + 1 < sweeps) prefetch(0);
      grid_barrier();
    }
  }
}

void gs_exact(Ctx& c, const CSRv& a, const Schedule& sch, const double* b, double* x, int K,
              int sweeps, bool backward, bool check) {
  if (a.n == 0 || sweeps <= 0) return;
  if (K == 1 && sch.max_len <= kLightRow && !getenv("LAMG_NO_LIGHT_FRONTS")) {
    const int threads = 256;
    int blocks = (int)std::min<int64_t>(c.max_coop_blocks((const void*)gs_fronts_light_kernel, threads),
                                        std::max<int64_t>(1, ((int64_t)sch.max_width + threads - 1) / threads));
    if (sch.max_width <= 2 * threads) blocks = 1;
    CSRv av = a;
    const int32_t* fp = sch.front_ptr.p;
    const int32_t* rw = sch.rows.p;
    int32_t nf = sch.nfronts;
    int bw = backward ? 1 : 0;
    void* args[] = {&av, (void*)&b, &x, (void*)&fp, (void*)&rw, &nf, &sweeps, &bw, &c.derr};
    if (check) c.checked([&] { coop_launch(c, (const void*)gs_fronts_light_kernel, blocks, threads, args); });
    else coop_launch(c, (const void*)gs_fronts_light_kernel, blocks, threads, args);
    return;
  }
  const int threads = 256;
  int64_t work = (int64_t)sch.max_width * K;
  int blocks = (int)std::min<int64_t>(c.max_coop_blocks((const void*)gs_fronts_kernel, threads),
                                      std::max<int64_t>(1, (work + threads - 1) / threads));
  // small fronts: a single CTA synchronises with __syncthreads only
  if (work <= 2 * threads) blocks = 1;
  CSRv av = a;
  const int32_t* fp = sch.front_ptr.p;
  const int32_t* rw = sch.rows.p;
  int32_t nf = sch.nfronts;
  int bw = backward ? 1 : 0;
  int t = (threads / K) * K;  // (row, k) pairs tile the grid exactly
  const int32_t* hv = sch.heavy.p;
  const int32_t* hp = sch.heavy_ptr.p;
  void* args[] = {&av, (void*)&b, &x, &K, (void*)&fp, (void*)&rw, &nf, &sweeps, &bw, &c.derr, (void*)&hv, (void*)&hp};
  if (check) c.checked([&] { coop_launch(c, (const void*)gs_fronts_kernel, blocks, t, args); });
  else coop_launch(c, (const void*)gs_fronts_kernel, blocks, t, args);
}

// ----------------------------------------------------------------- energy
__global__ void upper_flags_kernel(CSRv a, uint8_t* flag, int32_t* row_of) {
  int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= a.n) return;
  for (int64_t k = a.rp[u]; k < a.rp[u + 1]; ++k) {
    flag[k] = a.col[k] > u;
    row_of[k] = u;
  }
}
__global__ void gather_rows_kernel(const int64_t* entry, const int32_t* row_of, int64_t cnt,
                                   int32_t* out) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < cnt) out[j] = row_of[entry[j]];
}

void build_upper_index(Ctx& c, const CSRv& a, UpperIndex& out) {
  const int64_t nnz = 2 * a.m;
  out.entry.alloc(a.m, c.s);
  out.row.alloc(a.m, c.s);
  out.count = 0;
  if (nnz == 0) return;
  DVec<uint8_t> flag(nnz, c.s);
  DVec<int32_t> row_of(nnz, c.s);
  count_launch(), upper_flags_kernel<<<blocks_for(a.n), kThreads, 0, c.s>>>(a, flag.p, row_of.p);
  CK_LAUNCH();
  out.count = select_flagged_index64(c, flag.p, out.entry.p, nnz);
  count_launch(), gather_rows_kernel<<<blocks_for(out.count), kThreads, 0, c.s>>>(out.entry.p, row_of.p, out.count, out.row.p);
  CK_LAUNCH();
}

__global__ void energy_terms_kernel(CSRv a, const int64_t* entry, const int32_t* row, int64_t cnt,
                                    const double* __restrict__ x, double* t) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= cnt) return;
  int64_t k = entry[j];
  double d = x[row[j]] - x[a.col[k]];
  t[j] = -a.val[k] * d * d;
}

void energy_seq(Ctx& c, const CSRv& a, const UpperIndex& up, const double* x, double* d_out,
                DVec<double>& scratch) {
  if (scratch.n < up.count) scratch.alloc(up.count, c.s);
  if (up.count == 0) {
    CK(cudaMemsetAsync(d_out, 0, sizeof(double), c.s));
    return;
  }
  count_launch(), energy_terms_kernel<<<blocks_for(up.count), kThreads, 0, c.s>>>(a, up.entry.p, up.row.p, up.count, x, scratch.p);
  CK_LAUNCH();
  seq_sum(c, scratch.p, up.count, d_out);
}

// the same energy with a fixed-order tree sum of the terms (probe fast path)
void energy_tree(Ctx& c, const CSRv& a, const UpperIndex& up, const double* x, double* d_out,
                 DVec<double>& scratch) {
  if (scratch.n < up.count) scratch.alloc(up.count, c.s);
  if (up.count == 0) {
    CK(cudaMemsetAsync(d_out, 0, sizeof(double), c.s));
    return;
  }
  count_launch(), energy_terms_kernel<<<blocks_for(up.count), kThreads, 0, c.s>>>(a, up.entry.p, up.row.p, up.count, x, scratch.p);
  CK_LAUNCH();
  tree_sum(c, scratch.p, up.count, d_out);
}

// -------------------------------------------------------------------- rng
__device__ inline uint64_t splitmix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__global__ void fill_pm1_kernel(double* x, int64_t n, uint64_t s0, int stride, int offset) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t state = s0 + (uint64_t)(i + 3) * 0x9e3779b97f4a7c15ULL;
  double unit = (double)(splitmix(state) >> 11) * 0x1.0p-53;
  x[i * stride + offset] = 2.0 * unit - 1.0;
}
void fill_pm1(Ctx& c, double* x, int64_t n, uint64_t seed, int stride, int offset) {
  if (n == 0) return;
  uint64_t s0 = seed ? seed : 0x9e3779b97f4a7c15ULL;
  count_launch(), fill_pm1_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(x, n, s0, stride, offset);
  CK_LAUNCH();
}

// ------------------------------------------------------- mean subtraction
__global__ void sub_mean_kernel(double* x, int64_t n, int K, const double* sums) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n * K) return;
  int k = (int)(i % K);
  double mean = sums[k] / (double)n;
  x[i] = x[i] - mean;
}

void subtract_mean_seq(Ctx& c, double* x, int64_t n, int K) {
  if (n == 0) return;
  double* sums = c.dscal + 64;  // [64..80)
  if (K == 1) seq_sum(c, x, n, sums);
  else {
    seq_col_sums(c, x, n, K, sums);
  }
  count_launch(), sub_mean_kernel<<<blocks_for(n * K), kThreads, 0, c.s>>>(x, n, K, sums);
  CK_LAUNCH();
}

void subtract_mean_tree(Ctx& c, double* x, int64_t n) {
  if (n == 0) return;
  double* sums = c.dscal + 64;
  tree_sum(c, x, n, sums);
  count_launch(), sub_mean_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(x, n, 1, sums);
  CK_LAUNCH();
}

// ------------------------------------------------------------- validation
__global__ void abs_max_kernel(const double* __restrict__ d, int32_t n, unsigned long long* out) {
  __shared__ double sh[kThreads];
  double m = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs(d[i]));
  sh[threadIdx.x] = m;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) atomicMax(out, (unsigned long long)__double_as_longlong(sh[0]));
}

__device__ inline unsigned long long vkey(int32_t u, int64_t pos, int sub) {
  return ((unsigned long long)u << 32) | ((unsigned long long)pos << 3) | (unsigned long long)sub;
}

__global__ void validate_kernel(CSRv a, const unsigned long long* maxdiag_bits, DevErr* err) {
  int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= a.n) return;
  if (a.rp[u + 1] - a.rp[u] > kHeavyRowExact) return;  // validate_heavy_kernel
  const double md = __longlong_as_double((long long)*maxdiag_bits);
  const double tol = 1e-10 * (md < 1e-300 ? 1e-300 : md);
  double row_sum = a.diag[u];
  const int64_t b = a.rp[u], e = a.rp[u + 1];
  for (int64_t k = b; k < e; ++k) {
    const int32_t v = a.col[k];
    const int64_t pos = k - b;
    if (v == u) { dev_report(err, vkey(u, pos, 0), DE_VAL_SELF, u, v); return; }
    if (v < 0 || v >= a.n) { dev_report(err, vkey(u, pos, 1), DE_VAL_RANGE, u, v); return; }
    if (k > b && a.col[k - 1] >= v) { dev_report(err, vkey(u, pos, 2), DE_VAL_SORT, u, v); return; }
    int64_t lo = a.rp[v], hi = a.rp[v + 1];
    while (lo < hi) {
      int64_t mid = lo + (hi - lo) / 2;
      if (a.col[mid] < u) lo = mid + 1;
      else hi = mid;
    }
    if (lo == a.rp[v + 1] || a.col[lo] != u) { dev_report(err, vkey(u, pos, 3), DE_VAL_STRUCT, u, v); return; }
    if (a.val[lo] != a.val[k]) { dev_report(err, vkey(u, pos, 4), DE_VAL_VALUE, u, v); return; }
    row_sum = row_sum + a.val[k];
  }
  if (fabs(row_sum) > tol) { dev_report(err, vkey(u, e - b, 5), DE_VAL_ROWSUM, u, 0, row_sum); return; }
  if (e > b && a.diag[u] <= 0.0) dev_report(err, vkey(u, e - b, 6), DE_VAL_DIAG, u, 0);
}

// hub rows: one CTA per row; entry checks in parallel (the minimum key is
// the first failure, as in the sequential scan), row sum folded in order
__global__ void validate_heavy_kernel(CSRv a, const int32_t* heavy, const unsigned long long* maxdiag_bits,
                                      DevErr* err) {
  const int32_t u = heavy[blockIdx.x];
  const double md = __longlong_as_double((long long)*maxdiag_bits);
  const double tol = 1e-10 * (md < 1e-300 ? 1e-300 : md);
  const int64_t b = a.rp[u], e = a.rp[u + 1];
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int64_t k = b + threadIdx.x; k < e; k += blockDim.x) {
    const int32_t v = a.col[k];
    const int64_t pos = k - b;
    int kind = -1;
    if (v == u) kind = DE_VAL_SELF;
    else if (v < 0 || v >= a.n) kind = DE_VAL_RANGE;
    else if (k > b && a.col[k - 1] >= v) kind = DE_VAL_SORT;
    else {
      int64_t lo = a.rp[v], hi = a.rp[v + 1];
      while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (a.col[mid] < u) lo = mid + 1;
        else hi = mid;
      }
      if (lo == a.rp[v + 1] || a.col[lo] != u) kind = DE_VAL_STRUCT;
      else if (a.val[lo] != a.val[k]) kind = DE_VAL_VALUE;
    }
    if (kind >= 0) {
      dev_report(err, vkey(u, pos, kind - DE_VAL_SELF), kind, u, v);
      bad = 1;
    }
  }
  __syncthreads();
  if (bad) return;
  const double row_sum = block_seq_fold<false>(a.diag[u], a.col, a.val, nullptr, b, e);
  if (threadIdx.x != 0) return;
  if (fabs(row_sum) > tol) { dev_report(err, vkey(u, e - b, 5), DE_VAL_ROWSUM, u, 0, row_sum); return; }
  if (e > b && a.diag[u] <= 0.0) dev_report(err, vkey(u, e - b, 6), DE_VAL_DIAG, u, 0);
}

void validate_exact(Ctx& c, const CSRv& a) {
  if (a.n <= 0) throw LamgError(LAMG_E_INVALID_LAPLACIAN, "empty matrix");
  unsigned long long* md = (unsigned long long*)(c.dscal + 90);
  CK(cudaMemsetAsync(md, 0, sizeof(unsigned long long), c.s));
  count_launch(), abs_max_kernel<<<std::min(blocks_for(a.n), 1024), kThreads, 0, c.s>>>(a.diag, a.n, md);
  CK_LAUNCH();
  DVec<int32_t> heavy;
  const int32_t nh = heavy_rows(c, a, heavy);
  c.checked([&] {
    count_launch(), validate_kernel<<<blocks_for(a.n), kThreads, 0, c.s>>>(a, md, c.derr);
    if (nh) count_launch(), validate_heavy_kernel<<<nh, 256, 0, c.s>>>(a, heavy.p, md, c.derr);
    CK_LAUNCH();
  });
}

// -------------------------------------------------------------- transfers
__global__ void restrict_kernel(int32_t cn, const int64_t* __restrict__ mem_ptr,
                                const int32_t* __restrict__ mem, const double* __restrict__ r,
                                double mu, double* __restrict__ rc) {
  int32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= cn) return;
  double s = 0.0;
  for (int64_t j = mem_ptr[g]; j < mem_ptr[g + 1]; ++j) s = s + r[mem[j]];
  rc[g] = mu != 1.0 ? s * mu : s;
}
void restrict_exact(Ctx& c, int32_t coarse_n, const int64_t* mem_ptr, const int32_t* mem,
                    const double* r, double mu, double* rc) {
  if (coarse_n == 0) return;
  count_launch(), restrict_kernel<<<blocks_for(coarse_n), kThreads, 0, c.s>>>(coarse_n, mem_ptr, mem, r, mu, rc);
  CK_LAUNCH();
}

__global__ void interpolate_kernel(int32_t n, const int32_t* __restrict__ agg,
                                   const double* __restrict__ ec, double* __restrict__ x) {
  int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u < n) x[u] = x[u] + ec[agg[u]];
}
void interpolate(Ctx& c, int32_t fine_n, const int32_t* agg, const double* ec, double* x) {
  if (fine_n == 0) return;
  count_launch(), interpolate_kernel<<<blocks_for(fine_n), kThreads, 0, c.s>>>(fine_n, agg, ec, x);
  CK_LAUNCH();
}

__global__ void coarsen_rhs_kernel(StageV s, const double* __restrict__ b, double* __restrict__ bc) {
  int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= s.coarse_n) return;
  if (s.ntlong && s.t_ptr[k + 1] - s.t_ptr[k] > kLongT) return;  // coarsen_rhs_long_kernel
  double v = b[s.poc[k]];
  for (int64_t j = s.t_ptr[k]; j < s.t_ptr[k + 1]; ++j) {
    const int64_t p = s.t_p[j];
    const int32_t i = s.f_of_p[p];
    const double scaled = b[s.f_nodes[i]] / s.f_diag[i];
    v = v - s.f_val[p] * scaled;
  }
  bc[k] = v;
}
// coarse nodes with long contribution lists (hubs next to many eliminated
// nodes): one CTA each. The products f_val*(b_f/a_ff) are formed in parallel
// exactly as the sequential loop rounds them; VALIDATE folds them in (f, p)
// order with one thread (bit-exact), THROUGHPUT with a fixed block tree.
__global__ void coarsen_rhs_long_kernel(StageV s, const double* __restrict__ b, double* __restrict__ bc) {
  __shared__ double sh[kThreads];
  __shared__ double sh_v;
  const int32_t k = s.tlong[blockIdx.x];
  const int64_t j0 = s.t_ptr[k], j1 = s.t_ptr[k + 1];
  if (s.exact) {
    if (threadIdx.x == 0) sh_v = b[s.poc[k]];
    for (int64_t c0 = j0; c0 < j1; c0 += kThreads) {
      __syncthreads();
      const int64_t j = c0 + threadIdx.x;
      if (j < j1) {
        const int64_t p = s.t_p[j];
        const int32_t i = s.f_of_p[p];
        sh[threadIdx.x] = s.f_val[p] * (b[s.f_nodes[i]] / s.f_diag[i]);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        const int cnt = j1 - c0 < kThreads ? (int)(j1 - c0) : kThreads;
        double v = sh_v;
        for (int q = 0; q < cnt; ++q) v = v - sh[q];
        sh_v = v;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) bc[k] = sh_v;
    return;
  }
  double acc = 0.0;
  for (int64_t j = j0 + threadIdx.x; j < j1; j += kThreads) {
    const int64_t p = s.t_p[j];
    const int32_t i = s.f_of_p[p];
    acc += s.f_val[p] * (b[s.f_nodes[i]] / s.f_diag[i]);
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int w = kThreads / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) bc[k] = b[s.poc[k]] - sh[0];
}

void coarsen_rhs(Ctx& c, const StageV& s, const double* b, double* bc) {
  if (s.coarse_n == 0) return;
  count_launch(), coarsen_rhs_kernel<<<blocks_for(s.coarse_n), kThreads, 0, c.s>>>(s, b, bc);
  if (s.ntlong) count_launch(), coarsen_rhs_long_kernel<<<s.ntlong, kThreads, 0, c.s>>>(s, b, bc);
  CK_LAUNCH();
}

__global__ void long_t_flags_kernel(const int64_t* t_ptr, int32_t n, uint8_t* f) {
  const int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) f[k] = t_ptr[k + 1] - t_ptr[k] > kLongT;
}
int32_t stage_long_lists(Ctx& c, int32_t coarse_n, const int64_t* t_ptr, DVec<int32_t>& out) {
  out.alloc(std::max(coarse_n, 1), c.s);
  if (coarse_n == 0) return 0;
  DVec<uint8_t> f(coarse_n, c.s);
  count_launch(), long_t_flags_kernel<<<blocks_for(coarse_n), kThreads, 0, c.s>>>(t_ptr, coarse_n, f.p);
  CK_LAUNCH();
  return (int32_t)select_flagged_index(c, f.p, out.p, coarse_n);
}

__global__ void gather_kernel(double* dst, const double* src, const int32_t* idx, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}
__global__ void scatter_kernel(double* dst, const double* src, const int32_t* idx, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[idx[i]] = src[i];
}
void gather_d(Ctx& c, double* dst, const double* src, const int32_t* idx, int64_t n) {
  if (n == 0) return;
  count_launch(), gather_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(dst, src, idx, n);
  CK_LAUNCH();
}
void scatter_d(Ctx& c, double* dst, const double* src, const int32_t* idx, int64_t n) {
  if (n == 0) return;
  count_launch(), scatter_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(dst, src, idx, n);
  CK_LAUNCH();
}
void copy_d(Ctx& c, double* dst, const double* src, int64_t n) {
  if (n) CK(cudaMemcpyAsync(dst, src, sizeof(double) * (size_t)n, cudaMemcpyDeviceToDevice, c.s));
}

void inject(Ctx& c, const StageV& s, const double* x, double* xc) { gather_d(c, xc, x, s.poc, s.coarse_n); }

__global__ void backsub_f_kernel(StageV s, const double* __restrict__ b, double* x) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= s.nf) return;
  const int32_t f = s.f_nodes[i];
  double sum = b[f];
  for (int64_t p = s.f_ptr[i]; p < s.f_ptr[i + 1]; ++p) sum = sum - s.f_val[p] * x[s.f_nbr[p]];
  x[f] = sum / s.f_diag[i];
}
void backsub(Ctx& c, const StageV& s, const double* xc, const double* b, double* x) {
  scatter_d(c, x, xc, s.poc, s.coarse_n);
  if (s.nf == 0) return;
  count_launch(), backsub_f_kernel<<<blocks_for(s.nf), kThreads, 0, c.s>>>(s, b, x);
  CK_LAUNCH();
}

__global__ void stage_keys_kernel(int32_t nf, const int64_t* f_ptr, const int32_t* f_nbr,
                                  const int32_t* cop, uint32_t* key, int32_t* f_of_p) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nf) return;
  for (int64_t p = f_ptr[i]; p < f_ptr[i + 1]; ++p) {
    key[p] = (uint32_t)cop[f_nbr[p]];
    f_of_p[p] = i;
  }
}
__global__ void iota64_kernel(int64_t* x, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) x[i] = i;
}
__global__ void seg_bounds64_kernel(const uint64_t* sorted_key, int64_t n, int32_t nseg, int64_t* ptr) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > n) return;
  uint64_t lo = i == 0 ? 0ull : sorted_key[i - 1] + 1ull;
  uint64_t hi = i == n ? (uint64_t)nseg : sorted_key[i];
  for (uint64_t k = lo; k <= hi && k <= (uint64_t)nseg; ++k) ptr[k] = i;
}

__global__ void widen_kernel(const uint32_t* in, int64_t n, uint64_t* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i];
}

void build_stage_transpose(Ctx& c, int32_t coarse_n, int32_t nf, const int64_t* f_ptr,
                           const int32_t* f_nbr, const int32_t* cop, int64_t nnzf,
                           DVec<int64_t>& t_ptr, DVec<int64_t>& t_p, DVec<int32_t>& f_of_p) {
  t_ptr.alloc(coarse_n + 1, c.s);
  t_p.alloc(std::max<int64_t>(nnzf, 1), c.s);
  f_of_p.alloc(std::max<int64_t>(nnzf, 1), c.s);
  if (nnzf == 0) {
    t_ptr.zero();
    return;
  }
  DVec<uint32_t> key(nnzf, c.s);
  DVec<int64_t> ids(nnzf, c.s);
  count_launch(), stage_keys_kernel<<<blocks_for(nf), kThreads, 0, c.s>>>(nf, f_ptr, f_nbr, cop, key.p, f_of_p.p);
  count_launch(), iota64_kernel<<<blocks_for(nnzf), kThreads, 0, c.s>>>(ids.p, nnzf);
  CK_LAUNCH();
  // stable sort of contribution indices p by target coarse node: within a
  // target, p ascending == (f asc, p asc), the reference's accumulation order
  int bits = 1;
  while ((1ull << bits) <= (unsigned long long)coarse_n && bits < 32) ++bits;
  DVec<uint64_t> k64(nnzf, c.s), k64s(nnzf, c.s);
  count_launch(), widen_kernel<<<blocks_for(nnzf), kThreads, 0, c.s>>>(key.p, nnzf, k64.p);
  CK_LAUNCH();
  sort_pairs_u64(c, k64.p, k64s.p, ids.p, t_p.p, nnzf, bits);
  count_launch(), seg_bounds64_kernel<<<blocks_for(nnzf + 1), kThreads, 0, c.s>>>(k64s.p, nnzf, coarse_n, t_ptr.p);
  CK_LAUNCH();
}

__global__ void agg_keys_kernel(const int32_t* agg, int32_t n, uint64_t* key, int32_t* ids) {
  int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  key[u] = (uint64_t)(uint32_t)agg[u];
  ids[u] = u;
}
void build_members(Ctx& c, int32_t fine_n, int32_t coarse_n, const int32_t* agg,
                   DVec<int64_t>& mem_ptr, DVec<int32_t>& mem) {
  mem_ptr.alloc(coarse_n + 1, c.s);
  mem.alloc(fine_n, c.s);
  DVec<uint64_t> key(fine_n, c.s), key_sorted(fine_n, c.s);
  DVec<int32_t> ids(fine_n, c.s);
  count_launch(), agg_keys_kernel<<<blocks_for(fine_n), kThreads, 0, c.s>>>(agg, fine_n, key.p, ids.p);
  CK_LAUNCH();
  int bits = 1;
  while ((1ull << bits) <= (unsigned long long)coarse_n && bits < 32) ++bits;
  sort_pairs_u64_i32(c, key.p, key_sorted.p, ids.p, mem.p, fine_n, bits);
  count_launch(), seg_bounds64_kernel<<<blocks_for(fine_n + 1), kThreads, 0, c.s>>>(key_sorted.p, fine_n, coarse_n, mem_ptr.p);
  CK_LAUNCH();
}

}  // namespace lamgb
