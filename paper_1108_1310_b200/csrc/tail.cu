// tail.cu -- THROUGHPUT-mode coarse tail: one persistent cooperative kernel
// runs the whole recursive sub-cycle (cycle.cpp:115-209) below a size
// threshold.
//
// Coarse levels are small but visited geometrically often (gamma ~ 1.5 per
// level), and a coloured sweep is ~10 dependent colour phases. Host-driven,
// every phase is a kernel launch. Here the recursion, the per-level credits
// (LevelCredit::take, cycle.cpp:14-21) and every transfer run on the device:
//  - mid-size levels use the whole grid, a phase costs one grid barrier;
//  - levels of at most `small_rows` rows (and their whole subtree) run in
//    CTA 0 alone, a phase costs a __syncthreads, and the coloured operator,
//    x and b of a level are staged in shared memory for its sweeps.
// Every thread runs the same control flow on its own frame stack; credits
// live in shared memory (identical in every CTA for the mid levels).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "batch.cuh"
#include "solve.cuh"

namespace lamgb {

namespace {

constexpr int kTailThreads = 512;
constexpr int kTailThreadsBatch = 256;
constexpr int kTailThreadsSlice = 512;

// K-column node-major ops (nm_*): a thread owns one 4-column group of a row.
// The scope says how work items t map to (row, column group): the cluster
// and CTA scopes spread a row's K/4 groups over adjacent threads; the slice
// scope gives each CTA ONE group (its own 4 columns) of every row.
struct BlockScope {
  __device__ static int64_t tid() { return threadIdx.x; }
  __device__ static int64_t stride() { return blockDim.x; }
  __device__ static void sync() { __syncthreads(); }
  __device__ static bool leader() { return threadIdx.x == 0; }
  template <int K>
  __device__ static constexpr int groups() { return K / 4; }
  __device__ static int k0(int64_t t, int T) { return (int)(t % T) * 4; }
  template <int K>
  __device__ static int col0() { return 0; }
  template <int K>
  __device__ static constexpr int ncols() { return K; }
};
// The tail grid is a single thread-block cluster: its barrier is the
// hardware cluster barrier (barrier.cluster.arrive.release / wait.acquire),
// an order of magnitude cheaper than a software grid barrier.
struct GridScope {
  __device__ static int64_t tid() { return blockIdx.x * (int64_t)blockDim.x + threadIdx.x; }
  __device__ static int64_t stride() { return (int64_t)gridDim.x * blockDim.x; }
  __device__ static void sync() { cg::this_cluster().sync(); }
  __device__ static bool leader() { return blockIdx.x == 0 && threadIdx.x == 0; }
  template <int K>
  __device__ static constexpr int groups() { return K / 4; }
  __device__ static int k0(int64_t t, int T) { return (int)(t % T) * 4; }
  template <int K>
  __device__ static int col0() { return 0; }
  template <int K>
  __device__ static constexpr int ncols() { return K; }
};

// K > 1, node-major, one CTA (small levels of the cluster tail: CTA 0 runs
// them alone, a phase is a __syncthreads instead of a cluster barrier)
struct CtaScope : BlockScope {};

// K > 1, node-major, column slices: CTA g of K/4 owns columns 4g..4g+3 of
// every vector of the sub-cycle and runs the whole recursion for them alone
// (thread per row; a phase is a __syncthreads; no CTA waits on another, and
// x stays valid in this SM's L1 across phases -- only this CTA writes it)
__shared__ int g_slice_k0;  // first column of the 4-column slice this CTA is running
struct SliceScope {
  __device__ static int64_t tid() { return threadIdx.x; }
  __device__ static int64_t stride() { return blockDim.x; }
  __device__ static void sync() { __syncthreads(); }
  __device__ static bool leader() { return blockIdx.x == 0 && threadIdx.x == 0 && g_slice_k0 == 0; }
  template <int K>
  __device__ static constexpr int groups() { return 1; }
  __device__ static int k0(int64_t, int) { return g_slice_k0; }
  template <int K>
  __device__ static int col0() { return g_slice_k0; }
  template <int K>
  __device__ static constexpr int ncols() { return 4; }
};

// ---------------------------------------------------------------- sweeps
// shared-memory sweep (BlockScope only): every load of the sweep is an LDS
__device__ inline void gs_smem(const TLevel& L, const double* __restrict__ b, double* x, int sweeps,
                               TailCounters* ctr) {
  extern __shared__ __align__(16) unsigned char smem[];
  const long long t0 = clock64();
  const int32_t n = L.n;
  const int64_t nnz = 2 * L.m;
  double* s_x = (double*)smem;
  double* s_b = s_x + n;
  double* s_d = s_b + n;
  double* s_v = s_d + n;
  int32_t* s_c = (int32_t*)(s_v + nnz);
  int32_t* s_rp = s_c + nnz;
  int32_t* s_id = s_rp + n + 1;
  for (int32_t i = threadIdx.x; i < n; i += blockDim.x) {
    const int32_t u = L.row_ids[i];
    const double xi = x[i], di = L.pdiag[i];
    const int32_t ri = (int32_t)L.prp[i];
    s_x[i] = xi;
    s_id[i] = u;
    s_d[i] = di;
    s_rp[i] = ri;
    s_b[i] = b[u];
  }
  if (threadIdx.x == 0) s_rp[n] = (int32_t)L.prp[n];
  for (int64_t k0 = threadIdx.x; k0 < nnz; k0 += 4 * (int64_t)blockDim.x) {
    int32_t cv[4];
    double vv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t k = k0 + (int64_t)j * blockDim.x;
      cv[j] = k < nnz ? L.pcol[k] : 0;
      vv[j] = k < nnz ? L.pval[k] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t k = k0 + (int64_t)j * blockDim.x;
      if (k < nnz) {
        s_c[k] = cv[j];
        s_v[k] = vv[j];
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  // G = 4 lanes per row, tree-folded (deterministic)
  constexpr int G = 4;
  int32_t* s_cp = s_id + n;  // colour ranges (staged after the row ids)
  for (int32_t i = threadIdx.x; i <= L.ncolors; i += blockDim.x) s_cp[i] = L.cptr[i];
  __syncthreads();
  for (int sw = 0; sw < sweeps; ++sw)
    for (int32_t cc = 0; cc < L.ncolors; ++cc) {
      const int32_t i0 = s_cp[cc], i1 = s_cp[cc + 1];
      const int32_t span = ((i1 - i0) * G + 31) / 32 * 32;
      for (int32_t t = threadIdx.x; t < span; t += blockDim.x) {
        const int32_t i = i0 + t / G;
        const bool ok = i < i1;
        const int lane = t & (G - 1);
        double p = 0.0;
        if (ok) {
          const int32_t e = s_rp[i + 1];
          for (int32_t k = s_rp[i] + lane; k < e; k += G) p += s_v[k] * s_x[s_c[k]];
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o, G);
        if (ok && lane == 0) s_x[s_id[i]] = (s_b[i] - p) / s_d[i];
      }
      __syncthreads();
    }
  const long long t2 = clock64();
  for (int32_t i = threadIdx.x; i < n; i += blockDim.x) x[i] = s_x[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    ctr->smem_calls += 1;
    ctr->smem_phases += (long long)sweeps * L.ncolors;
    ctr->cyc_stage += (t1 - t0) + (clock64() - t2);
    ctr->cyc_phases += t2 - t1;
  }
}

// Coloured sweep with G lanes per row. The colour ranges are staged in shared
// memory, and each group's first row of the NEXT phase (row id, extent,
// diagonal, rhs and up to U entries per lane) is loaded before the barrier,
// so the barrier wait hides those dependent loads; after it only the x
// gathers and the fold remain on the critical path.
constexpr int kMaxColors = 256;

template <class S, int G>
__device__ inline void gs_group(const TLevel& L, const double* __restrict__ b, double* x, int sweeps,
                                int32_t* s_cptr, TailCounters* ctr_dbg) {
  constexpr int U = G == 1 ? 8 : 4;
  const int nc = L.ncolors;
  const bool cached = nc < kMaxColors;
  if (cached) {
    for (int i = threadIdx.x; i <= nc; i += blockDim.x) s_cptr[i] = L.cptr[i];
    __syncthreads();
  }
  const int lane = threadIdx.x & (G - 1);
  const int64_t slot = S::tid() / G;
  bool p_ok = false;
  int32_t p_u = 0;
  int64_t p_k0 = 0, p_k1 = 0;
  double p_d = 1.0, p_b = 0.0;
  int32_t p_c[U];
  double p_v[U];
  auto prefetch = [&](int c) {
    const int32_t c0 = cached ? s_cptr[c] : __ldg(L.cptr + c);
    const int32_t c1 = cached ? s_cptr[c + 1] : __ldg(L.cptr + c + 1);
    const int64_t i = c0 + slot;
    p_ok = i < c1;
    p_k0 = p_k1 = 0;
    if (p_ok) {
      p_u = __ldg(L.row_ids + i);
      p_k0 = __ldg(L.prp + i);
      p_k1 = __ldg(L.prp + i + 1);
      p_d = __ldg(L.pdiag + i);
      p_b = b[p_u];
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int64_t k = p_k0 + lane + (int64_t)j * G;
      const bool ok = k < p_k1;
      p_c[j] = ok ? __ldg(L.pcol + k) : 0;
      p_v[j] = ok ? __ldg(L.pval + k) : 0.0;
    }
  };
  prefetch(0);
  long long tA = clock64(), tB = 0, tC = 0, tD = 0;
  long long acc_fold = 0, acc_extra = 0, acc_pre = 0, acc_bar = 0;
  for (int sw = 0; sw < sweeps; ++sw)
    for (int32_t cc = 0; cc < nc; ++cc) {
      tA = clock64();
      const int32_t i0 = cached ? s_cptr[cc] : L.cptr[cc];
      const int32_t i1 = cached ? s_cptr[cc + 1] : L.cptr[cc + 1];
      {  // the prefetched row
        double xv[U];
#pragma unroll
        for (int j = 0; j < U; ++j) xv[j] = (p_k0 + lane + (int64_t)j * G < p_k1) ? x[p_c[j]] : 0.0;
        double acc;
        if (G == 1) {
          acc = p_b;
#pragma unroll
          for (int j = 0; j < U; ++j)
            if (p_k0 + j < p_k1) acc = acc - p_v[j] * xv[j];
          if (p_ok && p_k1 - p_k0 > U) acc = row_fold<8, true>(acc, L.pcol, L.pval, x, p_k0 + U, p_k1);
          if (p_ok) x[p_u] = acc / p_d;
        } else {
          acc = 0.0;
#pragma unroll
          for (int j = 0; j < U; ++j) acc += p_v[j] * xv[j];
          for (int64_t k = p_k0 + lane + (int64_t)U * G; k < p_k1; k += G) acc += __ldg(L.pval + k) * x[__ldg(L.pcol + k)];
#pragma unroll
          for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, G);
          if (p_ok && lane == 0) x[p_u] = (p_b - acc) / p_d;
        }
      }
      tB = clock64();
      // rows beyond the first slot of this colour (large levels only)
      const int64_t span = ((int64_t)(i1 - i0) * G + 31) / 32 * 32;
      for (int64_t t = S::tid() + S::stride(); t < span; t += S::stride()) {
        const int64_t i = i0 + t / G;
        const bool ok = i < i1;
        if (G == 1) {
          if (ok) {
            const int32_t u = L.row_ids[i];
            x[u] = row_fold<8, true>(b[u], L.pcol, L.pval, x, L.prp[i], L.prp[i + 1]) / L.pdiag[i];
          }
        } else {
          const double dot = group_dot<G>(L.pcol, L.pval, x, ok ? L.prp[i] : 0, ok ? L.prp[i + 1] : 0);
          if (ok && lane == 0) {
            const int32_t u = L.row_ids[i];
            x[u] = (b[u] - dot) / L.pdiag[i];
          }
        }
      }
      tC = clock64();
      const int next = cc + 1 < nc ? cc + 1 : (sw + 1 < sweeps ? 0 : -1);
      if (next >= 0) prefetch(next);
      // force the prefetched loads to land before timing the barrier
      if (p_ok && p_c[0] == -7) x[0] = p_v[0] + p_b;
      tD = clock64();
      S::sync();
      acc_fold += tB - tA;
      acc_extra += tC - tB;
      acc_pre += tD - tC;
      acc_bar += clock64() - tD;
    }
  if (blockIdx.x == 0 && threadIdx.x == 0 && std::is_same<S, GridScope>::value) {
    ctr_dbg->ph_fold += acc_fold;
    ctr_dbg->ph_extra += acc_extra;
    ctr_dbg->ph_prefetch += acc_pre;
    ctr_dbg->ph_barrier += acc_bar;
  }
}

template <class S>
__device__ inline void gs(const TLevel& L, const double* __restrict__ b, double* x, int sweeps, TailCounters* ctr,
                          int32_t xs_rows) {
  __shared__ int32_t s_cptr[kMaxColors];
  if (L.ncolors == 0 || sweeps == 0) return;
  const long long tg = clock64();
  if (S::leader()) ctr->phases += (long long)sweeps * L.ncolors;
  constexpr bool cta = !std::is_same<S, GridScope>::value;
  if (cta && L.smem_ok) {
    gs_smem(L, b, x, sweeps, ctr);
  } else if (cta && L.n <= xs_rows) {
    // x and b of the level in shared memory for the sweeps: every gather of
    // the dependent chain is an LDS; the matrix streams through L1
    extern __shared__ __align__(16) unsigned char smem[];
    double* sx = (double*)smem;
    double* sb = sx + L.n;
    for (int32_t i = threadIdx.x; i < L.n; i += blockDim.x) {
      sx[i] = x[i];
      sb[i] = b[i];
    }
    __syncthreads();
    if (L.group == 8) gs_group<S, 8>(L, sb, sx, sweeps, s_cptr, ctr);
    else if (L.group == 4) gs_group<S, 4>(L, sb, sx, sweeps, s_cptr, ctr);
    else gs_group<S, 1>(L, sb, sx, sweeps, s_cptr, ctr);
    for (int32_t i = threadIdx.x; i < L.n; i += blockDim.x) x[i] = sx[i];
    __syncthreads();
  } else {
    if (L.group == 8) gs_group<S, 8>(L, b, x, sweeps, s_cptr, ctr);
    else if (L.group == 4) gs_group<S, 4>(L, b, x, sweeps, s_cptr, ctr);
    else gs_group<S, 1>(L, b, x, sweeps, s_cptr, ctr);
  }
  if (S::leader()) {
    const long long dt = clock64() - tg;
    ctr->cyc_global_gs += dt;
    ctr->global_phases += (long long)sweeps * L.ncolors;
    ctr->lvl_gs_cyc[L.id] += dt;
    ctr->lvl_gs_calls[L.id] += 1;
  }
}

// -------------------------------------------------------------- transfers
template <class S, int G>
__device__ inline void residual_group(const TLevel& L, const double* __restrict__ b, const double* x, double* r) {
  const int64_t span = ((int64_t)L.n * G + 31) / 32 * 32;
  for (int64_t t = S::tid(); t < span; t += S::stride()) {
    const int64_t u = t / G;
    const bool ok = u < L.n;
    if (G == 1) {
      if (ok) {
        double s = L.diag[u] * x[u];
        s = row_fold<8, false>(s, L.col, L.val, x, L.rp[u], L.rp[u + 1]);
        r[u] = b[u] - s;
      }
    } else {
      const double dot = group_dot<G>(L.col, L.val, x, ok ? L.rp[u] : 0, ok ? L.rp[u + 1] : 0);
      if (ok && (threadIdx.x & (G - 1)) == 0) r[u] = b[u] - (L.diag[u] * x[u] + dot);
    }
  }
  S::sync();
}

template <class S>
__device__ inline void residual(const TLevel& L, const double* __restrict__ b, const double* x, double* r) {
  if (L.group == 8) residual_group<S, 8>(L, b, x, r);
  else if (L.group == 4) residual_group<S, 4>(L, b, x, r);
  else residual_group<S, 1>(L, b, x, r);
}

// restrict r into the child's rhs (member-ordered fold, times mu) and zero
// the child's iterate
template <class S>
__device__ inline void restrict_to(const TLevel& L, const TLevel& C, const double* r, double mu) {
  for (int64_t g = S::tid(); g < C.n; g += S::stride()) {
    double s = 0.0;
    for (int64_t j = L.mem_ptr[g]; j < L.mem_ptr[g + 1]; ++j) s = s + r[L.mem[j]];
    C.b[g] = mu != 1.0 ? s * mu : s;
    C.x[g] = 0.0;
  }
  S::sync();
}

template <class S>
__device__ inline void interpolate(const TLevel& L, const TLevel& C, double* x) {
  for (int64_t u = S::tid(); u < L.n; u += S::stride()) x[u] = x[u] + C.x[L.agg[u]];
  S::sync();
}

template <class S>
__device__ inline void coarsen(const StageV& s, const double* b, double* bc) {
  for (int64_t k = S::tid(); k < s.coarse_n; k += S::stride()) {
    double v = b[s.poc[k]];
    for (int64_t j = s.t_ptr[k]; j < s.t_ptr[k + 1]; ++j) {
      const int64_t p = s.t_p[j];
      const int32_t i = s.f_of_p[p];
      v = v - s.f_val[p] * (b[s.f_nodes[i]] / s.f_diag[i]);
    }
    bc[k] = v;
  }
  S::sync();
}

template <class S>
__device__ inline void inject(const StageV& s, const double* x, double* xc) {
  for (int64_t k = S::tid(); k < s.coarse_n; k += S::stride()) xc[k] = x[s.poc[k]];
  S::sync();
}

template <class S>
__device__ inline void backsub(const StageV& s, const double* xc, const double* b, double* x) {
  for (int64_t k = S::tid(); k < s.coarse_n; k += S::stride()) x[s.poc[k]] = xc[k];
  S::sync();
  for (int64_t i = S::tid(); i < s.nf; i += S::stride()) {
    const int32_t f = s.f_nodes[i];
    double sum = b[f];
    for (int64_t p = s.f_ptr[i]; p < s.f_ptr[i + 1]; ++p) sum = sum - s.f_val[p] * x[s.f_nbr[p]];
    x[f] = sum / s.f_diag[i];
  }
  S::sync();
}

// x = Minv[:n,:n] b per component: one warp per row, fixed-order lane folds
// (the coarsest level always runs in one CTA)
__device__ inline void direct(const TLevel& L, const double* b, double* x) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int32_t ci = 0; ci < L.ncomp; ++ci) {
    const int32_t s0 = L.comp_start[ci], cn = L.comp_start[ci + 1] - s0;
    const double* Mi = L.inv + L.inv_off[ci];
    for (int32_t i = warp; i < cn; i += nw) {
      double s = 0.0;
      for (int32_t j = lane; j < cn; j += 32) s += Mi[(int64_t)i * cn + j] * (L.whole ? b[j] : b[L.nodes[s0 + j]]);
      for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
      if (lane == 0) {
        if (L.whole) x[i] = s;
        else x[L.nodes[s0 + i]] = s;
      }
    }
  }
  __syncthreads();
}

// fixed-order reduction over the scope; every thread gets the same value
template <class S>
__device__ inline double scope_sum(double v, double* sh, double* part) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
    sh[32] = t;
    if (std::is_same<S, GridScope>::value) part[blockIdx.x] = t;
  }
  S::sync();
  double t = sh[32];
  if (std::is_same<S, GridScope>::value) {
    t = 0.0;
    for (unsigned g = 0; g < gridDim.x; ++g) t += ((volatile double*)part)[g];
  }
  S::sync();
  return t;
}

// RelaxationSolver::solve (coarse_solver.cpp:82-93)
template <class S>
__device__ inline void relax(const TLevel& L, const double* b, double* x, double* sh, double* part,
                             TailCounters* ctr, int32_t xs_rows) {
  residual<S>(L, b, x, L.r);
  double loc = 0.0;
  for (int64_t u = S::tid(); u < L.n; u += S::stride()) loc += L.r[u] * L.r[u];
  const double r0 = sqrt(scope_sum<S>(loc, sh, part));
  if (S::leader()) ctr->work += (double)L.m;
  if (r0 == 0.0) return;
  const double target = 1e-12 * r0;
  for (int sweep = 0; sweep < 400; ++sweep) {
    gs<S>(L, b, x, 1, ctr, xs_rows);
    loc = 0.0;
    for (int64_t u = S::tid(); u < L.n; u += S::stride()) loc += x[u];
    const double mean = scope_sum<S>(loc, sh, part) / (double)L.n;
    for (int64_t u = S::tid(); u < L.n; u += S::stride()) x[u] = x[u] - mean;
    S::sync();
    residual<S>(L, b, x, L.r);
    loc = 0.0;
    for (int64_t u = S::tid(); u < L.n; u += S::stride()) loc += L.r[u] * L.r[u];
    const double rn = sqrt(scope_sum<S>(loc, sh, part));
    if (S::leader()) {
      ctr->work += 2.0 * (double)L.m;
      ctr->relax_sweeps += 1;
    }
    if (rn <= target) break;
  }
}


// ------------------------------------------------- K right-hand sides
// (batch.cuh). Below the host-driven levels, a block of K columns runs as K/kc
// independent CTAs (subtree_kernel): each CTA runs the whole sub-cycle for
// its own kc columns, so a phase is a __syncthreads, and it never waits on
// another CTA. Inside the subtree every vector is COLUMN-major, v[k*n + u]:
// the CTAs' writes never share a cache sector (node-major rows would put all
// K columns of a node in one 256-byte segment written by K different SMs).
// The subtree's root level is transposed in at entry and out at exit.
struct ColSlice {
  int k0, kc, sh;  // kc = 1 << sh columns starting at k0
};
template <int K>
__device__ inline ColSlice my_cols() {
  const int kc = K >= (int)gridDim.x ? K / (int)gridDim.x : 1;  // powers of two
  return ColSlice{(int)blockIdx.x * kc, kc, __ffs(kc) - 1};
}

// Coloured sweep, column slice. The first (row, column) pair of each
// thread's next colour -- row id, extent, diagonal, rhs and up to kCU
// entries -- is loaded before the barrier; after it only the x gathers of
// the row remain, issued together and folded in entry order.
constexpr int kCU = 16;
template <int K>
__device__ inline void cs_gs(const TLevel& L, const double* __restrict__ b, double* x, int sweeps,
                             const int32_t* done, TailCounters* ctr) {
  __shared__ int32_t s_cp[kMaxColors + 1];
  if (L.ncolors == 0 || sweeps == 0) return;
  const long long tg = clock64();
  const ColSlice sl = my_cols<K>();
  const int nc = L.ncolors;
  const int64_t n = L.n;
  const bool cached = nc <= kMaxColors;
  if (cached)
    for (int i = threadIdx.x; i <= nc; i += blockDim.x) s_cp[i] = __ldg(L.cptr + i);
  __syncthreads();
  const int k = sl.k0 + (int)(threadIdx.x & (sl.kc - 1));
  const double* bk = b + k * n;
  double* xk = x + k * n;
  const bool frozen = done && done[k];
  const int64_t slot = threadIdx.x >> sl.sh;
  const int64_t warp_t0 = threadIdx.x & ~31u;
  auto cbounds = [&](int cc, int32_t& c0, int32_t& c1) {
    c0 = cached ? s_cp[cc] : __ldg(L.cptr + cc);
    c1 = cached ? s_cp[cc + 1] : __ldg(L.cptr + cc + 1);
  };
  bool p_ok = false;
  int32_t p_u = 0;
  int64_t p_e0 = 0, p_e1 = 0;
  double p_d = 1.0, p_b = 0.0;
  int32_t p_c[kCU];
  double p_v[kCU];
  auto prefetch = [&](int cc) {
    int32_t c0, c1;
    cbounds(cc, c0, c1);
    p_ok = false;
    p_e0 = p_e1 = 0;
    if (warp_t0 >= (int64_t)(c1 - c0) << sl.sh) return;  // whole warp idle in this colour
    const int64_t i = c0 + slot;
    p_ok = i < c1;
    if (p_ok) {
      p_u = __ldg(L.row_ids + i);
      p_e0 = __ldg(L.prp + i);
      p_e1 = __ldg(L.prp + i + 1);
      p_d = __ldg(L.pdiag + i);
      p_b = bk[p_u];
    }
#pragma unroll
    for (int j = 0; j < kCU; ++j) {
      const bool ok = p_e0 + j < p_e1;
      p_c[j] = ok ? __ldg(L.pcol + p_e0 + j) : 0;
      p_v[j] = ok ? __ldg(L.pval + p_e0 + j) : 0.0;
    }
  };
  prefetch(0);
  for (int sw = 0; sw < sweeps; ++sw)
    for (int32_t cc = 0; cc < nc; ++cc) {
      int32_t i0, i1;
      cbounds(cc, i0, i1);
      if (p_ok && !frozen) {
        double xv[kCU];
#pragma unroll
        for (int j = 0; j < kCU; ++j) xv[j] = p_e0 + j < p_e1 ? xk[p_c[j]] : 0.0;
        double s = p_b;
#pragma unroll
        for (int j = 0; j < kCU; ++j)
          if (p_e0 + j < p_e1) s = s - p_v[j] * xv[j];
        if (p_e1 - p_e0 > kCU) s = col_fold<1, true, 8>(s, L.pcol, L.pval, xk, p_e0 + kCU, p_e1, 0);
        xk[p_u] = s / p_d;
      }
      if (!frozen)  // pairs beyond the first of this colour (large colours only)
        for (int64_t t = threadIdx.x + blockDim.x; t < (int64_t)(i1 - i0) << sl.sh; t += blockDim.x) {
          const int64_t i = i0 + (t >> sl.sh);
          const int32_t u = __ldg(L.row_ids + i);
          const double s = col_fold<1, true, 8>(bk[u], L.pcol, L.pval, xk, __ldg(L.prp + i), __ldg(L.prp + i + 1), 0);
          xk[u] = s / __ldg(L.pdiag + i);
        }
      const int next = cc + 1 < nc ? cc + 1 : (sw + 1 < sweeps ? 0 : -1);
      if (next >= 0) prefetch(next);
      else p_ok = false;
      __syncthreads();
    }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctr->phases += (long long)sweeps * L.ncolors;
    ctr->lvl_gs_cyc[L.id] += clock64() - tg;
    ctr->lvl_gs_calls[L.id] += 1;
  }
}

// the whole sweep in shared memory: the coloured operator (int32 row
// pointers, column ids, values, diagonal, row ids) and this CTA's columns of
// x and b are staged once per call, every phase is LDS-only
inline int64_t cs_smem_bytes(int64_t n, int64_t nnz, int ncolors, int kc) {
  return n * kc * 16 + n * 8 + nnz * 8 + nnz * 4 + (n + 1) * 4 + n * 4 + (ncolors + 1) * 4 + 64;
}
template <int K>
__device__ inline void cs_gs_smem(const TLevel& L, const double* __restrict__ b, double* x, int sweeps,
                                  TailCounters* ctr) {
  extern __shared__ __align__(16) unsigned char smem[];
  const long long tg = clock64();
  const ColSlice sl = my_cols<K>();
  const int kc = sl.kc;
  const int32_t n = L.n;
  const int64_t nnz = 2 * L.m;
  const int nc = L.ncolors;
  double* s_x = (double*)smem;  // [kc][n]
  double* s_b = s_x + (int64_t)n * kc;
  double* s_d = s_b + (int64_t)n * kc;
  double* s_v = s_d + n;
  int32_t* s_c = (int32_t*)(s_v + nnz);
  int32_t* s_rp = s_c + nnz;
  int32_t* s_id = s_rp + n + 1;
  int32_t* s_cp = s_id + n;
  const int32_t e_base = (int32_t)__ldg(L.prp);
  for (int32_t i = threadIdx.x; i < n; i += blockDim.x) {
    s_d[i] = __ldg(L.pdiag + i);
    s_rp[i] = (int32_t)(__ldg(L.prp + i) - e_base);
    s_id[i] = __ldg(L.row_ids + i);
  }
  if (threadIdx.x == 0) s_rp[n] = (int32_t)(__ldg(L.prp + n) - e_base);
  for (int i = threadIdx.x; i <= nc; i += blockDim.x) s_cp[i] = __ldg(L.cptr + i);
  for (int64_t e = threadIdx.x; e < nnz; e += blockDim.x) {
    s_c[e] = __ldg(L.pcol + e_base + e);
    s_v[e] = __ldg(L.pval + e_base + e);
  }
  for (int64_t t = threadIdx.x; t < (int64_t)n * kc; t += blockDim.x) {  // my columns are contiguous
    s_x[t] = x[(int64_t)sl.k0 * n + t];
    s_b[t] = b[(int64_t)sl.k0 * n + t];
  }
  __syncthreads();
  for (int sw = 0; sw < sweeps; ++sw)
    for (int cc = 0; cc < nc; ++cc) {
      const int32_t i0 = s_cp[cc], i1 = s_cp[cc + 1];
      for (int32_t t = threadIdx.x; t < (i1 - i0) * kc; t += blockDim.x) {
        const int32_t i = i0 + (t >> sl.sh);
        const int j = t & (kc - 1);
        const double* sxj = s_x + (int64_t)j * n;
        const int32_t u = s_id[i];
        double s = s_b[(int64_t)j * n + u];
        const int32_t e1 = s_rp[i + 1];
        for (int32_t e0 = s_rp[i]; e0 < e1; e0 += 8) {  // loads of 8 entries ahead of their fold
          double xv[8], vv[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const bool ok = e0 + q < e1;
            vv[q] = ok ? s_v[e0 + q] : 0.0;
            xv[q] = ok ? sxj[s_c[e0 + q]] : 0.0;
          }
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (e0 + q < e1) s = s - vv[q] * xv[q];
        }
        s_x[(int64_t)j * n + u] = s / s_d[i];
      }
      __syncthreads();
    }
  for (int64_t t = threadIdx.x; t < (int64_t)n * kc; t += blockDim.x) x[(int64_t)sl.k0 * n + t] = s_x[t];
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctr->phases += (long long)sweeps * nc;
    ctr->smem_calls += 1;
    ctr->smem_phases += (long long)sweeps * nc;
    ctr->lvl_gs_cyc[L.id] += clock64() - tg;
    ctr->lvl_gs_calls[L.id] += 1;
  }
}

template <int K>
__device__ inline void cs_residual(const TLevel& L, const double* __restrict__ b, const double* x, double* r) {
  const ColSlice sl = my_cols<K>();
  const int64_t n = L.n;
  for (int64_t t = threadIdx.x; t < n << sl.sh; t += blockDim.x) {
    const int64_t u = t >> sl.sh;
    const int64_t k = sl.k0 + (t & (sl.kc - 1));
    const double* xk = x + k * n;
    const double s = col_fold<1, false, 16>(__ldg(L.diag + u) * xk[u], L.col, L.val, xk, __ldg(L.rp + u),
                                            __ldg(L.rp + u + 1), 0);
    r[k * n + u] = b[k * n + u] - s;
  }
  __syncthreads();
}

template <int K>
__device__ inline void cs_restrict(const TLevel& L, const TLevel& C, const double* r, double mu) {
  const ColSlice sl = my_cols<K>();
  for (int64_t t = threadIdx.x; t < (int64_t)C.n << sl.sh; t += blockDim.x) {
    const int64_t g = t >> sl.sh;
    const int64_t k = sl.k0 + (t & (sl.kc - 1));
    const double* rk = r + k * L.n;
    double s = 0.0;
    for (int64_t j = __ldg(L.mem_ptr + g); j < __ldg(L.mem_ptr + g + 1); ++j) s = s + rk[__ldg(L.mem + j)];
    C.b[k * C.n + g] = mu != 1.0 ? s * mu : s;
    C.x[k * C.n + g] = 0.0;
  }
  __syncthreads();
}

template <int K>
__device__ inline void cs_interp(const TLevel& L, const TLevel& C, double* x) {
  const ColSlice sl = my_cols<K>();
  for (int64_t t = threadIdx.x; t < (int64_t)L.n << sl.sh; t += blockDim.x) {
    const int64_t u = t >> sl.sh;
    const int64_t k = sl.k0 + (t & (sl.kc - 1));
    x[k * L.n + u] = x[k * L.n + u] + C.x[k * C.n + __ldg(L.agg + u)];
  }
  __syncthreads();
}

template <int K>
__device__ inline void cs_coarsen(const StageV& s, const double* b, double* bc) {
  const ColSlice sl = my_cols<K>();
  for (int64_t t = threadIdx.x; t < (int64_t)s.coarse_n << sl.sh; t += blockDim.x) {
    const int64_t q = t >> sl.sh;
    const int64_t k = sl.k0 + (t & (sl.kc - 1));
    const double* bk = b + k * s.parent_n;
    double v = bk[__ldg(s.poc + q)];
    for (int64_t j = __ldg(s.t_ptr + q); j < __ldg(s.t_ptr + q + 1); ++j) {
      const int64_t p = __ldg(s.t_p + j);
      const int32_t i = __ldg(s.f_of_p + p);
      v = v - __ldg(s.f_val + p) * (bk[__ldg(s.f_nodes + i)] / __ldg(s.f_diag + i));
    }
    bc[k * s.coarse_n + q] = v;
  }
  __syncthreads();
}

template <int K>
__device__ inline void cs_inject(const StageV& s, const double* x, double* xc) {
  const ColSlice sl = my_cols<K>();
  for (int64_t t = threadIdx.x; t < (int64_t)s.coarse_n << sl.sh; t += blockDim.x) {
    const int64_t q = t >> sl.sh;
    const int64_t k = sl.k0 + (t & (sl.kc - 1));
    xc[k * s.coarse_n + q] = x[k * s.parent_n + __ldg(s.poc + q)];
  }
  __syncthreads();
}

template <int K>
__device__ inline void cs_backsub(const StageV& s, const double* xc, const double* b, double* x) {
  const ColSlice sl = my_cols<K>();
  for (int64_t t = threadIdx.x; t < (int64_t)s.coarse_n << sl.sh; t += blockDim.x) {
    const int64_t q = t >> sl.sh;
    const int64_t k = sl.k0 + (t & (sl.kc - 1));
    x[k * s.parent_n + __ldg(s.poc + q)] = xc[k * s.coarse_n + q];
  }
  __syncthreads();
  for (int64_t t = threadIdx.x; t < (int64_t)s.nf << sl.sh; t += blockDim.x) {
    const int64_t i = t >> sl.sh;
    const int64_t k = sl.k0 + (t & (sl.kc - 1));
    double* xk = x + k * s.parent_n;
    const int32_t f = __ldg(s.f_nodes + i);
    double sum = b[k * s.parent_n + f];
    for (int64_t p = __ldg(s.f_ptr + i); p < __ldg(s.f_ptr + i + 1); ++p)
      sum = sum - __ldg(s.f_val + p) * xk[__ldg(s.f_nbr + p)];
    xk[f] = sum / __ldg(s.f_diag + i);
  }
  __syncthreads();
}

template <int K>
__device__ inline void cs_direct(const TLevel& L, const double* b, double* x) {
  const ColSlice sl = my_cols<K>();
  const int64_t n = L.n;
  for (int32_t ci = 0; ci < L.ncomp; ++ci) {
    const int32_t s0 = L.comp_start[ci], cn = L.comp_start[ci + 1] - s0;
    const double* Mi = L.inv + L.inv_off[ci];
    for (int64_t t = threadIdx.x; t < (int64_t)cn << sl.sh; t += blockDim.x) {
      const int32_t i = (int32_t)(t >> sl.sh);
      const int64_t k = sl.k0 + (t & (sl.kc - 1));
      const double* bk = b + k * n;
      double s = 0.0;
      for (int32_t j = 0; j < cn; ++j) s += __ldg(Mi + (int64_t)i * cn + j) * bk[L.whole ? j : L.nodes[s0 + j]];
      x[k * n + (L.whole ? i : L.nodes[s0 + i])] = s;
    }
    __syncthreads();
  }
}

// per-column sums of column-major X[k*n + u] in a K-independent order
// (chunks of R rows folded in sequence, chunk sums folded in sequence);
// part holds [K][kChunks]
constexpr int kChunks = 256;
template <bool SQ>
__device__ inline double chunk_colsum(const double* X, int64_t n, double* part, ColSlice sl, int64_t k) {
  const int64_t R = (n + kChunks - 1) / kChunks;
  const int np = (int)((n + R - 1) / R);
  for (int64_t t = threadIdx.x; t < (int64_t)np << sl.sh; t += blockDim.x) {
    const int64_t p = t >> sl.sh;
    const int64_t kk = sl.k0 + (t & (sl.kc - 1));
    const int64_t u1 = (p + 1) * R < n ? (p + 1) * R : n;
    double s = 0.0;
    for (int64_t u = p * R; u < u1; ++u) {
      const double v = X[kk * n + u];
      s += SQ ? v * v : v;
    }
    part[kk * kChunks + p] = s;
  }
  __syncthreads();
  double tot = 0.0;
  for (int p = 0; p < np; ++p) tot += part[k * kChunks + p];
  __syncthreads();
  return tot;
}

// RelaxationSolver::solve (coarse_solver.cpp:82-93) per column of the
// slice; each column freezes at its own tolerance
template <int K>
__device__ inline void cs_relax(const TLevel& L, const double* b, double* x, double* part, TailCounters* ctr) {
  __shared__ int32_t bdone[32];
  __shared__ double br0[32];
  const ColSlice sl = my_cols<K>();
  const int64_t n = L.n;
  const int64_t k = sl.k0 + (threadIdx.x & (sl.kc - 1));  // this thread's column
  cs_residual<K>(L, b, x, L.r);
  const double r0 = sqrt(chunk_colsum<true>(L.r, n, part, sl, k));
  if (threadIdx.x < 32) bdone[threadIdx.x] = 1;
  __syncthreads();
  if ((int)threadIdx.x < sl.kc) {
    br0[k] = r0;
    bdone[k] = r0 == 0.0;
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) ctr->work += (double)L.m;
  for (int sweep = 0; sweep < 400; ++sweep) {
    int active = 0;
    for (int j = 0; j < sl.kc; ++j) active += !bdone[sl.k0 + j];
    if (!active) break;
    cs_gs<K>(L, b, x, 1, bdone, ctr);
    const double mean = chunk_colsum<false>(x, n, part, sl, k) / (double)n;
    if (!bdone[k])
      for (int64_t t = threadIdx.x; t < n << sl.sh; t += blockDim.x) x[k * n + (t >> sl.sh)] -= mean;
    __syncthreads();
    cs_residual<K>(L, b, x, L.r);
    const double rn = sqrt(chunk_colsum<true>(L.r, n, part, sl, k));
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      ctr->work += 2.0 * (double)L.m;
      ctr->relax_sweeps += 1;
    }
    if ((int)threadIdx.x < sl.kc && !bdone[k] && rn <= 1e-12 * br0[k]) bdone[k] = 1;
    __syncthreads();
  }
}

// ----------------------------------- K columns, node-major, one cluster
// (batch.cuh) The block tail: the whole sub-cycle below the host-driven
// levels for all K columns in ONE thread-block cluster (GridScope: a colour
// phase costs one hardware cluster barrier), vectors node-major exactly as on
// the host-driven levels, so the root needs no transposition. A (row, group
// of 4 columns) pair is one thread: the row's entries are loaded once per
// group and each x gather is one 256-bit access. Every column folds in the
// row's entry (member, contribution) order -- the arithmetic of the batch.cu
// kernels -- so a column's bits do not depend on K.
template <bool SUB>
__device__ __forceinline__ void nm_fold(double (&s)[kV], const int32_t* __restrict__ col,
                                        const double* __restrict__ val, const double* X, int64_t e0, int64_t e1,
                                        int K, int k0) {
  constexpr int U = 8;
  for (int64_t b = e0; b < e1; b += U) {
    int32_t c[U];
    double v[U];
    d4 xv[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const bool ok = b + j < e1;
      c[j] = ok ? __ldg(col + b + j) : 0;
      v[j] = ok ? __ldg(val + b + j) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < U; ++j) xv[j] = b + j < e1 ? ld4(X + (int64_t)c[j] * K + k0) : d4{0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (b + j < e1) {
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
__device__ __forceinline__ void nm_store(double* p, const double (&s)[kV], double d, const bool (&fz)[kV], bool any) {
  if (!any) {
    st4(p, s[0] / d, s[1] / d, s[2] / d, s[3] / d);
  } else {
#pragma unroll
    for (int q = 0; q < kV; ++q)
      if (!fz[q]) p[q] = s[q] / d;
  }
}

// Coloured sweep. Each thread's first row of the NEXT colour (row id, extent,
// diagonal, b and the first 8 entries) is loaded before the barrier; after it
// only the x gathers, the fold and the store remain.
template <class S, int K>
__device__ inline void nm_gs(const TLevel& L, const double* __restrict__ b, double* x, int sweeps,
                             const int32_t* done, TailCounters* ctr) {
  __shared__ int32_t s_cp[kMaxColors + 1];
  if (L.ncolors == 0 || sweeps == 0) return;
  constexpr int T = S::template groups<K>();
  constexpr int U = 8;
  const long long tg = clock64();
  const int nc = L.ncolors;
  const bool cached = nc <= kMaxColors;
  if (cached)
    for (int i = threadIdx.x; i <= nc; i += blockDim.x) s_cp[i] = __ldg(L.cptr + i);
  __syncthreads();
  const int64_t slot = S::tid() / T;
  const int64_t rstride = S::stride() / T;
  const int k0 = S::k0(S::tid(), T);
  bool fz[kV];
  bool any = false;
#pragma unroll
  for (int q = 0; q < kV; ++q) {
    fz[q] = done && done[k0 + q];
    any = any || fz[q];
  }
  const bool all = fz[0] && fz[1] && fz[2] && fz[3];
  auto cbounds = [&](int cc, int32_t& c0, int32_t& c1) {
    c0 = cached ? s_cp[cc] : __ldg(L.cptr + cc);
    c1 = cached ? s_cp[cc + 1] : __ldg(L.cptr + cc + 1);
  };
  bool p_ok = false;
  int32_t p_u = 0;
  int64_t p_e0 = 0, p_e1 = 0;
  double p_d = 1.0;
  d4 p_b{0.0, 0.0, 0.0, 0.0};
  int32_t p_c[U];
  double p_v[U];
  auto prefetch = [&](int cc) {
    int32_t c0, c1;
    cbounds(cc, c0, c1);
    const int64_t i = c0 + slot;
    p_ok = i < c1;
    p_e0 = p_e1 = 0;
    if (p_ok) {
      p_u = __ldg(L.row_ids + i);
      p_e0 = __ldg(L.prp + i);
      p_e1 = __ldg(L.prp + i + 1);
      p_d = __ldg(L.pdiag + i);
      p_b = ld4(b + (int64_t)p_u * K + k0);
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const bool ok = p_e0 + j < p_e1;
      p_c[j] = ok ? __ldg(L.pcol + p_e0 + j) : 0;
      p_v[j] = ok ? __ldg(L.pval + p_e0 + j) : 0.0;
    }
  };
  prefetch(0);
  long long a_first = 0, a_extra = 0, a_pre = 0, a_bar = 0;
  for (int sw = 0; sw < sweeps; ++sw)
    for (int32_t cc = 0; cc < nc; ++cc) {
      const long long tA = clock64();
      int32_t i0, i1;
      cbounds(cc, i0, i1);
      if (p_ok && !all) {
        d4 xv[U];
#pragma unroll
        for (int j = 0; j < U; ++j)
          xv[j] = p_e0 + j < p_e1 ? ld4(x + (int64_t)p_c[j] * K + k0) : d4{0.0, 0.0, 0.0, 0.0};
        double sv[kV] = {p_b.x, p_b.y, p_b.z, p_b.w};
#pragma unroll
        for (int j = 0; j < U; ++j)
          if (p_e0 + j < p_e1) {
            sv[0] = sv[0] - p_v[j] * xv[j].x;
            sv[1] = sv[1] - p_v[j] * xv[j].y;
            sv[2] = sv[2] - p_v[j] * xv[j].z;
            sv[3] = sv[3] - p_v[j] * xv[j].w;
          }
        if (p_e1 - p_e0 > U) nm_fold<true>(sv, L.pcol, L.pval, x, p_e0 + U, p_e1, K, k0);
        nm_store(x + (int64_t)p_u * K + k0, sv, p_d, fz, any);
      }
      const long long tB = clock64();
      if (!all)  // rows beyond each thread's first of this colour
        for (int64_t i = i0 + slot + rstride; i < i1; i += rstride) {
          const int32_t u = __ldg(L.row_ids + i);
          const d4 bv = ld4(b + (int64_t)u * K + k0);
          double sv[kV] = {bv.x, bv.y, bv.z, bv.w};
          nm_fold<true>(sv, L.pcol, L.pval, x, __ldg(L.prp + i), __ldg(L.prp + i + 1), K, k0);
          nm_store(x + (int64_t)u * K + k0, sv, __ldg(L.pdiag + i), fz, any);
        }
      const long long tC = clock64();
      const int next = cc + 1 < nc ? cc + 1 : (sw + 1 < sweeps ? 0 : -1);
      if (next >= 0) prefetch(next);
      else p_ok = false;
      const long long tD = clock64();
      S::sync();
      a_first += tB - tA;
      a_extra += tC - tB;
      a_pre += tD - tC;
      a_bar += clock64() - tD;
    }
  if (S::leader()) {
    ctr->lvl_ph[L.id][0] += a_first;
    ctr->lvl_ph[L.id][1] += a_extra;
    ctr->lvl_ph[L.id][2] += a_pre;
    ctr->lvl_ph[L.id][3] += a_bar;
    ctr->phases += (long long)sweeps * nc;
    ctr->global_phases += (long long)sweeps * nc;
    ctr->lvl_gs_cyc[L.id] += clock64() - tg;
    ctr->lvl_gs_calls[L.id] += 1;
  }
}

// ---------------------------------------------- slice scope, shared memory
// Small levels of a slice (sl_ok): the CTA's four columns of x live in shared
// memory for the whole call, and the entries (col, val) of the NEXT colour --
// a contiguous range of the colour-permuted operator -- stream into a
// double buffer with cp.async while the current colour is folded from shared
// memory; each thread's next row (id, extent, diagonal, b) is loaded one phase
// ahead into registers. A phase then costs shared-memory gathers, the fold in
// entry order (the arithmetic of nm_gs), a division and a __syncthreads.
__device__ __forceinline__ void cp_async4(void* dst_smem, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst_smem)), "l"(src));
}
__device__ __forceinline__ void cp_async8(void* dst_smem, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst_smem)), "l"(src));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// shared memory of one slice call: x and b (32 B per row each), the stored
// rows' diagonal, extent and natural id, and nb colour buffers of cap entries
inline int64_t sl_smem_bytes(int64_t n, int64_t cap, int nb) { return 80 * n + 12 * nb * cap + 128; }

// RES = false: `sweeps` coloured Gauss-Seidel sweeps of the slice; RES = true:
// r = b - A x over the same colour-permuted rows (a row's entries keep their
// order, so both match nm_gs / nm_residual bit for bit)
template <int K, bool RES>
__device__ inline void sl_rows(const TLevel& L, const double* __restrict__ b, double* x, double* r, int sweeps,
                               const int32_t* done, TailCounters* ctr) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int32_t s_cp[kMaxColors + 1], s_e[kMaxColors + 1];
  const int nc = L.ncolors;
  if (nc == 0 || sweeps == 0) return;
  const long long tg = clock64();
  const int32_t n = L.n;
  const int64_t cap = L.sl_cap;
  const int nb = L.sl_nbuf;
  const int k0 = g_slice_k0;
  d4* s_x = (d4*)smem;
  d4* s_b = s_x + n;
  double* s_val = (double*)(s_b + n);               // [nb][cap]
  double* s_d = s_val + (int64_t)nb * cap;          // [n]
  int32_t* s_rp = (int32_t*)(s_d + n);              // [n+1]
  int32_t* s_id = s_rp + n + 1;                     // [n]
  int32_t* s_col = s_id + n;                        // [nb][cap]
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int i = tid; i <= nc; i += nt) {
    s_cp[i] = __ldg(L.sl_tab + i);
    s_e[i] = __ldg(L.sl_tab + nc + 1 + i);
  }
  for (int32_t i = tid; i < n; i += nt) {
    s_x[i] = ld4(x + (int64_t)i * K + k0);
    s_b[i] = ld4(b + (int64_t)i * K + k0);
    s_d[i] = __ldg(L.pdiag + i);
    s_rp[i] = (int32_t)__ldg(L.prp + i);
    s_id[i] = __ldg(L.row_ids + i);
  }
  if (tid == 0) s_rp[n] = (int32_t)__ldg(L.prp + n);
  bool fz[kV] = {false, false, false, false};
  bool any = false;
  if (!RES) {
#pragma unroll
    for (int q = 0; q < kV; ++q) {
      fz[q] = done && done[k0 + q];
      any = any || fz[q];
    }
  }
  __syncthreads();
  auto issue = [&](int cc, int buf) {  // the colour's entries -> buffer buf (asynchronous)
    const int32_t e0 = s_e[cc], e1 = s_e[cc + 1];
    double* dv = s_val + (int64_t)buf * cap;
    int32_t* dc = s_col + (int64_t)buf * cap;
    for (int32_t e = e0 + tid; e < e1; e += nt) {
      cp_async8(dv + (e - e0), L.pval + e);
      cp_async4(dc + (e - e0), L.pcol + e);
    }
    cp_async_commit();
  };
  const int P = sweeps * nc;
  long long a_stage = clock64() - tg, a_wait = 0, a_issue = 0, a_comp = 0;
  for (int q = 0; q < nb - 1; ++q) {  // nb - 1 colours in flight ahead of the one being folded
    if (q < P) issue(q % nc, q % nb);
    else cp_async_commit();
  }
  for (int p = 0; p < P; ++p) {
    const int cc = p % nc, buf = p % nb;
    // colour p's entries have landed once at most the nb - 2 newer groups are
    // pending; the barrier also orders phase p - 1's x writes and frees its buffer
    const long long t0 = clock64();
    if (nb == 3) cp_async_wait<1>();
    else cp_async_wait<0>();
    __syncthreads();
    const long long t1 = clock64();
    if (p + nb - 1 < P) issue((p + nb - 1) % nc, (p + nb - 1) % nb);
    else cp_async_commit();
    const long long t2 = clock64();
    const double* v = s_val + (int64_t)buf * cap;
    const int32_t* c = s_col + (int64_t)buf * cap;
    const int32_t c0 = s_cp[cc], c1 = s_cp[cc + 1], base = s_e[cc];
    for (int32_t i = c0 + tid; i < c1; i += nt) {
      const int32_t u = s_id[i];
      const int32_t r0 = s_rp[i] - base, r1 = s_rp[i + 1] - base;
      const double d = s_d[i];
      const d4 bv = s_b[u];
      double s0, s1, s2, s3;
      if (RES) {
        const d4 xu = s_x[u];
        s0 = d * xu.x, s1 = d * xu.y, s2 = d * xu.z, s3 = d * xu.w;
      } else {
        s0 = bv.x, s1 = bv.y, s2 = bv.z, s3 = bv.w;
      }
      // entries in batches of U: the batch's (col, val) and x reads are issued
      // together, then folded in entry order
      constexpr int U = 8;
      for (int32_t e0 = r0; e0 < r1; e0 += U) {
        int32_t cj[U];
        double w[U];
        d4 xv[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
          const bool ok = e0 + j < r1;
          cj[j] = ok ? c[e0 + j] : 0;
          w[j] = ok ? v[e0 + j] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < U; ++j) xv[j] = s_x[cj[j]];
#pragma unroll
        for (int j = 0; j < U; ++j)
          if (e0 + j < r1) {
            if (RES) {
              s0 = s0 + w[j] * xv[j].x;
              s1 = s1 + w[j] * xv[j].y;
              s2 = s2 + w[j] * xv[j].z;
              s3 = s3 + w[j] * xv[j].w;
            } else {
              s0 = s0 - w[j] * xv[j].x;
              s1 = s1 - w[j] * xv[j].y;
              s2 = s2 - w[j] * xv[j].z;
              s3 = s3 - w[j] * xv[j].w;
            }
          }
      }
      if (RES) {
        st4(r + (int64_t)u * K + k0, bv.x - s0, bv.y - s1, bv.z - s2, bv.w - s3);
      } else {
        d4 o{s0 / d, s1 / d, s2 / d, s3 / d};
        if (any) {
          const d4 old = s_x[u];
          if (fz[0]) o.x = old.x;
          if (fz[1]) o.y = old.y;
          if (fz[2]) o.z = old.z;
          if (fz[3]) o.w = old.w;
        }
        s_x[u] = o;
      }
    }
    a_wait += t1 - t0;
    a_issue += t2 - t1;
    a_comp += clock64() - t2;
  }
  cp_async_wait<0>();
  __syncthreads();
  if (!RES) {
    for (int32_t i = tid; i < n; i += nt) {
      const d4 o = s_x[i];
      st4(x + (int64_t)i * K + k0, o.x, o.y, o.z, o.w);
    }
  }
  __syncthreads();
  if (!RES && SliceScope::leader()) {
    ctr->phases += (long long)P;
    ctr->smem_calls += 1;
    ctr->smem_phases += (long long)P;
    ctr->lvl_gs_cyc[L.id] += clock64() - tg;
    ctr->lvl_gs_calls[L.id] += 1;
    ctr->lvl_ph[L.id][0] += a_stage;  // slice sweeps: staging, cp.async wait + barrier, issue, fold
    ctr->lvl_ph[L.id][1] += a_wait;
    ctr->lvl_ph[L.id][2] += a_issue;
    ctr->lvl_ph[L.id][3] += a_comp;
  }
}
template <int K>
__device__ inline void sl_gs(const TLevel& L, const double* __restrict__ b, double* x, int sweeps,
                             const int32_t* done, TailCounters* ctr) {
  sl_rows<K, false>(L, b, x, nullptr, sweeps, done, ctr);
}
template <int K>
__device__ inline void sl_residual(const TLevel& L, const double* __restrict__ b, const double* x, double* r) {
  sl_rows<K, true>(L, b, const_cast<double*>(x), r, 1, nullptr, nullptr);
}

template <class S, int K>
__device__ inline void nm_residual(const TLevel& L, const double* __restrict__ b, const double* x, double* r) {
  constexpr int T = S::template groups<K>();
  for (int64_t t = S::tid(); t < (int64_t)L.n * T; t += S::stride()) {
    const int64_t u = t / T;
    const int k0 = S::k0(t, T);
    const double d = __ldg(L.diag + u);
    const d4 xu = ld4(x + u * K + k0);
    double sv[kV] = {d * xu.x, d * xu.y, d * xu.z, d * xu.w};
    nm_fold<false>(sv, L.col, L.val, x, __ldg(L.rp + u), __ldg(L.rp + u + 1), K, k0);
    const d4 bv = ld4(b + u * K + k0);
    st4(r + u * K + k0, bv.x - sv[0], bv.y - sv[1], bv.z - sv[2], bv.w - sv[3]);
  }
  S::sync();
}

template <class S, int K>
__device__ inline void nm_restrict(const TLevel& L, const TLevel& C, const double* r, double mu) {
  constexpr int T = S::template groups<K>();
  for (int64_t t = S::tid(); t < (int64_t)C.n * T; t += S::stride()) {
    const int64_t g = t / T;
    const int k0 = S::k0(t, T);
    double sv[kV] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t j = __ldg(L.mem_ptr + g); j < __ldg(L.mem_ptr + g + 1); ++j) {
      const d4 rv = ld4(r + (int64_t)__ldg(L.mem + j) * K + k0);
      sv[0] = sv[0] + rv.x;
      sv[1] = sv[1] + rv.y;
      sv[2] = sv[2] + rv.z;
      sv[3] = sv[3] + rv.w;
    }
    if (mu != 1.0) st4(C.b + g * K + k0, sv[0] * mu, sv[1] * mu, sv[2] * mu, sv[3] * mu);
    else st4(C.b + g * K + k0, sv[0], sv[1], sv[2], sv[3]);
    st4(C.x + g * K + k0, 0.0, 0.0, 0.0, 0.0);
  }
  S::sync();
}

template <class S, int K>
__device__ inline void nm_interp(const TLevel& L, const TLevel& C, double* x) {
  constexpr int T = S::template groups<K>();
  for (int64_t t = S::tid(); t < (int64_t)L.n * T; t += S::stride()) {
    const int64_t u = t / T;
    const int k0 = S::k0(t, T);
    const d4 xv = ld4(x + u * K + k0);
    const d4 cv = ld4(C.x + (int64_t)__ldg(L.agg + u) * K + k0);
    st4(x + u * K + k0, xv.x + cv.x, xv.y + cv.y, xv.z + cv.z, xv.w + cv.w);
  }
  S::sync();
}

template <class S, int K>
__device__ inline void nm_coarsen(const StageV& s, const double* b, double* bc) {
  constexpr int T = S::template groups<K>();
  for (int64_t t = S::tid(); t < (int64_t)s.coarse_n * T; t += S::stride()) {
    const int64_t q = t / T;
    const int k0 = S::k0(t, T);
    const d4 bv = ld4(b + (int64_t)__ldg(s.poc + q) * K + k0);
    double v[kV] = {bv.x, bv.y, bv.z, bv.w};
    for (int64_t j = __ldg(s.t_ptr + q); j < __ldg(s.t_ptr + q + 1); ++j) {
      const int64_t p = __ldg(s.t_p + j);
      const int32_t i = __ldg(s.f_of_p + p);
      const double fv = __ldg(s.f_val + p), fd = __ldg(s.f_diag + i);
      const d4 fb = ld4(b + (int64_t)__ldg(s.f_nodes + i) * K + k0);
      v[0] = v[0] - fv * (fb.x / fd);
      v[1] = v[1] - fv * (fb.y / fd);
      v[2] = v[2] - fv * (fb.z / fd);
      v[3] = v[3] - fv * (fb.w / fd);
    }
    st4(bc + q * K + k0, v[0], v[1], v[2], v[3]);
  }
  S::sync();
}

template <class S, int K>
__device__ inline void nm_inject(const StageV& s, const double* x, double* xc) {
  constexpr int T = S::template groups<K>();
  for (int64_t t = S::tid(); t < (int64_t)s.coarse_n * T; t += S::stride()) {
    const int64_t q = t / T;
    const int k0 = S::k0(t, T);
    const d4 v = ld4(x + (int64_t)__ldg(s.poc + q) * K + k0);
    st4(xc + q * K + k0, v.x, v.y, v.z, v.w);
  }
  S::sync();
}

template <class S, int K>
__device__ inline void nm_backsub(const StageV& s, const double* xc, const double* b, double* x) {
  constexpr int T = S::template groups<K>();
  for (int64_t t = S::tid(); t < (int64_t)s.coarse_n * T; t += S::stride()) {
    const int64_t q = t / T;
    const int k0 = S::k0(t, T);
    const d4 v = ld4(xc + q * K + k0);
    st4(x + (int64_t)__ldg(s.poc + q) * K + k0, v.x, v.y, v.z, v.w);
  }
  S::sync();
  for (int64_t t = S::tid(); t < (int64_t)s.nf * T; t += S::stride()) {
    const int64_t i = t / T;
    const int k0 = S::k0(t, T);
    const int32_t f = __ldg(s.f_nodes + i);
    const d4 bv = ld4(b + (int64_t)f * K + k0);
    double sv[kV] = {bv.x, bv.y, bv.z, bv.w};
    for (int64_t p = __ldg(s.f_ptr + i); p < __ldg(s.f_ptr + i + 1); ++p) {
      const double fv = __ldg(s.f_val + p);
      const d4 xv = ld4(x + (int64_t)__ldg(s.f_nbr + p) * K + k0);
      sv[0] = sv[0] - fv * xv.x;
      sv[1] = sv[1] - fv * xv.y;
      sv[2] = sv[2] - fv * xv.z;
      sv[3] = sv[3] - fv * xv.w;
    }
    const double d = __ldg(s.f_diag + i);
    st4(x + (int64_t)f * K + k0, sv[0] / d, sv[1] / d, sv[2] / d, sv[3] / d);
  }
  S::sync();
}

// X = Minv[:n,:n] B per component (the throughput inverse; bdirect's order)
template <class S, int K>
__device__ inline void nm_direct(const TLevel& L, const double* b, double* x) {
  constexpr int T = S::template groups<K>();
  for (int32_t ci = 0; ci < L.ncomp; ++ci) {
    const int32_t s0 = __ldg(L.comp_start + ci), cn = __ldg(L.comp_start + ci + 1) - s0;
    const double* Mi = L.inv + __ldg(L.inv_off + ci);
    for (int64_t t = S::tid(); t < (int64_t)cn * T; t += S::stride()) {
      const int32_t i = (int32_t)(t / T);
      const int k0 = S::k0(t, T);
      double sv[kV] = {0.0, 0.0, 0.0, 0.0};
      for (int32_t j = 0; j < cn; ++j) {
        const double m = __ldg(Mi + (int64_t)i * cn + j);
        const d4 bv = ld4(b + (int64_t)(L.whole ? j : __ldg(L.nodes + s0 + j)) * K + k0);
        sv[0] += m * bv.x;
        sv[1] += m * bv.y;
        sv[2] += m * bv.z;
        sv[3] += m * bv.w;
      }
      st4(x + (int64_t)(L.whole ? i : __ldg(L.nodes + s0 + i)) * K + k0, sv[0], sv[1], sv[2], sv[3]);
    }
  }
  S::sync();
}

// per-column sums over the cluster in a K-independent order (kChunks chunks
// of R rows folded in sequence, chunk sums folded in sequence); every CTA
// gets all K sums in s_out (shared memory)
template <class S, int K, bool SQ>
__device__ inline void nm_colsum(const double* X, int64_t n, double* part, double* s_out) {
  const int64_t R = (n + kChunks - 1) / kChunks;
  const int np = (int)((n + R - 1) / R);
  constexpr int NC = S::template ncols<K>();  // the columns this scope's CTAs own
  const int c0 = S::template col0<K>();
  for (int64_t t = S::tid(); t < (int64_t)np * NC; t += S::stride()) {
    const int64_t p = t / NC;
    const int k = c0 + (int)(t % NC);
    const int64_t u1 = (p + 1) * R < n ? (p + 1) * R : n;
    double s = 0.0;
    for (int64_t u = p * R; u < u1; ++u) {
      const double v = X[u * K + k];
      s += SQ ? v * v : v;
    }
    part[(int64_t)k * kChunks + p] = s;
  }
  S::sync();
  if ((int)threadIdx.x < NC) {
    const int k = c0 + (int)threadIdx.x;
    double tot = 0.0;
    for (int p = 0; p < np; ++p) tot += ((volatile double*)part)[(int64_t)k * kChunks + p];
    s_out[k] = tot;
  }
  S::sync();  // part is reused by the next sum
}

// RelaxationSolver::solve (coarse_solver.cpp:82-93) per column; each column
// freezes at its own tolerance
template <class S, int K>
__device__ inline void nm_relax(const TLevel& L, const double* b, double* x, double* part, TailCounters* ctr) {
  __shared__ int32_t s_done[kMaxBlock];
  __shared__ double s_r0[kMaxBlock], s_sum[kMaxBlock];
  constexpr int T = S::template groups<K>();
  constexpr int NC = S::template ncols<K>();
  const int c0 = S::template col0<K>();
  const int64_t n = L.n;
  nm_residual<S, K>(L, b, x, L.r);
  nm_colsum<S, K, true>(L.r, n, part, s_sum);
  if ((int)threadIdx.x < NC) {
    const int k = c0 + (int)threadIdx.x;
    s_r0[k] = sqrt(s_sum[k]);
    s_done[k] = s_r0[k] == 0.0;
  }
  __syncthreads();
  if (S::leader()) ctr->work += (double)L.m;
  for (int sweep = 0; sweep < 400; ++sweep) {
    int active = 0;
    for (int k = c0; k < c0 + NC; ++k) active += !s_done[k];
    if (!active) break;
    if constexpr (std::is_same<S, SliceScope>::value) {
      if (L.sl_ok) sl_gs<K>(L, b, x, 1, s_done, ctr);
      else nm_gs<S, K>(L, b, x, 1, s_done, ctr);
    } else {
      nm_gs<S, K>(L, b, x, 1, s_done, ctr);
    }
    nm_colsum<S, K, false>(x, n, part, s_sum);
    for (int64_t t = S::tid(); t < n * T; t += S::stride()) {
      const int64_t u = t / T;
      const int k0 = S::k0(t, T);
#pragma unroll
      for (int q = 0; q < kV; ++q)
        if (!s_done[k0 + q]) x[u * K + k0 + q] -= s_sum[k0 + q] / (double)n;
    }
    S::sync();
    nm_residual<S, K>(L, b, x, L.r);
    nm_colsum<S, K, true>(L.r, n, part, s_sum);
    // (slice scope: every CTA sweeps until its own columns are done; the
    // counters follow CTA 0's columns)
    if (S::leader()) {
      ctr->work += 2.0 * (double)L.m;
      ctr->relax_sweeps += 1;
    }
    if ((int)threadIdx.x < NC) {
      const int k = c0 + (int)threadIdx.x;
      if (!s_done[k] && sqrt(s_sum[k]) <= 1e-12 * s_r0[k]) s_done[k] = 1;
    }
    __syncthreads();
  }
}

// single-column (any scope) or K-column column-slice (CTA scope) form of each
// operation of the recursion
template <class S, int K>
__device__ inline void op_gs(const TLevel& L, const double* b, double* x, int sweeps, TailCounters* ctr,
                             int32_t xs_rows) {
  if constexpr (K == 1) {
    gs<S>(L, b, x, sweeps, ctr, xs_rows);
  } else if constexpr (std::is_same<S, GridScope>::value) {
    if (L.gs_cta) {  // small level: CTA 0 sweeps, the cluster waits once
      if (blockIdx.x == 0) nm_gs<CtaScope, K>(L, b, x, sweeps, nullptr, ctr);
      GridScope::sync();
    } else {
      nm_gs<GridScope, K>(L, b, x, sweeps, nullptr, ctr);
    }
  } else if constexpr (std::is_same<S, SliceScope>::value) {
    if (L.sl_ok) sl_gs<K>(L, b, x, sweeps, nullptr, ctr);
    else nm_gs<S, K>(L, b, x, sweeps, nullptr, ctr);
  } else if constexpr (std::is_same<S, CtaScope>::value) {
    nm_gs<S, K>(L, b, x, sweeps, nullptr, ctr);
  }
  else if (L.smem_cs) cs_gs_smem<K>(L, b, x, sweeps, ctr);
  else cs_gs<K>(L, b, x, sweeps, nullptr, ctr);
}
template <class S, int K>
__device__ inline void op_residual(const TLevel& L, const double* b, const double* x, double* r) {
  if constexpr (K == 1) residual<S>(L, b, x, r);
  else if constexpr (std::is_same<S, SliceScope>::value) {
    if (L.sl_ok) sl_residual<K>(L, b, x, r);
    else nm_residual<S, K>(L, b, x, r);
  }
  else if constexpr (!std::is_same<S, BlockScope>::value) nm_residual<S, K>(L, b, x, r);
  else cs_residual<K>(L, b, x, r);
}
template <class S, int K>
__device__ inline void op_restrict(const TLevel& L, const TLevel& C, const double* r, double mu) {
  if constexpr (K == 1) restrict_to<S>(L, C, r, mu);
  else if constexpr (!std::is_same<S, BlockScope>::value) nm_restrict<S, K>(L, C, r, mu);
  else cs_restrict<K>(L, C, r, mu);
}
template <class S, int K>
__device__ inline void op_interp(const TLevel& L, const TLevel& C, double* x) {
  if constexpr (K == 1) interpolate<S>(L, C, x);
  else if constexpr (!std::is_same<S, BlockScope>::value) nm_interp<S, K>(L, C, x);
  else cs_interp<K>(L, C, x);
}
template <class S, int K>
__device__ inline void op_coarsen(const StageV& s, const double* b, double* bc) {
  if constexpr (K == 1) coarsen<S>(s, b, bc);
  else if constexpr (!std::is_same<S, BlockScope>::value) nm_coarsen<S, K>(s, b, bc);
  else cs_coarsen<K>(s, b, bc);
}
template <class S, int K>
__device__ inline void op_inject(const StageV& s, const double* x, double* xc) {
  if constexpr (K == 1) inject<S>(s, x, xc);
  else if constexpr (!std::is_same<S, BlockScope>::value) nm_inject<S, K>(s, x, xc);
  else cs_inject<K>(s, x, xc);
}
template <class S, int K>
__device__ inline void op_backsub(const StageV& s, const double* xc, const double* b, double* x) {
  if constexpr (K == 1) backsub<S>(s, xc, b, x);
  else if constexpr (!std::is_same<S, BlockScope>::value) nm_backsub<S, K>(s, xc, b, x);
  else cs_backsub<K>(s, xc, b, x);
}
template <class S, int K>
__device__ inline void op_direct(const TLevel& L, const double* b, double* x) {
  if constexpr (K == 1) direct(L, b, x);
  else if constexpr (!std::is_same<S, BlockScope>::value) nm_direct<S, K>(L, b, x);
  else cs_direct<K>(L, b, x);
}
template <class S, int K>
__device__ inline void op_relax(const TLevel& L, const double* b, double* x, double* sh, double* part,
                                TailCounters* ctr, int32_t xs_rows) {
  if constexpr (K == 1) relax<S>(L, b, x, sh, part, ctr, xs_rows);
  else if constexpr (!std::is_same<S, BlockScope>::value) nm_relax<S, K>(L, b, x, part, ctr);
  else cs_relax<K>(L, b, x, part, ctr);
}

struct Frame {
  int l, theta, it, step;
};

// per-operation cycle counters of the K-column tails (LAMG_TAIL_DEBUG)
__device__ inline long long now_cycles() { return clock64(); }
template <class S>
struct OpTimer {
  TailCounters* ctr;
  int op;
  long long t0;
  __device__ OpTimer(TailCounters* c, int o) : ctr(c), op(o), t0(now_cycles()) {}
  __device__ ~OpTimer() {
    if (S::leader()) {
      const int k = op + (std::is_same<S, SliceScope>::value ? 8 : 0);
      ctr->op_cyc[k] += now_cycles() - t0;
      ctr->op_calls[k] += 1;
    }
  }
};
#define OP_TIMED(op, call)     \
  do {                         \
    OpTimer<S> tm_(ctr, op);   \
    call;                      \
  } while (0)

// LevelCredit::take on the CTA's shared credits
__device__ inline int take(double* credits, int l, double gamma) {
  double cr = credits[l] + gamma;
  int th = (int)floor(cr);
  if (th < 1) th = 1;
  cr -= th;
  if (cr < 0.0) cr = 0.0;
  __syncthreads();
  if (threadIdx.x == 0) credits[l] = cr;
  __syncthreads();
  return th;
}

template <class S, int K>
__device__ void visit_loop(const TLevel* __restrict__ levels, int l0, int theta0, double* credits, double mu,
                           int32_t small_rows, double* sh, double* part, TailCounters* ctr, int32_t xs_rows);

// CTA 0 runs a small subtree alone; the other CTAs wait at the grid barrier
template <int K>
__device__ inline bool small_handoff(const TLevel* levels, const Frame& f, double* credits, double mu,
                                     int32_t small_rows, double* sh, double* part, TailCounters* ctr,
                                     int32_t xs_rows) {
  if constexpr (K > 1) {
    // K > 1: subtrees rooted at levels of at most xs_rows rows run as 4-column
    // slices, one per CTA (two rounds when there are more slices than CTAs):
    // no barrier between CTAs inside, x in shared memory (sl_gs)
    if (levels[f.l].n <= xs_rows) {
      __shared__ double credits0[kMaxLevels];
      const int nslices = K / kV;
      if (nslices > (int)gridDim.x) {
        for (int l = threadIdx.x; l < kMaxLevels; l += blockDim.x) credits0[l] = credits[l];
        __syncthreads();
      }
      for (int g = blockIdx.x; g < nslices; g += gridDim.x) {
        if (g != (int)blockIdx.x) {  // a second slice repeats the same visits: same credits
          __syncthreads();
          for (int l = threadIdx.x; l < kMaxLevels; l += blockDim.x) credits[l] = credits0[l];
        }
        if (threadIdx.x == 0) g_slice_k0 = g * kV;
        __syncthreads();
        visit_loop<SliceScope, K>(levels, f.l, f.theta, credits, mu, small_rows, sh, part, ctr, xs_rows);
      }
      GridScope::sync();
      return true;
    }
  }
  if (levels[f.l].n > small_rows) return false;
  // K > 1: CTA 0 runs the small subtree for all K columns, node-major
  using Small = typename std::conditional<K == 1, BlockScope, CtaScope>::type;
  if (blockIdx.x == 0) visit_loop<Small, K>(levels, f.l, f.theta, credits, mu, small_rows, sh, part, ctr, xs_rows);
  GridScope::sync();
  return true;
}

template <class S, int K>
__device__ void visit_loop(const TLevel* __restrict__ levels, int l0, int theta0, double* credits, double mu,
                           int32_t small_rows, double* sh, double* part, TailCounters* ctr, int32_t xs_rows) {
  Frame st[kMaxLevels];
  int sp = 0;
  st[sp++] = Frame{l0, theta0, 0, 0};
  while (sp > 0) {
    Frame& f = st[sp - 1];
    if (std::is_same<S, GridScope>::value && f.step == 0 && f.it == 0 &&
        small_handoff<K>(levels, f, credits, mu, small_rows, sh, part, ctr, xs_rows)) {
      --sp;
      continue;
    }
    const TLevel& L = levels[f.l];
    if (L.coarsest == CM_DIRECT) {
      OP_TIMED(7, (op_direct<S, K>(L, L.b, L.x)));
      if (S::leader()) ctr->work += (double)L.m;
      --sp;
      continue;
    }
    if (L.coarsest == CM_RELAX) {
      op_relax<S, K>(L, L.b, L.x, sh, part, ctr, xs_rows);
      --sp;
      continue;
    }
    const TLevel& C = levels[f.l + 1];
    if (L.child_kind == KIND_AGG) {
      if (f.step == 0) {
        if (f.it == f.theta) {
          --sp;
          continue;
        }
        if (C.nu_pre) OP_TIMED(0, (op_gs<S, K>(L, L.b, L.x, C.nu_pre, ctr, xs_rows)));
        OP_TIMED(1, (op_residual<S, K>(L, L.b, L.x, L.r)));
        OP_TIMED(2, (op_restrict<S, K>(L, C, L.r, mu)));
        if (S::leader()) ctr->work += (double)L.m * (C.nu_pre + 1);
        const int th = take(credits, f.l + 1, C.gamma);
        f.step = 1;
        st[sp++] = Frame{f.l + 1, th, 0, 0};
      } else {
        OP_TIMED(3, (op_interp<S, K>(L, C, L.x)));
        if (C.nu_post) OP_TIMED(0, (op_gs<S, K>(L, L.b, L.x, C.nu_post, ctr, xs_rows)));
        if (S::leader()) ctr->work += (double)L.m * C.nu_post;
        ++f.it;
        f.step = 0;
      }
    } else {  // elimination child (cycle.cpp:131-164)
      if (f.step == 0) {
        if (f.it == 0) {
          const double* in = L.b;
          for (int s = 0; s < L.nstages; ++s) {
            double* out = s + 1 < L.nstages ? L.stage_rhs[s + 1] : C.b;
            OP_TIMED(4, (op_coarsen<S, K>(L.stages[s], in, out)));
            in = out;
          }
          if (S::leader()) ctr->work += (double)L.elim_nnz;
        }
        if (f.it == f.theta) {
          --sp;
          continue;
        }
        const double* cur = L.x;
        for (int s = 0; s < L.nstages; ++s) {
          double* out = s + 1 < L.nstages ? L.stage_x[s + 1] : C.x;
          OP_TIMED(5, (op_inject<S, K>(L.stages[s], cur, out)));
          cur = out;
        }
        const int th = take(credits, f.l + 1, C.gamma);
        f.step = 1;
        st[sp++] = Frame{f.l + 1, th, 0, 0};
      } else {
        for (int s = L.nstages; s-- > 0;) {
          const double* xc = s + 1 < L.nstages ? L.stage_x[s + 1] : C.x;
          double* out = s == 0 ? L.x : L.stage_x[s];
          const double* rhs = s == 0 ? L.b : L.stage_rhs[s];
          OP_TIMED(6, (op_backsub<S, K>(L.stages[s], xc, rhs, out)));
        }
        if (S::leader()) ctr->work += (double)L.elim_nnz;
        ++f.it;
        f.step = 0;
      }
    }
  }
}

// MINB = 2 caps registers at 64 so two tail CTAs share an SM: best when
// many right-hand sides run concurrently; MINB = 1 (126 registers, no
// spills) gives the lowest single-solve latency. LAMG_TAIL_OCC selects.
template <int MINB, int K, int NT = kTailThreads>
__global__ void __launch_bounds__(NT, MINB) tail_kernel(const TLevel* __restrict__ levels, int nlevels, int l0,
                                                            int theta0, double* credits_g, double mu,
                                                            int32_t small_rows, double* part, TailCounters* ctr,
                                                            int32_t xs_rows) {
  __shared__ double credits[kMaxLevels];
  __shared__ double sh[64];
  const long long t_start = clock64();
  for (int l = threadIdx.x; l < nlevels; l += blockDim.x) credits[l] = credits_g[l];
  __syncthreads();
  visit_loop<GridScope, K>(levels, l0, theta0, credits, mu, small_rows, sh, part, ctr, xs_rows);
  if (blockIdx.x == 0) {
    for (int l = threadIdx.x; l < nlevels; l += blockDim.x) credits_g[l] = credits[l];
    if (threadIdx.x == 0) ctr->cyc_total += clock64() - t_start;
  }
}

// K > 1: the small-level subtree as a plain launch of K/kc CTAs, each the
// whole sub-cycle for its own kc columns -- no inter-CTA synchronisation
template <int K>
__global__ void __launch_bounds__(kTailThreadsBatch, 1) subtree_kernel(const TLevel* __restrict__ levels,
                                                                   int nlevels, int l0, int theta0,
                                                                   double* credits_g, double mu, int32_t small_rows,
                                                                   double* part, TailCounters* ctr, int32_t xs_rows) {
  __shared__ double credits[kMaxLevels];
  __shared__ double sh[64];
  const long long t_start = clock64();
  double* mine = credits_g + (int64_t)blockIdx.x * kMaxLevels;  // per-CTA copy (see slice_kernel)
  for (int l = threadIdx.x; l < nlevels; l += blockDim.x) credits[l] = mine[l];
  // the root level arrives node-major from the host-driven levels: my columns in
  const TLevel& R = levels[l0];
  const ColSlice sl = my_cols<K>();
  const int64_t n = R.n;
  for (int64_t t = threadIdx.x; t < n << sl.sh; t += blockDim.x) {
    const int64_t u = t >> sl.sh, k = sl.k0 + (t & (sl.kc - 1));
    R.b[k * n + u] = R.nm_b[u * K + k];
    R.x[k * n + u] = R.nm_x[u * K + k];
  }
  __syncthreads();
  visit_loop<BlockScope, K>(levels, l0, theta0, credits, mu, small_rows, sh, part, ctr, xs_rows);
  for (int64_t t = threadIdx.x; t < n << sl.sh; t += blockDim.x) {
    const int64_t u = t >> sl.sh, k = sl.k0 + (t & (sl.kc - 1));
    R.nm_x[u * K + k] = R.x[k * n + u];
  }
  for (int l = threadIdx.x; l < nlevels; l += blockDim.x) mine[l] = credits[l];
  if (blockIdx.x == 0 && threadIdx.x == 0) ctr->cyc_total += clock64() - t_start;
}

// K > 1, column slices (the default block tail): K/4 independent CTAs, CTA g
// the whole sub-cycle for columns 4g..4g+3 on the node-major vectors in place
// (its 32-byte sector of every row) -- no cluster, no barrier between CTAs
template <int K>
__global__ void __launch_bounds__(kTailThreadsSlice, 1) slice_kernel(const TLevel* __restrict__ levels, int nlevels,
                                                                    int l0, int theta0, double* credits_g, double mu,
                                                                    int32_t small_rows, double* part,
                                                                    TailCounters* ctr, int32_t xs_rows) {
  __shared__ double credits[kMaxLevels];
  __shared__ double sh[64];
  const long long t_start = clock64();
  // every CTA keeps its own copy of the (identical) credits: no CTA reads
  // what another writes, whenever each is scheduled
  double* mine = credits_g + (int64_t)blockIdx.x * kMaxLevels;
  for (int l = threadIdx.x; l < nlevels; l += blockDim.x) credits[l] = mine[l];
  if (threadIdx.x == 0) g_slice_k0 = (int)blockIdx.x * kV;
  __syncthreads();
  visit_loop<SliceScope, K>(levels, l0, theta0, credits, mu, small_rows, sh, part, ctr, xs_rows);
  for (int l = threadIdx.x; l < nlevels; l += blockDim.x) mine[l] = credits[l];
  if (blockIdx.x == 0 && threadIdx.x == 0) ctr->cyc_total += clock64() - t_start;
}

}  // namespace

void TailPlan::build(Ctx& c, const DHier& h, Workspace& ws, int32_t max_rows) {
  const int nl = (int)h.levels.size();
  // blocks of columns: by default the node-major cluster tail (nm_* ops);
  // LAMG_BATCH_TAIL=subtree selects the per-column CTA subtree below 4096 rows
  const char* et = getenv("LAMG_BATCH_TAIL");
  subtree = ws.K > 1 && ws.K <= 32 && et && strcmp(et, "subtree") == 0;
  slice = ws.K > 1 && !subtree && et && strcmp(et, "slice") == 0;
  const bool nm = ws.K > 1 && !subtree;
  if (subtree) {
    const char* eb = getenv("LAMG_BATCH_SMALL");
    max_rows = eb ? atoi(eb) : 4096;
  }
  first = nl;  // no tail
  for (int l = 1; l < nl; ++l)
    if (h.levels[l]->op.n <= max_rows) {
      first = l;
      break;
    }
  if (first >= nl || nl > kMaxLevels) {
    first = 1 << 30;
    return;
  }
  const char* e1 = getenv("LAMG_TAIL_SMALL");
  small_rows = subtree ? max_rows : e1 ? atoi(e1) : 4096;
  const char* e3 = getenv("LAMG_TAIL_SMEM_KB");
  smem = e3 ? std::min(kTailSmemMax, atoi(e3) * 1024) : 0;  // operators via L1/L2 unless set
  // x and b of the CTA-scope levels in shared memory (LAMG_TAIL_XSMEM=1; measured
  // neutral on cfg2: the phases are bound by the L2 chain of the operator rows)
  const char* e5 = getenv("LAMG_TAIL_XSMEM");
  xs_rows = (e5 && atoi(e5) == 1) ? small_rows : 0;
  const char* e2 = getenv(nm ? "LAMG_BATCH_CTAS" : "LAMG_TAIL_CTAS");
  ctas = std::max(1, std::min(e2 ? atoi(e2) : (nm ? 16 : 8), 16));  // one cluster (<= 16 CTAs)
  if (nm) {
    // subtrees rooted at levels of at most this many rows run in CTA 0 alone
    // (a phase is a __syncthreads instead of a cluster barrier)
    const char* es = getenv("LAMG_BATCH_SMALL");
    small_rows = es ? atoi(es) : 0;
    smem = 0;
    xs_rows = 0;
  }
  std::vector<TLevel> tl(nl);
  for (int l = first; l < nl; ++l) {
    const DLevel& L = *h.levels[l];
    TLevel& t = tl[l];
    memset(&t, 0, sizeof t);
    t.id = l;
    const CSRv a = L.op.view();
    t.n = a.n;
    t.m = a.m;
    t.rp = a.rp;
    t.col = a.col;
    t.val = a.val;
    t.diag = a.diag;
    t.b = ws.lv[l].b.p;
    t.x = ws.lv[l].x.p;
    t.r = ws.lv[l].r.p;
    t.gamma = L.gamma;
    t.nu_pre = L.nu_pre;
    t.nu_post = L.nu_post;
    t.coarsest = L.coarsest;
    t.group = row_group_for(a.n, a.m);
    if (L.color) {
      t.ncolors = L.color->ncolors;
      t.cptr = (const int32_t*)(L.color->rp.p + a.n + 1);
      t.row_ids = L.color->row_ids.p;
      t.prp = L.color->rp.p;
      t.pcol = L.color->col.p;
      t.pval = L.color->val.p;
      t.pdiag = L.color->diag.p;
      const int64_t bytes = (int64_t)a.n * (3 * 8 + 4 + 4) + 4 + 2 * a.m * 12 + 4 * (L.color->ncolors + 1);
      t.smem_ok = bytes <= smem;
    }
    if (L.direct) {
      const DDirect& d = *L.direct;
      t.ncomp = d.ncomp;
      t.comp_start = d.comp_start.p;
      t.nodes = d.nodes.p;
      t.inv = d.inv.p;
      t.inv_off = d.inv_off.p;
      t.whole = d.ncomp == 1;
      if (!nm && a.n > small_rows) small_rows = a.n;  // the one-column direct coarsest runs in one CTA
    }
    if (l + 1 < nl && L.coarsest == CM_NONE) {
      const DLevel& C = *h.levels[l + 1];
      t.child_kind = C.kind;
      if (C.kind == KIND_AGG) {
        t.agg = C.agg->aggregate_of.p;
        t.mem_ptr = C.agg->mem_ptr.p;
        t.mem = C.agg->mem.p;
      } else {
        t.nstages = (int)C.stages.size();
        if (t.nstages > kMaxStages) throw LamgError(LAMG_E_ERROR, "tail: too many elimination stages");
        for (int s = 0; s < t.nstages; ++s) {
          t.stages[s] = C.stages[s]->view();
          t.elim_nnz += C.stages[s]->nnzf;
          if (s >= 1) {
            t.stage_rhs[s] = ws.lv[l].stage_rhs[s].p;
            t.stage_x[s] = ws.lv[l].stage_x[s].p;
          }
        }
      }
    }
  }
  xs_rows = std::min(xs_rows, small_rows);
  smem = std::max(smem, (int)(2 * 8 * (int64_t)xs_rows));
  if (smem > kTailSmemMax) {
    xs_rows = 0;
    smem = std::min(smem, kTailSmemMax);
  }
  if (nm) {
    // slice scope (the standalone slice kernel, and the cluster tail's small
    // subtrees): levels whose x slice and two colour buffers fit the dynamic
    // shared memory sweep from it (sl_gs); the cluster hands a subtree to the
    // slices when every level in it does (LAMG_BATCH_SLICE_ROWS caps the root)
    const int64_t budget = kTailSmemMax;
    int64_t need = 0;
    std::vector<int32_t> sl_tab_h;
    std::vector<int64_t> sl_off(nl, -1);
    for (int l = first; l < nl; ++l) {
      const DLevel& L = *h.levels[l];
      if (!L.color) continue;
      const std::vector<int64_t> rp = L.color->rp.to_host();
      int64_t cap = 0;
      for (int32_t cc = 0; cc < L.color->ncolors; ++cc)
        cap = std::max(cap, rp[L.color->cptr_h[cc + 1]] - rp[L.color->cptr_h[cc]]);
      cap = (cap + 1) / 2 * 2;
      tl[l].sl_cap = (int32_t)cap;
      sl_off[l] = (int64_t)sl_tab_h.size();
      for (int32_t cc = 0; cc <= L.color->ncolors; ++cc) sl_tab_h.push_back(L.color->cptr_h[cc]);
      for (int32_t cc = 0; cc <= L.color->ncolors; ++cc) sl_tab_h.push_back((int32_t)rp[L.color->cptr_h[cc]]);
      tl[l].sl_nbuf = sl_smem_bytes(L.op.n, cap, 3) <= budget ? 3 : 2;
      tl[l].sl_ok = L.color->ncolors <= kMaxColors && 2 * L.op.m < (1ll << 31) &&
                    sl_smem_bytes(L.op.n, cap, tl[l].sl_nbuf) <= budget;
      if (tl[l].sl_ok) need = std::max(need, sl_smem_bytes(L.op.n, cap, tl[l].sl_nbuf));
    }
    sl_tabs.alloc(std::max<int64_t>((int64_t)sl_tab_h.size(), 1), c.s);
    sl_tabs.upload(sl_tab_h.data(), (int64_t)sl_tab_h.size());
    for (int l = first; l < nl; ++l) tl[l].sl_tab = sl_off[l] >= 0 ? sl_tabs.p + sl_off[l] : nullptr;
    const char* er = getenv("LAMG_BATCH_SLICE_ROWS");
    const int32_t cap_rows = er ? atoi(er) : 1 << 30;
    int root = nl;  // first level of the all-sl_ok suffix
    for (int l = nl - 1; l >= first; --l) {
      const DLevel& L = *h.levels[l];
      const bool ok = (!L.color || tl[l].sl_ok) && L.op.n <= cap_rows && L.coarsest != CM_RELAX;
      if (!ok) break;
      root = l;
    }
    xs_rows = !slice && root < nl ? h.levels[root]->op.n : 0;
    if (!slice && root >= nl) need = 0;
    smem = (int)need;
  }
  K = ws.K;
  if (subtree) {  // column-slice sweeps stage operator + slice in shared memory
    const char* e6 = getenv("LAMG_BATCH_SMEM_KB");
    smem = std::min(kTailSmemMax, (e6 ? atoi(e6) : 200) * 1024);
  }
  credits.alloc((int64_t)kMaxLevels * (kMaxBlock / kV), c.s);  // a slot per CTA of the slice / subtree forms
  ctr.alloc(1, c.s);
  const char* e4 = getenv("LAMG_TAIL_OCC");
  occ2 = !(e4 && atoi(e4) == 1);
  threads = K > 1 ? (slice ? kTailThreadsSlice : kTailThreadsBatch) : kTailThreads;
  if (slice) ctas = K / kV;
  if (subtree) {
    const char* ek = getenv("LAMG_BATCH_KC");
    int kc = ek ? std::max(1, atoi(ek)) : 1;
    while (K % kc) --kc;
    ctas = K / kc;
  }
  if (slice) {
    switch (K) {
      case 4: kernel = (const void*)slice_kernel<4>; break;
      case 8: kernel = (const void*)slice_kernel<8>; break;
      case 16: kernel = (const void*)slice_kernel<16>; break;
      case 32: kernel = (const void*)slice_kernel<32>; break;
      case 64: kernel = (const void*)slice_kernel<64>; break;
      case 128: kernel = (const void*)slice_kernel<128>; break;
      default: throw LamgError(LAMG_E_ARGUMENT, "tail: unsupported batch width");
    }
  } else
  switch (K) {
    case 1: kernel = occ2 ? (const void*)tail_kernel<2, 1> : (const void*)tail_kernel<1, 1>; break;
    // K > 1: 256 threads (255 registers) -- the column-slice phases are
    // latency-bound chains, more warps per CTA only add issue overhead
    case 4: kernel = subtree ? (const void*)subtree_kernel<4> : (const void*)tail_kernel<1, 4, kTailThreadsBatch>; break;
    case 8: kernel = subtree ? (const void*)subtree_kernel<8> : (const void*)tail_kernel<1, 8, kTailThreadsBatch>; break;
    case 16:
      kernel = subtree ? (const void*)subtree_kernel<16> : (const void*)tail_kernel<1, 16, kTailThreadsBatch>;
      break;
    case 32:
      kernel = subtree ? (const void*)subtree_kernel<32> : (const void*)tail_kernel<1, 32, kTailThreadsBatch>;
      break;
    case 64: kernel = (const void*)tail_kernel<1, 64, kTailThreadsBatch>; break;
    case 128: kernel = (const void*)tail_kernel<1, 128, kTailThreadsBatch>; break;
    default: throw LamgError(LAMG_E_ARGUMENT, "tail: unsupported batch width");
  }
  CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTailSmemMax));
  CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  // largest cluster the device can co-schedule with this footprint
  while (!subtree && !slice && ctas > 1) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = ctas;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, kernel, &cfg) == cudaSuccess && nclusters > 0) break;
    cudaGetLastError();
    ctas /= 2;
  }
  part.alloc(std::max<int64_t>(std::max(ctas, 1), kChunks) * K, c.s);
  if (subtree) {
    const int kc = K >= ctas ? K / ctas : 1;
    for (int l = first; l < nl; ++l) {
      const DLevel& L = *h.levels[l];
      tl[l].smem_cs = L.color && L.op.n <= small_rows &&
                      cs_smem_bytes(L.op.n, 2 * L.op.m, L.color->ncolors, kc) <= smem;
    }
  }
  if (nm) {  // LAMG_BATCH_GS_CTA=rows: sweeps of levels this small run in CTA 0 (tools/micro/phase_bench)
    const char* eg = getenv("LAMG_BATCH_GS_CTA");
    const int32_t gs_rows = eg ? atoi(eg) : 0;  // off: slower in the full kernel (extra-row chains)
    for (int l = first; l < nl; ++l) tl[l].gs_cta = h.levels[l]->op.n <= gs_rows;
  }
  if (subtree) {  // column-major copies of the root level's b and x (see subtree_kernel)
    const int64_t rn = (int64_t)h.levels[first]->op.n * K;
    root_b.alloc(rn, c.s);
    root_x.alloc(rn, c.s);
    tl[first].nm_b = tl[first].b;
    tl[first].nm_x = tl[first].x;
    tl[first].b = root_b.p;
    tl[first].x = root_x.p;
  }
  dlevels.alloc(nl, c.s);
  CK(cudaMemcpyAsync(dlevels.p, tl.data(), sizeof(TLevel) * nl, cudaMemcpyHostToDevice, c.s));
  c.sync();
}

void TailPlan::reset(Ctx& c) {
  if (!credits.n) return;
  credits.zero();
  ctr.zero();
}

void TailPlan::run(Ctx& c, int l, int theta, double mu, int nlevels) {
  // LAMG_SKIP_TAIL=1 (timing experiments only: wrong results): the sub-cycle below
  // the host-driven levels is not run, which isolates the cost of the levels above
  static const bool skip = getenv("LAMG_SKIP_TAIL") && atoi(getenv("LAMG_SKIP_TAIL")) == 1;
  if (skip) return;
  const TLevel* lv = dlevels.p;
  double* cr = credits.p;
  double* pt = part.p;
  TailCounters* ct = ctr.p;
  int32_t sr = small_rows;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c.s;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = ctas;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = subtree || slice ? 0 : 1;
  count_launch();
  int32_t xr = xs_rows;
  void* args[] = {(void*)&lv, &nlevels, &l, &theta, &cr, &mu, &sr, &pt, &ct, &xr};
  CK(cudaLaunchKernelExC(&cfg, kernel, args));
}

void TailPlan::collect(Ctx& c, double* work, int* relax_sweeps) {
  if (!ctr.n) return;
  TailCounters h;
  CK(cudaMemcpyAsync(&h, ctr.p, sizeof h, cudaMemcpyDeviceToHost, c.s));
  c.sync();
  *work += h.work;
  *relax_sweeps += (int)h.relax_sweeps;
  if (getenv("LAMG_TAIL_DEBUG"))
    fprintf(stderr,
            "[tail] first %d ctas %d small %d: phases %lld, %lld cycles in tail kernels; smem: %lld calls %lld "
            "phases, stage %.0f cyc/call, %.0f cyc/phase; global gs: %lld phases %.0f cyc/phase\n",
            first, ctas, small_rows, h.phases, h.cyc_total, h.smem_calls, h.smem_phases,
            h.smem_calls ? (double)h.cyc_stage / h.smem_calls : 0.0,
            h.smem_phases ? (double)h.cyc_phases / h.smem_phases : 0.0, h.global_phases,
            h.global_phases ? (double)h.cyc_global_gs / h.global_phases : 0.0);
  if (getenv("LAMG_TAIL_DEBUG")) print_debug(h);
}

void TailPlan::print_debug(const TailCounters& h) const {
  if (h.global_phases)
    fprintf(stderr, "[tail] grid phase breakdown (CTA0 thread0, cycles/phase): fold %.0f extra %.0f prefetch %.0f barrier %.0f\n",
            (double)h.ph_fold / h.global_phases, (double)h.ph_extra / h.global_phases,
            (double)h.ph_prefetch / h.global_phases, (double)h.ph_barrier / h.global_phases);
  static const char* names[8] = {"gs", "residual", "restrict", "interp", "coarsen", "inject", "backsub", "direct"};
  for (int k = 0; k < 16; ++k)
    if (h.op_calls[k])
      fprintf(stderr, "[tail]   %-7s %-8s calls %8lld  %9.0f cycles/call  %5.1f%% of tail cycles\n",
              k < 8 ? "cluster" : "slice", names[k & 7], h.op_calls[k], (double)h.op_cyc[k] / h.op_calls[k],
              100.0 * h.op_cyc[k] / std::max(1LL, h.cyc_total));
  for (int l = 0; l < kMaxLevels; ++l)
    if (h.lvl_gs_calls[l])
      fprintf(stderr,
              "[tail]   level %2d: gs calls %8lld  %10.0f cycles/call  %5.1f%% of tail cycles; per call: first %.0f "
              "extra %.0f prefetch %.0f barrier %.0f\n",
              l, h.lvl_gs_calls[l], (double)h.lvl_gs_cyc[l] / h.lvl_gs_calls[l],
              100.0 * h.lvl_gs_cyc[l] / std::max(1LL, h.cyc_total), (double)h.lvl_ph[l][0] / h.lvl_gs_calls[l],
              (double)h.lvl_ph[l][1] / h.lvl_gs_calls[l], (double)h.lvl_ph[l][2] / h.lvl_gs_calls[l],
              (double)h.lvl_ph[l][3] / h.lvl_gs_calls[l]);
}

}  // namespace lamgb
