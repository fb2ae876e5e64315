// setup.cu -- device setup phase: elimination, probe, test vectors, affinity,
// hubs, aggregation, Galerkin, coarsest factorisation, and the setup driver.
//
// Decision rules are the reference's, made order-free where the reference is
// sequential (SURVEY.md Appendix A "Verified equivalences"):
//  - the low-degree independent set is the lexicographically-first MIS of the
//    candidates, resolved in rounds (a row decides once every lower candidate
//    neighbour has);
//  - greedy aggregation visits nodes in (min affinity, index) order; a node
//    decides once every earlier-ordered neighbour has, reading the same
//    statuses the sequential scan would;
//  - hash-map accumulations (Schur, Galerkin) become a stable sort by key of
//    the contributions in emission order followed by an in-order fold.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <limits>

#include <math_constants.h>

#include "hier.cuh"

namespace lamgb {

static uint64_t rng_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
// Rng::derive (rng.hpp:34-37): third draw of Rng(seed ^ c*(stream+1))
uint64_t rng_derive_host(uint64_t seed, uint64_t stream) {
  uint64_t s = seed ^ (0xd1342543de82ef95ULL * (stream + 1));
  if (!s) s = 0x9e3779b97f4a7c15ULL;
  return rng_mix(s + 3 * 0x9e3779b97f4a7c15ULL);
}

static int bits_for(uint64_t maxval) {
  int b = 1;
  while (b < 64 && (1ull << b) <= maxval) ++b;
  return b;
}

// ====================================================================
// assemble_canonical on the device (sparse_laplacian.cpp:60-104) from an
// edge list sorted by (u,v), u<v, merged, zero weights dropped. Row x holds
// its lower neighbours (edges (u,x), u ascending) then its upper ones
// ((x,v), v ascending); diag[x] folds w in that order, as the reference's
// edge-ordered fill does.
// ====================================================================
__global__ void seg_bounds_i32_kernel(const int32_t* sorted_key, int64_t n, int32_t nseg,
                                      int64_t* ptr) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > n) return;
  int64_t lo = i == 0 ? 0 : (int64_t)sorted_key[i - 1] + 1;
  int64_t hi = i == n ? nseg : sorted_key[i];
  for (int64_t k = lo; k <= hi && k <= nseg; ++k) ptr[k] = i;
}

__global__ void row_counts_kernel(int32_t n, const int64_t* uptr, const int64_t* vptr, int64_t* cnt) {
  int32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x < n) cnt[x] = (uptr[x + 1] - uptr[x]) + (vptr[x + 1] - vptr[x]);
}

__global__ void assemble_fill_kernel(int32_t n, int64_t E, const int32_t* eu, const int32_t* ev,
                                     const double* ew, const int64_t* uptr, const int64_t* vptr,
                                     const int32_t* vperm, const int64_t* rp, int32_t* col,
                                     double* val, double* diag) {
  int32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n) return;
  int64_t o = rp[x];
  double d = 0.0;
  for (int64_t j = vptr[x]; j < vptr[x + 1]; ++j) {  // edges (u, x), u ascending
    int32_t e = vperm[j];
    col[o] = eu[e];
    val[o] = -ew[e];
    d = d + ew[e];
    ++o;
  }
  for (int64_t e = uptr[x]; e < uptr[x + 1]; ++e) {  // edges (x, v), v ascending
    col[o] = ev[e];
    val[o] = -ew[e];
    d = d + ew[e];
    ++o;
  }
  diag[x] = d;
}

__global__ void ev_keys_kernel(const int32_t* ev, int64_t E, uint64_t* key, int32_t* ids) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= E) return;
  key[i] = (uint64_t)(uint32_t)ev[i];
  ids[i] = (int32_t)i;
}
__global__ void narrow_kernel(const uint64_t* in, int64_t n, int32_t* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = (int32_t)in[i];
}

void assemble_canonical_dev(Ctx& c, int32_t n, int64_t E, const int32_t* eu,
                                   const int32_t* ev, const double* ew, DCSR& out) {
  if (n <= 0) throw LamgError(LAMG_E_EMPTY_GRAPH, "cannot assemble a Laplacian with n = 0");
  out.alloc(n, E, c.s);
  DVec<int64_t> uptr(n + 1, c.s), vptr(n + 1, c.s), cnt(n + 1, c.s);
  DVec<int32_t> vperm(std::max<int64_t>(E, 1), c.s);
  if (E > 0) {
    // u-segments: eu is sorted
    count_launch(), seg_bounds_i32_kernel<<<blocks_for(E + 1), kThreads, 0, c.s>>>(eu, E, n, uptr.p);
    // v-segments: stable sort of edge ids by v
    DVec<uint64_t> k(E, c.s), ks(E, c.s);
    DVec<int32_t> ids(E, c.s), vs(E, c.s);
    count_launch(), ev_keys_kernel<<<blocks_for(E), kThreads, 0, c.s>>>(ev, E, k.p, ids.p);
    CK_LAUNCH();
    sort_pairs_u64_i32(c, k.p, ks.p, ids.p, vperm.p, E, bits_for((uint64_t)n));
    count_launch(), narrow_kernel<<<blocks_for(E), kThreads, 0, c.s>>>(ks.p, E, vs.p);
    count_launch(), seg_bounds_i32_kernel<<<blocks_for(E + 1), kThreads, 0, c.s>>>(vs.p, E, n, vptr.p);
    CK_LAUNCH();
  } else {
    uptr.zero();
    vptr.zero();
  }
  count_launch(), row_counts_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(n, uptr.p, vptr.p, cnt.p);
  CK_LAUNCH();
  CK(cudaMemsetAsync(cnt.p + n, 0, sizeof(int64_t), c.s));
  exclusive_scan_i64(c, cnt.p, out.rp.p, n + 1);
  count_launch(), assemble_fill_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(n, E, eu, ev, ew, uptr.p, vptr.p, vperm.p,
                                                          out.rp.p, out.col.p, out.val.p, out.diag.p);
  CK_LAUNCH();
}

// Sorted-contribution fold shared by Schur and Galerkin: keys are
// (min<<32 | max) in emission order; a stable sort groups equal keys with
// their emission order intact, each group folds from 0.0 and exact zeros are
// dropped (elimination.cpp:93-101, aggregation.cpp:293-501).
__global__ void seg_heads_kernel(const uint64_t* k, int64_t n, uint8_t* head) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) head[i] = (i == 0 || k[i] != k[i - 1]);
}
__global__ void seg_fold_kernel(const uint64_t* k, const double* w, const int64_t* heads,
                                int64_t nseg, int64_t n, double* sum, uint8_t* keep) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  int64_t b = heads[s], e = s + 1 < nseg ? heads[s + 1] : n;
  double acc = 0.0;
  for (int64_t i = b; i < e; ++i) acc = acc + w[i];
  sum[s] = acc;
  keep[s] = acc != 0.0;
}
__global__ void emit_edges_kernel(const int64_t* keep_idx, int64_t ne, const int64_t* heads,
                                  const uint64_t* k, const double* sum, int32_t* eu, int32_t* ev,
                                  double* ew) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= ne) return;
  int64_t s = keep_idx[j];
  uint64_t key = k[heads[s]];
  eu[j] = (int32_t)(key >> 32);
  ev[j] = (int32_t)(key & 0xffffffffu);
  ew[j] = sum[s];
}

static void fold_contribs_and_assemble(Ctx& c, int32_t coarse_n, int64_t nc, DVec<uint64_t>& keys,
                                       DVec<double>& w, DCSR& out) {
  if (nc == 0) {
    assemble_canonical_dev(c, coarse_n, 0, nullptr, nullptr, nullptr, out);
    return;
  }
  DVec<uint64_t> ks(nc, c.s);
  DVec<double> ws(nc, c.s);
  sort_pairs_u64_d(c, keys.p, ks.p, w.p, ws.p, nc, 32 + bits_for((uint64_t)coarse_n));
  keys.release();
  w.release();
  DVec<uint8_t> head(nc, c.s);
  count_launch(), seg_heads_kernel<<<blocks_for(nc), kThreads, 0, c.s>>>(ks.p, nc, head.p);
  CK_LAUNCH();
  DVec<int64_t> heads(nc, c.s);
  int64_t nseg = select_flagged_index64(c, head.p, heads.p, nc);
  DVec<double> sum(nseg, c.s);
  DVec<uint8_t> keep(nseg, c.s);
  count_launch(), seg_fold_kernel<<<blocks_for(nseg), kThreads, 0, c.s>>>(ks.p, ws.p, heads.p, nseg, nc, sum.p, keep.p);
  CK_LAUNCH();
  DVec<int64_t> kidx(nseg, c.s);
  int64_t ne = select_flagged_index64(c, keep.p, kidx.p, nseg);
  DVec<int32_t> eu(std::max<int64_t>(ne, 1), c.s), ev(std::max<int64_t>(ne, 1), c.s);
  DVec<double> ew(std::max<int64_t>(ne, 1), c.s);
  count_launch(), emit_edges_kernel<<<blocks_for(ne), kThreads, 0, c.s>>>(kidx.p, ne, heads.p, ks.p, sum.p, eu.p, ev.p, ew.p);
  CK_LAUNCH();
  assemble_canonical_dev(c, coarse_n, ne, eu.p, ev.p, ew.p, out);
}

__device__ inline uint64_t pair_key(int32_t a, int32_t b) {
  if (a > b) {
    int32_t t = a;
    a = b;
    b = t;
  }
  return ((uint64_t)(uint32_t)a << 32) | (uint32_t)b;
}

// ====================================================================
// Galerkin P^T A P (aggregation.cpp:280-313)
// ====================================================================
__global__ void galerkin_flags_kernel(CSRv a, const int64_t* up_entry, const int32_t* up_row,
                                      int64_t cnt, const int32_t* agg, uint8_t* flag) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= cnt) return;
  flag[j] = agg[up_row[j]] != agg[a.col[up_entry[j]]];
}
__global__ void galerkin_emit_kernel(CSRv a, const int64_t* up_entry, const int32_t* up_row,
                                     const int64_t* sel, int64_t nc, const int32_t* agg,
                                     uint64_t* key, double* w) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nc) return;
  int64_t j = sel[i];
  int64_t e = up_entry[j];
  key[i] = pair_key(agg[up_row[j]], agg[a.col[e]]);
  w[i] = -a.val[e];
}

void galerkin(Ctx& c, const CSRv& a, const int32_t* agg, int32_t coarse_n, DCSR& out) {
  UpperIndex up;
  build_upper_index(c, a, up);
  DVec<uint8_t> flag(std::max<int64_t>(up.count, 1), c.s);
  count_launch(), galerkin_flags_kernel<<<blocks_for(up.count), kThreads, 0, c.s>>>(a, up.entry.p, up.row.p, up.count, agg, flag.p);
  CK_LAUNCH();
  DVec<int64_t> sel(std::max<int64_t>(up.count, 1), c.s);
  int64_t nc = select_flagged_index64(c, flag.p, sel.p, up.count);
  DVec<uint64_t> keys(std::max<int64_t>(nc, 1), c.s);
  DVec<double> w(std::max<int64_t>(nc, 1), c.s);
  count_launch(), galerkin_emit_kernel<<<blocks_for(nc), kThreads, 0, c.s>>>(a, up.entry.p, up.row.p, sel.p, nc, agg, keys.p, w.p);
  CK_LAUNCH();
  fold_contribs_and_assemble(c, coarse_n, nc, keys, w, out);
  c.work += (double)a.m;
}

// ====================================================================
// Low-degree independent set (elimination.cpp:11-27): the sequential greedy
// in index order picks u iff u is a candidate (1 <= deg <= 4, diag > 0) and
// no lower candidate neighbour was picked. Rounds: an undecided candidate
// becomes OUT as soon as a lower candidate neighbour is IN, and IN once all
// its lower candidate neighbours are OUT.
// ====================================================================
enum { MIS_UNDEC = 0, MIS_IN = 1, MIS_OUT = 2, MIS_NONCAND = 3 };

__global__ void mis_init_kernel(CSRv a, int32_t maxdeg, int8_t* state, int32_t* undecided) {
  int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= a.n) return;
  int64_t deg = a.rp[u + 1] - a.rp[u];
  bool cand = deg > 0 && deg <= maxdeg && a.diag[u] > 0.0;
  state[u] = cand ? MIS_UNDEC : MIS_NONCAND;
  if (cand) atomicAdd(undecided, 1);
}

__global__ void mis_rounds_kernel(CSRv a, int8_t* state, int32_t* undecided) {
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  volatile int8_t* vs = state;
  while (true) {
    grid_barrier();
    int32_t left = *(volatile int32_t*)undecided;
    grid_barrier();
    if (left == 0) break;
    for (int64_t u = gtid; u < a.n; u += gstride) {
      if (vs[u] != MIS_UNDEC) continue;
      bool any_in = false, all_dec = true;
      for (int64_t k = a.rp[u]; k < a.rp[u + 1]; ++k) {
        int32_t v = a.col[k];
        if (v >= u) continue;
        int8_t s = vs[v];
        if (s == MIS_IN) {
          any_in = true;
          break;
        }
        if (s == MIS_UNDEC) all_dec = false;
      }
      if (any_in) {
        vs[u] = MIS_OUT;
        atomicSub(undecided, 1);
      } else if (all_dec) {
        vs[u] = MIS_IN;
        atomicSub(undecided, 1);
      }
    }
  }
}

__global__ void mis_flags_kernel(const int8_t* state, int32_t n, uint8_t* fflag, uint8_t* cflag) {
  int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  fflag[u] = state[u] == MIS_IN;
  cflag[u] = state[u] != MIS_IN;
}

void select_low_degree(Ctx& c, const CSRv& a, int32_t max_degree, SelectResult& out) {
  const int32_t n = a.n;
  DVec<int8_t> state(n, c.s);
  int32_t* undecided = c.dflag + 16;
  CK(cudaMemsetAsync(undecided, 0, sizeof(int32_t), c.s));
  count_launch(), mis_init_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(a, max_degree, state.p, undecided);
  CK_LAUNCH();
  const int threads = 256;
  int blocks = std::min(c.max_coop_blocks((const void*)mis_rounds_kernel, threads), blocks_for(n, threads));
  if (n < 8192) blocks = 1;
  CSRv av = a;
  void* args[] = {&av, &state.p, &undecided};
  coop_launch(c, (const void*)mis_rounds_kernel, blocks, threads, args);
  DVec<uint8_t> ff(n, c.s), cf(n, c.s);
  count_launch(), mis_flags_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(state.p, n, ff.p, cf.p);
  CK_LAUNCH();
  out.f.alloc(n, c.s);
  out.c.alloc(n, c.s);
  out.nf = (int32_t)select_flagged_index(c, ff.p, out.f.p, n);
  out.nc = (int32_t)select_flagged_index(c, cf.p, out.c.p, n);
}

// ====================================================================
// Schur complement (elimination.cpp:29-105)
// ====================================================================
__global__ void cop_init_kernel(int32_t n, int32_t* cop) {
  int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u < n) cop[u] = -1;
}
__global__ void cop_set_kernel(const int32_t* cset, int32_t nc, int32_t* cop) {
  int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nc) cop[cset[k]] = k;
}
__global__ void f_deg_kernel(CSRv a, const int32_t* f, int32_t nf, int64_t* deg, int64_t* pairs) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nf) return;
  int64_t d = a.rp[f[i] + 1] - a.rp[f[i]];
  deg[i] = d;
  pairs[i] = d * (d - 1) / 2;
}
__global__ void schur_check_kernel(CSRv a, const int32_t* f, int32_t nf, const int32_t* cop, DevErr* err) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nf) return;
  int32_t fu = f[i];
  unsigned long long base = (unsigned long long)i << 32;
  if (cop[fu] >= 0) { dev_report(err, base | 0, DE_SCHUR_OVERLAP, fu, 0); return; }
  if (a.diag[fu] <= 0.0) { dev_report(err, base | 1, DE_SCHUR_PIVOT, fu, 0); return; }
  for (int64_t k = a.rp[fu]; k < a.rp[fu + 1]; ++k) {
    if (cop[a.col[k]] < 0) {
      dev_report(err, base | ((unsigned long long)(k - a.rp[fu] + 1) << 2) | 2, DE_SCHUR_DEPENDENT, fu, a.col[k]);
      return;
    }
  }
}
__global__ void stage_fill_kernel(CSRv a, const int32_t* f, int32_t nf, const int64_t* f_ptr,
                                  double* f_diag, int32_t* f_nbr, double* f_val) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nf) return;
  int32_t fu = f[i];
  f_diag[i] = a.diag[fu];
  int64_t o = f_ptr[i];
  for (int64_t k = a.rp[fu]; k < a.rp[fu + 1]; ++k, ++o) {
    f_nbr[o] = a.col[k];
    f_val[o] = a.val[k];
  }
}
// retained C-C edges in (c order, column) order
__global__ void cc_count_kernel(CSRv a, const int32_t* cset, int32_t nc, const int32_t* cop, int64_t* cnt) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nc) return;
  int32_t cu = cset[i];
  int64_t n = 0;
  for (int64_t k = a.rp[cu]; k < a.rp[cu + 1]; ++k) {
    int32_t v = a.col[k];
    if (cop[v] >= 0 && v > cu) ++n;
  }
  cnt[i] = n;
}
__global__ void cc_emit_kernel(CSRv a, const int32_t* cset, int32_t nc, const int32_t* cop,
                               const int64_t* off, uint64_t* key, double* w) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nc) return;
  int32_t cu = cset[i];
  int64_t o = off[i];
  for (int64_t k = a.rp[cu]; k < a.rp[cu + 1]; ++k) {
    int32_t v = a.col[k];
    if (cop[v] >= 0 && v > cu) {
      key[o] = pair_key(cop[cu], cop[v]);
      w[o] = -a.val[k];
      ++o;
    }
  }
}
// fill cliques in (f order, p < q) order: w_fp w_fq / a_ff
__global__ void fill_emit_kernel(int32_t nf, const int64_t* f_ptr, const int32_t* f_nbr,
                                 const double* f_val, const double* f_diag, const int32_t* cop,
                                 const int64_t* poff, int64_t base, uint64_t* key, double* w) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nf) return;
  int64_t o = base + poff[i];
  double aff = f_diag[i];
  for (int64_t p = f_ptr[i]; p < f_ptr[i + 1]; ++p)
    for (int64_t q = p + 1; q < f_ptr[i + 1]; ++q) {
      key[o] = pair_key(cop[f_nbr[p]], cop[f_nbr[q]]);
      w[o] = (f_val[p] * f_val[q]) / aff;
      ++o;
    }
}

void schur_reduce(Ctx& c, const CSRv& a, const int32_t* f, int32_t nf, const int32_t* cset,
                  int32_t nc, DStage& st, DCSR& coarse, bool check_inputs) {
  const int32_t n = a.n;
  st.parent_n = n;
  st.coarse_n = nc;
  st.nf = nf;
  st.cop.alloc(n, c.s);
  count_launch(), cop_init_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(n, st.cop.p);
  count_launch(), cop_set_kernel<<<blocks_for(nc), kThreads, 0, c.s>>>(cset, nc, st.cop.p);
  CK_LAUNCH();
  st.poc.alloc(std::max(nc, 1), c.s);
  if (nc) CK(cudaMemcpyAsync(st.poc.p, cset, sizeof(int32_t) * nc, cudaMemcpyDeviceToDevice, c.s));
  st.f_nodes.alloc(std::max(nf, 1), c.s);
  if (nf) CK(cudaMemcpyAsync(st.f_nodes.p, f, sizeof(int32_t) * nf, cudaMemcpyDeviceToDevice, c.s));
  if (check_inputs && nf) {
    CSRv av = a;
    c.checked([&] {
      count_launch(), schur_check_kernel<<<blocks_for(nf), kThreads, 0, c.s>>>(av, f, nf, st.cop.p, c.derr);
      CK_LAUNCH();
    });
  }
  DVec<int64_t> deg(nf + 1, c.s), pairs(nf + 1, c.s), poff(nf + 1, c.s);
  st.f_ptr.alloc(nf + 1, c.s);
  if (nf) {
    count_launch(), f_deg_kernel<<<blocks_for(nf), kThreads, 0, c.s>>>(a, f, nf, deg.p, pairs.p);
    CK_LAUNCH();
  }
  CK(cudaMemsetAsync(deg.p + nf, 0, sizeof(int64_t), c.s));
  CK(cudaMemsetAsync(pairs.p + nf, 0, sizeof(int64_t), c.s));
  exclusive_scan_i64(c, deg.p, st.f_ptr.p, nf + 1);
  exclusive_scan_i64(c, pairs.p, poff.p, nf + 1);
  st.nnzf = read_i64(c, st.f_ptr.p + nf);
  int64_t npairs = read_i64(c, poff.p + nf);
  st.f_diag.alloc(std::max(nf, 1), c.s);
  st.f_nbr.alloc(std::max<int64_t>(st.nnzf, 1), c.s);
  st.f_val.alloc(std::max<int64_t>(st.nnzf, 1), c.s);
  if (nf) {
    count_launch(), stage_fill_kernel<<<blocks_for(nf), kThreads, 0, c.s>>>(a, f, nf, st.f_ptr.p, st.f_diag.p, st.f_nbr.p, st.f_val.p);
    CK_LAUNCH();
  }
  // emission: C-C edges first, then the fill cliques
  DVec<int64_t> ccnt(nc + 1, c.s), coff(nc + 1, c.s);
  if (nc) {
    count_launch(), cc_count_kernel<<<blocks_for(nc), kThreads, 0, c.s>>>(a, cset, nc, st.cop.p, ccnt.p);
    CK_LAUNCH();
  }
  CK(cudaMemsetAsync(ccnt.p + nc, 0, sizeof(int64_t), c.s));
  exclusive_scan_i64(c, ccnt.p, coff.p, nc + 1);
  int64_t ncc = read_i64(c, coff.p + nc);
  int64_t total = ncc + npairs;
  DVec<uint64_t> keys(std::max<int64_t>(total, 1), c.s);
  DVec<double> w(std::max<int64_t>(total, 1), c.s);
  if (nc) count_launch(), cc_emit_kernel<<<blocks_for(nc), kThreads, 0, c.s>>>(a, cset, nc, st.cop.p, coff.p, keys.p, w.p);
  if (nf)
    count_launch(), fill_emit_kernel<<<blocks_for(nf), kThreads, 0, c.s>>>(nf, st.f_ptr.p, st.f_nbr.p, st.f_val.p, st.f_diag.p,
                                                           st.cop.p, poff.p, ncc, keys.p, w.p);
  CK_LAUNCH();
  fold_contribs_and_assemble(c, nc, total, keys, w, coarse);
  c.work += (double)(a.m + coarse.m);
  build_stage_transpose(c, nc, nf, st.f_ptr.p, st.f_nbr.p, st.cop.p, st.nnzf, st.t_ptr, st.t_p, st.f_of_p);
  st.ntlong = stage_long_lists(c, nc, st.t_ptr.p, st.tlong);
}

// elimination.cpp:107-124
bool eliminate_rounds(Ctx& c, const CSRv& a, std::vector<std::unique_ptr<DStage>>& stages, DCSR& coarse) {
  stages.clear();
  DCSR cur_store;
  CSRv cur = a;
  while (cur.n > 1) {
    SelectResult sel;
    select_low_degree(c, cur, 4, sel);
    if ((double)sel.nf < 0.01 * cur.n || sel.nf == 0 || sel.nc == 0) break;
    auto st = std::make_unique<DStage>();
    DCSR next;
    schur_reduce(c, cur, sel.f.p, sel.nf, sel.c.p, sel.nc, *st, next, false);
    stages.push_back(std::move(st));
    cur_store = std::move(next);
    cur = cur_store.view();
  }
  if (stages.empty()) return false;
  coarse = std::move(cur_store);
  return true;
}

// ====================================================================
// probe_relaxation (smoothing.cpp:59-89) and generate_tvs (:42-57)
// ====================================================================
double probe_factor(Ctx& c, const CSRv& a, const Schedule& sch, const UpperIndex& up, int sweeps, uint64_t seed,
                    bool exact);

// The probe's output is one threshold decision (factor <= 0.7, hierarchy.cpp
// setup loop); its folds (means, energies) are the reference's sequential
// ones only to reproduce that decision. They run as fixed-order tree sums
// first: a sequential and a tree sum of the same terms differ by at most
// (n-1) eps sum|t| (2 m eps ~ 1e-7 relative at m = 5e8), which moves the
// factor (an 8th root of an energy ratio) by far less than the 1e-6 margin;
// inside the margin the probe is rerun with the exact folds. The decision --
// and so the hierarchy -- is the reference's either way.
double probe_relaxation(Ctx& c, const CSRv& a, const Schedule& sch, const UpperIndex& up,
                        int sweeps, uint64_t seed) {
  const double w0 = c.work;  // the work counter is charged for one probe, as the reference's
  const double fast = probe_factor(c, a, sch, up, sweeps, seed, false);
  if (std::fabs(fast - 0.7) > 1e-6 * 0.7) return fast;
  c.work = w0;
  return probe_factor(c, a, sch, up, sweeps, seed, true);
}

double probe_factor(Ctx& c, const CSRv& a, const Schedule& sch, const UpperIndex& up, int sweeps, uint64_t seed,
                    bool exact) {
  DVec<double> x(a.n, c.s), scratch;
  auto sub_mean = [&] {
    if (exact) subtract_mean_seq(c, x.p, a.n);
    else subtract_mean_tree(c, x.p, a.n);
  };
  auto energy = [&](double* out) {
    if (exact) energy_seq(c, a, up, x.p, out, scratch);
    else energy_tree(c, a, up, x.p, out, scratch);
  };
  fill_pm1(c, x.p, a.n, rng_derive_host(seed, 0x9));
  sub_mean();
  const int half = sweeps / 2;
  double* e_mid = c.dscal + 100;
  double* e_end = c.dscal + 101;
  CK(cudaMemsetAsync(e_mid, 0, sizeof(double), c.s));
  bool have_mid = false;
  for (int s = 0; s < sweeps; ++s) {
    gs_exact(c, a, sch, nullptr, x.p, 1, 1);
    c.work += (double)a.m;
    sub_mean();
    if (s + 1 == half) {
      energy(e_mid);
      c.work += (double)a.m;
      have_mid = true;
    }
  }
  energy(e_end);
  c.work += (double)a.m;
  CK(cudaMemcpyAsync(c.hscal, e_mid, 2 * sizeof(double), cudaMemcpyDeviceToHost, c.s));
  c.sync();
  double em = c.hscal[0], ee = c.hscal[1];
  double norm_mid = have_mid ? (em > 0.0 ? std::sqrt(em) : 0.0) : 0.0;
  double norm_end = ee > 0.0 ? std::sqrt(ee) : 0.0;
  if (half == 0) norm_mid = 0.0;
  if (norm_end == 0.0 || norm_mid == 0.0) return 0.0;
  return std::pow(norm_end / norm_mid, 1.0 / (double)(sweeps - half));
}

void generate_tvs(Ctx& c, const CSRv& a, const Schedule& sch, int K, int sweeps, uint64_t seed,
                  DVec<double>& X) {
  X.alloc((int64_t)a.n * K, c.s);
  for (int k = 0; k < K; ++k) fill_pm1(c, X.p, a.n, rng_derive_host(seed, (uint64_t)k), K, k);
  gs_exact(c, a, sch, nullptr, X.p, K, sweeps);
  c.work += (double)K * sweeps * (double)a.m;
  subtract_mean_seq(c, X.p, a.n, K);
}

// ====================================================================
// affinities (aggregation.cpp:83-116) and hubs (:118-134)
// ====================================================================
__global__ void node_norm_kernel(const double* __restrict__ X, int32_t n, int K, double* nn) {
  int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  double s = 0.0;
  for (int k = 0; k < K; ++k) {
    double x = X[(int64_t)u * K + k];
    s = s + x * x;
  }
  nn[u] = s;
}
__global__ void affinity_kernel(CSRv a, const double* __restrict__ X, int K,
                                const double* __restrict__ nn, double* aff) {
  int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= a.n) return;
  for (int64_t e = a.rp[u]; e < a.rp[u + 1]; ++e) {
    int32_t v = a.col[e];
    int32_t lo = u < v ? u : v, hi = u < v ? v : u;  // the reference evaluates at (u<v)
    double c;
    if (nn[lo] == 0.0 || nn[hi] == 0.0) {
      c = 1.0;
    } else {
      double dot = 0.0;
      for (int k = 0; k < K; ++k) dot = dot + X[(int64_t)lo * K + k] * X[(int64_t)hi * K + k];
      c = 1.0 - (dot * dot) / (nn[lo] * nn[hi]);
      c = c < 0.0 ? 0.0 : (1.0 < c ? 1.0 : c);
    }
    aff[e] = c;
  }
}

void compute_affinities(Ctx& c, const CSRv& a, int K, const double* X, double* aff, double* nn) {
  count_launch(), node_norm_kernel<<<blocks_for(a.n), kThreads, 0, c.s>>>(X, a.n, K, nn);
  count_launch(), affinity_kernel<<<blocks_for(a.n), kThreads, 0, c.s>>>(a, X, K, nn, aff);
  CK_LAUNCH();
  c.work += (double)K * (double)a.m;
}

__global__ void hub_flags_kernel(CSRv a, uint8_t* flag) {
  int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= a.n) return;
  flag[u] = 0;
  int64_t b = a.rp[u], e = a.rp[u + 1];
  if (b == e) return;
  double num = 0.0, den = 0.0;
  for (int64_t k = b; k < e; ++k) {
    double aw = fabs(a.val[k]);
    int32_t v = a.col[k];
    num = num + aw * (double)(a.rp[v + 1] - a.rp[v]);
    den = den + aw;
  }
  if (den == 0.0) return;
  flag[u] = (double)(e - b) >= 8.0 * num / den;
}

int32_t detect_hubs(Ctx& c, const CSRv& a, DVec<int32_t>& hubs) {
  DVec<uint8_t> flag(a.n, c.s);
  count_launch(), hub_flags_kernel<<<blocks_for(a.n), kThreads, 0, c.s>>>(a, flag.p);
  CK_LAUNCH();
  hubs.alloc(a.n, c.s);
  return (int32_t)select_flagged_index(c, flag.p, hubs.p, a.n);
}

// ====================================================================
// aggregation (aggregation.cpp:142-278)
// ====================================================================
enum { ST_UNDEC = 0, ST_SEED = 1, ST_ASSOC = 2 };

__global__ void strongest_kernel(CSRv a, double* strongest) {
  int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= a.n) return;
  double s = 0.0;
  for (int64_t k = a.rp[u]; k < a.rp[u + 1]; ++k) {
    double e = fabs(a.val[k]);
    if (s < e) s = e;
  }
  strongest[u] = s;
}

__device__ inline bool edge_usable(const double* strongest, int32_t u, int32_t v, double entry) {
  double su = strongest[u], sv = strongest[v];
  double mn = sv < su ? sv : su;  // std::min(su, sv)
  return fabs(entry) >= 1e-3 * mn;
}

__global__ void dummy_kernel(CSRv a, const double* strongest, uint8_t* dummy) {
  int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= a.n) return;
  bool any = false;
  for (int64_t k = a.rp[u]; k < a.rp[u + 1] && !any; ++k) any = edge_usable(strongest, u, a.col[k], a.val[k]);
  dummy[u] = any ? 0 : 1;
}

__global__ void status_init_kernel(int32_t n, int8_t* status, int32_t* seed_ref) {
  int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  status[u] = ST_UNDEC;
  seed_ref[u] = -1;
}
__global__ void hubs_seed_kernel(const int32_t* hubs, int32_t nh, const uint8_t* dummy, int8_t* status) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nh && !dummy[hubs[i]]) status[hubs[i]] = ST_SEED;
}

// order key: minimal usable non-dummy affinity (aggregation.cpp:192-204)
__global__ void order_key_kernel(CSRv a, const double* strongest, const uint8_t* dummy,
                                 const int8_t* status, const double* aff, uint8_t* inorder,
                                 uint64_t* key) {
  int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= a.n) return;
  inorder[u] = 0;
  if (dummy[u] || status[u] != ST_UNDEC) return;
  double best = CUDART_INF;
  for (int64_t k = a.rp[u]; k < a.rp[u + 1]; ++k) {
    int32_t v = a.col[k];
    if (!edge_usable(strongest, u, v, a.val[k]) || dummy[v]) continue;
    double c = aff[k];
    if (c < best) best = c;
  }
  if (best < CUDART_INF) {
    inorder[u] = 1;
    key[u] = (uint64_t)__double_as_longlong(best + 0.0);  // affinities are >= 0: bits are monotone
  }
}
__global__ void gather_keys_kernel(const int32_t* idx, int64_t cnt, const uint64_t* key, uint64_t* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < cnt) out[i] = key[idx[i]];
}
__global__ void order_pos_kernel(const int32_t* order, int64_t cnt, int32_t* pos) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < cnt) pos[order[i]] = (int32_t)i;
}
__global__ void fill_i32_kernel(int32_t* x, int64_t n, int32_t v) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) x[i] = v;
}

// Status-free candidate flag per directed entry u->s: s not dummy, edge
// usable, and the nodal-energy inflation of aggregating u with s is <= 2.5
// (NodalQuadratic::build / inflation_vs, aggregation.cpp:26-79).
constexpr int kMaxK = 16;
__global__ void candidate_kernel(CSRv a, const double* __restrict__ X, int K,
                                 const double* strongest, const uint8_t* dummy, uint8_t* cand) {
  int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= a.n) return;
  const int64_t b0 = a.rp[u], e0 = a.rp[u + 1];
  if (dummy[u]) {
    for (int64_t j = b0; j < e0; ++j) cand[j] = 0;
    return;
  }
  const double a_uu = a.diag[u];
  double bq[kMaxK], cq[kMaxK], rm[kMaxK];
  for (int k = 0; k < K; ++k) bq[k] = cq[k] = 0.0;
  for (int64_t j = b0; j < e0; ++j) {
    double w = -a.val[j];
    int32_t v = a.col[j];
    for (int k = 0; k < K; ++k) {
      double xv = X[(int64_t)v * K + k];
      bq[k] = bq[k] + w * xv;
      cq[k] = cq[k] + 0.5 * w * xv * xv;
    }
  }
  for (int k = 0; k < K; ++k) rm[k] = a_uu > 0.0 ? cq[k] - bq[k] * bq[k] / (2.0 * a_uu) : cq[k];
  for (int64_t j = b0; j < e0; ++j) {
    int32_t s = a.col[j];
    if (dummy[s] || !edge_usable(strongest, u, s, a.val[j])) {
      cand[j] = 0;
      continue;
    }
    double q = -CUDART_INF;
    for (int k = 0; k < K; ++k) {
      double relaxed = rm[k];
      if (relaxed <= 0.0) continue;
      double y = X[(int64_t)s * K + k];
      double at = 0.5 * a_uu * y * y - bq[k] * y + cq[k];
      double v = at / relaxed;
      if (q < v) q = v;
    }
    if (q == -CUDART_INF) q = 1.0;
    cand[j] = q <= 2.5;
  }
}

// Greedy seed/associate scan, resolved in rounds (aggregation.cpp:206-230).
__global__ void greedy_rounds_kernel(CSRv a, const int32_t* order, int32_t norder, const int32_t* pos,
                                     const uint8_t* cand, const double* aff, int8_t* status,
                                     int32_t* seed_ref, int8_t* done, int32_t* remaining) {
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  volatile int8_t* vst = status;
  volatile int8_t* vdone = done;
  while (true) {
    grid_barrier();
    int32_t left = *(volatile int32_t*)remaining;
    grid_barrier();
    if (left == 0) break;
    for (int64_t i = gtid; i < norder; i += gstride) {
      const int32_t u = order[i];
      if (vdone[u]) continue;
      bool ready = true;
      for (int64_t k = a.rp[u]; k < a.rp[u + 1]; ++k) {
        int32_t p = pos[a.col[k]];
        if (p >= 0 && p < i && !vdone[a.col[k]]) {
          ready = false;
          break;
        }
      }
      if (!ready) continue;
      __threadfence();
      if (vst[u] == ST_UNDEC) {
        int32_t best_s = -1;
        double best_c = CUDART_INF;
        for (int64_t k = a.rp[u]; k < a.rp[u + 1]; ++k) {
          if (!cand[k]) continue;
          int32_t s = a.col[k];
          if (vst[s] == ST_ASSOC) continue;
          double c = aff[k];
          if (c < best_c || (c == best_c && s < best_s)) {
            best_c = c;
            best_s = s;
          }
        }
        if (best_s >= 0) {
          if (vst[best_s] == ST_UNDEC) vst[best_s] = ST_SEED;
          vst[u] = ST_ASSOC;
          seed_ref[u] = best_s;
        }
      }
      __threadfence();
      vdone[u] = 1;
      atomicSub(remaining, 1);
    }
  }
}

__global__ void root_flags_kernel(int32_t n, const uint8_t* dummy, const int8_t* status,
                                  const int32_t* first_dummy, int32_t* root, int32_t* count_nonassoc) {
  int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  int32_t r;
  if (dummy[u]) r = (u == *first_dummy);
  else r = status[u] != ST_ASSOC;
  root[u] = r;
  if (!dummy[u] && status[u] != ST_ASSOC) atomicAdd(count_nonassoc, 1);
}
__global__ void first_dummy_kernel(int32_t n, const uint8_t* dummy, int32_t* first) {
  int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u < n && dummy[u]) atomicMin(first, u);
}
__global__ void number_roots_kernel(int32_t n, const uint8_t* dummy, const int8_t* status,
                                    const int32_t* root, const int32_t* ids, const int32_t* first_dummy,
                                    int32_t* agg, int32_t* seed_of) {
  int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  if (dummy[u]) {
    agg[u] = ids[*first_dummy];
    if (root[u]) seed_of[ids[u]] = -1;
  } else if (status[u] != ST_ASSOC) {
    agg[u] = ids[u];
    seed_of[ids[u]] = u;
  }
}
__global__ void number_assoc_kernel(int32_t n, const uint8_t* dummy, const int8_t* status,
                                    const int32_t* seed_ref, int32_t* agg) {
  int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  if (!dummy[u] && status[u] == ST_ASSOC) agg[u] = agg[seed_ref[u]];
}

void aggregate(Ctx& c, const CSRv& a, int K, const double* X, double gamma, const int32_t* hubs,
               int32_t nhubs, DAgg& out, int* stages_run) {
  if (K > kMaxK) throw LamgError(LAMG_E_ARGUMENT, "aggregate: at most 16 test vectors supported");
  const int32_t n = a.n;
  const int64_t nnz = 2 * a.m;
  DVec<double> aff(std::max<int64_t>(nnz, 1), c.s), nn(n, c.s), strongest(n, c.s);
  compute_affinities(c, a, K, X, aff.p, nn.p);
  count_launch(), strongest_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(a, strongest.p);
  DVec<uint8_t> dummy(n, c.s);
  count_launch(), dummy_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(a, strongest.p, dummy.p);
  DVec<int8_t> status(n, c.s), done(n, c.s);
  DVec<int32_t> seed_ref(n, c.s);
  count_launch(), status_init_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(n, status.p, seed_ref.p);
  if (nhubs) count_launch(), hubs_seed_kernel<<<blocks_for(nhubs), kThreads, 0, c.s>>>(hubs, nhubs, dummy.p, status.p);
  CK_LAUNCH();
  // stage-1 visiting order: (min affinity, node) ascending
  DVec<uint8_t> inorder(n, c.s);
  DVec<uint64_t> key(n, c.s);
  count_launch(), order_key_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(a, strongest.p, dummy.p, status.p, aff.p, inorder.p, key.p);
  CK_LAUNCH();
  DVec<int32_t> members(n, c.s);
  int32_t norder = (int32_t)select_flagged_index(c, inorder.p, members.p, n);
  DVec<int32_t> order(std::max(norder, 1), c.s), pos(n, c.s);
  count_launch(), fill_i32_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(pos.p, n, -1);
  CK_LAUNCH();
  if (norder) {
    DVec<uint64_t> k1(norder, c.s), k2(norder, c.s);
    count_launch(), gather_keys_kernel<<<blocks_for(norder), kThreads, 0, c.s>>>(members.p, norder, key.p, k1.p);
    CK_LAUNCH();
    sort_pairs_u64_i32(c, k1.p, k2.p, members.p, order.p, norder, 64);  // stable: ties by node
    count_launch(), order_pos_kernel<<<blocks_for(norder), kThreads, 0, c.s>>>(order.p, norder, pos.p);
    CK_LAUNCH();
  }
  DVec<uint8_t> cand(std::max<int64_t>(nnz, 1), c.s);
  count_launch(), candidate_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(a, X, K, strongest.p, dummy.p, cand.p);
  CK_LAUNCH();
  done.zero();
  int32_t* remaining = c.dflag + 20;
  CK(cudaMemcpyAsync(remaining, &norder, sizeof(int32_t), cudaMemcpyHostToDevice, c.s));
  if (norder) {
    const int threads = 256;
    int blocks = std::min(c.max_coop_blocks((const void*)greedy_rounds_kernel, threads), blocks_for(norder, threads));
    if (norder < 8192) blocks = 1;
    CSRv av = a;
    void* args[] = {&av, &order.p, &norder, &pos.p, &cand.p, &aff.p, &status.p, &seed_ref.p, &done.p, &remaining};
    coop_launch(c, (const void*)greedy_rounds_kernel, blocks, threads, args);
  }
  // numbering (aggregation.cpp:249-276): ids by an exclusive scan over roots
  int32_t* first_dummy = c.dflag + 24;
  int32_t* nonassoc = c.dflag + 25;
  int32_t init[2] = {std::numeric_limits<int32_t>::max(), 0};
  CK(cudaMemcpyAsync(first_dummy, init, sizeof init, cudaMemcpyHostToDevice, c.s));
  count_launch(), first_dummy_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(n, dummy.p, first_dummy);
  DVec<int32_t> root(n + 1, c.s), ids(n + 1, c.s);
  count_launch(), root_flags_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(n, dummy.p, status.p, first_dummy, root.p, nonassoc);
  CK_LAUNCH();
  CK(cudaMemsetAsync(root.p + n, 0, sizeof(int32_t), c.s));
  exclusive_scan_i32(c, root.p, ids.p, n + 1);
  int32_t coarse_n = read_i32(c, ids.p + n);
  int32_t hv[2];
  CK(cudaMemcpyAsync(hv, first_dummy, sizeof hv, cudaMemcpyDeviceToHost, c.s));
  c.sync();
  const bool has_dummy = hv[0] != std::numeric_limits<int32_t>::max();
  out.fine_n = n;
  out.coarse_n = coarse_n;
  out.aggregate_of.alloc(n, c.s);
  out.seed_of.alloc(std::max(coarse_n, 1), c.s);
  count_launch(), number_roots_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(n, dummy.p, status.p, root.p, ids.p, first_dummy,
                                                         out.aggregate_of.p, out.seed_of.p);
  count_launch(), number_assoc_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(n, dummy.p, status.p, seed_ref.p, out.aggregate_of.p);
  CK_LAUNCH();
  if (has_dummy) out.dummy_aggregate = read_i32(c, ids.p + hv[0]);
  else out.dummy_aggregate = -1;
  // stage-1 coarsening ratio; the reference's second stage never changes the
  // result (statuses only move Undecided -> Seed/Associate, so its candidate
  // sets only shrink) and is charged but not re-run
  const int32_t count = (has_dummy ? 1 : 0) + hv[1];
  const double alpha1 = n > 0 ? (double)count / (double)n : 1.0;
  *stages_run = alpha1 <= 0.7 / gamma ? 1 : 2;
  out.stage_used = 1;
  out.alpha = n > 0 ? (double)coarse_n / (double)n : 1.0;
  c.work += (double)K * (double)a.m * (double)(*stages_run);
}

// ====================================================================
// coarsest direct solver (coarse_solver.cpp:26-76): components, bordered
// matrices, unblocked partial-pivot LU -- one CTA
// ====================================================================
__global__ void labels_kernel(CSRv a, int32_t* label) {
  // min-label propagation to a fixed point (one CTA; n is small)
  __shared__ int changed;
  for (int32_t u = threadIdx.x; u < a.n; u += blockDim.x) label[u] = u;
  __syncthreads();
  do {
    __syncthreads();
    if (threadIdx.x == 0) changed = 0;
    __syncthreads();
    for (int32_t u = threadIdx.x; u < a.n; u += blockDim.x) {
      int32_t l = label[u];
      for (int64_t k = a.rp[u]; k < a.rp[u + 1]; ++k) l = min(l, label[a.col[k]]);
      if (l < label[u]) {
        label[u] = l;
        changed = 1;
      }
    }
    __syncthreads();
  } while (changed);
}

// builds the bordered matrix of one component in `M` (N = cn + 1, row major):
// single-component: from the operator as is; multi-component: from the
// extracted sub-Laplacian, whose diagonal assemble_canonical recomputes as
// the ascending-column fold of the weights (components.cpp:35-56)
__global__ void bordered_kernel(CSRv a, const int32_t* nodes, int32_t cn, bool whole,
                                const int32_t* local, double* M) {
  const int32_t N = cn + 1;
  for (int64_t i = threadIdx.x; i < (int64_t)N * N; i += blockDim.x) M[i] = 0.0;
  __syncthreads();
  for (int32_t lu = threadIdx.x; lu < cn; lu += blockDim.x) {
    int32_t u = whole ? lu : nodes[lu];
    double d = 0.0;
    for (int64_t k = a.rp[u]; k < a.rp[u + 1]; ++k) {
      int32_t lv = whole ? a.col[k] : local[a.col[k]];
      M[(int64_t)lu * N + lv] = a.val[k];
      d = d + -a.val[k];
    }
    M[(int64_t)lu * N + lu] = whole ? a.diag[u] : d;
    M[(int64_t)lu * N + cn] = 1.0;
    M[(int64_t)cn * N + lu] = 1.0;
  }
}

__global__ void lu_kernel(double* M, int32_t N, int32_t* perm) {
  __shared__ double sv[1024];
  __shared__ int32_t si[1024];
  __shared__ int32_t piv_row;
  for (int32_t i = threadIdx.x; i < N; i += blockDim.x) perm[i] = i;
  __syncthreads();
  for (int32_t k = 0; k < N; ++k) {
    // pivot: first row of maximal |M[i][k]|, i >= k
    double best = -1.0;
    int32_t bi = N;
    for (int32_t i = k + threadIdx.x; i < N; i += blockDim.x) {
      double v = fabs(M[(int64_t)i * N + k]);
      if (v > best || (v == best && i < bi)) {
        best = v;
        bi = i;
      }
    }
    sv[threadIdx.x] = best;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
      if (threadIdx.x < w) {
        double ov = sv[threadIdx.x + w];
        int32_t oi = si[threadIdx.x + w];
        if (ov > sv[threadIdx.x] || (ov == sv[threadIdx.x] && oi < si[threadIdx.x])) {
          sv[threadIdx.x] = ov;
          si[threadIdx.x] = oi;
        }
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      // the sequential scan keeps the first maximum: it starts from row k
      // and only replaces on strictly greater values
      int32_t p = si[0];
      if (fabs(M[(int64_t)k * N + k]) == sv[0]) p = k;
      piv_row = p;
    }
    __syncthreads();
    const int32_t p = piv_row;
    if (p != k) {
      for (int32_t j = threadIdx.x; j < N; j += blockDim.x) {
        double t = M[(int64_t)k * N + j];
        M[(int64_t)k * N + j] = M[(int64_t)p * N + j];
        M[(int64_t)p * N + j] = t;
      }
      if (threadIdx.x == 0) {
        int32_t t = perm[k];
        perm[k] = perm[p];
        perm[p] = t;
      }
    }
    __syncthreads();
    const double piv = M[(int64_t)k * N + k];
    if (piv == 0.0) continue;
    for (int32_t i = k + 1 + threadIdx.x; i < N; i += blockDim.x) M[(int64_t)i * N + k] = M[(int64_t)i * N + k] / piv;
    __syncthreads();
    const int64_t rows = N - k - 1;
    for (int64_t t = threadIdx.x; t < rows * rows; t += blockDim.x) {
      int32_t i = k + 1 + (int32_t)(t / rows), j = k + 1 + (int32_t)(t % rows);
      M[(int64_t)i * N + j] = M[(int64_t)i * N + j] - M[(int64_t)i * N + k] * M[(int64_t)k * N + j];
    }
    __syncthreads();
  }
}

__global__ void local_index_kernel(const int32_t* nodes, int32_t cn, int32_t* local) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cn) local[nodes[i]] = i;
}

void make_direct(Ctx& c, const CSRv& a, DDirect& d) {
  const int32_t n = a.n;
  d.n = n;
  d.m = a.m;
  DVec<int32_t> label(n, c.s);
  count_launch(), labels_kernel<<<1, 1024, 0, c.s>>>(a, label.p);
  CK_LAUNCH();
  std::vector<int32_t> lab = label.to_host();
  // components in order of their smallest node, nodes ascending (BFS order of
  // connected_components, components.cpp:9-33)
  std::vector<int32_t> comp_id(n, -1), order;
  std::vector<int32_t> start;
  std::vector<std::vector<int32_t>> comps;
  for (int32_t u = 0; u < n; ++u) {
    if (lab[u] == u) {
      comp_id[u] = (int32_t)comps.size();
      comps.emplace_back();
    }
  }
  for (int32_t u = 0; u < n; ++u) comps[comp_id[lab[u]]].push_back(u);
  d.ncomp = (int32_t)comps.size();
  std::vector<int32_t> hstart(d.ncomp + 1, 0), hnodes;
  std::vector<int64_t> hoff(d.ncomp, 0);
  int64_t lu_total = 0;
  d.comp_size.clear();
  d.maxN = 0;
  for (int32_t ci = 0; ci < d.ncomp; ++ci) {
    hstart[ci + 1] = hstart[ci] + (int32_t)comps[ci].size();
    hnodes.insert(hnodes.end(), comps[ci].begin(), comps[ci].end());
    int64_t N = (int64_t)comps[ci].size() + 1;
    hoff[ci] = lu_total;
    lu_total += N * N;
    d.comp_size.push_back((int32_t)comps[ci].size());
    d.maxN = std::max<int32_t>(d.maxN, (int32_t)N);
  }
  d.comp_start.alloc(d.ncomp + 1, c.s);
  d.comp_start.upload(hstart.data(), d.ncomp + 1);
  d.nodes.alloc(std::max(n, 1), c.s);
  d.nodes.upload(hnodes.data(), n);
  d.lu_off.alloc(d.ncomp, c.s);
  d.lu_off.upload(hoff.data(), d.ncomp);
  d.lu.alloc(lu_total, c.s);
  d.perm.alloc(n + d.ncomp, c.s);
  DVec<int32_t> local(n, c.s);
  for (int32_t ci = 0; ci < d.ncomp; ++ci) {
    const int32_t cn = d.comp_size[ci];
    const bool whole = d.ncomp == 1;
    const int32_t* nodes = d.nodes.p + hstart[ci];
    if (!whole) {
      count_launch(), local_index_kernel<<<blocks_for(cn), kThreads, 0, c.s>>>(nodes, cn, local.p);
      CK_LAUNCH();
    }
    double* M = d.lu.p + hoff[ci];
    count_launch(), bordered_kernel<<<1, 1024, 0, c.s>>>(a, nodes, cn, whole, local.p, M);
    count_launch(), lu_kernel<<<1, 1024, 0, c.s>>>(M, cn + 1, d.perm.p + hstart[ci] + ci);
    CK_LAUNCH();
  }
  const double nn1 = (double)n + 1.0;
  c.work += nn1 * nn1 * nn1 / 3.0;
}

// Per-visit solve with the cached factors (coarse_solver.cpp:47-66). The
// forward sweep runs column-wise (each y_i still receives its subtractions in
// ascending j), the backward sweep row-wise as a single chain, so the result
// is bit-identical to the sequential substitution.
__global__ void direct_solve_kernel(const int32_t* comp_start, int32_t ncomp, const int32_t* nodes,
                                    const int64_t* lu_off, const double* lu, const int32_t* perm,
                                    bool whole, const double* b, double* x, double* work_y,
                                    double* work_rhs) {
  for (int32_t ci = 0; ci < ncomp; ++ci) {
    const int32_t s0 = comp_start[ci], cn = comp_start[ci + 1] - s0, N = cn + 1;
    const double* M = lu + lu_off[ci];
    const int32_t* P = perm + s0 + ci;
    double* y = work_y;
    double* rhs = work_rhs;
    for (int32_t k = threadIdx.x; k < cn; k += blockDim.x) rhs[k] = whole ? b[k] : b[nodes[s0 + k]];
    if (threadIdx.x == 0) rhs[cn] = 0.0;
    __syncthreads();
    for (int32_t i = threadIdx.x; i < N; i += blockDim.x) y[i] = rhs[P[i]];
    __syncthreads();
    for (int32_t j = 0; j < N; ++j) {
      const double yj = y[j];
      for (int32_t i = j + 1 + threadIdx.x; i < N; i += blockDim.x) y[i] = y[i] - M[(int64_t)i * N + j] * yj;
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      for (int32_t i = N; i-- > 0;) {
        double s = y[i];
        for (int32_t j = i + 1; j < N; ++j) s = s - M[(int64_t)i * N + j] * y[j];
        y[i] = s / M[(int64_t)i * N + i];
      }
    }
    __syncthreads();
    for (int32_t k = threadIdx.x; k < cn; k += blockDim.x) {
      if (whole) x[k] = y[k];
      else x[nodes[s0 + k]] = y[k];
    }
    __syncthreads();
  }
}

// throughput variant: x = Minv[:n,:n] b per component (precomputed inverse rows)
__global__ void direct_inv_kernel(const int32_t* comp_start, int32_t ncomp, const int32_t* nodes,
                                  const int64_t* inv_off, const double* inv, bool whole,
                                  const double* b, double* x) {
  for (int32_t ci = 0; ci < ncomp; ++ci) {
    const int32_t s0 = comp_start[ci], cn = comp_start[ci + 1] - s0;
    const double* Mi = inv + inv_off[ci];
    for (int32_t i = threadIdx.x; i < cn; i += blockDim.x) {
      double s = 0.0;
      for (int32_t j = 0; j < cn; ++j) s += Mi[(int64_t)i * cn + j] * (whole ? b[j] : b[nodes[s0 + j]]);
      if (whole) x[i] = s;
      else x[nodes[s0 + i]] = s;
    }
    __syncthreads();
  }
}

void direct_solve(Ctx& c, const DDirect& d, const double* b, double* x, bool exact, double* scratch) {
  if (exact || d.inv.n == 0) {
    count_launch(), direct_solve_kernel<<<1, 256, 0, c.s>>>(d.comp_start.p, d.ncomp, d.nodes.p, d.lu_off.p, d.lu.p, d.perm.p,
                                            d.ncomp == 1, b, x, scratch, scratch + d.maxN + 1);
  } else {
    count_launch(), direct_inv_kernel<<<1, 256, 0, c.s>>>(d.comp_start.p, d.ncomp, d.nodes.p, d.inv_off.p, d.inv.p,
                                          d.ncomp == 1, b, x);
  }
  CK_LAUNCH();
  c.work += (double)d.m;
}

// RelaxationSolver::solve (coarse_solver.cpp:82-93); validate mode: exact-order
// sweeps and sequential folds, one host check per sweep
void relax_solve(Ctx& c, const CSRv& a, const Schedule& sch, const DColor* col, const LongRows* nat,
                 const double* b, double* x, DVec<double>& r, int* sweeps_out, bool exact) {
  if (r.n < a.n) r.alloc(a.n, c.s);
  if (!exact && col && nat) {
    // LAMG_RELAX_PATH=coop|graph overrides the size rule
    const char* path = getenv("LAMG_RELAX_PATH");
    const bool graph = path ? std::string(path) == "graph" : a.n >= (1 << 20);
    const int sw = graph ? relax_colored_graph(c, a, *col, *nat, b, x, r.p)
                         : relax_colored_coop(c, a, *col, *nat, b, x, r.p);
    c.work += (double)a.m * (1.0 + 2.0 * sw);
    *sweeps_out = sw;
    return;
  }
  double* nrm = c.dscal + 110;
  residual_exact(c, a, b, x, r.p, sch.heavy_nat.p, sch.nheavy_nat);
  c.work += (double)a.m;
  seq_norm2(c, r.p, a.n, nrm);
  const double r0 = read_scalar(c, nrm);
  *sweeps_out = 0;
  if (r0 == 0.0) return;
  const double target = 1e-12 * r0;
  for (int sweep = 0; sweep < 400; ++sweep) {
    if (!exact && col) gs_colored(c, *col, a.n, b, x, 1);
    else gs_exact(c, a, sch, b, x, 1, 1);
    c.work += (double)a.m;
    if (exact) subtract_mean_seq(c, x, a.n);
    else subtract_mean_tree(c, x, a.n);
    residual_exact(c, a, b, x, r.p, sch.heavy_nat.p, sch.nheavy_nat);
    c.work += (double)a.m;
    if (exact) seq_norm2(c, r.p, a.n, nrm);
    else tree_norm2(c, r.p, a.n, nrm);
    ++*sweeps_out;
    if (read_scalar(c, nrm) <= target) break;
  }
}

// ====================================================================
// setup driver (hierarchy.cpp:59-138)
// ====================================================================
double level_cycle_index(const DHier& h, size_t l, double gamma) {
  if (l + 1 >= h.levels.size()) return 1.0;
  if (h.levels[l + 1]->kind == KIND_ELIM) return 1.0;
  const double m1 = (double)h.levels[0]->op.m;
  const double ml = (double)h.levels[l]->op.m;
  const double mc = (double)h.levels[l + 1]->op.m;
  if (ml > 0.1 * m1) return gamma;
  if (mc <= 0.0) return 1.0;
  return std::min(2.0, 0.7 * ml / mc);
}

static void finish_level(Ctx& c, DLevel& L) {
  build_schedule(c, L.op.view(), false, L.sched);
  build_upper_index(c, L.op.view(), L.upper);
}

static void mark_coarsest(Ctx& c, DHier& h, int mode) {
  DLevel& L = *h.levels.back();
  L.coarsest = mode;
  if (mode == CM_DIRECT) {
    L.direct = std::make_unique<DDirect>();
    make_direct(c, L.op.view(), *L.direct);
  }
}

std::unique_ptr<DHier> setup_device(Ctx& c, const CSRv& a, const SetupOpts& o) {
  auto t0 = std::chrono::steady_clock::now();
  validate_exact(c, a);
  const double w0 = c.work = 0.0;
  auto h = std::make_unique<DHier>();
  h->seed = o.seed;
  h->device = c.device;
  {
    auto L0 = std::make_unique<DLevel>();
    L0->kind = KIND_FINEST;
    L0->op.alloc(a.n, a.m, c.s);
    CK(cudaMemcpyAsync(L0->op.rp.p, a.rp, sizeof(int64_t) * (a.n + 1), cudaMemcpyDeviceToDevice, c.s));
    CK(cudaMemcpyAsync(L0->op.col.p, a.col, sizeof(int32_t) * 2 * a.m, cudaMemcpyDeviceToDevice, c.s));
    CK(cudaMemcpyAsync(L0->op.val.p, a.val, sizeof(double) * 2 * a.m, cudaMemcpyDeviceToDevice, c.s));
    CK(cudaMemcpyAsync(L0->op.diag.p, a.diag, sizeof(double) * a.n, cudaMemcpyDeviceToDevice, c.s));
    finish_level(c, *L0);
    h->levels.push_back(std::move(L0));
  }
  int stagnant_rounds = 0;
  while (h->levels.size() < 100) {
    DLevel& cur = *h->levels.back();
    const CSRv cv = cur.op.view();
    if (cv.n <= o.coarsest_n) {
      mark_coarsest(c, *h, CM_DIRECT);
      break;
    }
    {
      std::vector<std::unique_ptr<DStage>> stages;
      DCSR coarse;
      if (eliminate_rounds(c, cv, stages, coarse)) {
        auto L = std::make_unique<DLevel>();
        L->kind = KIND_ELIM;
        L->op = std::move(coarse);
        validate_exact(c, L->op.view());
        L->stages = std::move(stages);
        L->gamma = 1.0;
        finish_level(c, *L);
        h->levels.push_back(std::move(L));
        continue;
      }
    }
    const uint64_t level_seed = rng_derive_host(o.seed, (uint64_t)h->levels.size());
    const double factor = probe_relaxation(c, cv, cur.sched, cur.upper, 8, level_seed);
    if (factor <= 0.7) {
      mark_coarsest(c, *h, CM_RELAX);
      break;
    }
    const int k = std::min(o.tv_count_finest + 2 * (int)(h->levels.size() - 1), o.tv_count_max);
    DVec<double> X;
    generate_tvs(c, cv, cur.sched, k, o.tv_sweeps, level_seed, X);
    DVec<int32_t> hubs;
    int32_t nh = detect_hubs(c, cv, hubs);
    auto agg = std::make_unique<DAgg>();
    int stages_run = 1;
    aggregate(c, cv, k, X.p, o.gamma, hubs.p, nh, *agg, &stages_run);
    X.release();
    if (agg->coarse_n >= cv.n) {
      h->warnings.push_back("aggregation made no progress at level " + std::to_string(h->levels.size()) +
                            "; level becomes coarsest");
      mark_coarsest(c, *h, CM_DIRECT);
      break;
    }
    auto L = std::make_unique<DLevel>();
    L->kind = KIND_AGG;
    galerkin(c, cv, agg->aggregate_of.p, agg->coarse_n, L->op);
    validate_exact(c, L->op.view());
    L->gamma = 1.0;
    L->nu_pre = 1;
    L->nu_post = 2;
    L->tv_count = k;
    const bool stagnant = agg->alpha > 0.95;
    build_members(c, agg->fine_n, agg->coarse_n, agg->aggregate_of.p, agg->mem_ptr, agg->mem);
    L->agg = std::move(agg);
    finish_level(c, *L);
    h->levels.push_back(std::move(L));
    if (stagnant && ++stagnant_rounds >= 2) {
      h->warnings.push_back("aggregation stagnated twice; stopping coarsening");
      mark_coarsest(c, *h, CM_DIRECT);
      break;
    }
  }
  if (h->levels.back()->coarsest == CM_NONE) {
    h->warnings.push_back("level cap reached before the coarsening terminated");
    mark_coarsest(c, *h, CM_DIRECT);
  }
  for (size_t l = 0; l + 1 < h->levels.size(); ++l) h->levels[l + 1]->gamma = level_cycle_index(*h, l, o.gamma);
  h->setup_work = (c.work - w0) / (double)h->levels[0]->op.m;
  c.sync();
  h->setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return h;
}

}  // namespace lamgb
