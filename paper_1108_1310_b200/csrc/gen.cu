// gen.cu -- graph ingest on the device: the seeded
// R-MAT generator of BASELINE.json config 5, duplicate merging, and the
// largest-connected-component extraction, producing the reference's CSR
// Laplacian directly in HBM.
//
// Definitions follow SURVEY.md 8(d) (the reference's generators cannot
// produce these graphs, generators.hpp:9-34); the host restatement is
// paper_1108_1310_b200/graphs.py (rmat, largest_component), and the device
// result is bit-identical to it:
//  * sample i, bit t draws U = unit(seed, t*S + i) of the counter-form
//    lamg::Rng (rng.hpp:10-41); quadrant by U against a, a+b, a+b+c;
//  * self-loops dropped, duplicates merged into integer multiplicities
//    (exact in f64: the weight fold order cannot matter);
//  * the largest component (ties: smallest node id) is kept in ascending node
//    order (components.cpp:35-56 extract_component) and re-assembled with
//    assemble_canonical (sparse_laplacian.cpp:60-104).
#include <algorithm>

#include "hier.cuh"

namespace lamgb {

namespace {

__device__ inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__device__ inline double unit_at(uint64_t s0, uint64_t idx) {
  return (double)(mix64(s0 + (idx + 3) * 0x9e3779b97f4a7c15ULL) >> 11) * 0x1.0p-53;
}

// key = lo << scale | hi for u != v; all-ones for self-loops (sorted last)
__global__ void rmat_kernel(int scale, int64_t S, uint64_t s0, double a, double ab, double abc, uint64_t* key) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= S) return;
  uint64_t u = 0, v = 0;
  for (int t = 0; t < scale; ++t) {
    const double r = unit_at(s0, (uint64_t)t * (uint64_t)S + (uint64_t)i);
    const uint64_t ub = r >= ab;
    const uint64_t vb = (r >= a && r < ab) || r >= abc;
    u |= ub << t;
    v |= vb << t;
  }
  key[i] = u == v ? ~0ull : (u < v ? (u << scale) | v : (v << scale) | u);
}

// Chung-Lu (config 4): pair j's endpoints are searchsorted(cdf, U, 'right')
// of draws j and pairs + j (graphs.chung_lu), clamped to n - 1
__device__ inline int32_t upper_bound_f64(const double* cdf, int32_t n, double u) {
  int32_t lo = 0, hi = n;  // first index with cdf[i] > u
  while (lo < hi) {
    const int32_t mid = lo + (hi - lo) / 2;
    if (cdf[mid] <= u) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
__global__ void chunglu_kernel(const double* __restrict__ cdf, int32_t n, int bits, int64_t pairs, uint64_t s0,
                               uint64_t* key) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= pairs) return;
  uint64_t u = (uint64_t)min(upper_bound_f64(cdf, n, unit_at(s0, (uint64_t)j)), n - 1);
  uint64_t v = (uint64_t)min(upper_bound_f64(cdf, n, unit_at(s0, (uint64_t)(pairs + j))), n - 1);
  key[j] = u == v ? ~0ull : (u < v ? (u << bits) | v : (v << bits) | u);
}

__global__ void ones_kernel(double* w, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) w[i] = 1.0;
}

__global__ void run_heads_kernel(const uint64_t* k, int64_t n, uint8_t* head) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) head[i] = k[i] != ~0ull && (i == 0 || k[i] != k[i - 1]);
}

__global__ void runs_to_edges_kernel(const uint64_t* k, const int64_t* start, int64_t E, int64_t total, int scale,
                                     int32_t* eu, int32_t* ev, double* ew) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= E) return;
  const int64_t s = start[e];
  const int64_t t = e + 1 < E ? start[e + 1] : total;
  const uint64_t key = k[s];
  eu[e] = (int32_t)(key >> scale);
  ev[e] = (int32_t)(key & ((1ull << scale) - 1));
  ew[e] = (double)(t - s);
}

// ---------------------------------------------------------- components
__global__ void iota_i32_kernel(int32_t* p, int32_t n) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = i;
}
// parent links only ever point to smaller ids; reads bypass L1 (another SM
// may have linked a root since this SM cached the line)
__device__ inline int32_t find_root(int32_t* parent_, int32_t x) {
  volatile int32_t* parent = parent_;
  int32_t p = parent[x];
  while (p != x) {  // path halving; racing writes only shorten paths
    const int32_t g = parent[p];
    if (g != p) parent[x] = g;
    x = p;
    p = parent[x];
  }
  return x;
}
// union by minimum root: a tree's root is the smallest node id it holds
__global__ void hook_kernel(const int32_t* eu, const int32_t* ev, int64_t E, int32_t* parent) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= E) return;
  int32_t a = eu[e], b = ev[e];
  while (true) {
    a = find_root(parent, a);
    b = find_root(parent, b);
    if (a == b) return;
    const int32_t lo = a < b ? a : b, hi = a < b ? b : a;
    if (atomicCAS(parent + hi, hi, lo) == hi) return;
    a = lo;
    b = hi;
  }
}
// edges whose endpoints still have different roots (union retry guard)
__global__ void unjoined_kernel(const int32_t* eu, const int32_t* ev, int64_t E, int32_t* parent, int32_t* flag) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < E && find_root(parent, eu[e]) != find_root(parent, ev[e])) *flag = 1;
}
__global__ void compress_kernel(int32_t* parent, int32_t n, int32_t* size) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t r = find_root(parent, i);
  parent[i] = r;
  atomicAdd(size + r, 1);
}
// largest component; ties to the smallest root (= smallest node id)
__global__ void pick_kernel(const int32_t* size, int32_t n, unsigned long long* best) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || size[i] == 0) return;
  atomicMax(best, ((unsigned long long)size[i] << 32) | (unsigned long long)(0xffffffffu - (uint32_t)i));
}
__global__ void keep_flags_kernel(const int32_t* parent, int32_t n, int32_t root, int32_t* flag) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flag[i] = parent[i] == root;
}
__global__ void edge_keep_kernel(const int32_t* eu, int64_t E, const int32_t* parent, int32_t root, uint8_t* f) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < E) f[e] = parent[eu[e]] == root;
}
__global__ void relabel_kernel(const int64_t* sel, int64_t E2, const int32_t* eu, const int32_t* ev, const double* ew,
                               const int32_t* local, int32_t* ou, int32_t* ov, double* ow) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= E2) return;
  const int64_t e = sel[j];
  ou[j] = local[eu[e]];
  ov[j] = local[ev[e]];
  ow[j] = ew[e];
}
__global__ void csr_edges_kernel(CSRv a, int32_t* eu, int32_t* ev, double* ew, const int64_t* upos) {
  // u < v entries of each row, in (u, v) order: upos[u] = first output slot of row u
  const int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= a.n) return;
  int64_t o = upos[u];
  for (int64_t k = a.rp[u]; k < a.rp[u + 1]; ++k)
    if (a.col[k] > u) {
      eu[o] = u;
      ev[o] = a.col[k];
      ew[o] = -a.val[k];
      ++o;
    }
}
__global__ void upper_count_kernel(CSRv a, int64_t* cnt) {
  const int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= a.n) return;
  int64_t c = 0;
  for (int64_t k = a.rp[u]; k < a.rp[u + 1]; ++k) c += a.col[k] > u;
  cnt[u] = c;
}

}  // namespace

// largest_component (graphs.py; components.cpp:9-56): keeps the largest
// connected component of `a` in ascending node order. Returns false (and
// leaves `out` empty) when `a` is already connected.
bool largest_component_dev(Ctx& c, const CSRv& a, DCSR& out) {
  const int32_t n = a.n;
  // edge list u < v in (u, v) order
  DVec<int64_t> cnt(n + 1, c.s), upos(n + 1, c.s);
  count_launch(), upper_count_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(a, cnt.p);
  CK(cudaMemsetAsync(cnt.p + n, 0, sizeof(int64_t), c.s));
  exclusive_scan_i64(c, cnt.p, upos.p, n + 1);
  const int64_t E = read_i64(c, upos.p + n);
  DVec<int32_t> eu(std::max<int64_t>(E, 1), c.s), ev(std::max<int64_t>(E, 1), c.s);
  DVec<double> ew(std::max<int64_t>(E, 1), c.s);
  count_launch(), csr_edges_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(a, eu.p, ev.p, ew.p, upos.p);
  DVec<int32_t> parent(n, c.s), size(n, c.s);
  count_launch(), iota_i32_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(parent.p, n);
  size.zero();
  // hook until every edge joins one tree (one pass in practice; the check
  // makes the result independent of any interleaving)
  int32_t* unjoined = c.dflag + 40;
  for (int pass = 0; E && pass < 64; ++pass) {
    count_launch(), hook_kernel<<<blocks_for(E), kThreads, 0, c.s>>>(eu.p, ev.p, E, parent.p);
    CK(cudaMemsetAsync(unjoined, 0, sizeof(int32_t), c.s));
    count_launch(), unjoined_kernel<<<blocks_for(E), kThreads, 0, c.s>>>(eu.p, ev.p, E, parent.p, unjoined);
    CK_LAUNCH();
    if (read_i32(c, unjoined) == 0) break;
    if (pass == 63) throw LamgError(LAMG_E_ERROR, "largest component: union-find did not converge");
  }
  count_launch(), compress_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(parent.p, n, size.p);
  unsigned long long* best = (unsigned long long*)(c.dscal + 96);
  CK(cudaMemsetAsync(best, 0, sizeof(unsigned long long), c.s));
  count_launch(), pick_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(size.p, n, best);
  CK_LAUNCH();
  const unsigned long long hb = (unsigned long long)read_i64(c, (const int64_t*)best);
  const int32_t root = (int32_t)(0xffffffffu - (uint32_t)(hb & 0xffffffffu));
  const int32_t nk = (int32_t)(hb >> 32);
  if (nk == n) return false;
  DVec<int32_t> flag(n + 1, c.s), local(n + 1, c.s);
  count_launch(), keep_flags_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(parent.p, n, root, flag.p);
  CK(cudaMemsetAsync(flag.p + n, 0, sizeof(int32_t), c.s));
  exclusive_scan_i32(c, flag.p, local.p, n + 1);
  DVec<uint8_t> ef(std::max<int64_t>(E, 1), c.s);
  DVec<int64_t> sel(std::max<int64_t>(E, 1), c.s);
  if (E) count_launch(), edge_keep_kernel<<<blocks_for(E), kThreads, 0, c.s>>>(eu.p, E, parent.p, root, ef.p);
  const int64_t E2 = E ? select_flagged_index64(c, ef.p, sel.p, E) : 0;
  DVec<int32_t> ou(std::max<int64_t>(E2, 1), c.s), ov(std::max<int64_t>(E2, 1), c.s);
  DVec<double> ow(std::max<int64_t>(E2, 1), c.s);
  if (E2)
    count_launch(), relabel_kernel<<<blocks_for(E2), kThreads, 0, c.s>>>(sel.p, E2, eu.p, ev.p, ew.p, local.p, ou.p,
                                                                       ov.p, ow.p);
  CK_LAUNCH();
  assemble_canonical_dev(c, nk, E2, ou.p, ov.p, ow.p, out);
  c.sync();
  return true;
}

// R-MAT (BASELINE.json config 5; graphs.py rmat): 2^scale nodes,
// edge_factor * 2^scale samples, duplicates summed, optional LCC.
// sampled edge keys (lo << bits | hi, all-ones for self-loops) -> merged
// edges (weights = multiplicities, or 1 with unit_weights) -> canonical CSR
// -> largest component
static void keys_to_graph(Ctx& c, int32_t n, int scale, DVec<uint64_t>& k, int64_t S, bool unit_weights, bool lcc,
                          DCSR& out) {
  DCSR full;
  {
    DVec<uint64_t> ks(std::max<int64_t>(S, 1), c.s);
    sort_keys_u64(c, k.p, ks.p, S, 64);
    k.release();
    DVec<uint8_t> head(S, c.s);
    count_launch(), run_heads_kernel<<<blocks_for(S), kThreads, 0, c.s>>>(ks.p, S, head.p);
    DVec<int64_t> start(S, c.s);
    const int64_t E = select_flagged_index64(c, head.p, start.p, S);
    head.release();
    // run e ends at the next run's start; the last at the first self-loop key
    int64_t total = S;
    DVec<int32_t> eu(std::max<int64_t>(E, 1), c.s), ev(std::max<int64_t>(E, 1), c.s);
    DVec<double> ew(std::max<int64_t>(E, 1), c.s);
    if (E) {
      // the last run ends where the self-loop block starts: find it from the sorted keys
      int64_t lo = 0, hi = S;  // first index with key == ~0 (host binary search over a few reads)
      while (lo < hi) {
        const int64_t mid = lo + (hi - lo) / 2;
        uint64_t kv;
        CK(cudaMemcpyAsync(&kv, ks.p + mid, sizeof kv, cudaMemcpyDeviceToHost, c.s));
        c.sync();
        if (kv == ~0ull) hi = mid;
        else lo = mid + 1;
      }
      total = lo;  // self-loop keys (all ones) sort last
      count_launch(), runs_to_edges_kernel<<<blocks_for(E), kThreads, 0, c.s>>>(ks.p, start.p, E, total, scale, eu.p,
                                                                               ev.p, ew.p);
      CK_LAUNCH();
      if (unit_weights) count_launch(), ones_kernel<<<blocks_for(E), kThreads, 0, c.s>>>(ew.p, E);
    }
    ks.release();
    start.release();
    assemble_canonical_dev(c, n, E, eu.p, ev.p, ew.p, full);
  }
  c.sync();
  if (lcc) {
    DCSR sub;
    if (largest_component_dev(c, full.view(), sub)) {
      out = std::move(sub);
      return;
    }
  }
  out = std::move(full);
}

void gen_rmat(Ctx& c, int scale, int edge_factor, double a, double b, double cc, uint64_t seed, bool lcc,
              DCSR& out) {
  if (scale < 1 || scale > 30) throw LamgError(LAMG_E_ARGUMENT, "rmat: scale must be in [1, 30]");
  const int32_t n = (int32_t)(1u << scale);
  const int64_t S = (int64_t)edge_factor << scale;
  const double ab = a + b, abc = a + b + cc;  // graphs.py evaluates a + b + c left to right
  const uint64_t s0 = seed ? seed : 0x9e3779b97f4a7c15ULL;
  DVec<uint64_t> k(std::max<int64_t>(S, 1), c.s);
  count_launch(), rmat_kernel<<<blocks_for(S), kThreads, 0, c.s>>>(scale, S, s0, a, ab, abc, k.p);
  CK_LAUNCH();
  keys_to_graph(c, n, scale, k, S, false, lcc, out);
}

// BASELINE config 4 (graphs.chung_lu): the normalised cumulative weights
// come from the host (numpy's pairwise mean and sequential cumsum define
// them); sampling, merging and the component step run here
void gen_chung_lu(Ctx& c, int32_t n, const double* cdf_host, int64_t pairs, uint64_t seed, bool lcc, DCSR& out) {
  if (n < 2) throw LamgError(LAMG_E_ARGUMENT, "chung_lu: n must be at least 2");
  int bits = 1;
  while ((1ll << bits) < n) ++bits;
  const uint64_t s0 = seed ? seed : 0x9e3779b97f4a7c15ULL;
  DVec<double> cdf(n, c.s);
  cdf.upload(cdf_host, n);
  DVec<uint64_t> k(std::max<int64_t>(pairs, 1), c.s);
  if (pairs) count_launch(), chunglu_kernel<<<blocks_for(pairs), kThreads, 0, c.s>>>(cdf.p, n, bits, pairs, s0, k.p);
  CK_LAUNCH();
  cdf.release();
  keys_to_graph(c, n, bits, k, pairs, true, lcc, out);
}

}  // namespace lamgb
