// part.cu -- fine-level node-block partition with halo exchange (SURVEY.md
// 8(e) mode 2): the finest operator split into contiguous row blocks, one
// per GPU, each block a local CSR whose columns index [owned rows | ghosts];
// a coloured Gauss-Seidel sweep exchanges the ghost values after every
// colour, a residual after the sweep. Rows keep their entry order and every
// kernel is the single-device one, so a partitioned sweep or residual is
// bit-identical to the unpartitioned THROUGHPUT smoother (gs_colored_one /
// residual_tp / residual_tasks) -- the parity test pins exactly that.
//
// Transports: NCCL point-to-point (one process per GPU; the library dlopens
// libnccl so it loads without it) or in-process (all parts owned by one
// process on one device, ghosts written by a gather kernel between the
// colour launches -- no kernel ever waits on another).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include "part.cuh"

namespace lamgb {

// ------------------------------------------------------------ host plan
void part_bounds(int32_t n, const int64_t* rp, int32_t nparts, std::vector<int32_t>& bounds) {
  if (nparts < 1) throw LamgError(LAMG_E_ARGUMENT, "partition needs at least one part");
  bounds.assign(nparts + 1, 0);
  const int64_t nnz = rp[n];
  for (int32_t p = 1; p < nparts; ++p) {
    // balance rows + entries (a row costs its entries plus a vector update)
    const int64_t target = (nnz + n) * p / nparts;
    int32_t lo = bounds[p - 1], hi = n;
    while (lo < hi) {
      const int32_t mid = lo + (hi - lo) / 2;
      if (rp[mid] + mid < target) lo = mid + 1;
      else hi = mid;
    }
    bounds[p] = lo;
  }
  bounds[nparts] = n;
}

PartPlan build_part_plan(int32_t n, const int64_t* rp, const int32_t* col, const double* val, const double* diag,
                         const std::vector<int32_t>& bounds, int32_t part) {
  const int32_t P = (int32_t)bounds.size() - 1;
  if (part < 0 || part >= P) throw LamgError(LAMG_E_ARGUMENT, "part index out of range");
  PartPlan pl;
  pl.nparts = P;
  pl.part = part;
  pl.lo = bounds[part];
  pl.hi = bounds[part + 1];
  pl.nloc = pl.hi - pl.lo;
  const int64_t k0 = rp[pl.lo], k1 = rp[pl.hi];
  for (int64_t k = k0; k < k1; ++k)
    if (col[k] < pl.lo || col[k] >= pl.hi) pl.ghost_gid.push_back(col[k]);
  std::sort(pl.ghost_gid.begin(), pl.ghost_gid.end());
  pl.ghost_gid.erase(std::unique(pl.ghost_gid.begin(), pl.ghost_gid.end()), pl.ghost_gid.end());
  pl.nghost = (int32_t)pl.ghost_gid.size();
  pl.rp.resize(pl.nloc + 1);
  pl.col.resize(k1 - k0);
  pl.val.assign(val + k0, val + k1);
  pl.diag.assign(diag + pl.lo, diag + pl.hi);
  for (int32_t i = 0; i <= pl.nloc; ++i) pl.rp[i] = rp[pl.lo + i] - k0;
  for (int64_t k = k0; k < k1; ++k) {
    const int32_t g = col[k];
    pl.col[k - k0] = (g >= pl.lo && g < pl.hi)
                         ? g - pl.lo
                         : pl.nloc + (int32_t)(std::lower_bound(pl.ghost_gid.begin(), pl.ghost_gid.end(), g) -
                                               pl.ghost_gid.begin());
  }
  // ghosts are sorted by global id and parts are contiguous: the ghosts owned
  // by part q are one range
  pl.recv_ptr.resize(P + 1);
  for (int32_t q = 0; q <= P; ++q)
    pl.recv_ptr[q] = (int32_t)(std::lower_bound(pl.ghost_gid.begin(), pl.ghost_gid.end(), bounds[q]) -
                               pl.ghost_gid.begin());
  // the operator is symmetric, so part q's ghosts from this part are exactly
  // the owned rows with a neighbour in q's block, in ascending order
  pl.send_ptr.assign(P + 1, 0);
  for (int32_t q = 0; q < P; ++q) {
    pl.send_ptr[q] = (int32_t)pl.send_idx.size();
    if (q == part) continue;
    for (int32_t v = pl.lo; v < pl.hi; ++v)
      for (int64_t k = rp[v]; k < rp[v + 1]; ++k)
        if (col[k] >= bounds[q] && col[k] < bounds[q + 1]) {
          pl.send_idx.push_back(v - pl.lo);
          break;
        }
  }
  pl.send_ptr[P] = (int32_t)pl.send_idx.size();
  return pl;
}

// ------------------------------------------------------------ NCCL (dlopen)
namespace {
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      a.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (a.h) break;
    }
    if (!a.h) return a;
    a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(a.h, "ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))dlsym(a.h, "ncclCommInitRank");
    a.CommDestroy = (decltype(a.CommDestroy))dlsym(a.h, "ncclCommDestroy");
    a.Send = (decltype(a.Send))dlsym(a.h, "ncclSend");
    a.Recv = (decltype(a.Recv))dlsym(a.h, "ncclRecv");
    a.GroupStart = (decltype(a.GroupStart))dlsym(a.h, "ncclGroupStart");
    a.GroupEnd = (decltype(a.GroupEnd))dlsym(a.h, "ncclGroupEnd");
    a.Broadcast = (decltype(a.Broadcast))dlsym(a.h, "ncclBroadcast");
    a.GetErrorString = (decltype(a.GetErrorString))dlsym(a.h, "ncclGetErrorString");
    return a;
  }();
  if (!api.h || !api.GetUniqueId || !api.CommInitRank || !api.Send || !api.Recv || !api.GroupStart ||
      !api.GroupEnd || !api.Broadcast)
    throw LamgError(LAMG_E_NCCL, "libnccl.so.2 could not be loaded");
  return api;
}
void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw LamgError(LAMG_E_NCCL, std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "?"));
}
}  // namespace

void comm_unique_id(char out[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  nck(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  memcpy(out, &id, 128);
}

Comm::Comm(int32_t nranks_, int32_t rank_, const char id[128]) : nranks(nranks_), rank(rank_) {
  ncclUniqueId uid;
  memcpy(&uid, id, 128);
  ncclComm_t cm;
  nck(nccl().CommInitRank(&cm, nranks, uid, rank), "ncclCommInitRank");
  handle = cm;
}
Comm::~Comm() {
  if (handle) nccl().CommDestroy((ncclComm_t)handle);
}

// ------------------------------------------------------------ kernels
namespace {
// ghost values for a peer: dst[i] = x[idx[i]]
__global__ void pack_kernel(const double* __restrict__ x, const int32_t* __restrict__ idx, int32_t cnt,
                            double* __restrict__ dst) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cnt) dst[i] = x[idx[i]];
}
// global <-> local slices
__global__ void take_kernel(const double* __restrict__ g, int32_t lo, int32_t cnt, double* __restrict__ l) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cnt) l[i] = g[lo + i];
}
__global__ void put_kernel(const double* __restrict__ l, int32_t lo, int32_t cnt, double* __restrict__ g) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cnt) g[lo + i] = l[i];
}
__global__ void part_interp_kernel(double* __restrict__ x, const int32_t* __restrict__ agg, int32_t lo, int32_t n,
                                   const double* __restrict__ xc) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = x[i] + xc[agg[lo + i]];
}
__global__ void local_perm_fill_kernel(const int64_t* rp, const int32_t* col, const double* val, const double* diag,
                                       const int32_t* rows, int32_t n, const int64_t* prp, int32_t* pcol,
                                       double* pval, double* pdiag) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= n) return;
  const int32_t u = rows[w];
  const int64_t o = prp[w] - rp[u];
  for (int64_t k = rp[u] + lane; k < rp[u + 1]; k += 32) {
    pcol[o + k] = col[k];
    pval[o + k] = val[k];
  }
  if (lane == 0) pdiag[w] = diag[u];
}
}  // namespace

// ------------------------------------------------------------ one part on the device
struct PartLevel::Part {
  PartPlan plan;
  DVec<int64_t> rp;
  DVec<int32_t> col;
  DVec<double> val, diag;
  DColor color;        // local colour-permuted copy, global colour ids
  LongRows nat;        // local natural long rows (hub residuals)
  DVec<int32_t> send_idx;
  DVec<double> x, b, r, sendbuf;
  CSRv view() const { return CSRv{plan.nloc, (int64_t)(plan.col.size() + 1) / 2, rp.p, col.p, val.p, diag.p}; }
};

PartLevel::~PartLevel() = default;

PartLevel::PartLevel(Ctx& c_, const CSRv& full_dev, const std::vector<int64_t>& rp_h, const std::vector<int32_t>& col_h,
                     const std::vector<double>& val_h, const std::vector<double>& diag_h,
                     const std::vector<int32_t>& bounds_, int32_t first_part, int32_t nown, Comm* comm_)
    : c(c_), bounds(bounds_), comm(comm_) {
  const int32_t P = (int32_t)bounds.size() - 1;
  if (nown < 1 || first_part < 0 || first_part + nown > P)
    throw LamgError(LAMG_E_ARGUMENT, "owned parts out of range");
  if (!comm && nown != P) throw LamgError(LAMG_E_ARGUMENT, "the in-process transport owns every part");
  if (comm && (nown != 1 || comm->nranks != P || comm->rank != first_part))
    throw LamgError(LAMG_E_ARGUMENT, "an NCCL rank owns exactly its own part");
  // the global THROUGHPUT colouring (deterministic: every rank computes the same)
  Schedule sch;
  build_schedule(c, full_dev, false, sch);
  std::unique_ptr<DColor> gcol = make_color(c, full_dev, sch);
  ncolors = gcol->ncolors;
  group = gcol->group;
  {
    LongRows full_nat;
    build_natural_long_rows(c, full_dev, full_nat);
    use_tasks = has_long_rows(full_nat);
    task_group = residual_tasks_group(full_dev, full_nat);
  }
  std::vector<int32_t> grow = gcol->row_ids.to_host();  // stored position -> global row
  std::vector<int32_t> colour_of(full_dev.n), pos_of(full_dev.n);
  for (int32_t cc = 0; cc < ncolors; ++cc)
    for (int32_t i = gcol->cptr_h[cc]; i < gcol->cptr_h[cc + 1]; ++i) colour_of[grow[i]] = cc;
  for (int32_t i = 0; i < full_dev.n; ++i) pos_of[grow[i]] = i;
  for (int32_t q = first_part; q < first_part + nown; ++q) {
    auto pt = std::make_unique<Part>();
    Part& p = *pt;
    p.plan = build_part_plan(full_dev.n, rp_h.data(), col_h.data(), val_h.data(), diag_h.data(), bounds, q);
    const PartPlan& pl = p.plan;
    const int64_t nnz = (int64_t)pl.col.size();
    p.rp.alloc(pl.nloc + 1, c.s);
    p.rp.upload(pl.rp.data(), pl.nloc + 1);
    p.col.alloc(std::max<int64_t>(nnz, 1), c.s);
    p.col.upload(pl.col.data(), nnz);
    p.val.alloc(std::max<int64_t>(nnz, 1), c.s);
    p.val.upload(pl.val.data(), nnz);
    p.diag.alloc(std::max(pl.nloc, 1), c.s);
    p.diag.upload(pl.diag.data(), pl.nloc);
    // local stored order: owned rows in their global colour-permuted order
    std::vector<int32_t> rows(pl.nloc);
    std::iota(rows.begin(), rows.end(), 0);
    std::sort(rows.begin(), rows.end(), [&](int32_t a, int32_t b) { return pos_of[pl.lo + a] < pos_of[pl.lo + b]; });
    DColor& cl = p.color;
    cl.ncolors = ncolors;
    cl.group = group;
    cl.cptr_h.assign(ncolors + 1, 0);
    for (int32_t i = 0; i < pl.nloc; ++i) ++cl.cptr_h[colour_of[pl.lo + rows[i]] + 1];
    for (int32_t cc = 0; cc < ncolors; ++cc) cl.cptr_h[cc + 1] += cl.cptr_h[cc];
    cl.row_ids.alloc(std::max(pl.nloc, 1), c.s);
    cl.row_ids.upload(rows.data(), pl.nloc);
    std::vector<int64_t> prp(pl.nloc + 1, 0);
    for (int32_t i = 0; i < pl.nloc; ++i) prp[i + 1] = prp[i] + (pl.rp[rows[i] + 1] - pl.rp[rows[i]]);
    cl.rp.alloc(pl.nloc + 1, c.s);
    cl.rp.upload(prp.data(), pl.nloc + 1);
    cl.col.alloc(std::max<int64_t>(nnz, 1), c.s);
    cl.val.alloc(std::max<int64_t>(nnz, 1), c.s);
    cl.diag.alloc(std::max(pl.nloc, 1), c.s);
    if (pl.nloc)
      count_launch(), local_perm_fill_kernel<<<blocks_for((int64_t)pl.nloc * 32), kThreads, 0, c.s>>>(
          p.rp.p, p.col.p, p.val.p, p.diag.p, cl.row_ids.p, pl.nloc, cl.rp.p, cl.col.p, cl.val.p, cl.diag.p);
    CK_LAUNCH();
    // heavy rows (one CTA each) per colour, as build_coloring lists them
    std::vector<int32_t> hv, hn;
    cl.hptr_h.assign(ncolors + 1, 0);
    for (int32_t cc = 0; cc < ncolors; ++cc) {
      cl.hptr_h[cc] = (int32_t)hv.size();
      for (int32_t i = cl.cptr_h[cc]; i < cl.cptr_h[cc + 1]; ++i)
        if (prp[i + 1] - prp[i] > kHeavyRow) hv.push_back(i);
    }
    cl.hptr_h[ncolors] = (int32_t)hv.size();
    for (int32_t u = 0; u < pl.nloc; ++u)
      if (pl.rp[u + 1] - pl.rp[u] > kHeavyRow) hn.push_back(u);
    cl.heavy.alloc(std::max<size_t>(hv.size(), 1), c.s);
    if (!hv.empty()) cl.heavy.upload(hv.data(), (int64_t)hv.size());
    cl.heavy_nat.alloc(std::max<size_t>(hn.size(), 1), c.s);
    if (!hn.empty()) cl.heavy_nat.upload(hn.data(), (int64_t)hn.size());
    cl.nheavy_nat = (int32_t)hn.size();
    build_long_rows(c, pl.rp, std::vector<int32_t>{0, pl.nloc}, p.nat);
    p.send_idx.alloc(std::max<size_t>(pl.send_idx.size(), 1), c.s);
    if (!pl.send_idx.empty()) p.send_idx.upload(pl.send_idx.data(), (int64_t)pl.send_idx.size());
    p.x.alloc(std::max(pl.nloc + pl.nghost, 1), c.s);
    p.x.zero();
    p.b.alloc(std::max(pl.nloc, 1), c.s);
    p.b.zero();
    p.r.alloc(std::max(pl.nloc, 1), c.s);
    p.sendbuf.alloc(std::max<size_t>(pl.send_idx.size(), 1), c.s);
    parts.push_back(std::move(pt));
  }
  c.sync();
}

int32_t PartLevel::nparts() const { return (int32_t)bounds.size() - 1; }

PartLevel::Part& PartLevel::local(int32_t part) {
  for (auto& p : parts)
    if (p->plan.part == part) return *p;
  throw LamgError(LAMG_E_ARGUMENT, "part not owned here");
}

void PartLevel::exchange() {
  const int32_t P = nparts();
  if (!comm) {
    // in-process: each part's send list is gathered straight into the
    // peer's ghost slots (same device, same stream, ordered launches)
    for (auto& pp : parts) {
      const PartPlan& pl = pp->plan;
      for (int32_t q = 0; q < P; ++q) {
        const int32_t cnt = pl.send_ptr[q + 1] - pl.send_ptr[q];
        if (!cnt) continue;
        Part& dst = local(q);
        count_launch(), pack_kernel<<<blocks_for(cnt), kThreads, 0, c.s>>>(
            pp->x.p, pp->send_idx.p + pl.send_ptr[q], cnt, dst.x.p + dst.plan.nloc + dst.plan.recv_ptr[pl.part]);
      }
    }
    CK_LAUNCH();
    return;
  }
  Part& p = *parts[0];
  const PartPlan& pl = p.plan;
  const int32_t ns = pl.send_ptr[P];
  if (ns) count_launch(), pack_kernel<<<blocks_for(ns), kThreads, 0, c.s>>>(p.x.p, p.send_idx.p, ns, p.sendbuf.p);
  CK_LAUNCH();
  NcclApi& api = nccl();
  nck(api.GroupStart(), "ncclGroupStart");
  for (int32_t q = 0; q < P; ++q) {
    if (q == pl.part) continue;
    const int32_t sc = pl.send_ptr[q + 1] - pl.send_ptr[q];
    const int32_t rc = pl.recv_ptr[q + 1] - pl.recv_ptr[q];
    if (sc) nck(api.Send(p.sendbuf.p + pl.send_ptr[q], sc, ncclFloat64, q, (ncclComm_t)comm->handle, c.s), "ncclSend");
    if (rc)
      nck(api.Recv(p.x.p + pl.nloc + pl.recv_ptr[q], rc, ncclFloat64, q, (ncclComm_t)comm->handle, c.s), "ncclRecv");
  }
  nck(api.GroupEnd(), "ncclGroupEnd");
}

void PartLevel::sweep(int sweeps) {
  for (int s = 0; s < sweeps; ++s)
    for (int32_t cc = 0; cc < ncolors; ++cc) {
      for (auto& p : parts) gs_colored_one(c, p->color, p->b.p, p->x.p, cc);
      exchange();  // the next colour reads this colour's new values across blocks
    }
}

void PartLevel::residual() {
  for (auto& p : parts) {
    const CSRv a = p->view();
    // the single-device choice (solve.cu Driver::resid), made on the whole level
    if (use_tasks) residual_tasks(c, a, p->nat, p->b.p, p->x.p, p->r.p, task_group);
    else residual_tp(c, a, p->b.p, p->x.p, p->r.p, p->color);
  }
}

void PartLevel::load(const double* b_global_dev, const double* x_global_dev) {
  for (auto& p : parts) {
    const PartPlan& pl = p->plan;
    if (!pl.nloc) continue;
    if (b_global_dev)
      count_launch(), take_kernel<<<blocks_for(pl.nloc), kThreads, 0, c.s>>>(b_global_dev, pl.lo, pl.nloc, p->b.p);
    if (x_global_dev)
      count_launch(), take_kernel<<<blocks_for(pl.nloc), kThreads, 0, c.s>>>(x_global_dev, pl.lo, pl.nloc, p->x.p);
  }
  CK_LAUNCH();
  if (x_global_dev) exchange();
}

void PartLevel::store(double* x_global_dev, double* r_global_dev) {
  for (auto& p : parts) {
    const PartPlan& pl = p->plan;
    if (!pl.nloc) continue;
    if (x_global_dev)
      count_launch(), put_kernel<<<blocks_for(pl.nloc), kThreads, 0, c.s>>>(p->x.p, pl.lo, pl.nloc, x_global_dev);
    if (r_global_dev)
      count_launch(), put_kernel<<<blocks_for(pl.nloc), kThreads, 0, c.s>>>(p->r.p, pl.lo, pl.nloc, r_global_dev);
  }
  CK_LAUNCH();
}

void PartLevel::allgather(bool residual, double* full) {
  if (!comm) {
    store(residual ? nullptr : full, residual ? full : nullptr);
    return;
  }
  Part& p = *parts[0];
  NcclApi& api = nccl();
  nck(api.GroupStart(), "ncclGroupStart");
  for (int32_t q = 0; q < nparts(); ++q) {
    const int32_t cnt = bounds[q + 1] - bounds[q];
    if (!cnt) continue;
    const double* src = q == comm->rank ? (residual ? p.r.p : p.x.p) : nullptr;
    nck(api.Broadcast(src, full + bounds[q], cnt, ncclFloat64, q, (ncclComm_t)comm->handle, c.s), "ncclBroadcast");
  }
  nck(api.GroupEnd(), "ncclGroupEnd");
}

void PartLevel::interpolate(const int32_t* agg, const double* xc) {
  for (auto& p : parts)
    if (p->plan.nloc)
      count_launch(), part_interp_kernel<<<blocks_for(p->plan.nloc), kThreads, 0, c.s>>>(p->x.p, agg, p->plan.lo,
                                                                                      p->plan.nloc, xc);
  CK_LAUNCH();
  exchange();
}

}  // namespace lamgb
