// capi.cu -- the extern "C" boundary (include/lamg_b200.h).
//
// Every entry point catches the library's C++ exceptions and returns the
// status code of the reference exception type, with the reference's message
// available from lamg_last_error().
#include <cmath>
#include <cstring>
#include <string>

#include "batch.cuh"
#include "part.cuh"
#include "mmio.cuh"
#include "solve.cuh"

using namespace lamgb;

namespace lamgb {
uint64_t rng_derive_host(uint64_t seed, uint64_t stream);
}

struct lamg_ctx {
  Ctx c;
};
struct lamg_hier {
  std::unique_ptr<DHier> h;
};

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return LAMG_OK;
  } catch (const LamgError& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host out of memory";
    return LAMG_E_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return LAMG_E_ERROR;
  }
}

void set_device(Ctx& c) { CK(cudaSetDevice(c.device)); }

// host CSR -> owning device CSR
void upload_csr(Ctx& c, const lamg_csr* a, DCSR& d) {
  if (!a) throw LamgError(LAMG_E_ARGUMENT, "null CSR");
  d.alloc(a->n, a->m, c.s);
  d.rp.upload(a->row_ptr, a->n + 1);
  d.col.upload(a->col, 2 * a->m);
  d.val.upload(a->val, 2 * a->m);
  d.diag.upload(a->diag, a->n);
}

void download_csr(Ctx& c, const DCSR& d, int64_t* rp, int32_t* col, double* val, double* diag) {
  if (rp) d.rp.download(rp, d.n + 1);
  if (col) d.col.download(col, 2 * d.m);
  if (val) d.val.download(val, 2 * d.m);
  if (diag) d.diag.download(diag, d.n);
  c.sync();
}

template <typename T>
DVec<T> up(Ctx& c, const T* h, int64_t n) {
  DVec<T> d(std::max<int64_t>(n, 1), c.s);
  if (n && h) d.upload(h, n);
  return d;
}

const DLevel& level_of(const lamg_hier* h, int32_t l) {
  if (!h || !h->h) throw LamgError(LAMG_E_ARGUMENT, "null hierarchy");
  if (l < 0 || l >= (int32_t)h->h->levels.size()) throw LamgError(LAMG_E_ARGUMENT, "level out of range");
  return *h->h->levels[l];
}

// stage arrays given as host pointers -> device stage (for the transfer kernels)
void upload_stage(Ctx& c, int32_t parent_n, int32_t coarse_n, int32_t nf, const int32_t* f_nodes,
                  const double* f_diag, const int64_t* f_ptr, const int32_t* f_nbr, const double* f_val,
                  const int32_t* cop, const int32_t* poc, DStage& s) {
  s.parent_n = parent_n;
  s.coarse_n = coarse_n;
  s.nf = nf;
  s.nnzf = f_ptr[nf];
  s.f_nodes = up(c, f_nodes, nf);
  s.f_diag = up(c, f_diag, nf);
  s.f_ptr = up(c, f_ptr, nf + 1);
  s.f_nbr = up(c, f_nbr, s.nnzf);
  s.f_val = up(c, f_val, s.nnzf);
  s.cop = up(c, cop, parent_n);
  s.poc = up(c, poc, coarse_n);
  build_stage_transpose(c, coarse_n, nf, s.f_ptr.p, s.f_nbr.p, s.cop.p, s.nnzf, s.t_ptr, s.t_p, s.f_of_p);
  s.ntlong = stage_long_lists(c, coarse_n, s.t_ptr.p, s.tlong);
}

int solve_common(lamg_ctx* ctx, const lamg_hier* h, const double* b, const double* x0, bool dev,
                 const lamg_cycle_cfg* cfg, double* x, lamg_solve_stats* stats, double* residuals,
                 int32_t cap, PartLevel* part = nullptr) {
  SolveResult res;
  int rc = guarded([&] {
    if (!ctx || !h || !h->h) throw LamgError(LAMG_E_ARGUMENT, "null context or hierarchy");
    Ctx& c = ctx->c;
    set_device(c);
    const int64_t n = h->h->levels[0]->op.n;
    CycleCfg cc;
    if (cfg) {
      cc.correction = cfg->correction;
      cc.mu = cfg->mu;
      cc.max_cycles = cfg->max_cycles;
      cc.target_reduction = cfg->target_reduction;
      cc.divergence_factor = cfg->divergence_factor;
    }
    auto run = [&](const double* bb, const double* xx0, double* xx) {
      return part ? solve_partitioned(c, *h->h, *part, bb, xx0, cc, xx, res)
                  : solve_device(c, *h->h, bb, xx0, cc, xx, res);
    };
    int r;
    if (dev) {
      r = run(b, x0, x);
    } else {
      DVec<double> db(n, c.s), dx0(n, c.s), dx(n, c.s);
      db.upload(b, n);
      dx0.upload(x0, n);
      r = run(db.p, dx0.p, dx.p);
      dx.download(x, n);
      c.sync();
    }
    if (r != LAMG_OK) throw LamgError(r, res.message);
  });
  if (stats) {
    stats->acf = res.acf;
    stats->solve_work = res.solve_work;
    stats->cycles = res.cycles;
    stats->converged = res.converged ? 1 : 0;
    stats->recombinations = res.recombinations;
    stats->recomb_max_growth = res.recomb_max_growth;
    stats->nresiduals = (int32_t)res.residuals.size();
    stats->relax_sweeps = res.relax_sweeps;
  }
  if (residuals)
    for (int32_t i = 0; i < cap && i < (int32_t)res.residuals.size(); ++i) residuals[i] = res.residuals[i];
  return rc;
}

void fill_stats(const SolveResult& res, lamg_solve_stats* stats, double* residuals, int32_t cap) {
  if (stats) {
    stats->acf = res.acf;
    stats->solve_work = res.solve_work;
    stats->cycles = res.cycles;
    stats->converged = res.converged ? 1 : 0;
    stats->recombinations = res.recombinations;
    stats->recomb_max_growth = res.recomb_max_growth;
    stats->nresiduals = (int32_t)res.residuals.size();
    stats->relax_sweeps = res.relax_sweeps;
  }
  if (residuals)
    for (int32_t i = 0; i < cap && i < (int32_t)res.residuals.size(); ++i) residuals[i] = res.residuals[i];
}

// nrhs right-hand sides, RHS-major [nrhs][n]: blocks of <= kMaxBlock columns in
// THROUGHPUT mode (batch.cuh), one reference-order solve per column otherwise
int solve_batch_common(lamg_ctx* ctx, const lamg_hier* h, int32_t nrhs, const double* b, const double* x0, bool dev,
                       const lamg_cycle_cfg* cfg, double* x, lamg_solve_stats* stats, double* residuals,
                       int32_t cap) {
  std::vector<SolveResult> all;
  int status = LAMG_OK;
  int rc = guarded([&] {
    if (!ctx || !h || !h->h) throw LamgError(LAMG_E_ARGUMENT, "null context or hierarchy");
    if (nrhs < 0 || (nrhs > 0 && (!b || !x0 || !x))) throw LamgError(LAMG_E_ARGUMENT, "bad batch arguments");
    Ctx& c = ctx->c;
    set_device(c);
    const int64_t n = h->h->levels[0]->op.n;
    CycleCfg cc;
    if (cfg) {
      cc.correction = cfg->correction;
      cc.mu = cfg->mu;
      cc.max_cycles = cfg->max_cycles;
      cc.target_reduction = cfg->target_reduction;
      cc.divergence_factor = cfg->divergence_factor;
    }
    const bool blocked = c.mode == LAMG_MODE_THROUGHPUT && cc.correction == 0 && nrhs > 1;
    const int chunk = blocked ? kMaxBlock : 1;
    DVec<double> db, dx0, dx;
    if (!dev) {
      const int64_t w = std::min<int64_t>(nrhs, chunk) * n;
      db.alloc(w, c.s);
      dx0.alloc(w, c.s);
      dx.alloc(w, c.s);
    }
    for (int32_t j0 = 0; j0 < nrhs; j0 += chunk) {
      const int cnt = std::min<int32_t>(chunk, nrhs - j0);
      const double* bj = dev ? b + j0 * n : db.p;
      const double* xj0 = dev ? x0 + j0 * n : dx0.p;
      double* xj = dev ? x + j0 * n : dx.p;
      if (!dev) {
        db.upload(b + j0 * n, cnt * n);
        dx0.upload(x0 + j0 * n, cnt * n);
      }
      std::vector<SolveResult> part;
      int r;
      if (blocked) {
        r = solve_batch_device(c, *h->h, cnt, bj, xj0, cc, xj, part);
      } else {
        part.resize(1);
        r = solve_device(c, *h->h, bj, xj0, cc, xj, part[0]);
      }
      if (r != LAMG_OK && status == LAMG_OK) status = r;
      if (!dev) {
        dx.download(x + j0 * n, cnt * n);
        c.sync();
      }
      for (auto& p : part) all.push_back(std::move(p));
    }
    if (status != LAMG_OK) {
      for (auto& p : all)
        if (!p.message.empty()) throw LamgError(status, p.message);
      throw LamgError(status, "batched solve failed");
    }
  });
  for (size_t j = 0; j < all.size(); ++j)
    fill_stats(all[j], stats ? stats + j : nullptr, residuals ? residuals + (int64_t)j * cap : nullptr, cap);
  return rc;
}

}  // namespace

namespace lamgb {
void gen_rmat(Ctx& c, int scale, int edge_factor, double a, double b, double cc, uint64_t seed, bool lcc, DCSR& out);
bool largest_component_dev(Ctx& c, const CSRv& a, DCSR& out);
void gen_chung_lu(Ctx& c, int32_t n, const double* cdf_host, int64_t pairs, uint64_t seed, bool lcc, DCSR& out);
}  // namespace lamgb

struct lamg_graph {
  int device = 0;
  DCSR a;
};

extern "C" {

const char* lamg_last_error(void) { return g_err.c_str(); }
const char* lamg_version(void) { return "lamg_b200 0.1 (sm_100a)"; }

int64_t lamg_launch_count(void) { return (int64_t)g_launches.load(); }
void lamg_guard_report(int64_t* checked, int64_t* overruns) {
  long long c = 0, o = 0;
  guard_report(&c, &o);
  if (checked) *checked = c;
  if (overruns) *overruns = o;
}

void* lamg_ctx_stream(lamg_ctx* ctx) { return ctx ? (void*)ctx->c.s : nullptr; }

int lamg_ctx_create(int device, int mode, lamg_ctx** out) {
  *out = nullptr;
  return guarded([&] {
    auto* x = new lamg_ctx();
    Ctx& c = x->c;
    c.device = device;
    c.mode = mode;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
      delete x;
      throw LamgError(LAMG_E_CUDA, "no CUDA device available (liblamg_b200 has no CPU path)");
    }
    CK(cudaSetDevice(device));
    CK(cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, device));
    CK(cudaStreamCreateWithFlags(&c.s, cudaStreamNonBlocking));
    CK(cudaMalloc(&c.derr, sizeof(DevErr)));
    CK(cudaMallocHost(&c.herr, sizeof(DevErr)));
    CK(cudaMallocHost(&c.hscal, 4 * kMaxBlock * sizeof(double)));
    CK(cudaMalloc(&c.dflag, 64 * sizeof(int)));
    CK(cudaMalloc(&c.dscal, 256 * sizeof(double)));
    CK(cudaMalloc(&c.dpart, 256 * sizeof(double)));
    CK(cudaMalloc(&c.dbpart, (size_t)kMaxBlock * kColChunks * sizeof(double)));
    CK(cudaMalloc(&c.dbscal, 8 * kMaxBlock * sizeof(double)));
    CK(cudaMalloc(&c.dbdone, kMaxBlock * sizeof(int32_t)));
    c.clear_err();
    *out = x;
  });
}

int lamg_ctx_set_mode(lamg_ctx* ctx, int mode) {
  return guarded([&] {
    if (mode != LAMG_MODE_VALIDATE && mode != LAMG_MODE_THROUGHPUT) throw LamgError(LAMG_E_ARGUMENT, "bad mode");
    ctx->c.mode = mode;
  });
}

int lamg_ctx_set_exact_levels(lamg_ctx* ctx, int32_t levels) {
  return guarded([&] {
    if (!ctx || levels < 0) throw LamgError(LAMG_E_ARGUMENT, "bad context or level count");
    if (ctx->c.exact_levels != levels && (ctx->c.ws || ctx->c.bws)) {
      set_device(ctx->c);
      ctx->c.sync();
      // captured cycles hold the previous smoother choice
      if (ctx->c.ws) ctx->c.ws->clear_graphs();
      if (ctx->c.bws) ctx->c.bws->clear_graphs();
    }
    ctx->c.exact_levels = levels;
  });
}

void lamg_ctx_destroy(lamg_ctx* ctx) {
  if (!ctx) return;
  Ctx& c = ctx->c;
  cudaSetDevice(c.device);
  cudaStreamSynchronize(c.s);
  delete c.ws;
  c.ws = nullptr;
  delete c.bws;
  c.bws = nullptr;
  c.bscratch.release();
  c.rpart.release();
  c.rcnt.release();
  if (c.relax_graph.exec) cudaGraphExecDestroy(c.relax_graph.exec);
  c.relax_graph.exec = nullptr;
  c.ripart.release();
  c.rcptr.release();
  c.rtpart.release();
  c.rtcptr.release();
  c.res_csr = DCSR();
  c.res_stage.f_diag.release();
  c.res_stage.f_ptr.release();
  c.res_stage.f_nbr.release();
  c.res_stage.f_val.release();
  c.res_stage.cop.release();
  for (auto& v : c.prof.ev)
    for (auto e : v) cudaEventDestroy(e);
  cudaStreamSynchronize(c.s);
  cudaFree(c.derr);
  cudaFreeHost(c.herr);
  cudaFreeHost(c.hscal);
  cudaFree(c.dflag);
  cudaFree(c.dscal);
  cudaFree(c.dpart);
  cudaFree(c.dbpart);
  cudaFree(c.dbscal);
  cudaFree(c.dbdone);
  cudaStreamDestroy(c.s);
  delete ctx;
}

// ------------------------------------------------------------------ setup
int lamg_setup(lamg_ctx* ctx, const lamg_csr* a, int on_device, const lamg_setup_opts* opts,
               lamg_hier** out) {
  *out = nullptr;
  return guarded([&] {
    Ctx& c = ctx->c;
    set_device(c);
    SetupOpts o;
    if (opts) {
      o.gamma = opts->gamma;
      o.seed = opts->rng_seed;
      o.coarsest_n = opts->coarsest_n;
      o.tv_sweeps = opts->tv_sweeps;
      o.tv_count_finest = opts->tv_count_finest;
      o.tv_count_max = opts->tv_count_max;
    }
    if (a->n <= 0) throw LamgError(LAMG_E_INVALID_LAPLACIAN, "empty matrix");
    auto* h = new lamg_hier();
    try {
      if (on_device) {
        CSRv v{a->n, a->m, a->row_ptr, a->col, a->val, a->diag};
        h->h = setup_device(c, v, o);
      } else {
        DCSR d;
        upload_csr(c, a, d);
        h->h = setup_device(c, d.view(), o);
      }
    } catch (...) {
      delete h;
      throw;
    }
    h->h->mark_ready(c.s);
    *out = h;
  });
}

void lamg_hier_destroy(lamg_hier* h) {
  if (!h) return;
  if (h->h) {
    cudaSetDevice(h->h->device);
    cudaDeviceSynchronize();
  }
  g_free_sync = true;
  delete h;
  g_free_sync = false;
}

int lamg_hier_info(const lamg_hier* h, int32_t* nlevels, double* setup_work, int32_t* nwarnings,
                   double* setup_seconds) {
  return guarded([&] {
    if (!h || !h->h) throw LamgError(LAMG_E_ARGUMENT, "null hierarchy");
    if (nlevels) *nlevels = (int32_t)h->h->levels.size();
    if (setup_work) *setup_work = h->h->setup_work;
    if (nwarnings) *nwarnings = (int32_t)h->h->warnings.size();
    if (setup_seconds) *setup_seconds = h->h->setup_seconds;
  });
}

int lamg_hier_warning(const lamg_hier* h, int32_t i, char* buf, int32_t cap) {
  return guarded([&] {
    if (!h || i < 0 || i >= (int32_t)h->h->warnings.size()) throw LamgError(LAMG_E_ARGUMENT, "bad warning index");
    snprintf(buf, (size_t)cap, "%s", h->h->warnings[i].c_str());
  });
}

int lamg_hier_level_info(const lamg_hier* h, int32_t l, lamg_level_info* o) {
  return guarded([&] {
    const DLevel& L = level_of(h, l);
    memset(o, 0, sizeof *o);
    o->kind = L.kind;
    o->n = L.op.n;
    o->m = L.op.m;
    o->gamma = L.gamma;
    o->nu_pre = L.nu_pre;
    o->nu_post = L.nu_post;
    o->tv_count = L.tv_count;
    o->coarsest = L.coarsest;
    o->nstages = (int32_t)L.stages.size();
    o->dummy_aggregate = -1;
    if (L.agg) {
      o->coarse_n = L.agg->coarse_n;
      o->alpha = L.agg->alpha;
      o->stage_used = L.agg->stage_used;
      o->dummy_aggregate = L.agg->dummy_aggregate;
    }
    o->gs_fronts = L.sched.nfronts;
    o->colors = L.color ? L.color->ncolors : 0;
  });
}

int lamg_level_cycle_index(const lamg_hier* h, int32_t l, double gamma, double* out) {
  return guarded([&] {
    if (!h || !h->h) throw LamgError(LAMG_E_ARGUMENT, "null hierarchy");
    *out = level_cycle_index(*h->h, (size_t)l, gamma);
  });
}

int lamg_hier_download_op(const lamg_hier* h, int32_t l, int64_t* rp, int32_t* col, double* val,
                          double* diag) {
  return guarded([&] {
    const DLevel& L = level_of(h, l);
    CK(cudaSetDevice(h->h->device));
    h->h->wait_ready();
    if (rp) CK(cudaMemcpy(rp, L.op.rp.p, sizeof(int64_t) * (L.op.n + 1), cudaMemcpyDeviceToHost));
    if (col) CK(cudaMemcpy(col, L.op.col.p, sizeof(int32_t) * 2 * L.op.m, cudaMemcpyDeviceToHost));
    if (val) CK(cudaMemcpy(val, L.op.val.p, sizeof(double) * 2 * L.op.m, cudaMemcpyDeviceToHost));
    if (diag) CK(cudaMemcpy(diag, L.op.diag.p, sizeof(double) * L.op.n, cudaMemcpyDeviceToHost));
  });
}

int lamg_hier_download_agg(const lamg_hier* h, int32_t l, int32_t* aggregate_of, int32_t* seed_of) {
  return guarded([&] {
    const DLevel& L = level_of(h, l);
    if (!L.agg) throw LamgError(LAMG_E_ARGUMENT, "level is not an aggregation level");
    CK(cudaSetDevice(h->h->device));
    h->h->wait_ready();
    if (aggregate_of)
      CK(cudaMemcpy(aggregate_of, L.agg->aggregate_of.p, sizeof(int32_t) * L.agg->fine_n, cudaMemcpyDeviceToHost));
    if (seed_of) CK(cudaMemcpy(seed_of, L.agg->seed_of.p, sizeof(int32_t) * L.agg->coarse_n, cudaMemcpyDeviceToHost));
  });
}

int lamg_hier_stage_info(const lamg_hier* h, int32_t l, int32_t s, int32_t* parent_n, int32_t* coarse_n,
                         int32_t* nf, int64_t* nnz_f) {
  return guarded([&] {
    const DLevel& L = level_of(h, l);
    if (s < 0 || s >= (int32_t)L.stages.size()) throw LamgError(LAMG_E_ARGUMENT, "stage out of range");
    const DStage& st = *L.stages[s];
    *parent_n = st.parent_n;
    *coarse_n = st.coarse_n;
    *nf = st.nf;
    *nnz_f = st.nnzf;
  });
}

int lamg_hier_download_stage(const lamg_hier* h, int32_t l, int32_t s, int32_t* f_nodes, double* f_diag,
                             int64_t* f_ptr, int32_t* f_nbr, double* f_val, int32_t* cop, int32_t* poc) {
  return guarded([&] {
    const DLevel& L = level_of(h, l);
    if (s < 0 || s >= (int32_t)L.stages.size()) throw LamgError(LAMG_E_ARGUMENT, "stage out of range");
    const DStage& st = *L.stages[s];
    CK(cudaSetDevice(h->h->device));
    h->h->wait_ready();
    auto cp = [](void* dst, const void* src, size_t bytes) {
      if (dst && bytes) CK(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
    };
    cp(f_nodes, st.f_nodes.p, sizeof(int32_t) * st.nf);
    cp(f_diag, st.f_diag.p, sizeof(double) * st.nf);
    cp(f_ptr, st.f_ptr.p, sizeof(int64_t) * (st.nf + 1));
    cp(f_nbr, st.f_nbr.p, sizeof(int32_t) * st.nnzf);
    cp(f_val, st.f_val.p, sizeof(double) * st.nnzf);
    cp(cop, st.cop.p, sizeof(int32_t) * st.parent_n);
    cp(poc, st.poc.p, sizeof(int32_t) * st.coarse_n);
  });
}

// ------------------------------------------------------------------ solve
int lamg_solve(lamg_ctx* ctx, const lamg_hier* h, const double* b, const double* x0, const lamg_cycle_cfg* cfg,
               double* x, lamg_solve_stats* stats, double* residuals, int32_t cap) {
  return solve_common(ctx, h, b, x0, false, cfg, x, stats, residuals, cap);
}

int lamg_solve_dev(lamg_ctx* ctx, const lamg_hier* h, const double* b, const double* x0, const lamg_cycle_cfg* cfg,
                   double* x, lamg_solve_stats* stats, double* residuals, int32_t cap) {
  return solve_common(ctx, h, b, x0, true, cfg, x, stats, residuals, cap);
}

int lamg_solve_batch(lamg_ctx* ctx, const lamg_hier* h, int32_t nrhs, const double* b, const double* x0,
                     const lamg_cycle_cfg* cfg, double* x, lamg_solve_stats* stats, double* residuals,
                     int32_t cap) {
  return solve_batch_common(ctx, h, nrhs, b, x0, false, cfg, x, stats, residuals, cap);
}

int lamg_solve_batch_dev(lamg_ctx* ctx, const lamg_hier* h, int32_t nrhs, const double* b, const double* x0,
                         const lamg_cycle_cfg* cfg, double* x, lamg_solve_stats* stats, double* residuals,
                         int32_t cap) {
  return solve_batch_common(ctx, h, nrhs, b, x0, true, cfg, x, stats, residuals, cap);
}

// ------------------------------------------------------ graph ingest (gen.cu)
int lamg_gen_rmat(lamg_ctx* ctx, int32_t scale, int32_t edge_factor, double a, double b, double c_, uint64_t seed,
                  int32_t keep_lcc, lamg_graph** out) {
  *out = nullptr;
  return guarded([&] {
    Ctx& c = ctx->c;
    set_device(c);
    auto* g = new lamg_graph();
    g->device = c.device;
    try {
      gen_rmat(c, scale, edge_factor, a, b, c_, seed, keep_lcc != 0, g->a);
      c.sync();
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

int lamg_gen_chung_lu(lamg_ctx* ctx, int32_t n, const double* cdf, int64_t pairs, uint64_t seed, int32_t keep_lcc,
                      lamg_graph** out) {
  *out = nullptr;
  return guarded([&] {
    Ctx& c = ctx->c;
    set_device(c);
    auto* g = new lamg_graph();
    g->device = c.device;
    try {
      gen_chung_lu(c, n, cdf, pairs, seed, keep_lcc != 0, g->a);
      c.sync();
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

int lamg_graph_lcc(lamg_ctx* ctx, const lamg_csr* a, int on_device, lamg_graph** out) {
  *out = nullptr;
  return guarded([&] {
    Ctx& c = ctx->c;
    set_device(c);
    auto* g = new lamg_graph();
    g->device = c.device;
    try {
      DCSR up;
      CSRv v{a->n, a->m, a->row_ptr, a->col, a->val, a->diag};
      if (!on_device) {
        upload_csr(c, a, up);
        v = up.view();
      }
      if (!largest_component_dev(c, v, g->a)) {  // already connected: a copy
        g->a.alloc(v.n, v.m, c.s);
        CK(cudaMemcpyAsync(g->a.rp.p, v.rp, sizeof(int64_t) * (v.n + 1), cudaMemcpyDefault, c.s));
        CK(cudaMemcpyAsync(g->a.col.p, v.col, sizeof(int32_t) * 2 * v.m, cudaMemcpyDefault, c.s));
        CK(cudaMemcpyAsync(g->a.val.p, v.val, sizeof(double) * 2 * v.m, cudaMemcpyDefault, c.s));
        CK(cudaMemcpyAsync(g->a.diag.p, v.diag, sizeof(double) * v.n, cudaMemcpyDefault, c.s));
      }
      c.sync();
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

int lamg_graph_csr(const lamg_graph* g, lamg_csr* out) {
  return guarded([&] {
    if (!g) throw LamgError(LAMG_E_ARGUMENT, "null graph");
    *out = lamg_csr{g->a.n, g->a.m, g->a.rp.p, g->a.col.p, g->a.val.p, g->a.diag.p};
  });
}

int lamg_graph_download(const lamg_graph* g, int64_t* row_ptr, int32_t* col, double* val, double* diag) {
  return guarded([&] {
    if (!g) throw LamgError(LAMG_E_ARGUMENT, "null graph");
    CK(cudaSetDevice(g->device));
    CK(cudaDeviceSynchronize());
    if (row_ptr) CK(cudaMemcpy(row_ptr, g->a.rp.p, sizeof(int64_t) * (g->a.n + 1), cudaMemcpyDeviceToHost));
    if (col) CK(cudaMemcpy(col, g->a.col.p, sizeof(int32_t) * 2 * g->a.m, cudaMemcpyDeviceToHost));
    if (val) CK(cudaMemcpy(val, g->a.val.p, sizeof(double) * 2 * g->a.m, cudaMemcpyDeviceToHost));
    if (diag) CK(cudaMemcpy(diag, g->a.diag.p, sizeof(double) * g->a.n, cudaMemcpyDeviceToHost));
  });
}

void lamg_graph_destroy(lamg_graph* g) {
  if (!g) return;
  cudaSetDevice(g->device);
  cudaDeviceSynchronize();
  g_free_sync = true;
  delete g;
  g_free_sync = false;
}

int lamg_hier_prepare_throughput(lamg_ctx* ctx, lamg_hier* h) {
  return guarded([&] {
    if (!ctx || !h || !h->h) throw LamgError(LAMG_E_ARGUMENT, "null context or hierarchy");
    set_device(ctx->c);
    h->h->ensure_throughput([&] { prepare_throughput(ctx->c, *h->h); });
  });
}

static const DColor& color_of(const lamg_hier* h, int32_t l) {
  const DLevel& L = level_of(h, l);
  if (!L.color) throw LamgError(LAMG_E_ARGUMENT, "level " + std::to_string(l) + " has no throughput smoother");
  return *L.color;
}

int lamg_hier_color_count(const lamg_hier* h, int32_t l, int32_t* ncolors) {
  return guarded([&] { *ncolors = color_of(h, l).ncolors; });
}

int lamg_hier_download_colors(const lamg_hier* h, int32_t l, int32_t* row_ids, int32_t* color_ptr) {
  return guarded([&] {
    const DColor& cl = color_of(h, l);
    CK(cudaSetDevice(h->h->device));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(row_ids, cl.row_ids.p, sizeof(int32_t) * level_of(h, l).op.n, cudaMemcpyDeviceToHost));
    memcpy(color_ptr, cl.cptr_h.data(), sizeof(int32_t) * (cl.ncolors + 1));
  });
}

int lamg_hier_smooth(lamg_ctx* ctx, const lamg_hier* h, int32_t l, int32_t nrhs, const double* b, double* x,
                     int32_t sweeps) {
  return guarded([&] {
    if (!ctx || !h || !h->h) throw LamgError(LAMG_E_ARGUMENT, "null context or hierarchy");
    Ctx& c = ctx->c;
    set_device(c);
    const DColor& cl = color_of(h, l);
    const int64_t len = (int64_t)level_of(h, l).op.n * nrhs;
    DVec<double> db(len, c.s), dx(len, c.s);
    db.upload(b, len);
    dx.upload(x, len);
    if (nrhs == 1) {
      gs_colored(c, cl, level_of(h, l).op.n, db.p, dx.p, sweeps);
    } else {
      DVec<int32_t> done(nrhs, c.s);
      done.fill_bytes(0);
      bgs_colored(c, cl, level_of(h, l).op.n, db.p, dx.p, sweeps, nrhs, done.p);
    }
    dx.download(x, len);
    c.sync();
  });
}

int lamg_hier_smooth_exact(lamg_ctx* ctx, const lamg_hier* h, int32_t l, int32_t nrhs, const double* b, double* x,
                           int32_t sweeps) {
  return guarded([&] {
    if (!ctx || !h || !h->h) throw LamgError(LAMG_E_ARGUMENT, "null context or hierarchy");
    Ctx& c = ctx->c;
    set_device(c);
    const DLevel& L = level_of(h, l);
    const int64_t len = (int64_t)L.op.n * nrhs;
    DVec<double> db(len, c.s), dx(len, c.s);
    db.upload(b, len);
    dx.upload(x, len);
    if (nrhs == 1) {
      gs_exact(c, L.op.view(), L.sched, db.p, dx.p, 1, sweeps);
    } else {
      if (!batch_width_ok(nrhs)) throw LamgError(LAMG_E_ARGUMENT, "batch width must be 4, 8, 16, 32, 64 or 128");
      ExactItems it;
      build_exact_items(c, L.sched, 32 >> exact_table_for(nrhs), it);
      DVec<int32_t> ctl(1 + (int64_t)kMaxExactSweeps * std::max(1, it.nfronts), c.s);
      bgs_exact(c, L.op.view(), L.sched, it, db.p, dx.p, sweeps, nrhs, ctl.p);
    }
    dx.download(x, len);
    c.sync();
  });
}

// -------------------------------------------------------------- profiling
int lamg_ctx_profile(lamg_ctx* ctx, int enable) {
  return guarded([&] {
    Ctx& c = ctx->c;
    c.prof.enabled = enable != 0;
    for (int k = 0; k < kProfClasses; ++k) {
      c.prof.used[k] = 0;
      c.prof.bytes[k] = 0.0;
    }
  });
}

int lamg_ctx_profile_read(lamg_ctx* ctx, int kernel, int64_t* launches, double* total_ms, double* bytes) {
  return guarded([&] {
    Ctx& c = ctx->c;
    if (kernel < 0 || kernel >= kProfClasses) throw LamgError(LAMG_E_ARGUMENT, "bad profile class");
    c.sync();
    double tot = 0.0;
    for (int64_t i = 0; i < c.prof.used[kernel]; ++i) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, c.prof.ev[kernel][2 * i], c.prof.ev[kernel][2 * i + 1]));
      tot += ms;
    }
    *launches = c.prof.used[kernel];
    *total_ms = tot;
    *bytes = c.prof.used[kernel] ? c.prof.bytes[kernel] / (double)c.prof.used[kernel] : 0.0;  // mean per launch
  });
}

// ------------------------------------------------------- per-kernel API
#define WITH_CSR(ctx, a)        \
  Ctx& c = (ctx)->c;            \
  set_device(c);                \
  DCSR A_;                      \
  upload_csr(c, a, A_);         \
  const CSRv av = A_.view();

int lamg_k_validate(lamg_ctx* ctx, const lamg_csr* a) {
  return guarded([&] {
    WITH_CSR(ctx, a);
    validate_exact(c, av);
  });
}

int lamg_k_mvm(lamg_ctx* ctx, const lamg_csr* a, const double* x, double* y) {
  return guarded([&] {
    WITH_CSR(ctx, a);
    auto dx = up(c, x, a->n);
    DVec<double> dy(std::max(a->n, 1), c.s);
    residual_exact(c, av, nullptr, dx.p, dy.p);
    dy.download(y, a->n);
    c.sync();
  });
}

int lamg_k_residual(lamg_ctx* ctx, const lamg_csr* a, const double* b, const double* x, double* r) {
  return guarded([&] {
    WITH_CSR(ctx, a);
    auto dx = up(c, x, a->n);
    auto db = up(c, b, a->n);
    DVec<double> dr(std::max(a->n, 1), c.s);
    residual_exact(c, av, db.p, dx.p, dr.p);
    dr.download(r, a->n);
    c.sync();
  });
}

int lamg_k_energy(lamg_ctx* ctx, const lamg_csr* a, const double* x, double* e) {
  return guarded([&] {
    WITH_CSR(ctx, a);
    auto dx = up(c, x, a->n);
    UpperIndex upi;
    build_upper_index(c, av, upi);
    DVec<double> scratch;
    energy_seq(c, av, upi, dx.p, c.dscal + 160, scratch);
    *e = read_scalar(c, c.dscal + 160);
  });
}

int lamg_k_gs_sweep(lamg_ctx* ctx, const lamg_csr* a, const double* b, double* x, int backward) {
  return guarded([&] {
    WITH_CSR(ctx, a);
    auto dx = up(c, x, a->n);
    DVec<double> db;
    if (b) db = up(c, b, a->n);
    Schedule sch;
    build_schedule(c, av, backward != 0, sch);
    gs_exact(c, av, sch, b ? db.p : nullptr, dx.p, 1, 1, backward != 0, true);
    dx.download(x, a->n);
    c.sync();
  });
}

int lamg_k_generate_tvs(lamg_ctx* ctx, const lamg_csr* a, int32_t count, int32_t sweeps, uint64_t seed,
                        double* out) {
  return guarded([&] {
    WITH_CSR(ctx, a);
    Schedule sch;
    build_schedule(c, av, false, sch);
    DVec<double> X;
    generate_tvs(c, av, sch, count, sweeps, seed, X);
    std::vector<double> h = X.to_host();
    for (int32_t k = 0; k < count; ++k)
      for (int32_t u = 0; u < a->n; ++u) out[(int64_t)k * a->n + u] = h[(int64_t)u * count + k];
  });
}

int lamg_k_probe(lamg_ctx* ctx, const lamg_csr* a, int32_t sweeps, uint64_t seed, double* factor) {
  return guarded([&] {
    WITH_CSR(ctx, a);
    Schedule sch;
    build_schedule(c, av, false, sch);
    UpperIndex upi;
    build_upper_index(c, av, upi);
    *factor = probe_factor(c, av, sch, upi, sweeps, seed, true);  // the value, bit for bit
  });
}

static DVec<double> upload_tvs_node_major(Ctx& c, int32_t n, int32_t K, const double* tvs) {
  std::vector<double> h((size_t)n * K);
  for (int32_t k = 0; k < K; ++k)
    for (int32_t u = 0; u < n; ++u) h[(size_t)u * K + k] = tvs[(int64_t)k * n + u];
  return up(c, h.data(), (int64_t)n * K);
}

int lamg_k_affinities(lamg_ctx* ctx, const lamg_csr* a, int32_t K, const double* tvs, double* aff,
                      double* nn, int32_t* degenerate, int32_t* ndeg) {
  return guarded([&] {
    WITH_CSR(ctx, a);
    auto X = upload_tvs_node_major(c, a->n, K, tvs);
    DVec<double> daff(std::max<int64_t>(2 * a->m, 1), c.s), dnn(std::max(a->n, 1), c.s);
    compute_affinities(c, av, K, X.p, daff.p, dnn.p);
    daff.download(aff, 2 * a->m);
    std::vector<double> hn(a->n);
    dnn.download(hn.data(), a->n);
    c.sync();
    if (nn) memcpy(nn, hn.data(), sizeof(double) * a->n);
    int32_t nd = 0;
    for (int32_t u = 0; u < a->n; ++u)
      if (hn[u] == 0.0) {
        if (degenerate) degenerate[nd] = u;
        ++nd;
      }
    if (ndeg) *ndeg = nd;
  });
}

int lamg_k_detect_hubs(lamg_ctx* ctx, const lamg_csr* a, int32_t* hubs, int32_t* nhubs) {
  return guarded([&] {
    WITH_CSR(ctx, a);
    DVec<int32_t> dh;
    int32_t nh = detect_hubs(c, av, dh);
    if (nh) dh.download(hubs, nh);
    c.sync();
    *nhubs = nh;
  });
}

int lamg_k_aggregate(lamg_ctx* ctx, const lamg_csr* a, int32_t K, const double* tvs, double gamma,
                     const int32_t* hubs, int32_t nhubs, int32_t* aggregate_of, int32_t* seed_of,
                     int32_t* coarse_n, double* alpha, int32_t* stage_used, int32_t* dummy_aggregate) {
  return guarded([&] {
    WITH_CSR(ctx, a);
    auto X = upload_tvs_node_major(c, a->n, K, tvs);
    auto dh = up(c, hubs, nhubs);
    DAgg t;
    int stages = 1;
    aggregate(c, av, K, X.p, gamma, dh.p, nhubs, t, &stages);
    t.aggregate_of.download(aggregate_of, a->n);
    if (seed_of && t.coarse_n) t.seed_of.download(seed_of, t.coarse_n);
    c.sync();
    *coarse_n = t.coarse_n;
    *alpha = t.alpha;
    *stage_used = t.stage_used;
    *dummy_aggregate = t.dummy_aggregate;
  });
}

int lamg_k_galerkin(lamg_ctx* ctx, const lamg_csr* a, const int32_t* aggregate_of, int32_t coarse_n) {
  return guarded([&] {
    WITH_CSR(ctx, a);
    auto dagg = up(c, aggregate_of, a->n);
    galerkin(c, av, dagg.p, coarse_n, c.res_csr);
    c.res_stage.nf = 0;
    c.sync();
  });
}

int lamg_k_select_low_degree(lamg_ctx* ctx, const lamg_csr* a, int32_t max_degree, int32_t* f, int32_t* nf,
                             int32_t* cc, int32_t* nc) {
  return guarded([&] {
    WITH_CSR(ctx, a);
    SelectResult r;
    select_low_degree(c, av, max_degree, r);
    if (r.nf) r.f.download(f, r.nf);
    if (r.nc) r.c.download(cc, r.nc);
    c.sync();
    *nf = r.nf;
    *nc = r.nc;
  });
}

int lamg_k_schur(lamg_ctx* ctx, const lamg_csr* a, const int32_t* f, int32_t nf, const int32_t* cset, int32_t nc,
                 int32_t* unused) {
  (void)unused;
  return guarded([&] {
    WITH_CSR(ctx, a);
    auto df = up(c, f, nf);
    auto dc = up(c, cset, nc);
    DStage st;
    schur_reduce(c, av, df.p, nf, dc.p, nc, st, c.res_csr, true);
    c.res_stage.nf = nf;
    c.res_stage.f_diag = std::move(st.f_diag);
    c.res_stage.f_ptr = std::move(st.f_ptr);
    c.res_stage.f_nbr = std::move(st.f_nbr);
    c.res_stage.f_val = std::move(st.f_val);
    c.res_stage.cop = std::move(st.cop);
    c.sync();
  });
}

int lamg_k_result_dims(lamg_ctx* ctx, int32_t* n, int64_t* m, int64_t* nnz_f) {
  return guarded([&] {
    Ctx& c = ctx->c;
    *n = c.res_csr.n;
    *m = c.res_csr.m;
    *nnz_f = c.res_stage.nf ? read_i64(c, c.res_stage.f_ptr.p + c.res_stage.nf) : 0;
  });
}

int lamg_k_take_csr(lamg_ctx* ctx, int64_t* rp, int32_t* col, double* val, double* diag) {
  return guarded([&] {
    Ctx& c = ctx->c;
    download_csr(c, c.res_csr, rp, col, val, diag);
  });
}

int lamg_k_take_stage(lamg_ctx* ctx, double* f_diag, int64_t* f_ptr, int32_t* f_nbr, double* f_val, int32_t* cop) {
  return guarded([&] {
    Ctx& c = ctx->c;
    auto& s = c.res_stage;
    int64_t nnz = s.nf ? read_i64(c, s.f_ptr.p + s.nf) : 0;
    if (s.nf) {
      s.f_diag.download(f_diag, s.nf);
      s.f_ptr.download(f_ptr, s.nf + 1);
    } else if (f_ptr) {
      f_ptr[0] = 0;
    }
    if (nnz) {
      s.f_nbr.download(f_nbr, nnz);
      s.f_val.download(f_val, nnz);
    }
    if (cop && s.cop.n) s.cop.download(cop, s.cop.n);
    c.sync();
  });
}

int lamg_k_restrict(lamg_ctx* ctx, const int32_t* agg, int32_t fine_n, int32_t coarse_n, const double* r,
                    double* rc) {
  return guarded([&] {
    Ctx& c = ctx->c;
    set_device(c);
    auto da = up(c, agg, fine_n);
    auto dr = up(c, r, fine_n);
    DVec<int64_t> mp;
    DVec<int32_t> mem;
    build_members(c, fine_n, coarse_n, da.p, mp, mem);
    DVec<double> drc(std::max(coarse_n, 1), c.s);
    restrict_exact(c, coarse_n, mp.p, mem.p, dr.p, 1.0, drc.p);
    drc.download(rc, coarse_n);
    c.sync();
  });
}

int lamg_k_interpolate(lamg_ctx* ctx, const int32_t* agg, int32_t fine_n, int32_t coarse_n, const double* ec,
                       double* x) {
  return guarded([&] {
    Ctx& c = ctx->c;
    set_device(c);
    auto da = up(c, agg, fine_n);
    auto de = up(c, ec, coarse_n);
    auto dx = up(c, x, fine_n);
    interpolate(c, fine_n, da.p, de.p, dx.p);
    dx.download(x, fine_n);
    c.sync();
  });
}

int lamg_k_coarsen_rhs(lamg_ctx* ctx, int32_t parent_n, int32_t coarse_n, int32_t nf, const int32_t* f_nodes,
                       const double* f_diag, const int64_t* f_ptr, const int32_t* f_nbr, const double* f_val,
                       const int32_t* cop, const int32_t* poc, const double* b, double* bc) {
  return guarded([&] {
    Ctx& c = ctx->c;
    set_device(c);
    DStage s;
    upload_stage(c, parent_n, coarse_n, nf, f_nodes, f_diag, f_ptr, f_nbr, f_val, cop, poc, s);
    auto db = up(c, b, parent_n);
    DVec<double> dbc(std::max(coarse_n, 1), c.s);
    coarsen_rhs(c, s.view(), db.p, dbc.p);
    dbc.download(bc, coarse_n);
    c.sync();
  });
}

int lamg_k_backsub(lamg_ctx* ctx, int32_t parent_n, int32_t coarse_n, int32_t nf, const int32_t* f_nodes,
                   const double* f_diag, const int64_t* f_ptr, const int32_t* f_nbr, const double* f_val,
                   const int32_t* cop, const int32_t* poc, const double* xc, const double* b, double* x) {
  return guarded([&] {
    Ctx& c = ctx->c;
    set_device(c);
    DStage s;
    upload_stage(c, parent_n, coarse_n, nf, f_nodes, f_diag, f_ptr, f_nbr, f_val, cop, poc, s);
    auto dxc = up(c, xc, coarse_n);
    auto db = up(c, b, parent_n);
    DVec<double> dx(std::max(parent_n, 1), c.s);
    dx.zero();
    backsub(c, s.view(), dxc.p, db.p, dx.p);
    dx.download(x, parent_n);
    c.sync();
  });
}

int lamg_k_coarsest_direct(lamg_ctx* ctx, const lamg_csr* a, const double* b, double* x) {
  return guarded([&] {
    WITH_CSR(ctx, a);
    DDirect d;
    make_direct(c, av, d);
    auto db = up(c, b, a->n);
    auto dx = up(c, x, a->n);
    DVec<double> scratch(2 * (int64_t)d.maxN + 2, c.s);
    // THROUGHPUT contexts solve with the precomputed inverse, as their solves do
    const bool exact = c.mode == LAMG_MODE_VALIDATE;
    if (!exact) build_direct_inverse(c, d);
    direct_solve(c, d, db.p, dx.p, exact, scratch.p);
    dx.download(x, a->n);
    c.sync();
  });
}

int lamg_k_coarsest_relax(lamg_ctx* ctx, const lamg_csr* a, const double* b, double* x) {
  return guarded([&] {
    WITH_CSR(ctx, a);
    Schedule sch;
    build_schedule(c, av, false, sch);
    auto db = up(c, b, a->n);
    auto dx = up(c, x, a->n);
    DVec<double> r;
    int sw = 0;
    const bool exact = c.mode == LAMG_MODE_VALIDATE;
    // THROUGHPUT contexts run the coloured relaxation their solves use
    std::unique_ptr<DColor> col;
    LongRows nat;
    if (!exact) {
      col = make_color(c, av, sch);
      build_natural_long_rows(c, av, nat);
    }
    relax_solve(c, av, sch, col.get(), exact ? nullptr : &nat, db.p, dx.p, r, &sw, exact);
    dx.download(x, a->n);
    c.sync();
    // the cached sweep graph points at this call's temporaries
    if (c.relax_graph.exec) CK(cudaGraphExecDestroy(c.relax_graph.exec));
    c.relax_graph.exec = nullptr;
  });
}

int lamg_k_recombine(lamg_ctx* ctx, const lamg_csr* a, const double* b, int32_t cols, const double* saved_x,
                     const double* saved_r, double* x, double* before, double* after) {
  return guarded([&] {
    if (cols < 1 || cols > 2) throw LamgError(LAMG_E_ERROR, "recombine supports one or two columns");
    WITH_CSR(ctx, a);
    const int64_t n = a->n;
    auto db = up(c, b, n);
    auto dx = up(c, x, n);
    LevelWS w;
    w.r.alloc(n, c.s);
    w.tmp.alloc(n, c.s);
    for (int i = 0; i < cols; ++i) {
      w.saved_x[i] = up(c, saved_x + i * n, n);
      w.saved_r[i] = up(c, saved_r + i * n, n);
    }
    double* growth = c.dscal + 170;
    CK(cudaMemsetAsync(growth, 0, sizeof(double), c.s));
    recombine_api(c, av, db.p, cols, w, dx.p, c.mode == LAMG_MODE_VALIDATE, growth);
    dx.download(x, n);
    CK(cudaMemcpyAsync(c.hscal, c.dscal + 120, 7 * sizeof(double), cudaMemcpyDeviceToHost, c.s));
    c.sync();
    *before = std::sqrt(c.hscal[0]);
    double nn = c.hscal[6];
    *after = std::sqrt(nn < 0.0 ? 0.0 : nn);
  });
}

int lamg_credit_takes(double gamma, int32_t count, int32_t* out) {
  LevelCredits cr;
  for (int32_t i = 0; i < count; ++i) out[i] = cr.take(0, gamma);
  return LAMG_OK;
}

double lamg_flat_mu(double q) { return 2.0 * q / (q + 1.0); }

uint64_t lamg_rng_derive(uint64_t seed, uint64_t stream) { return rng_derive_host(seed, stream); }

// ------------------------------------------------- fine-level partition
struct lamg_comm {
  std::unique_ptr<Comm> c;
};
struct lamg_part_level {
  lamg_ctx* ctx;
  std::unique_ptr<PartLevel> pl;
  int32_t n;
  uint64_t hier_uid = 0;  // DHier::uid of the hierarchy whose finest level this is (0: built from a CSR)
};

int lamg_comm_unique_id(char id[128]) {
  return guarded([&] { comm_unique_id(id); });
}

int lamg_comm_create(lamg_ctx* ctx, int32_t nranks, int32_t rank, const char id[128], lamg_comm** out) {
  *out = nullptr;
  return guarded([&] {
    set_device(ctx->c);
    auto* cm = new lamg_comm();
    try {
      cm->c = std::make_unique<Comm>(nranks, rank, id);
    } catch (...) {
      delete cm;
      throw;
    }
    *out = cm;
  });
}

void lamg_comm_destroy(lamg_comm* comm) { delete comm; }

static std::vector<int32_t> bounds_of(const int32_t* bounds, int32_t nparts, int32_t n) {
  if (nparts < 1) throw LamgError(LAMG_E_ARGUMENT, "partition needs at least one part");
  std::vector<int32_t> b(bounds, bounds + nparts + 1);
  if (b[0] != 0 || b[nparts] != n) throw LamgError(LAMG_E_ARGUMENT, "bounds must run from 0 to n");
  for (int32_t p = 0; p < nparts; ++p)
    if (b[p + 1] < b[p]) throw LamgError(LAMG_E_ARGUMENT, "bounds must be ascending");
  return b;
}

int lamg_part_bounds(int32_t n, const int64_t* row_ptr, int32_t nparts, int32_t* bounds) {
  return guarded([&] {
    std::vector<int32_t> b;
    part_bounds(n, row_ptr, nparts, b);
    std::copy(b.begin(), b.end(), bounds);
  });
}

int lamg_part_plan_sizes(const lamg_csr* a, const int32_t* bounds, int32_t nparts, int32_t part, int32_t* nloc,
                         int32_t* nghost, int64_t* nnz, int32_t* nsend) {
  return guarded([&] {
    const PartPlan pl = build_part_plan(a->n, a->row_ptr, a->col, a->val, a->diag, bounds_of(bounds, nparts, a->n),
                                        part);
    *nloc = pl.nloc;
    *nghost = pl.nghost;
    *nnz = (int64_t)pl.col.size();
    *nsend = (int32_t)pl.send_idx.size();
  });
}

int lamg_part_plan(const lamg_csr* a, const int32_t* bounds, int32_t nparts, int32_t part, int64_t* row_ptr,
                   int32_t* col, int32_t* ghost_gid, int32_t* recv_ptr, int32_t* send_ptr, int32_t* send_idx) {
  return guarded([&] {
    const PartPlan pl = build_part_plan(a->n, a->row_ptr, a->col, a->val, a->diag, bounds_of(bounds, nparts, a->n),
                                        part);
    std::copy(pl.rp.begin(), pl.rp.end(), row_ptr);
    std::copy(pl.col.begin(), pl.col.end(), col);
    std::copy(pl.ghost_gid.begin(), pl.ghost_gid.end(), ghost_gid);
    std::copy(pl.recv_ptr.begin(), pl.recv_ptr.end(), recv_ptr);
    std::copy(pl.send_ptr.begin(), pl.send_ptr.end(), send_ptr);
    std::copy(pl.send_idx.begin(), pl.send_idx.end(), send_idx);
  });
}

int lamg_part_level_create(lamg_ctx* ctx, const lamg_csr* a, const int32_t* bounds, int32_t nparts,
                           int32_t first_part, int32_t nown, lamg_comm* comm, lamg_part_level** out) {
  *out = nullptr;
  return guarded([&] {
    WITH_CSR(ctx, a);
    const std::vector<int32_t> b = bounds_of(bounds, nparts, a->n);
    std::vector<int64_t> rp(a->row_ptr, a->row_ptr + a->n + 1);
    std::vector<int32_t> col(a->col, a->col + 2 * a->m);
    std::vector<double> val(a->val, a->val + 2 * a->m), diag(a->diag, a->diag + a->n);
    auto* h = new lamg_part_level();
    h->ctx = ctx;
    h->n = a->n;
    try {
      h->pl = std::make_unique<PartLevel>(c, av, rp, col, val, diag, b, first_part, nown, comm ? comm->c.get() : nullptr);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

void lamg_part_level_destroy(lamg_part_level* pl) {
  if (!pl) return;
  cudaStreamSynchronize(pl->ctx->c.s);
  delete pl;
}

int32_t lamg_part_level_n(const lamg_part_level* pl) { return pl ? pl->n : 0; }

int lamg_part_level_from_hier(lamg_ctx* ctx, const lamg_hier* hier, int32_t nparts, int32_t first_part,
                              int32_t nown, lamg_comm* comm, lamg_part_level** out) {
  *out = nullptr;
  return guarded([&] {
    if (!ctx || !hier || !hier->h) throw LamgError(LAMG_E_ARGUMENT, "null context or hierarchy");
    Ctx& c = ctx->c;
    set_device(c);
    const DCSR& op = hier->h->levels[part_level_of(*hier->h)]->op;
    std::vector<int64_t> rp = op.rp.to_host();
    std::vector<int32_t> col(2 * op.m);
    std::vector<double> val(2 * op.m), diag(op.n);
    op.col.download(col.data(), 2 * op.m);
    op.val.download(val.data(), 2 * op.m);
    op.diag.download(diag.data(), op.n);
    c.sync();
    std::vector<int32_t> b;
    part_bounds(op.n, rp.data(), nparts, b);
    auto* h = new lamg_part_level();
    h->ctx = ctx;
    h->n = op.n;
    h->hier_uid = hier->h->uid;
    try {
      h->pl = std::make_unique<PartLevel>(c, op.view(), rp, col, val, diag, b, first_part, nown,
                                          comm ? comm->c.get() : nullptr);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int lamg_part_solve(lamg_ctx* ctx, const lamg_hier* h, lamg_part_level* pl, const double* b, const double* x0,
                    const lamg_cycle_cfg* cfg, double* x, lamg_solve_stats* stats, double* residuals, int32_t cap) {
  if (!pl) return guarded([] { throw LamgError(LAMG_E_ARGUMENT, "null partition"); });
  // the parts enqueue on their own context's stream, the coarse levels on ctx's
  if (pl->ctx != ctx)
    return guarded([] { throw LamgError(LAMG_E_ARGUMENT, "partition was built on another context"); });
  if (h && h->h && pl->hier_uid && pl->hier_uid != h->h->uid)
    return guarded([] { throw LamgError(LAMG_E_ARGUMENT, "partition was built from another hierarchy"); });
  return solve_common(ctx, h, b, x0, false, cfg, x, stats, residuals, cap, pl->pl.get());
}

int lamg_part_smooth(lamg_part_level* h, const double* b, double* x, int32_t sweeps) {
  return guarded([&] {
    Ctx& c = h->ctx->c;
    set_device(c);
    auto db = up(c, b, h->n);
    auto dx = up(c, x, h->n);
    h->pl->load(db.p, dx.p);
    h->pl->sweep(sweeps);
    h->pl->store(dx.p, nullptr);
    dx.download(x, h->n);
    c.sync();
  });
}

int lamg_part_residual(lamg_part_level* h, const double* b, const double* x, double* r) {
  return guarded([&] {
    Ctx& c = h->ctx->c;
    set_device(c);
    auto db = up(c, b, h->n);
    auto dx = up(c, x, h->n);
    auto dr = up(c, r, h->n);
    h->pl->load(db.p, dx.p);
    h->pl->residual();
    h->pl->store(nullptr, dr.p);
    dr.download(r, h->n);
    c.sync();
  });
}

int lamg_part_time(lamg_part_level* h, int32_t sweeps, float* ms) {
  return guarded([&] {
    Ctx& c = h->ctx->c;
    set_device(c);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, c.s));
    h->pl->sweep(sweeps);
    h->pl->residual();
    CK(cudaEventRecord(e1, c.s));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

// ------------------------------------------------------ Matrix Market files
struct lamg_mm {
  MMProblem p;
  std::vector<int64_t> rp;
  std::vector<int32_t> col;
  std::vector<double> val, diag;
};

int lamg_mm_read(const char* path, int32_t kind, int32_t absolute_weight_policy, lamg_mm** out) {
  *out = nullptr;
  return guarded([&] {
    if (!path) throw LamgError(LAMG_E_ARGUMENT, "null path");
    auto* mm = new lamg_mm();
    try {
      mm->p = read_matrix_market_file(path, kind, absolute_weight_policy != 0);
      assemble_problem(mm->p, mm->rp, mm->col, mm->val, mm->diag);
    } catch (...) {
      delete mm;
      throw;
    }
    *out = mm;
  });
}

int lamg_mm_info(const lamg_mm* mm, int32_t* n, int64_t* m, int32_t* was_laplacian, int32_t* nwarnings) {
  return guarded([&] {
    if (!mm) throw LamgError(LAMG_E_ARGUMENT, "null problem");
    *n = mm->p.n;
    *m = (int64_t)mm->p.edges.size();
    *was_laplacian = mm->p.was_laplacian ? 1 : 0;
    *nwarnings = (int32_t)mm->p.warnings.size();
  });
}

int lamg_mm_warning(const lamg_mm* mm, int32_t i, char* buf, int32_t cap) {
  return guarded([&] {
    if (!mm || i < 0 || i >= (int32_t)mm->p.warnings.size()) throw LamgError(LAMG_E_ARGUMENT, "no such warning");
    snprintf(buf, cap, "%s", mm->p.warnings[i].c_str());
  });
}

int lamg_mm_csr(const lamg_mm* mm, int64_t* row_ptr, int32_t* col, double* val, double* diag) {
  return guarded([&] {
    if (!mm) throw LamgError(LAMG_E_ARGUMENT, "null problem");
    if (row_ptr) memcpy(row_ptr, mm->rp.data(), sizeof(int64_t) * mm->rp.size());
    if (col) memcpy(col, mm->col.data(), sizeof(int32_t) * mm->col.size());
    if (val) memcpy(val, mm->val.data(), sizeof(double) * mm->val.size());
    if (diag) memcpy(diag, mm->diag.data(), sizeof(double) * mm->diag.size());
  });
}

void lamg_mm_destroy(lamg_mm* mm) { delete mm; }

int lamg_mm_write(const char* path, const lamg_csr* a, int32_t as_laplacian) {
  return guarded([&] {
    if (!path || !a) throw LamgError(LAMG_E_ARGUMENT, "null argument");
    write_matrix_market_file(path, a->n, a->m, a->row_ptr, a->col, a->val, a->diag, as_laplacian != 0);
  });
}

}  // extern "C"
