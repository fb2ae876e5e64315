// solve.cu -- the solve phase: energy-corrected cycle (cycle.cpp:107-273).
//
// Control flow is host C++ mirroring CycleDriver: per-level credits decide
// the fan-out, each level's work is a short sequence of device kernels on
// the context stream. Vectors never leave the device; the host reads one
// scalar per cycle (the residual norm that drives convergence/divergence).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <string>

#include "batch.cuh"
#include "solve.cuh"
#include "part.cuh"

namespace lamgb {

uint64_t rng_derive_host(uint64_t seed, uint64_t stream);

int LevelCredits::take(size_t l, double gamma) {
  if (credit.size() <= l) credit.resize(l + 1, 0.0);
  credit[l] += gamma;
  int theta = std::max(1, (int)std::floor(credit[l]));
  credit[l] -= theta;
  if (credit[l] < 0.0) credit[l] = 0.0;
  return theta;
}

// ---------------------------------------------------------------- profiling
static void prof_mark(Ctx& c, int cls, bool begin, double bytes = 0.0) {
  if (!c.prof.enabled) return;
  auto& ev = c.prof.ev[cls];
  int64_t idx = 2 * c.prof.used[cls] + (begin ? 0 : 1);
  while ((int64_t)ev.size() <= idx) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    ev.push_back(e);
  }
  CK(cudaEventRecord(ev[idx], c.s));
  if (!begin) {
    ++c.prof.used[cls];
    c.prof.bytes[cls] += bytes;  // total over the profiled launches
  }
}

// ------------------------------------------------------------- workspace
void Workspace::clear_graphs() {
  for (auto& g : graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  graphs.clear();
}

void Workspace::ensure(Ctx& c, const DHier& h, int K_) {
  if (owner == h.uid && lv.size() == h.levels.size() && K == K_) return;
  owner = h.uid;
  K = K_;
  tail_built = false;
  clear_graphs();
  lv.clear();
  lv.resize(h.levels.size());
  int32_t maxN = 0;
  for (size_t l = 0; l < h.levels.size(); ++l) {
    const DLevel& L = *h.levels[l];
    LevelWS& w = lv[l];
    const int64_t n = (int64_t)L.op.n * K;
    w.b.alloc(n, c.s);  // level 0: fixed-address copies of the solve's b and x (graph replay)
    w.x.alloc(n, c.s);
    w.r.alloc(n, c.s);
    if (L.direct) maxN = std::max(maxN, L.direct->maxN);
    if (K_ > 1 && L.xitems[0].nitems) w.xctl.alloc(1 + (int64_t)kMaxExactSweeps * L.xitems[0].nfronts, c.s);
    if (l + 1 < h.levels.size() && h.levels[l + 1]->kind == KIND_ELIM) {
      const auto& st = h.levels[l + 1]->stages;
      w.stage_rhs.resize(st.size());
      w.stage_x.resize(st.size());
      for (size_t s = 1; s < st.size(); ++s) {
        w.stage_rhs[s].alloc((int64_t)st[s]->parent_n * K, c.s);
        w.stage_x[s].alloc((int64_t)st[s]->parent_n * K, c.s);
      }
    }
  }
  direct_scratch.alloc(2 * (int64_t)maxN + 2, c.s);
  top_rhs_valid = false;
}

void Workspace::ensure_adaptive(Ctx& c, const DHier& h) {
  for (size_t l = 0; l < h.levels.size(); ++l) {
    LevelWS& w = lv[l];
    const int32_t n = h.levels[l]->op.n;
    if (w.saved_x[0].n >= n) continue;
    for (int i = 0; i < 2; ++i) {
      w.saved_x[i].alloc(n, c.s);
      w.saved_r[i].alloc(n, c.s);
    }
    w.tmp.alloc(n, c.s);
  }
}

// -------------------------------------------------------------- reductions
static void fold_sum(Ctx& c, bool exact, const double* x, int64_t n, double* d_out) {
  if (exact) seq_sum(c, x, n, d_out);
  else tree_sum(c, x, n, d_out);
}
static void fold_norm2(Ctx& c, bool exact, const double* x, int64_t n, double* d_out) {
  if (exact) seq_norm2(c, x, n, d_out);
  else tree_norm2(c, x, n, d_out);
}
static void sub_mean(Ctx& c, bool exact, double* x, int64_t n) {
  if (exact) subtract_mean_seq(c, x, n);
  else subtract_mean_tree(c, x, n);
}

// ------------------------------------------------------------ recombination
__global__ void diff_kernel(const double* a, const double* b, double* out, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = a[i] - b[i];
}
__global__ void prod_kernel(const double* a, const double* b, double* out, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = a[i] * b[i];
}
// dots[0]=r.r, [1+i]=c_i, [3..6]=g00,g01,g11 -> alpha[0..1] (cycle.cpp:216-257)
__global__ void recomb_alpha_kernel(const double* dots, int cols, double* alpha) {
  double r_norm2 = dots[0];
  double c[2] = {dots[1], dots[2]};
  double g[2][2] = {{dots[3], dots[4]}, {dots[4], dots[5]}};
  double al[2] = {0.0, 0.0};
  if (cols == 1) {
    if (g[0][0] > 0.0) al[0] = c[0] / g[0][0];
  } else if (cols == 2) {
    double det = g[0][0] * g[1][1] - g[0][1] * g[0][1];
    double gg = g[0][0] * g[1][1];
    if (det > 1e-14 * (gg < 1e-300 ? 1e-300 : gg)) {
      al[0] = (c[0] * g[1][1] - c[1] * g[0][1]) / det;
      al[1] = (c[1] * g[0][0] - c[0] * g[0][1]) / det;
    } else {
      double gain0 = g[0][0] > 0.0 ? c[0] * c[0] / g[0][0] : 0.0;
      double gain1 = g[1][1] > 0.0 ? c[1] * c[1] / g[1][1] : 0.0;
      if (gain0 >= gain1 && g[0][0] > 0.0) al[0] = c[0] / g[0][0];
      else if (g[1][1] > 0.0) al[1] = c[1] / g[1][1];
    }
  }
  for (int i = 0; i < cols; ++i) al[i] = al[i] < -2.0 ? -2.0 : (2.0 < al[i] ? 2.0 : al[i]);
  double predicted = r_norm2;
  for (int i = 0; i < cols; ++i) {
    predicted -= 2.0 * al[i] * c[i];
    for (int j = 0; j < cols; ++j) predicted += al[i] * g[i][j] * al[j];
  }
  if (predicted > r_norm2) al[0] = al[1] = 0.0;
  alpha[0] = al[0];
  alpha[1] = al[1];
}
// rk = r - sum alpha_i ad_i (ad_i = r - saved_r_i); x += sum alpha_i (saved_x_i - x)
__global__ void recomb_update_kernel(int64_t n, int cols, const double* alpha, const double* r,
                                     const double* sr0, const double* sr1, const double* sx0,
                                     const double* sx1, double* x, double* rk2) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  double rk = r[k], xk = x[k], delta = 0.0;
  const double* sr[2] = {sr0, sr1};
  const double* sx[2] = {sx0, sx1};
  for (int i = 0; i < cols; ++i) {
    double ad = r[k] - sr[i][k];
    rk -= alpha[i] * ad;
    delta += alpha[i] * (sx[i][k] - xk);
  }
  rk2[k] = rk * rk;
  x[k] = xk + delta;
}
__global__ void recomb_finish_kernel(const double* dots, const double* new2, double* growth) {
  double before = sqrt(dots[0]);
  double nn = *new2;
  double after = sqrt(nn < 0.0 ? 0.0 : nn);
  if (before > 0.0) {
    double g = after / before;
    if (*growth < g) *growth = g;
  }
}

// recombine (cycle.cpp:23-103) with the reference's fold order in every dot
static void recombine(Ctx& c, const CSRv& a, const double* b, int cols, LevelWS& w, double* x,
                      bool exact, double* growth, const Schedule* sch = nullptr) {
  const int64_t n = a.n;
  if (sch) residual_exact(c, a, b, x, w.r.p, sch->heavy_nat.p, sch->nheavy_nat);
  else residual_exact(c, a, b, x, w.r.p);
  c.work += (double)a.m;
  double* dots = c.dscal + 120;  // [120..126]
  CK(cudaMemsetAsync(dots, 0, 7 * sizeof(double), c.s));
  count_launch(), prod_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(w.r.p, w.r.p, w.tmp.p, n);
  fold_sum(c, exact, w.tmp.p, n, dots + 0);
  DVec<double> ad[2];
  for (int i = 0; i < cols; ++i) {
    ad[i].alloc(n, c.s);
    count_launch(), diff_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(w.r.p, w.saved_r[i].p, ad[i].p, n);
  }
  for (int i = 0; i < cols; ++i) {
    count_launch(), prod_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(w.r.p, ad[i].p, w.tmp.p, n);
    fold_sum(c, exact, w.tmp.p, n, dots + 1 + i);
    for (int j = 0; j <= i; ++j) {
      count_launch(), prod_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(ad[i].p, ad[j].p, w.tmp.p, n);
      int slot = (i == 0 && j == 0) ? 3 : (i == 1 && j == 0) ? 4 : 5;
      fold_sum(c, exact, w.tmp.p, n, dots + slot);
    }
  }
  double* alpha = c.dscal + 130;
  count_launch(), recomb_alpha_kernel<<<1, 1, 0, c.s>>>(dots, cols, alpha);
  count_launch(), recomb_update_kernel<<<blocks_for(n), kThreads, 0, c.s>>>(n, cols, alpha, w.r.p, w.saved_r[0].p,
                                                            cols > 1 ? w.saved_r[1].p : w.saved_r[0].p,
                                                            w.saved_x[0].p, cols > 1 ? w.saved_x[1].p : w.saved_x[0].p,
                                                            x, w.tmp.p);
  fold_sum(c, exact, w.tmp.p, n, dots + 6);
  count_launch(), recomb_finish_kernel<<<1, 1, 0, c.s>>>(dots, dots + 6, growth);
  CK_LAUNCH();
  c.work += (double)cols * (double)n;
}

void recombine_api(Ctx& c, const CSRv& a, const double* b, int cols, LevelWS& w, double* x, bool exact,
                   double* growth) {
  recombine(c, a, b, cols, w, x, exact, growth);
}

// ------------------------------------------------------------------ driver
struct Driver {
  Ctx& c;
  const DHier& h;
  const CycleCfg& cfg;
  Workspace& ws;
  LevelCredits credits;
  bool exact;
  double* growth;
  int64_t recombinations = 0;
  int relax_sweeps = 0;
  int K = 1;                     // right-hand sides per block (batch.cuh)
  std::vector<int> relax_cols;   // K > 1: relaxation sweeps per column

  // LAMG_TRACE=1 (debugging aid, one column, host-driven levels): norms of b
  // and x around every level visit
  double tnorm(const double* v, int64_t n) {
    double* d = c.dscal + 160;
    tree_norm2(c, v, n, d);
    return read_scalar(c, d);
  }
  void visit(size_t l, const double* b, double* x, int theta) {
    static const bool trace = getenv("LAMG_TRACE") && atoi(getenv("LAMG_TRACE")) == 1;
    if (trace && K == 1) {
      const int64_t n = h.levels[l]->op.n;
      fprintf(stderr, "[trace] enter l=%zu theta=%d |b|=%.6e |x|=%.6e\n", l, theta, tnorm(b, n), tnorm(x, n));
      visit_(l, b, x, theta);
      fprintf(stderr, "[trace] leave l=%zu |x|=%.6e\n", l, tnorm(x, n));
      return;
    }
    visit_(l, b, x, theta);
  }
  void visit_(size_t l, const double* b, double* x, int theta) {
    if (!exact && (int)l >= ws.tail.first) {
      prof_mark(c, pcls(l, 3), true);
      ws.tail.run(c, (int)l, theta, cfg.mu, (int)h.levels.size());
      prof_mark(c, pcls(l, 3), false);
      return;
    }
    const DLevel& L = *h.levels[l];
    if (L.coarsest != CM_NONE) {
      coarsest(l, b, x);
      return;
    }
    if (h.levels[l + 1]->kind == KIND_ELIM) visit_elimination(l, b, x, theta);
    else visit_aggregation(l, b, x, theta);
  }

  void coarsest(size_t l, const double* b, double* x) {
    const DLevel& L = *h.levels[l];
    if (K > 1) {
      if (L.coarsest == CM_DIRECT) {
        bdirect(c, *L.direct, b, x, K);
      } else {
        if (!L.color) throw LamgError(LAMG_E_ERROR, "batched relaxation needs the coloured operator");
        std::vector<int> sw;
        brelax(c, L.op.view(), *L.color, L.blong_nat, b, x, ws.lv[l].r.p, K, sw);
        relax_cols.resize(K, 0);
        for (int k = 0; k < K; ++k) relax_cols[k] += sw[k];
      }
      return;
    }
    if (L.coarsest == CM_DIRECT) {
      direct_solve(c, *L.direct, b, x, exact, ws.direct_scratch.p);
    } else {
      int sw = 0;
      relax_solve(c, L.op.view(), L.sched, L.color.get(), &L.blong_nat, b, x, ws.lv[l].r, &sw, exact);
      relax_sweeps += sw;
    }
  }

  // the finest level's coarsened right-hand sides are cached for the whole
  // solve (cycle.cpp:139-148); computing them before the first cycle keeps
  // every cycle's kernel schedule identical
  void prepare_top(const double* b) {
    if (h.levels.size() < 2 || h.levels[1]->kind != KIND_ELIM || ws.top_rhs_valid) return;
    const auto& st = h.levels[1]->stages;
    const size_t S = st.size();
    const double* in = b;
    for (size_t s = 0; s < S; ++s) {
      double* out = s + 1 < S ? ws.lv[0].stage_rhs[s + 1].p : ws.lv[1].b.p;
      if (K > 1) bcoarsen_rhs(c, st[s]->view(), in, out, K);
      else coarsen_rhs(c, st[s]->view(exact), in, out);
      c.work += (double)st[s]->nnzf;
      in = out;
    }
    ws.top_rhs_valid = true;
  }

  // cycle.cpp:131-164
  void visit_elimination(size_t l, const double* b, double* x, int theta) {
    const DLevel& child = *h.levels[l + 1];
    const auto& st = child.stages;
    const size_t S = st.size();
    LevelWS& w = ws.lv[l];
    LevelWS& wc = ws.lv[l + 1];
    // stage_rhs[0] = b; stage_rhs[s] = coarsened; coarse rhs -> child's b
    std::vector<const double*> rhs(S);
    rhs[0] = b;
    const bool cached = l == 0 && ws.top_rhs_valid;
    for (size_t s = 0; s < S; ++s) {
      double* out = s + 1 < S ? w.stage_rhs[s + 1].p : wc.b.p;
      if (!cached) {
        if (K > 1) bcoarsen_rhs(c, st[s]->view(), rhs[s], out, K);
        else coarsen_rhs(c, st[s]->view(exact), rhs[s], out);
        c.work += (double)st[s]->nnzf;
      }
      if (s + 1 < S) rhs[s + 1] = out;
    }
    if (l == 0) ws.top_rhs_valid = true;
    for (int i = 0; i < theta; ++i) {
      prof_mark(c, pcls(l, 2), true);
      const double* cur = x;
      for (size_t s = 0; s < S; ++s) {
        double* out = s + 1 < S ? w.stage_x[s + 1].p : wc.x.p;
        if (K > 1) binject(c, st[s]->view(), cur, out, K);
        else inject(c, st[s]->view(), cur, out);
        cur = out;
      }
      prof_mark(c, pcls(l, 2), false);
      int theta_child = credits.take(l + 1, child.gamma);
      visit(l + 1, wc.b.p, wc.x.p, theta_child);
      prof_mark(c, pcls(l, 2), true);
      for (size_t s = S; s-- > 0;) {
        const double* xc = s + 1 < S ? w.stage_x[s + 1].p : wc.x.p;
        double* out = s == 0 ? x : w.stage_x[s].p;
        if (K > 1) bbacksub(c, st[s]->view(), xc, rhs[s], out, K);
        else backsub(c, st[s]->view(), xc, rhs[s], out);
        c.work += (double)st[s]->nnzf;
      }
      prof_mark(c, pcls(l, 2), false);
    }
  }

  // THROUGHPUT solves (one column and K-column blocks) sweep the
  // c.exact_levels finest levels in the reference's exact order: on config 2
  // the finest level's order alone moves the cycle count from the
  // reference's 129 to 141 coloured; exact on level 0 restores 129 (one
  // column: the light wavefront kernel; blocks: bgs_exact's ticketed items)
  // levels below first_smooth + c.exact_levels sweep exactly, where
  // first_smooth is the finest level that smooths (level 0 on 3D grids; level
  // 1 when the finest is eliminated, as on RGG and 2D grids)
  int exact_levels() const {
    int first = (int)h.levels.size();
    for (size_t l = 0; l + 1 < h.levels.size(); ++l)
      if (h.levels[l + 1]->kind == KIND_AGG) {
        first = (int)l;
        break;
      }
    return first + c.exact_levels;
  }
  static int pcls(size_t l, int k) { return 2 + 4 * (int)std::min<size_t>(l, 63) + k; }
  void gs(size_t l, const double* b, double* x, int sweeps) {
    const DLevel& L = *h.levels[l];
    // profile class 0: the sweeps of the finest level that smooths (level 1 below a finest elimination)
    const bool p = (int)l == exact_levels() - c.exact_levels;
    if (p) prof_mark(c, 0, true);
    prof_mark(c, pcls(l, 0), true);
    if (K > 1) {
      if (!L.color) throw LamgError(LAMG_E_ERROR, "batched smoothing needs the coloured operator");
      const ExactItems& xi = L.xitems[exact_table_for(K)];
      if ((int)l < exact_levels() && L.fcolor) bgs_colored(c, *L.fcolor, L.op.n, b, x, sweeps, K);
      else if ((int)l < exact_levels() && xi.nitems) bgs_exact(c, L.op.view(), L.sched, xi, b, x, sweeps, K, ws.lv[l].xctl.p);
      else bgs_colored(c, *L.color, L.op.n, b, x, sweeps, K);
    } else if (!exact && L.fcolor && (int)l < exact_levels()) gs_colored(c, *L.fcolor, L.op.n, b, x, sweeps);
    else if (!exact && L.color && (int)l >= exact_levels()) gs_colored(c, *L.color, L.op.n, b, x, sweeps);
    else gs_exact(c, L.op.view(), L.sched, b, x, 1, sweeps);
    // algorithmic bytes: operator once (8(n+1) + 24m + 8n) + per column x
    // read, b read, x write (24n); K = 1 gives SURVEY.md 8(d)'s 24m + 40n + 8
    if (p) prof_mark(c, 0, false, (24.0 * L.op.m + 16.0 * L.op.n + 8.0 + 24.0 * L.op.n * K) * sweeps);
    prof_mark(c, pcls(l, 0), false, (24.0 * L.op.m + 16.0 * L.op.n + 8.0 + 24.0 * L.op.n * K) * sweeps);
    c.work += (double)L.op.m * sweeps;
  }
  void resid(size_t l, const double* b, const double* x, double* r) {
    const DLevel& L = *h.levels[l];
    const bool p = l == 0;
    if (p) prof_mark(c, 1, true);
    prof_mark(c, pcls(l, 1), true);
    if (K > 1) bresidual(c, L.op.view(), L.blong_nat, b, x, r, K);
    else if (!exact && has_long_rows(L.blong_nat)) residual_tasks(c, L.op.view(), L.blong_nat, b, x, r);
    else if (!exact && L.color) residual_tp(c, L.op.view(), b, x, r, *L.color);
    else residual_exact(c, L.op.view(), b, x, r, L.sched.heavy_nat.p, L.sched.nheavy_nat);
    if (p) prof_mark(c, 1, false, 24.0 * L.op.m + 16.0 * L.op.n + 8.0 + 24.0 * L.op.n * K);
    prof_mark(c, pcls(l, 1), false, 24.0 * L.op.m + 16.0 * L.op.n + 8.0 + 24.0 * L.op.n * K);
    c.work += (double)L.op.m;
  }

  // cycle.cpp:176-209
  void visit_aggregation(size_t l, const double* b, double* x, int theta) {
    const DLevel& L = *h.levels[l];
    const DLevel& child = *h.levels[l + 1];
    const DAgg& t = *child.agg;
    LevelWS& w = ws.lv[l];
    LevelWS& wc = ws.lv[l + 1];
    const bool adaptive = cfg.correction == 1;
    static const bool trace = getenv("LAMG_TRACE") != nullptr;
    int nsaved = 0;
    for (int i = 0; i < theta; ++i) {
      if (child.nu_pre) gs(l, b, x, child.nu_pre);
      // K-column blocks: residual and restriction in one kernel where the level has no long rows
      bool fused = false;
      if (K > 1 && !adaptive && !c.prof.enabled) {
        fused = bresidual_restrict(c, L.op.view(), L.blong_nat, t.coarse_n, t.mem_ptr.p, t.mem.p, b, x, cfg.mu,
                                   wc.b.p, wc.x.p, K);
        if (fused) c.work += (double)L.op.m;
      }
      if (!fused) resid(l, b, x, w.r.p);
      if (trace && K == 1)
        fprintf(stderr, "[trace]   l=%zu pre-smoothed |x|=%.6e |r|=%.6e\n", l, tnorm(x, L.op.n), tnorm(w.r.p, L.op.n));
      if (adaptive) {
        if (nsaved >= 2) throw LamgError(LAMG_E_ERROR, "recombination supports at most two saved iterates");
        copy_d(c, w.saved_x[nsaved].p, x, L.op.n);
        copy_d(c, w.saved_r[nsaved].p, w.r.p, L.op.n);
        ++nsaved;
      }
      prof_mark(c, pcls(l, 2), true);
      if (fused) {
      } else if (K > 1) {
        brestrict(c, t.coarse_n, t.mem_ptr.p, t.mem.p, w.r.p, cfg.mu, wc.b.p, wc.x.p, K);
      } else {
        restrict_exact(c, t.coarse_n, t.mem_ptr.p, t.mem.p, w.r.p, cfg.mu, wc.b.p);
        wc.x.zero();
      }
      prof_mark(c, pcls(l, 2), false);
      int theta_child = credits.take(l + 1, child.gamma);
      visit(l + 1, wc.b.p, wc.x.p, theta_child);
      prof_mark(c, pcls(l, 2), true);
      if (K > 1) binterpolate(c, L.op.n, t.aggregate_of.p, wc.x.p, x, K);
      else interpolate(c, L.op.n, t.aggregate_of.p, wc.x.p, x);
      prof_mark(c, pcls(l, 2), false);
      if (trace && K == 1) {
        resid(l, b, x, w.r.p);
        fprintf(stderr, "[trace]   l=%zu corrected |x|=%.6e |r|=%.6e\n", l, tnorm(x, L.op.n), tnorm(w.r.p, L.op.n));
      }
      if (child.nu_post) gs(l, b, x, child.nu_post);
      if (trace && K == 1) {
        resid(l, b, x, w.r.p);
        fprintf(stderr, "[trace]   l=%zu post-smoothed |x|=%.6e |r|=%.6e\n", l, tnorm(x, L.op.n), tnorm(w.r.p, L.op.n));
      }
    }
    if (adaptive && nsaved > 0) {
      recombine(c, L.op.view(), b, nsaved, w, x, exact, growth, &L.sched);
      ++recombinations;
    }
  }
};

// ------------------------------------------------------------ solve entry
__global__ void absmax_kernel(const double* x, int64_t n, unsigned long long* out) {
  __shared__ double sh[kThreads];
  double m = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs(x[i]));
  sh[threadIdx.x] = m;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) atomicMax(out, (unsigned long long)__double_as_longlong(sh[0]));
}

static std::string to_string_f(double v) {
  char buf[64];
  snprintf(buf, sizeof buf, "%f", v);
  return buf;
}

// compatibility: |sum b| <= 1e-10 ||b||_inf (sequential fold, exact max); the
// test is a threshold decision: sequential in VALIDATE mode (bit-exact with
// the reference), fixed-order tree otherwise
static void check_compatible(Ctx& c, const double* b, int64_t n, bool exact) {
  unsigned long long* bmax = (unsigned long long*)(c.dscal + 140);
  double* bsum = c.dscal + 141;
  CK(cudaMemsetAsync(bmax, 0, sizeof(unsigned long long), c.s));
  count_launch(), absmax_kernel<<<std::min(blocks_for(n), 1024), kThreads, 0, c.s>>>(b, n, bmax);
  CK_LAUNCH();
  if (exact) seq_sum(c, b, n, bsum);
  else tree_sum(c, b, n, bsum);
  CK(cudaMemcpyAsync(c.hscal, c.dscal + 140, 2 * sizeof(double), cudaMemcpyDeviceToHost, c.s));
  c.sync();
  double b_inf, b_sum = c.hscal[1];
  {
    unsigned long long bits;
    memcpy(&bits, &c.hscal[0], sizeof bits);
    memcpy(&b_inf, &bits, sizeof b_inf);
  }
  if (std::fabs(b_sum) > 1e-10 * b_inf)
    throw LamgError(LAMG_E_INCOMPATIBLE_RHS, "right-hand side sum " + to_string_f(b_sum) + " is not zero");
}

// THROUGHPUT data, workspace and the on-device tail of a one-column solve;
// returns whether the tail runs the coarse levels
static bool prepare_solve(Ctx& c, const DHier& h, const CycleCfg& cfg, bool exact) {
  if (!exact) const_cast<DHier&>(h).ensure_throughput([&] { prepare_throughput(c, const_cast<DHier&>(h)); });
  if (!c.ws) c.ws = new Workspace();
  Workspace& ws = *c.ws;
  ws.ensure(c, h);
  ws.top_rhs_valid = false;
  if (cfg.correction == 1) ws.ensure_adaptive(c, h);
  // the on-device tail needs the flat cycle (recombination stays host-driven)
  const bool use_tail = !exact && cfg.correction == 0;
  if (use_tail && !ws.tail_built) {
    const char* env = getenv("LAMG_TAIL_ROWS");
    ws.tail.build(c, h, ws, env ? atoi(env) : 40000);
    ws.tail_built = true;
  }
  if (!use_tail) ws.tail.first = 1 << 30;
  else ws.tail.reset(c);
  return use_tail;
}

// a captured cycle depends on the credits at its start and on mu (baked
// into the restriction and tail kernel arguments)
static std::vector<double> graph_key(const std::vector<double>& credits, const CycleCfg& cfg) {
  std::vector<double> k = credits;
  k.push_back(cfg.mu);
  return k;
}

// cycle.cpp:221-273; b, x0, x are device pointers of the finest size
int solve_device(Ctx& c, const DHier& h, const double* b, const double* x0, const CycleCfg& cfg,
                 double* x, SolveResult& res) {
  const DLevel& L0 = *h.levels[0];
  const CSRv a = L0.op.view();
  const int64_t n = a.n;
  const bool exact = c.mode == LAMG_MODE_VALIDATE;
  res = SolveResult{};
  check_compatible(c, b, n, exact);
  const bool use_tail = prepare_solve(c, h, cfg, exact);
  Workspace& ws = *c.ws;
  const double w0 = c.work = 0.0;
  // the solve runs on fixed-address copies of b and x (CUDA-graph replay)
  double* xw = ws.lv[0].x.p;
  const double* bw = ws.lv[0].b.p;
  copy_d(c, ws.lv[0].b.p, b, n);
  copy_d(c, xw, x0, n);
  double* rn_d = c.dscal + 150;
  double* growth = c.dscal + 151;
  CK(cudaMemsetAsync(growth, 0, sizeof(double), c.s));
  Driver d{c, h, cfg, ws, LevelCredits{}, exact, growth};
  d.credits.credit.assign(h.levels.size(), 0.0);
  d.resid(0, bw, xw, ws.lv[0].r.p);
  fold_norm2(c, exact, ws.lv[0].r.p, n, rn_d);
  const double r0 = read_scalar(c, rn_d);
  res.residuals.push_back(r0);
  if (r0 == 0.0) {
    sub_mean(c, exact, xw, n);
    copy_d(c, x, xw, n);
    c.sync();
    res.converged = true;
    res.acf = 0.0;
    res.solve_work = (c.work - w0) / (double)a.m;
    return LAMG_OK;
  }
  // graphs need a host-sync-free cycle: flat correction, coarsest in the tail
  const char* eg = getenv("LAMG_GRAPHS");
  const bool use_graphs = use_tail && !c.prof.enabled && (int)h.levels.size() - 1 >= ws.tail.first &&
                          !(eg && atoi(eg) == 0);
  if (use_graphs) d.prepare_top(bw);
  const double target = r0 / cfg.target_reduction;
  int rc = LAMG_OK;
  for (int cycle = 1; cycle <= cfg.max_cycles; ++cycle) {
    auto one_cycle = [&] {
      d.visit(0, bw, xw, 1);
      sub_mean(c, exact, xw, n);
      d.resid(0, bw, xw, ws.lv[0].r.p);
      fold_norm2(c, exact, ws.lv[0].r.p, n, rn_d);
    };
    if (use_graphs) {
      // the captured kernels bake in the credits and CycleConfig::mu
      const std::vector<double> key = graph_key(d.credits.credit, cfg);
      Workspace::CycleGraph* g = nullptr;
      for (auto& e : ws.graphs)
        if (e.key == key) g = &e;
      if (!g) {
        Workspace::CycleGraph e;
        e.key = key;
        const double wc = c.work;
        const long long l0 = t_launches;
        cudaGraph_t graph;
        CK(cudaStreamBeginCapture(c.s, cudaStreamCaptureModeThreadLocal));
        one_cycle();
        CK(cudaStreamEndCapture(c.s, &graph));
        CK(cudaGraphInstantiate(&e.exec, graph, 0));
        CK(cudaGraphDestroy(graph));
        e.work = c.work - wc;
        e.launches = t_launches - l0;
        g_launches -= e.launches;  // counted when the graph runs
        t_launches = l0;
        e.credits_after = d.credits.credit;
        c.work = wc;
        ws.graphs.push_back(std::move(e));
        g = &ws.graphs.back();
      }
      CK(cudaGraphLaunch(g->exec, c.s));
      g_launches += g->launches;
      c.work += g->work;
      d.credits.credit = g->credits_after;
    } else {
      one_cycle();
    }
    const double rn = read_scalar(c, rn_d);
    res.residuals.push_back(rn);
    res.cycles = cycle;
    if (rn <= target) {
      res.converged = true;
      break;
    }
    if (rn > cfg.divergence_factor * r0 || !std::isfinite(rn)) {
      res.acf = std::pow(rn / r0, 1.0 / cycle);
      res.solve_work = (c.work - w0) / (double)a.m;
      res.message = "solve diverged: residual grew from " + to_string_f(r0) + " to " + to_string_f(rn);
      rc = LAMG_E_DIVERGED;
      break;
    }
  }
  copy_d(c, x, xw, n);
  if (rc == LAMG_OK) {
    const double rp = res.residuals.back();
    res.acf = std::pow(rp / r0, 1.0 / (double)res.cycles);
    res.solve_work = (c.work - w0) / (double)a.m;
  }
  if (use_tail) ws.tail.collect(c, &c.work, &d.relax_sweeps);
  if (use_tail) res.solve_work = (c.work - w0) / (double)a.m;
  res.recombinations = d.recombinations;
  res.recomb_max_growth = read_scalar(c, growth);
  res.relax_sweeps = d.relax_sweeps;
  return rc;
}

// ------------------------------------------------------- batched solve
// cycle.cpp:221-273 for nrhs <= 32 right-hand sides at once (THROUGHPUT
// mode). The visit sequence is data-independent (LevelCredit), so one cycle
// schedule -- one CUDA graph per credit state -- serves every column; each
// column is copied out at the cycle where its own test (r <= r0/1e10, or
// divergence) fires. A column's bits do not depend on the batch it rides in.
int solve_batch_device(Ctx& c, const DHier& h, int nrhs, const double* B, const double* X0, const CycleCfg& cfg,
                       double* X, std::vector<SolveResult>& res) {
  if (nrhs < 1 || nrhs > kMaxBlock) throw LamgError(LAMG_E_ARGUMENT, "batched solve takes 1..128 right-hand sides");
  if (c.mode != LAMG_MODE_THROUGHPUT || cfg.correction != 0)
    throw LamgError(LAMG_E_ARGUMENT, "batched solve runs the flat THROUGHPUT cycle");
  const DLevel& L0 = *h.levels[0];
  const int64_t n = L0.op.n;
  const int K = batch_width_for(nrhs);
  res.assign(nrhs, SolveResult{});
  const_cast<DHier&>(h).ensure_throughput([&] { prepare_throughput(c, const_cast<DHier&>(h)); });
  if (!c.bws) c.bws = new Workspace();
  Workspace& ws = *c.bws;
  ws.ensure(c, h, K);
  ws.top_rhs_valid = false;
  if (!ws.tail_built) {
    // levels of at most this many rows run in the K-column cluster tail
    const char* env = getenv("LAMG_BATCH_TAIL_ROWS");
    ws.tail.build(c, h, ws, env ? atoi(env) : 16384);
    ws.tail_built = true;
  }
  ws.tail.reset(c);
  double* Xw = ws.lv[0].x.p;
  double* Bw = ws.lv[0].b.p;
  double* Rw = ws.lv[0].r.p;
  to_node_major(c, B, n, nrhs, K, Bw);
  to_node_major(c, X0, n, nrhs, K, Xw);
  // compatibility per column: |sum b| <= 1e-10 ||b||_inf
  unsigned long long* bmax = (unsigned long long*)c.dbscal;  // [K]
  double* bsum = c.dbscal + kMaxBlock;                       // [K]
  double* rn_d = c.dbscal + 2 * kMaxBlock;                   // [K]
  double* xsum = c.dbscal + 3 * kMaxBlock;                   // [K]
  bcolabsmax(c, Bw, n, K, bmax);
  bcolsum(c, Bw, n, K, false, bsum);
  CK(cudaMemcpyAsync(c.hscal, c.dbscal, 2 * kMaxBlock * sizeof(double), cudaMemcpyDeviceToHost, c.s));
  c.sync();
  for (int j = 0; j < nrhs; ++j) {
    double b_inf;
    memcpy(&b_inf, &c.hscal[j], sizeof b_inf);
    const double b_sum = c.hscal[kMaxBlock + j];
    if (std::fabs(b_sum) > 1e-10 * b_inf)
      throw LamgError(LAMG_E_INCOMPATIBLE_RHS, "right-hand side sum " + to_string_f(b_sum) + " is not zero");
  }
  const double w0 = c.work = 0.0;
  Driver d{c, h, cfg, ws, LevelCredits{}, false, c.dscal + 151};
  d.K = K;
  d.credits.credit.assign(h.levels.size(), 0.0);
  CK(cudaMemsetAsync(c.dscal + 151, 0, sizeof(double), c.s));
  std::vector<double> rn(K), r0(K), target(K);
  auto read_norms = [&] {
    CK(cudaMemcpyAsync(c.hscal, rn_d, K * sizeof(double), cudaMemcpyDeviceToHost, c.s));
    c.sync();
    for (int k = 0; k < K; ++k) rn[k] = std::sqrt(c.hscal[k]);
  };
  d.resid(0, Bw, Xw, Rw);
  bcolsum(c, Rw, n, K, true, rn_d);
  read_norms();
  std::vector<char> done(nrhs, 0);
  int active = nrhs;
  bool any_zero = false;
  for (int j = 0; j < nrhs; ++j) {
    r0[j] = rn[j];
    target[j] = r0[j] / cfg.target_reduction;
    res[j].residuals.push_back(r0[j]);
    if (r0[j] == 0.0) any_zero = true;
  }
  if (any_zero) {  // r0 == 0: the answer is x0 minus its mean (cycle.cpp:234-238)
    bcolsum(c, Xw, n, K, false, xsum);
    for (int j = 0; j < nrhs; ++j)
      if (r0[j] == 0.0) {
        column_out(c, Xw, n, K, j, X + j * n, xsum);
        res[j].converged = true;
        done[j] = 1;
        --active;
      }
  }
  const char* eg = getenv("LAMG_GRAPHS");
  const bool use_graphs = (int)h.levels.size() - 1 >= ws.tail.first && !c.prof.enabled && !(eg && atoi(eg) == 0);
  if (use_graphs) d.prepare_top(Bw);
  std::vector<double> work_at(1, 0.0);
  int cycle = 0;
  for (cycle = 1; cycle <= cfg.max_cycles && active > 0; ++cycle) {
    auto one_cycle = [&] {
      d.visit(0, Bw, Xw, 1);
      bcolsum(c, Xw, n, K, false, xsum);
      bsub_mean(c, Xw, n, K, xsum);
      d.resid(0, Bw, Xw, Rw);
      bcolsum(c, Rw, n, K, true, rn_d);
    };
    if (use_graphs) {
      // the captured kernels bake in the credits and CycleConfig::mu
      const std::vector<double> key = graph_key(d.credits.credit, cfg);
      Workspace::CycleGraph* g = nullptr;
      for (auto& e : ws.graphs)
        if (e.key == key) g = &e;
      if (!g) {
        Workspace::CycleGraph e;
        e.key = key;
        const double wc = c.work;
        const long long l0 = t_launches;
        cudaGraph_t graph;
        CK(cudaStreamBeginCapture(c.s, cudaStreamCaptureModeThreadLocal));
        one_cycle();
        CK(cudaStreamEndCapture(c.s, &graph));
        CK(cudaGraphInstantiate(&e.exec, graph, 0));
        CK(cudaGraphDestroy(graph));
        e.work = c.work - wc;
        e.launches = t_launches - l0;
        g_launches -= e.launches;
        t_launches = l0;
        e.credits_after = d.credits.credit;
        c.work = wc;
        ws.graphs.push_back(std::move(e));
        g = &ws.graphs.back();
      }
      CK(cudaGraphLaunch(g->exec, c.s));
      g_launches += g->launches;
      c.work += g->work;
      d.credits.credit = g->credits_after;
    } else {
      one_cycle();
    }
    work_at.push_back(c.work);
    read_norms();
    for (int j = 0; j < nrhs; ++j) {
      if (done[j]) continue;
      res[j].residuals.push_back(rn[j]);
      res[j].cycles = cycle;
      if (rn[j] <= target[j]) {
        res[j].converged = true;
      } else if (rn[j] > cfg.divergence_factor * r0[j] || !std::isfinite(rn[j])) {
        res[j].message = "solve diverged: residual grew from " + to_string_f(r0[j]) + " to " + to_string_f(rn[j]);
      } else {
        continue;
      }
      column_out(c, Xw, n, K, j, X + j * n);
      done[j] = 1;
      --active;
    }
  }
  for (int j = 0; j < nrhs; ++j)
    if (!done[j]) column_out(c, Xw, n, K, j, X + j * n);  // max_cycles reached
  // the on-device tail's work is read once at the end; cycles are identical in
  // structure, so a column's share is proportional to its cycle count
  double tail_work = 0.0;
  int tail_relax = 0;
  ws.tail.collect(c, &tail_work, &tail_relax);
  const int ran = std::max(1, cycle - 1);
  for (int j = 0; j < nrhs; ++j) {
    SolveResult& r = res[j];
    const int cj = r.cycles;
    const double wj = work_at[std::min<size_t>(cj, work_at.size() - 1)] - w0 + tail_work * cj / ran;
    r.solve_work = wj / (double)L0.op.m;
    r.acf = cj > 0 && r0[j] > 0.0 ? std::pow(r.residuals.back() / r0[j], 1.0 / cj) : 0.0;
    r.relax_sweeps = (j < (int)d.relax_cols.size() ? d.relax_cols[j] : 0) + tail_relax;
  }
  c.sync();
  for (int j = 0; j < nrhs; ++j)
    if (!res[j].message.empty()) return LAMG_E_DIVERGED;
  return LAMG_OK;
}


// ------------------------------------------------ partitioned finest level
// lamg::solve with the finest level split across parts (part.cuh). Level 0's
// visit (cycle.cpp:176-209, theta = 1) runs its sweeps and residual on the
// parts; the residual is allgathered so restrict_residual, the whole coarse
// recursion (Driver::visit from level 1, tail included) and the coarse
// correction are exactly the single-device ones on every rank; the
// interpolation lands on the owned rows. Every kernel and fold order matches
// solve_device, so the result is bit-identical to it.
// The partitioned level lp is the finest level that smooths: level 0 when its
// child is an aggregation level (3D grids), level 1 when level 0 is reduced
// by elimination first (2D grids, geometric and power-law graphs) -- then the
// finest level's work is the RHS coarsening (cached, cycle.cpp:139-148), the
// injection and the back-substitution, replicated on every rank. A level lp
// that is the relaxation coarsest (configs 4 and 5) runs RelaxationSolver::solve
// (coarse_solver.cpp:82-93) on the parts: sweep, mean, residual, norm.
int part_level_of(const DHier& h) {
  if (h.levels.size() < 2) return 0;
  return h.levels[1]->kind == KIND_ELIM ? 1 : 0;
}

int solve_partitioned(Ctx& c, const DHier& h, PartLevel& pl, const double* b, const double* x0, const CycleCfg& cfg,
                      double* x, SolveResult& res) {
  const DLevel& L0 = *h.levels[0];
  const int64_t n = L0.op.n;
  res = SolveResult{};
  if (c.mode != LAMG_MODE_THROUGHPUT || cfg.correction != 0)
    throw LamgError(LAMG_E_ARGUMENT, "the partitioned solve runs THROUGHPUT mode with the flat cycle");
  const int lp = part_level_of(h);
  const DLevel& LP = *h.levels[lp];
  const int64_t np = LP.op.n;
  const bool relax = LP.coarsest == CM_RELAX;
  if (h.levels.size() < 2 || (!relax && (LP.coarsest != CM_NONE || h.levels[lp + 1]->kind != KIND_AGG)))
    throw LamgError(LAMG_E_ARGUMENT,
                    "the partitioned solve needs a smoothing level (aggregation child or relaxation coarsest) at "
                    "the top of the hierarchy");
  if (pl.bounds.back() != np)
    throw LamgError(LAMG_E_DIMENSION_MISMATCH, "partition does not match the hierarchy's first smoothing level");
  check_compatible(c, b, n, false);
  const bool use_tail = prepare_solve(c, h, cfg, false);
  Workspace& ws = *c.ws;
  ws.top_rhs_valid = false;
  const double w0 = c.work = 0.0;
  double* xw = ws.lv[0].x.p;
  double* bw = ws.lv[0].b.p;
  double* rw = ws.lv[0].r.p;
  copy_d(c, bw, b, n);
  copy_d(c, xw, x0, n);
  double* rn_d = c.dscal + 150;
  double* growth = c.dscal + 151;
  double* rl_d = c.dscal + 152;  // relaxation norms of the partitioned level
  CK(cudaMemsetAsync(growth, 0, sizeof(double), c.s));
  Driver d{c, h, cfg, ws, LevelCredits{}, false, growth};
  d.credits.credit.assign(h.levels.size(), 0.0);
  const double m0 = (double)L0.op.m;
  const double mp = (double)LP.op.m;
  // vectors of the partitioned level (level 0's own, or level 1's workspace)
  double* xp = lp == 0 ? xw : ws.lv[lp].x.p;
  double* bp = lp == 0 ? bw : ws.lv[lp].b.p;
  double* rp = ws.lv[lp].r.p;
  const std::vector<std::unique_ptr<DStage>>* stages = lp == 1 ? &h.levels[1]->stages : nullptr;
  const size_t S = stages ? stages->size() : 0;
  std::vector<const double*> rhs(S);
  if (lp == 1) {  // coarsen the right-hand side once (cycle.cpp:139-148)
    rhs[0] = bw;
    for (size_t s = 0; s < S; ++s) {
      double* out = s + 1 < S ? ws.lv[0].stage_rhs[s + 1].p : bp;
      coarsen_rhs(c, (*stages)[s]->view(false), rhs[s], out);
      c.work += (double)(*stages)[s]->nnzf;
      if (s + 1 < S) rhs[s + 1] = out;
    }
  }
  // one visit of the partitioned level (theta = 1): b in bp, x in xp (full vectors, in and out)
  auto visit_part = [&] {
    pl.load(bp, xp);
    if (relax) {
      pl.residual();
      c.work += mp;
      pl.allgather(true, rp);
      tree_norm2(c, rp, np, rl_d);
      const double r0 = read_scalar(c, rl_d);
      if (r0 == 0.0) return;
      for (int sweep = 0; sweep < 400; ++sweep) {
        pl.sweep(1);
        pl.allgather(false, xp);
        subtract_mean_tree(c, xp, np);
        pl.load(nullptr, xp);
        pl.residual();
        c.work += 2.0 * mp;
        pl.allgather(true, rp);
        tree_norm2(c, rp, np, rl_d);
        ++d.relax_sweeps;
        if (read_scalar(c, rl_d) <= 1e-12 * r0) break;
      }
      return;
    }
    const DLevel& child = *h.levels[lp + 1];
    const DAgg& t = *child.agg;
    LevelWS& wc = ws.lv[lp + 1];
    if (child.nu_pre) {
      pl.sweep(child.nu_pre);
      c.work += mp * child.nu_pre;
    }
    pl.residual();
    c.work += mp;
    pl.allgather(true, rp);
    restrict_exact(c, t.coarse_n, t.mem_ptr.p, t.mem.p, rp, cfg.mu, wc.b.p);
    wc.x.zero();
    const int theta_child = d.credits.take(lp + 1, child.gamma);
    d.visit(lp + 1, wc.b.p, wc.x.p, theta_child);
    pl.interpolate(t.aggregate_of.p, wc.x.p);
    if (child.nu_post) {
      pl.sweep(child.nu_post);
      c.work += mp * child.nu_post;
    }
    pl.allgather(false, xp);
  };
  // r = b - A x on the finest level and its norm: on the parts when they hold
  // the finest level, replicated otherwise
  auto residual_norm = [&] {
    if (lp == 0) {
      pl.load(nullptr, xw);
      pl.residual();
      pl.allgather(true, rw);
    } else {
      d.resid(0, bw, xw, rw);
      c.work -= m0;  // counted below
    }
    c.work += m0;
    tree_norm2(c, rw, n, rn_d);
  };
  if (lp == 0) pl.load(bw, xw);
  residual_norm();
  const double r0 = read_scalar(c, rn_d);
  res.residuals.push_back(r0);
  if (r0 != 0.0) {
    const double target = r0 / cfg.target_reduction;
    for (int cycle = 1; cycle <= cfg.max_cycles; ++cycle) {
      if (lp == 0) {
        visit_part();
      } else {  // visit_elimination(0) with theta = 1 (cycle.cpp:131-164)
        const double* cur = xw;
        for (size_t s = 0; s < S; ++s) {
          double* out = s + 1 < S ? ws.lv[0].stage_x[s + 1].p : xp;
          inject(c, (*stages)[s]->view(), cur, out);
          cur = out;
        }
        d.credits.take(1, h.levels[1]->gamma);
        visit_part();
        for (size_t s = S; s-- > 0;) {
          const double* xc = s + 1 < S ? ws.lv[0].stage_x[s + 1].p : xp;
          double* out = s == 0 ? xw : ws.lv[0].stage_x[s].p;
          backsub(c, (*stages)[s]->view(), xc, rhs[s], out);
          c.work += (double)(*stages)[s]->nnzf;
        }
      }
      // subtract_mean over the whole iterate, then the cycle's residual
      subtract_mean_tree(c, xw, n);
      residual_norm();
      const double rn = read_scalar(c, rn_d);
      res.residuals.push_back(rn);
      res.cycles = cycle;
      if (rn <= target) {
        res.converged = true;
        break;
      }
      if (rn > cfg.divergence_factor * r0 || !std::isfinite(rn)) {
        res.acf = std::pow(rn / r0, 1.0 / cycle);
        res.solve_work = (c.work - w0) / m0;
        res.message = "solve diverged: residual grew from " + to_string_f(r0) + " to " + to_string_f(rn);
        copy_d(c, x, xw, n);
        c.sync();
        return LAMG_E_DIVERGED;
      }
    }
  } else {
    res.converged = true;
    subtract_mean_tree(c, xw, n);
  }
  if (r0 != 0.0) {
    const double rp_ = res.residuals.back();
    res.acf = std::pow(rp_ / r0, 1.0 / (double)res.cycles);
  }
  copy_d(c, x, xw, n);
  if (use_tail) ws.tail.collect(c, &c.work, &d.relax_sweeps);
  res.solve_work = (c.work - w0) / m0;
  res.recombinations = d.recombinations;
  res.recomb_max_growth = read_scalar(c, growth);
  res.relax_sweeps = d.relax_sweeps;
  return LAMG_OK;
}

}  // namespace lamgb
