// oracle/ref_capi.cpp -- TEST INFRASTRUCTURE ONLY (the parity checker).
//
// C-ABI wrapper over the UNMODIFIED reference implementation. The reference
// sources are compiled where they lie (/root/reference/proj/core/src/*.cpp)
// with -Dlamg=lamg_ref (oracle/Makefile), so every `lamg::` below resolves to
// the reference's own code. Output goes to oracle/_ref/liblamg_ref.so, which
// is git-ignored and only used by tests/, smoke() and bench.py's CPU arms.
#define ORACLE_PREFIX ref_
#include "oracle_api.h"

#include <chrono>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "lamg/aggregation.hpp"
#include "lamg/coarse_solver.hpp"
#include "lamg/cycle.hpp"
#include "lamg/elimination.hpp"
#include "lamg/errors.hpp"
#include "lamg/generators.hpp"
#include "lamg/hierarchy.hpp"
#include "lamg/rng.hpp"
#include "lamg/smoothing.hpp"
#include "lamg/solver.hpp"
#include "lamg/sparse_laplacian.hpp"
#include "lamg/work.hpp"

namespace {

thread_local std::string g_err;
thread_local int g_setup_status = 0;

int fail(int code, const char* what) {
  g_err = what;
  return code;
}

// Maps the reference's exception types (errors.hpp:8-42, cycle.hpp:50-53) to status codes.
template <typename F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return ORC_OK;
  } catch (const lamg::DivergedError& e) {
    return fail(ORC_E_DIVERGED, e.what());
  } catch (const lamg::EmptyGraphError& e) {
    return fail(ORC_E_EMPTY_GRAPH, e.what());
  } catch (const lamg::SingularDiagonalError& e) {
    return fail(ORC_E_SINGULAR_DIAGONAL, e.what());
  } catch (const lamg::InvalidLaplacianError& e) {
    return fail(ORC_E_INVALID_LAPLACIAN, e.what());
  } catch (const lamg::DimensionMismatchError& e) {
    return fail(ORC_E_DIMENSION_MISMATCH, e.what());
  } catch (const lamg::IncompatibleRhsError& e) {
    return fail(ORC_E_INCOMPATIBLE_RHS, e.what());
  } catch (const std::exception& e) {
    return fail(ORC_E_ERROR, e.what());
  }
}

lamg::SparseLaplacian make_csr(CSR_ARGS) {
  lamg::SparseLaplacian a;
  a.n = n;
  a.m = m;
  a.row_ptr.assign(rp, rp + n + 1);
  a.col.assign(col, col + 2 * m);
  a.val.assign(val, val + 2 * m);
  a.diag.assign(diag, diag + n);
  return a;
}

#define CSR_PASS n, m, rp, col, val, diag

void put_csr(bag* b, const std::string& p, const lamg::SparseLaplacian& a) {
  bag_put_i32(b, (p + "n").c_str(), a.n);
  bag_put_i64(b, (p + "m").c_str(), a.m);
  bag_put(b, (p + "row_ptr").c_str(), BAG_I64, a.row_ptr.data(), (int64_t)a.row_ptr.size());
  bag_put(b, (p + "col").c_str(), BAG_I32, a.col.data(), (int64_t)a.col.size());
  bag_put(b, (p + "val").c_str(), BAG_F64, a.val.data(), (int64_t)a.val.size());
  bag_put(b, (p + "diag").c_str(), BAG_F64, a.diag.data(), (int64_t)a.diag.size());
}

void put_stage(bag* b, const std::string& p, const lamg::ElimStage& s) {
  bag_put_i32(b, (p + "parent_n").c_str(), s.parent_n);
  bag_put_i32(b, (p + "coarse_n").c_str(), s.coarse_n);
  bag_put(b, (p + "f_nodes").c_str(), BAG_I32, s.f_nodes.data(), (int64_t)s.f_nodes.size());
  bag_put(b, (p + "f_diag").c_str(), BAG_F64, s.f_diag.data(), (int64_t)s.f_diag.size());
  bag_put(b, (p + "f_ptr").c_str(), BAG_I64, s.f_ptr.data(), (int64_t)s.f_ptr.size());
  bag_put(b, (p + "f_nbr").c_str(), BAG_I32, s.f_nbr.data(), (int64_t)s.f_nbr.size());
  bag_put(b, (p + "f_val").c_str(), BAG_F64, s.f_val.data(), (int64_t)s.f_val.size());
  bag_put(b, (p + "coarse_of_parent").c_str(), BAG_I32, s.coarse_of_parent.data(),
          (int64_t)s.coarse_of_parent.size());
  bag_put(b, (p + "parent_of_coarse").c_str(), BAG_I32, s.parent_of_coarse.data(),
          (int64_t)s.parent_of_coarse.size());
}

void put_agg(bag* b, const std::string& p, const lamg::AggregationTransfer& t) {
  bag_put(b, (p + "aggregate_of").c_str(), BAG_I32, t.aggregate_of.data(),
          (int64_t)t.aggregate_of.size());
  bag_put(b, (p + "seed_of").c_str(), BAG_I32, t.seed_of.data(), (int64_t)t.seed_of.size());
  bag_put_i32(b, (p + "coarse_n").c_str(), t.coarse_n);
  bag_put_f64(b, (p + "alpha").c_str(), t.alpha);
  bag_put_i32(b, (p + "stage_used").c_str(), t.stage_used);
  bag_put_i32(b, (p + "dummy_aggregate").c_str(), t.dummy_aggregate);
}

lamg::ElimStage make_stage(STAGE_ARGS) {
  lamg::ElimStage s;
  s.parent_n = parent_n;
  s.coarse_n = coarse_n;
  s.f_nodes.assign(f_nodes, f_nodes + nf);
  s.f_diag.assign(f_diag, f_diag + nf);
  s.f_ptr.assign(f_ptr, f_ptr + nf + 1);
  s.f_nbr.assign(f_nbr, f_nbr + f_ptr[nf]);
  s.f_val.assign(f_val, f_val + f_ptr[nf]);
  s.coarse_of_parent.assign(coarse_of_parent, coarse_of_parent + parent_n);
  s.parent_of_coarse.assign(parent_of_coarse, parent_of_coarse + coarse_n);
  return s;
}

lamg::TestVectorSet make_tvs(int32_t n, int K, const double* tvs) {
  lamg::TestVectorSet t;
  t.n = n;
  t.count = K;
  for (int k = 0; k < K; ++k) t.columns.emplace_back(tvs + (int64_t)k * n, tvs + (int64_t)(k + 1) * n);
  return t;
}

lamg::CycleConfig make_cfg(int correction, double mu, int max_cycles, double target_reduction,
                           double divergence_factor, double gamma, uint64_t seed) {
  lamg::CycleConfig c;
  c.correction = correction ? lamg::CorrectionMode::AdaptiveRecombination : lamg::CorrectionMode::Flat;
  c.mu = mu;
  c.max_cycles = max_cycles;
  c.target_reduction = target_reduction;
  c.divergence_factor = divergence_factor;
  c.gamma = gamma;
  c.rng_seed = seed;
  return c;
}

void put_stats(bag* b, const lamg::SolveStats& s) {
  bag_put(b, "residuals", BAG_F64, s.residuals.data(), (int64_t)s.residuals.size());
  bag_put_f64(b, "acf", s.acf);
  bag_put_f64(b, "solve_work", s.solve_work);
  bag_put_i32(b, "cycles", s.cycles);
  bag_put_i32(b, "converged", s.converged ? 1 : 0);
  bag_put_i64(b, "recombinations", s.recombinations);
  bag_put_f64(b, "recomb_max_growth", s.recomb_max_growth);
}

void export_hierarchy(bag* b, const std::string& pfx, const lamg::Hierarchy& h) {
  bag_put_i32(b, (pfx + "nlevels").c_str(), (int32_t)h.levels.size());
  bag_put_f64(b, (pfx + "setup_work").c_str(), h.setup_work);
  bag_put_i32(b, (pfx + "nwarnings").c_str(), (int32_t)h.warnings.size());
  for (std::size_t l = 0; l < h.levels.size(); ++l) {
    const lamg::Level& L = h.levels[l];
    std::string p = pfx + "L" + std::to_string(l) + ".";
    bag_put_i32(b, (p + "kind").c_str(), (int32_t)L.kind);
    put_csr(b, p, L.op);
    bag_put_f64(b, (p + "gamma").c_str(), L.gamma);
    bag_put_i32(b, (p + "nu_pre").c_str(), L.nu_pre);
    bag_put_i32(b, (p + "nu_post").c_str(), L.nu_post);
    bag_put_i32(b, (p + "tv_count").c_str(), L.tv_count);
    bag_put_i32(b, (p + "coarsest").c_str(), (int32_t)L.coarsest);
    if (const auto* t = std::get_if<lamg::AggregationTransfer>(&L.transfer)) put_agg(b, p, *t);
    if (const auto* t = std::get_if<lamg::EliminationTransfer>(&L.transfer)) {
      bag_put_i32(b, (p + "nstages").c_str(), (int32_t)t->stages.size());
      for (std::size_t s = 0; s < t->stages.size(); ++s)
        put_stage(b, p + "S" + std::to_string(s) + ".", t->stages[s]);
    }
  }
}

}  // namespace

extern "C" {

int64_t ref_bag_len(const bag* b, const char* name) { return bag_len(b, name); }
int ref_bag_type(const bag* b, const char* name) { return bag_type(b, name); }
int ref_bag_get(const bag* b, const char* name, void* dst) { return bag_get(b, name, dst); }
int ref_bag_count(const bag* b) { return bag_count(b); }
const char* ref_bag_name(const bag* b, int i) { return bag_name(b, i); }
void ref_bag_free(bag* b) { bag_free(b); }
const char* ref_last_error(void) { return g_err.c_str(); }

uint64_t ref_rng_derive(uint64_t seed, uint64_t stream) { return lamg::Rng::derive(seed, stream); }

void ref_rng_draws(uint64_t seed, int64_t count, int kind, void* out) {
  lamg::Rng r(seed);
  for (int64_t i = 0; i < count; ++i) {
    if (kind == 0) ((uint64_t*)out)[i] = r.next_u64();
    else if (kind == 1) ((double*)out)[i] = r.next_unit();
    else ((double*)out)[i] = r.next_pm1();
  }
}

int ref_validate(CSR_ARGS) {
  return guarded([&] { lamg::validate_laplacian(make_csr(CSR_PASS)); });
}

int ref_mvm(CSR_ARGS, const double* x, double* y) {
  return guarded([&] {
    auto a = make_csr(CSR_PASS);
    lamg::mvm(a, std::span<const double>(x, n), std::span<double>(y, n));
  });
}

int ref_residual(CSR_ARGS, const double* b, const double* x, double* r) {
  return guarded([&] {
    auto a = make_csr(CSR_PASS);
    auto rr = lamg::residual(a, std::span<const double>(b, n), std::span<const double>(x, n));
    std::memcpy(r, rr.data(), sizeof(double) * n);
  });
}

int ref_energy(CSR_ARGS, const double* x, double* e) {
  return guarded([&] { *e = lamg::energy(make_csr(CSR_PASS), std::span<const double>(x, n)); });
}

int ref_vec_stats(int64_t len, const double* x, double* sum, double* norm2) {
  std::span<const double> s(x, (std::size_t)len);
  *sum = lamg::vec_sum(s);
  *norm2 = lamg::norm2(s);
  return ORC_OK;
}

int ref_subtract_mean(int64_t len, double* x) {
  lamg::subtract_mean(std::span<double>(x, (std::size_t)len));
  return ORC_OK;
}

int ref_gs_sweep(CSR_ARGS, const double* b, double* x, int backward) {
  return guarded([&] {
    auto a = make_csr(CSR_PASS);
    std::span<const double> bs = b ? std::span<const double>(b, n) : std::span<const double>();
    lamg::gauss_seidel_sweep(a, bs, std::span<double>(x, n),
                             backward ? lamg::SweepOrder::Backward : lamg::SweepOrder::Forward);
  });
}

int ref_generate_tvs(CSR_ARGS, int count, int sweeps, uint64_t seed, double* out) {
  return guarded([&] {
    auto t = lamg::generate_tvs(make_csr(CSR_PASS), count, sweeps, seed);
    for (int k = 0; k < count; ++k) std::memcpy(out + (int64_t)k * n, t.columns[k].data(), sizeof(double) * n);
  });
}

int ref_probe(CSR_ARGS, int sweeps, uint64_t seed, double* factor) {
  return guarded([&] { *factor = lamg::probe_relaxation(make_csr(CSR_PASS), sweeps, seed).factor; });
}

int ref_affinities(CSR_ARGS, int K, const double* tvs, bag** out) {
  *out = nullptr;
  return guarded([&] {
    auto v = lamg::compute_affinities(make_csr(CSR_PASS), make_tvs(n, K, tvs));
    bag* b = bag_new();
    bag_put(b, "edge_affinity", BAG_F64, v.edge_affinity.data(), (int64_t)v.edge_affinity.size());
    bag_put(b, "node_norm", BAG_F64, v.node_norm.data(), (int64_t)v.node_norm.size());
    bag_put(b, "degenerate", BAG_I32, v.degenerate.data(), (int64_t)v.degenerate.size());
    *out = b;
  });
}

int ref_detect_hubs(CSR_ARGS, bag** out) {
  *out = nullptr;
  return guarded([&] {
    auto h = lamg::detect_hubs(make_csr(CSR_PASS));
    bag* b = bag_new();
    bag_put(b, "hubs", BAG_I32, h.data(), (int64_t)h.size());
    *out = b;
  });
}

int ref_energy_ratio_qus(CSR_ARGS, int K, const double* tvs, int32_t u, int32_t s, double* q) {
  return guarded([&] { *q = lamg::energy_ratio_qus(make_csr(CSR_PASS), make_tvs(n, K, tvs), u, s); });
}

int ref_aggregate(CSR_ARGS, int K, const double* tvs, double gamma, const int32_t* hubs,
                  int32_t nhubs, bag** out) {
  *out = nullptr;
  return guarded([&] {
    auto t = lamg::aggregate(make_csr(CSR_PASS), make_tvs(n, K, tvs), gamma,
                             std::span<const lamg::Index>(hubs, (std::size_t)nhubs));
    bag* b = bag_new();
    put_agg(b, "", t);
    *out = b;
  });
}

int ref_galerkin(CSR_ARGS, const int32_t* aggregate_of, int32_t coarse_n, bag** out) {
  *out = nullptr;
  return guarded([&] {
    lamg::AggregationTransfer t;
    t.fine_n = n;
    t.coarse_n = coarse_n;
    t.aggregate_of.assign(aggregate_of, aggregate_of + n);
    auto c = lamg::galerkin_coarse_operator(make_csr(CSR_PASS), t);
    bag* b = bag_new();
    put_csr(b, "", c);
    *out = b;
  });
}

int ref_restrict_residual(const int32_t* aggregate_of, int32_t fine_n, int32_t coarse_n,
                          const double* r, double* rc) {
  return guarded([&] {
    lamg::AggregationTransfer t;
    t.fine_n = fine_n;
    t.coarse_n = coarse_n;
    t.aggregate_of.assign(aggregate_of, aggregate_of + fine_n);
    auto v = lamg::restrict_residual(t, std::span<const double>(r, fine_n));
    std::memcpy(rc, v.data(), sizeof(double) * coarse_n);
  });
}

int ref_add_interpolated(const int32_t* aggregate_of, int32_t fine_n, const double* ec, double* x) {
  return guarded([&] {
    lamg::AggregationTransfer t;
    t.fine_n = fine_n;
    t.aggregate_of.assign(aggregate_of, aggregate_of + fine_n);
    int32_t cn = 0;
    for (int32_t u = 0; u < fine_n; ++u) cn = std::max(cn, aggregate_of[u] + 1);
    t.coarse_n = cn;
    lamg::add_interpolated(t, std::span<const double>(ec, cn), std::span<double>(x, fine_n));
  });
}

int ref_select_low_degree(CSR_ARGS, int32_t max_degree, bag** out) {
  *out = nullptr;
  return guarded([&] {
    std::vector<lamg::Index> f, c;
    lamg::select_low_degree_set(make_csr(CSR_PASS), max_degree, f, c);
    bag* b = bag_new();
    bag_put(b, "f", BAG_I32, f.data(), (int64_t)f.size());
    bag_put(b, "c", BAG_I32, c.data(), (int64_t)c.size());
    *out = b;
  });
}

int ref_schur(CSR_ARGS, const int32_t* f, int32_t nf, const int32_t* c, int32_t nc, bag** out) {
  *out = nullptr;
  return guarded([&] {
    auto [coarse, stage] = lamg::schur_reduce(make_csr(CSR_PASS),
                                              std::span<const lamg::Index>(f, (std::size_t)nf),
                                              std::span<const lamg::Index>(c, (std::size_t)nc));
    bag* b = bag_new();
    put_csr(b, "", coarse);
    put_stage(b, "S.", stage);
    *out = b;
  });
}

int ref_eliminate_rounds(CSR_ARGS, bag** out) {
  *out = nullptr;
  return guarded([&] {
    auto t = lamg::eliminate_rounds(make_csr(CSR_PASS));
    bag* b = bag_new();
    bag_put_i32(b, "nstages", t ? (int32_t)t->stages.size() : 0);
    if (t) {
      put_csr(b, "", t->coarse_op);
      for (std::size_t s = 0; s < t->stages.size(); ++s) put_stage(b, "S" + std::to_string(s) + ".", t->stages[s]);
    }
    *out = b;
  });
}

int ref_coarsen_rhs_stage(STAGE_ARGS, const double* b, double* bc) {
  return guarded([&] {
    auto s = make_stage(parent_n, coarse_n, nf, f_nodes, f_diag, f_ptr, f_nbr, f_val,
                        coarse_of_parent, parent_of_coarse);
    auto v = lamg::coarsen_rhs_elim(s, std::span<const double>(b, parent_n));
    std::memcpy(bc, v.data(), sizeof(double) * coarse_n);
  });
}

int ref_backsub_stage(STAGE_ARGS, const double* xc, const double* b, double* x) {
  return guarded([&] {
    auto s = make_stage(parent_n, coarse_n, nf, f_nodes, f_diag, f_ptr, f_nbr, f_val,
                        coarse_of_parent, parent_of_coarse);
    auto v = lamg::backsubstitute_elim(s, std::span<const double>(xc, coarse_n),
                                       std::span<const double>(b, parent_n));
    std::memcpy(x, v.data(), sizeof(double) * parent_n);
  });
}

int ref_coarsest_direct(CSR_ARGS, const double* b, double* x) {
  return guarded([&] {
    auto s = lamg::CoarsestSolver::make_direct(make_csr(CSR_PASS));
    s->solve(std::span<const double>(b, n), std::span<double>(x, n));
  });
}

int ref_coarsest_relax(CSR_ARGS, const double* b, double* x) {
  return guarded([&] {
    auto s = lamg::CoarsestSolver::make_relaxation(make_csr(CSR_PASS));
    s->solve(std::span<const double>(b, n), std::span<double>(x, n));
  });
}

double ref_flat_mu(double q) { return lamg::flat_mu(q); }

int ref_credit_takes(double gamma, int count, int32_t* out) {
  lamg::LevelCredit c;
  for (int i = 0; i < count; ++i) out[i] = c.take(0, gamma);
  return ORC_OK;
}

int ref_recombine(CSR_ARGS, const double* b, int cols, const double* saved_x,
                  const double* saved_r, double* x, double* before, double* after) {
  return guarded([&] {
    auto a = make_csr(CSR_PASS);
    std::vector<lamg::Vector> sx, sr;
    for (int i = 0; i < cols; ++i) {
      sx.emplace_back(saved_x + (int64_t)i * n, saved_x + (int64_t)(i + 1) * n);
      sr.emplace_back(saved_r + (int64_t)i * n, saved_r + (int64_t)(i + 1) * n);
    }
    *after = lamg::recombine(a, std::span<const double>(b, n), sx, sr, std::span<double>(x, n), before);
  });
}

void* ref_setup(CSR_ARGS, double gamma, uint64_t seed, int32_t coarsest_n, int tv_sweeps,
                int tv_count_finest, int tv_count_max) {
  lamg::Hierarchy* out = nullptr;
  g_setup_status = guarded([&] {
    lamg::SetupOptions o;
    o.gamma = gamma;
    o.rng_seed = seed;
    o.coarsest_n = coarsest_n;
    o.tv_sweeps = tv_sweeps;
    o.tv_count_finest = tv_count_finest;
    o.tv_count_max = tv_count_max;
    lamg::work::reset();  // work is a thread-local running total: start each driver call at 0
    out = new lamg::Hierarchy(lamg::setup(make_csr(CSR_PASS), o));
  });
  return out;
}

int ref_setup_status(void) { return g_setup_status; }

int ref_hier_export(void* h, bag** out) {
  bag* b = bag_new();
  export_hierarchy(b, "", *(lamg::Hierarchy*)h);
  *out = b;
  return ORC_OK;
}

double ref_level_cycle_index(void* h, int32_t l, double gamma) {
  return lamg::level_cycle_index(*(lamg::Hierarchy*)h, (std::size_t)l, gamma);
}

int ref_solve(void* h, const double* b, const double* x0, int correction, double mu,
              int max_cycles, double target_reduction, double divergence_factor, double gamma,
              uint64_t seed, double* x, bag** stats) {
  auto* H = (lamg::Hierarchy*)h;
  int32_t n = H->finest_n();
  bag* sb = bag_new();
  *stats = sb;
  try {
    auto cfg = make_cfg(correction, mu, max_cycles, target_reduction, divergence_factor, gamma, seed);
    lamg::work::reset();
    auto [xv, st] = lamg::solve(*H, std::span<const double>(b, n), std::span<const double>(x0, n), cfg);
    std::memcpy(x, xv.data(), sizeof(double) * n);
    put_stats(sb, st);
    g_err.clear();
    return ORC_OK;
  } catch (const lamg::DivergedError& e) {
    put_stats(sb, e.stats);
    return fail(ORC_E_DIVERGED, e.what());
  } catch (...) {
    return guarded([] { throw; });
  }
}

void ref_hier_free(void* h) { delete (lamg::Hierarchy*)h; }

void* ref_prepare(CSR_ARGS, double gamma, uint64_t seed, int32_t coarsest_n, int tv_sweeps,
                  int tv_count_finest, int tv_count_max, int correction, double mu,
                  int max_cycles, double target_reduction, double divergence_factor,
                  double cycle_gamma, uint64_t cycle_seed) {
  lamg::Prepared* out = nullptr;
  g_setup_status = guarded([&] {
    lamg::SolverOptions o;
    o.setup.gamma = gamma;
    o.setup.rng_seed = seed;
    o.setup.coarsest_n = coarsest_n;
    o.setup.tv_sweeps = tv_sweeps;
    o.setup.tv_count_finest = tv_count_finest;
    o.setup.tv_count_max = tv_count_max;
    o.cycle = make_cfg(correction, mu, max_cycles, target_reduction, divergence_factor, cycle_gamma, cycle_seed);
    lamg::work::reset();
    out = new lamg::Prepared(lamg::prepare(make_csr(CSR_PASS), o));
  });
  return out;
}

int ref_prepared_export(void* p, bag** out) {
  auto* P = (lamg::Prepared*)p;
  bag* b = bag_new();
  bag_put_i32(b, "ncomponents", (int32_t)P->components.size());
  bag_put_f64(b, "setup_work", P->setup_work);
  for (std::size_t c = 0; c < P->components.size(); ++c) {
    std::string p = "C" + std::to_string(c) + ".";
    const auto& run = P->components[c];
    bag_put(b, (p + "nodes").c_str(), BAG_I32, run.nodes.data(), (int64_t)run.nodes.size());
    if (run.nodes.size() > 1) export_hierarchy(b, p, run.hierarchy);
  }
  *out = b;
  return ORC_OK;
}

int ref_solve_prepared(void* p, const double* b, const double* x0, double* x, bag** report) {
  auto* P = (lamg::Prepared*)p;
  int32_t n = P->a.n;
  bag* rb = bag_new();
  *report = rb;
  return guarded([&] {
    std::span<const double> xs = x0 ? std::span<const double>(x0, n) : std::span<const double>();
    lamg::work::reset();
    auto r = lamg::solve_prepared(*P, std::span<const double>(b, n), xs);
    std::memcpy(x, r.x.data(), sizeof(double) * n);
    put_stats(rb, r.stats);
    bag_put_f64(rb, "total_solve_work", r.solve_work);
    bag_put_i32(rb, "all_converged", r.converged ? 1 : 0);
    bag_put_f64(rb, "reduction", r.reduction);
  });
}

void ref_prepared_free(void* p) { delete (lamg::Prepared*)p; }

int ref_solve_batch(void* h, int nrhs, const double* B, const double* X0, int correction,
                    double mu, int max_cycles, double target_reduction, double divergence_factor,
                    double gamma, uint64_t seed, int nthreads, double* seconds, int32_t* cycles) {
  auto* H = (lamg::Hierarchy*)h;
  const int64_t n = H->finest_n();
  auto cfg = make_cfg(correction, mu, max_cycles, target_reduction, divergence_factor, gamma, seed);
  std::vector<int> status(nrhs, 0);
  auto worker = [&](int t) {
    for (int i = t; i < nrhs; i += nthreads) {
      try {
        auto [xv, st] = lamg::solve(*H, std::span<const double>(B + i * n, n),
                                    std::span<const double>(X0 + i * n, n), cfg);
        cycles[i] = st.cycles;
      } catch (...) {
        status[i] = 1;
        cycles[i] = -1;
      }
    }
  };
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 1; t < nthreads; ++t) pool.emplace_back(worker, t);
  worker(0);
  for (auto& th : pool) th.join();
  *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  for (int s : status)
    if (s) return fail(ORC_E_ERROR, "solve_batch: a solve failed");
  return ORC_OK;
}

// Reference generators and assembly, used only to pin the numpy input
// builders in paper_1108_1310_b200/graphs.py (generators.cpp:19-127,
// sparse_laplacian.cpp:106-135).
int ref_gen(const char* name, int32_t p0, double p1, double p2, int32_t p3, bag** out) {
  *out = nullptr;
  return guarded([&] {
    std::string g(name);
    lamg::SparseLaplacian a;
    if (g == "grid_5pt") a = lamg::gen::grid_5pt(p0);
    else if (g == "grid_13pt_4th") a = lamg::gen::grid_13pt_4th(p0);
    else if (g == "grid_anis_rotated")
      a = lamg::gen::grid_anis_rotated(p0, p1, p2, p3 ? lamg::gen::CrossAlignment::Northeast
                                                     : lamg::gen::CrossAlignment::Agnostic);
    else if (g == "path") a = lamg::gen::path(p0);
    else if (g == "star") a = lamg::gen::star(p0);
    else if (g == "complete") a = lamg::gen::complete(p0);
    else if (g == "two_hubs") a = lamg::gen::two_hubs(p0);
    else if (g == "binary_tree") a = lamg::gen::binary_tree(p0);
    else throw lamg::Error("unknown generator " + g);
    bag* b = bag_new();
    put_csr(b, "", a);
    *out = b;
  });
}

int ref_assemble(int32_t n, int64_t ne, const int32_t* u, const int32_t* v, const double* w,
                 bag** out) {
  *out = nullptr;
  return guarded([&] {
    lamg::EdgeList el;
    el.n = n;
    for (int64_t i = 0; i < ne; ++i) el.edges.push_back({u[i], v[i], w[i]});
    auto a = lamg::assemble_laplacian(el);
    bag* b = bag_new();
    put_csr(b, "", a);
    *out = b;
  });
}

}  // extern "C"
