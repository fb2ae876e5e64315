// include/lamg_b200/lamg.hpp -- drop-in C++ facade over liblamg_b200.so.
//
// Re-exposes the reference LAMG C++ API (/root/reference/proj/core/include/
// lamg/*.hpp) with the same names, types and signatures, implemented on the
// C-ABI in include/lamg_b200.h. Existing host code keeps calling
//
//   lamg::Hierarchy h = lamg::setup(a, opts);                  // hierarchy.hpp:65
//   auto [x, stats]   = lamg::solve(h, b, x0, cfg);            // cycle.hpp:58-59
//   lamg::Prepared p  = lamg::prepare(a, solver_opts);         // solver.hpp:36
//   lamg::SolveReport r = lamg::solve_prepared(p, b, x0);      // solver.hpp:49-50
//
// and the setup and solve run on the GPU. Failures raise the reference's
// exception types with the reference's message text. The default execution
// mode is VALIDATE (bit-identical to the reference); lamg::b200::set_mode
// selects THROUGHPUT (coloured Gauss-Seidel smoother, same hierarchy).
// The hierarchy stays in HBM: Level::op, Level::transfer and
// Level::coarsest_solver are views whose arrays are downloaded on first use
// (n, m and every scalar are known at once), so setup() moves no operator to
// the host. Header-only: include it and link -llamg_b200.
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <functional>
#include <limits>
#include <memory>
#include <mutex>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <variant>
#include <vector>

#include "lamg_b200.h"

namespace lamg {

using Index = std::int32_t;
using EntryCount = std::int64_t;
using Real = double;
using Vector = std::vector<Real>;

// ---- errors.hpp:8-42 ----------------------------------------------------
struct Error : std::runtime_error {
  explicit Error(const std::string& what) : std::runtime_error(what) {}
};
struct EmptyGraphError : Error { using Error::Error; };
struct SingularDiagonalError : Error { using Error::Error; };
struct InvalidLaplacianError : Error { using Error::Error; };
struct DimensionMismatchError : Error { using Error::Error; };
struct IncompatibleRhsError : Error { using Error::Error; };
struct ParseError : Error { using Error::Error; };
struct IoError : Error { using Error::Error; };

// ---- sparse_laplacian.hpp:18-39 -----------------------------------------
struct SparseLaplacian {
  Index n = 0;
  EntryCount m = 0;
  std::vector<EntryCount> row_ptr;
  std::vector<Index> col;
  std::vector<Real> val;
  std::vector<Real> diag;
  Index degree(Index u) const { return static_cast<Index>(row_ptr[u + 1] - row_ptr[u]); }
};

// ---- hierarchy.hpp ------------------------------------------------------
enum class LevelKind { Finest, Elimination, Aggregation, Coarsest };
enum class CoarsestMode { None, Direct, Relaxation };

struct SetupOptions {
  double gamma = 1.5;
  std::uint64_t rng_seed = 1;
  Index coarsest_n = 150;
  int tv_sweeps = 3;
  int tv_count_finest = 4;
  int tv_count_max = 10;
};

namespace b200 {
// A device array of the hierarchy, downloaded (once, thread-safely) on first
// use; reads like the reference's std::vector member it stands in for.
template <class T>
class LazyArray {
 public:
  LazyArray() = default;
  explicit LazyArray(std::function<const std::vector<T>&()> get) : get_(std::move(get)) {}
  const std::vector<T>& vec() const { return get_ ? get_() : own_; }
  operator const std::vector<T>&() const { return vec(); }
  const T& operator[](std::size_t i) const { return vec()[i]; }
  std::size_t size() const { return vec().size(); }
  bool empty() const { return vec().empty(); }
  const T* data() const { return vec().data(); }
  auto begin() const { return vec().begin(); }
  auto end() const { return vec().end(); }
  bool operator==(const std::vector<T>& o) const { return vec() == o; }

 private:
  std::function<const std::vector<T>&()> get_;
  std::vector<T> own_;
};

// a group of arrays filled by one download
template <class D>
struct Lazy {
  std::once_flag once;
  std::function<void(D&)> load;
  D data;
  const D& get() {
    std::call_once(once, [this] { load(data); });
    return data;
  }
};
}  // namespace b200

// Level::op: sparse_laplacian.hpp's fields, arrays fetched from HBM on first use
struct LevelOperator {
  Index n = 0;
  EntryCount m = 0;
  b200::LazyArray<EntryCount> row_ptr;
  b200::LazyArray<Index> col;
  b200::LazyArray<Real> val;
  b200::LazyArray<Real> diag;
  std::shared_ptr<b200::Lazy<SparseLaplacian>> src;
  Index degree(Index u) const { return static_cast<Index>(row_ptr[u + 1] - row_ptr[u]); }
  const SparseLaplacian& laplacian() const { return src->get(); }
  operator const SparseLaplacian&() const { return laplacian(); }
};

// elimination.hpp:16-31
struct ElimStage {
  Index parent_n = 0;
  Index coarse_n = 0;
  b200::LazyArray<Index> f_nodes;
  b200::LazyArray<Real> f_diag;
  b200::LazyArray<EntryCount> f_ptr;
  b200::LazyArray<Index> f_nbr;
  b200::LazyArray<Real> f_val;
  b200::LazyArray<Index> coarse_of_parent;
  b200::LazyArray<Index> parent_of_coarse;
};
struct EliminationTransfer {
  std::vector<ElimStage> stages;
  LevelOperator coarse_op;  // the eliminated level's operator (the same device arrays as Level::op)
};

// aggregation.hpp:36-44
struct AggregationTransfer {
  Index fine_n = 0;
  Index coarse_n = 0;
  b200::LazyArray<Index> aggregate_of;
  b200::LazyArray<Index> seed_of;
  int stage_used = 0;
  double alpha = 1.0;
  Index dummy_aggregate = -1;
};

// coarse_solver.hpp:15-24 -- the coarsest-level solvers run on the GPU
// (direct: bordered LU per component; relaxation: Gauss-Seidel to 1e-12)
class CoarsestSolver {
 public:
  static std::shared_ptr<const CoarsestSolver> make_direct(const SparseLaplacian& a);
  static std::shared_ptr<const CoarsestSolver> make_relaxation(const SparseLaplacian& a);
  virtual ~CoarsestSolver() = default;
  virtual void solve(std::span<const Real> b, std::span<Real> x) const = 0;
};

// hierarchy.hpp:24-37
struct Level {
  LevelKind kind = LevelKind::Finest;
  LevelOperator op;  // device-resident; arrays downloaded on first use
  std::variant<std::monostate, EliminationTransfer, AggregationTransfer> transfer;
  double gamma = 1.0;
  int nu_pre = 0;
  int nu_post = 0;
  int tv_count = 0;
  CoarsestMode coarsest = CoarsestMode::None;
  std::shared_ptr<const CoarsestSolver> coarsest_solver;
  bool is_elimination() const { return kind == LevelKind::Elimination; }
  bool is_aggregation() const { return kind == LevelKind::Aggregation; }
};

struct Hierarchy {
  std::vector<Level> levels;
  double setup_work = 0.0;
  std::uint64_t seed = 0;
  std::vector<std::string> warnings;
  std::shared_ptr<lamg_hier> device;  // the GPU-resident hierarchy

  Index finest_n() const { return levels.front().op.n; }
  EntryCount finest_m() const { return levels.front().op.m; }
  EntryCount total_stored_edges() const {
    EntryCount t = 0;
    for (const auto& l : levels) t += l.op.m;
    return t;
  }
  double storage_per_edge() const {
    double t = 0.0;
    for (const auto& l : levels) t += 2.0 * static_cast<double>(l.op.m) + static_cast<double>(l.op.n);
    return t / static_cast<double>(finest_m());
  }
  double edge_ratio() const {
    return static_cast<double>(total_stored_edges()) / static_cast<double>(finest_m());
  }
};

struct LevelStats {
  int level = 0;
  std::string kind;
  bool coarsest = false;
  Index n = 0;
  EntryCount m = 0;
  double gamma = 0.0;
  int nu_pre = 0;
  int nu_post = 0;
  int tv_count = 0;
};
struct HierarchyStats {
  std::vector<LevelStats> levels;
  double edge_ratio = 0.0;
  double storage_per_edge = 0.0;
  double setup_work = 0.0;
};

// ---- cycle.hpp ----------------------------------------------------------
enum class CorrectionMode { Flat, AdaptiveRecombination };

struct CycleConfig {
  double gamma = 1.5;
  CorrectionMode correction = CorrectionMode::Flat;
  double mu = 4.0 / 3.0;
  int max_cycles = 300;
  double target_reduction = 1e10;
  double divergence_factor = 1e3;
  std::uint64_t rng_seed = 1;
};

struct SolveStats {
  std::vector<double> residuals;
  double acf = 0.0;
  double solve_work = 0.0;
  int cycles = 0;
  bool converged = false;
  std::int64_t recombinations = 0;
  double recomb_max_growth = 0.0;
};

struct DivergedError : Error {
  SolveStats stats;
  DivergedError(const std::string& what, SolveStats s) : Error(what), stats(std::move(s)) {}
};

inline double flat_mu(double q) { return lamg_flat_mu(q); }

// ---- device context (one per host thread) --------------------------------
namespace b200 {

inline int& mode_ref() {
  static thread_local int mode = LAMG_MODE_VALIDATE;
  return mode;
}

inline lamg_ctx* context() {
  struct Holder {
    lamg_ctx* p = nullptr;
    ~Holder() { lamg_ctx_destroy(p); }
  };
  static thread_local Holder h;
  if (!h.p) {
    if (lamg_ctx_create(0, mode_ref(), &h.p) != LAMG_OK) throw Error(lamg_last_error());
  }
  return h.p;
}

// selects VALIDATE (bit-identical to the reference) or THROUGHPUT
inline void set_mode(int mode) {
  mode_ref() = mode;
  if (lamg_ctx_set_mode(context(), mode) != LAMG_OK) throw Error(lamg_last_error());
}

[[noreturn]] inline void raise(int code) {
  std::string msg = lamg_last_error();
  switch (code) {
    case LAMG_E_EMPTY_GRAPH: throw EmptyGraphError(msg);
    case LAMG_E_SINGULAR_DIAGONAL: throw SingularDiagonalError(msg);
    case LAMG_E_INVALID_LAPLACIAN: throw InvalidLaplacianError(msg);
    case LAMG_E_DIMENSION_MISMATCH: throw DimensionMismatchError(msg);
    case LAMG_E_INCOMPATIBLE_RHS: throw IncompatibleRhsError(msg);
    case LAMG_E_PARSE: throw ParseError(msg);
    case LAMG_E_IO: throw IoError(msg);
    default: throw Error(msg);
  }
}
inline void check(int code) {
  if (code != LAMG_OK) raise(code);
}

inline lamg_csr view(const SparseLaplacian& a) {
  return lamg_csr{a.n, a.m, a.row_ptr.data(), a.col.data(), a.val.data(), a.diag.data()};
}

}  // namespace b200

namespace b200 {
inline LevelOperator level_operator(std::shared_ptr<lamg_hier> dev, int32_t l, Index n, EntryCount m) {
  LevelOperator op;
  op.n = n;
  op.m = m;
  auto src = std::make_shared<Lazy<SparseLaplacian>>();
  src->load = [dev, l, n, m](SparseLaplacian& a) {
    a.n = n;
    a.m = m;
    a.row_ptr.resize(static_cast<std::size_t>(n) + 1);
    a.col.resize(static_cast<std::size_t>(2 * m));
    a.val.resize(static_cast<std::size_t>(2 * m));
    a.diag.resize(static_cast<std::size_t>(n));
    check(lamg_hier_download_op(dev.get(), l, a.row_ptr.data(), a.col.data(), a.val.data(), a.diag.data()));
  };
  op.src = src;
  op.row_ptr = LazyArray<EntryCount>([src]() -> const std::vector<EntryCount>& { return src->get().row_ptr; });
  op.col = LazyArray<Index>([src]() -> const std::vector<Index>& { return src->get().col; });
  op.val = LazyArray<Real>([src]() -> const std::vector<Real>& { return src->get().val; });
  op.diag = LazyArray<Real>([src]() -> const std::vector<Real>& { return src->get().diag; });
  return op;
}

inline ElimStage elim_stage(std::shared_ptr<lamg_hier> dev, int32_t l, int32_t s) {
  ElimStage st;
  int32_t pn = 0, cn = 0, nf = 0;
  int64_t nnz = 0;
  check(lamg_hier_stage_info(dev.get(), l, s, &pn, &cn, &nf, &nnz));
  st.parent_n = pn;
  st.coarse_n = cn;
  struct D {
    std::vector<Index> f_nodes, f_nbr, cop, poc;
    std::vector<Real> f_diag, f_val;
    std::vector<EntryCount> f_ptr;
  };
  auto src = std::make_shared<Lazy<D>>();
  src->load = [dev, l, s, pn, cn, nf, nnz](D& d) {
    d.f_nodes.resize(nf);
    d.f_diag.resize(nf);
    d.f_ptr.resize(static_cast<std::size_t>(nf) + 1);
    d.f_nbr.resize(static_cast<std::size_t>(nnz));
    d.f_val.resize(static_cast<std::size_t>(nnz));
    d.cop.resize(pn);
    d.poc.resize(cn);
    check(lamg_hier_download_stage(dev.get(), l, s, d.f_nodes.data(), d.f_diag.data(), d.f_ptr.data(),
                                   d.f_nbr.data(), d.f_val.data(), d.cop.data(), d.poc.data()));
  };
  st.f_nodes = LazyArray<Index>([src]() -> const std::vector<Index>& { return src->get().f_nodes; });
  st.f_diag = LazyArray<Real>([src]() -> const std::vector<Real>& { return src->get().f_diag; });
  st.f_ptr = LazyArray<EntryCount>([src]() -> const std::vector<EntryCount>& { return src->get().f_ptr; });
  st.f_nbr = LazyArray<Index>([src]() -> const std::vector<Index>& { return src->get().f_nbr; });
  st.f_val = LazyArray<Real>([src]() -> const std::vector<Real>& { return src->get().f_val; });
  st.coarse_of_parent = LazyArray<Index>([src]() -> const std::vector<Index>& { return src->get().cop; });
  st.parent_of_coarse = LazyArray<Index>([src]() -> const std::vector<Index>& { return src->get().poc; });
  return st;
}

// coarse_solver.cpp:26-98 through lamg_k_coarsest_direct / lamg_k_coarsest_relax
class DeviceCoarsest final : public CoarsestSolver {
 public:
  DeviceCoarsest(std::function<const SparseLaplacian&()> op, bool direct) : op_(std::move(op)), direct_(direct) {}
  void solve(std::span<const Real> b, std::span<Real> x) const override {
    const SparseLaplacian& a = op_();
    if (b.size() != static_cast<std::size_t>(a.n) || x.size() != static_cast<std::size_t>(a.n))
      throw DimensionMismatchError("coarsest solve: vector length does not match the level");
    const lamg_csr v = view(a);
    check(direct_ ? lamg_k_coarsest_direct(context(), &v, b.data(), x.data())
                  : lamg_k_coarsest_relax(context(), &v, b.data(), x.data()));
  }

 private:
  std::function<const SparseLaplacian&()> op_;
  bool direct_;
};

inline std::shared_ptr<const CoarsestSolver> level_coarsest(const LevelOperator& op, CoarsestMode mode) {
  auto src = op.src;
  return std::make_shared<DeviceCoarsest>([src]() -> const SparseLaplacian& { return src->get(); },
                                          mode == CoarsestMode::Direct);
}
}  // namespace b200

inline std::shared_ptr<const CoarsestSolver> CoarsestSolver::make_direct(const SparseLaplacian& a) {
  auto own = std::make_shared<SparseLaplacian>(a);
  return std::make_shared<b200::DeviceCoarsest>([own]() -> const SparseLaplacian& { return *own; }, true);
}
inline std::shared_ptr<const CoarsestSolver> CoarsestSolver::make_relaxation(const SparseLaplacian& a) {
  auto own = std::make_shared<SparseLaplacian>(a);
  return std::make_shared<b200::DeviceCoarsest>([own]() -> const SparseLaplacian& { return *own; }, false);
}

// hierarchy.hpp:65 -- lamg::setup on the GPU
inline Hierarchy setup(const SparseLaplacian& a, const SetupOptions& opts = {}) {
  lamg_ctx* ctx = b200::context();
  lamg_setup_opts o{opts.gamma, opts.rng_seed, opts.coarsest_n, opts.tv_sweeps, opts.tv_count_finest,
                    opts.tv_count_max};
  lamg_csr v = b200::view(a);
  lamg_hier* raw = nullptr;
  b200::check(lamg_setup(ctx, &v, 0, &o, &raw));
  Hierarchy h;
  h.device = std::shared_ptr<lamg_hier>(raw, lamg_hier_destroy);
  h.seed = opts.rng_seed;
  int32_t nl = 0, nw = 0;
  double secs = 0.0;
  b200::check(lamg_hier_info(raw, &nl, &h.setup_work, &nw, &secs));
  for (int32_t i = 0; i < nw; ++i) {
    char buf[512];
    b200::check(lamg_hier_warning(raw, i, buf, sizeof buf));
    h.warnings.emplace_back(buf);
  }
  std::shared_ptr<lamg_hier> dev = h.device;
  for (int32_t l = 0; l < nl; ++l) {
    lamg_level_info li;
    b200::check(lamg_hier_level_info(raw, l, &li));
    Level L;
    L.kind = static_cast<LevelKind>(li.kind);
    L.gamma = li.gamma;
    L.nu_pre = li.nu_pre;
    L.nu_post = li.nu_post;
    L.tv_count = li.tv_count;
    L.coarsest = static_cast<CoarsestMode>(li.coarsest);
    L.op = b200::level_operator(dev, l, li.n, li.m);
    if (L.kind == LevelKind::Aggregation) {
      AggregationTransfer t;
      t.fine_n = h.levels.back().op.n;
      t.coarse_n = li.n;
      t.stage_used = li.stage_used;
      t.alpha = li.alpha;
      t.dummy_aggregate = li.dummy_aggregate;
      struct Agg {
        std::vector<Index> aggregate_of, seed_of;
      };
      auto src = std::make_shared<b200::Lazy<Agg>>();
      const Index fn = t.fine_n, cn = li.n;
      src->load = [dev, l, fn, cn](Agg& d) {
        d.aggregate_of.resize(static_cast<std::size_t>(fn));
        d.seed_of.resize(static_cast<std::size_t>(cn));
        b200::check(lamg_hier_download_agg(dev.get(), l, d.aggregate_of.data(), d.seed_of.data()));
      };
      t.aggregate_of = b200::LazyArray<Index>([src]() -> const std::vector<Index>& { return src->get().aggregate_of; });
      t.seed_of = b200::LazyArray<Index>([src]() -> const std::vector<Index>& { return src->get().seed_of; });
      L.transfer = std::move(t);
    } else if (L.kind == LevelKind::Elimination) {
      EliminationTransfer t;
      for (int32_t s = 0; s < li.nstages; ++s) t.stages.push_back(b200::elim_stage(dev, l, s));
      t.coarse_op = L.op;
      L.transfer = std::move(t);
    }
    if (L.coarsest != CoarsestMode::None) L.coarsest_solver = b200::level_coarsest(L.op, L.coarsest);
    h.levels.push_back(std::move(L));
  }
  return h;
}

// hierarchy.hpp:91 / hierarchy.cpp:31-40
inline double level_cycle_index(const Hierarchy& h, std::size_t l, double gamma) {
  double out = 0.0;
  b200::check(lamg_level_cycle_index(h.device.get(), static_cast<int32_t>(l), gamma, &out));
  return out;
}

// hierarchy.cpp:140-168
inline HierarchyStats hierarchy_stats(const Hierarchy& h) {
  HierarchyStats s;
  for (std::size_t l = 0; l < h.levels.size(); ++l) {
    const Level& L = h.levels[l];
    LevelStats ls;
    ls.level = static_cast<int>(l) + 1;
    ls.coarsest = L.coarsest != CoarsestMode::None;
    switch (L.kind) {
      case LevelKind::Finest: ls.kind = ls.coarsest ? "coarsest" : "finest"; break;
      case LevelKind::Elimination: ls.kind = "elimination"; break;
      case LevelKind::Aggregation: ls.kind = "aggregation"; break;
      case LevelKind::Coarsest: ls.kind = "coarsest"; break;
    }
    ls.n = L.op.n;
    ls.m = L.op.m;
    ls.gamma = l + 1 < h.levels.size() ? h.levels[l + 1].gamma : 0.0;
    if (l + 1 < h.levels.size()) {
      ls.nu_pre = h.levels[l + 1].is_aggregation() ? 1 : 0;
      ls.nu_post = h.levels[l + 1].is_aggregation() ? 2 : 0;
    }
    ls.tv_count = L.tv_count;
    s.levels.push_back(std::move(ls));
  }
  s.edge_ratio = h.edge_ratio();
  s.storage_per_edge = h.storage_per_edge();
  s.setup_work = h.setup_work;
  return s;
}

// cycle.hpp:58-59 -- lamg::solve on the GPU
inline std::pair<Vector, SolveStats> solve(const Hierarchy& h, std::span<const Real> b,
                                           std::span<const Real> x0, const CycleConfig& cfg = {}) {
  const auto n = static_cast<std::size_t>(h.finest_n());
  if (b.size() != n || x0.size() != n)
    throw DimensionMismatchError("solve: vector length does not match the finest level");
  lamg_cycle_cfg c{cfg.gamma, cfg.correction == CorrectionMode::AdaptiveRecombination ? 1 : 0, cfg.mu,
                   cfg.max_cycles, cfg.target_reduction, cfg.divergence_factor, cfg.rng_seed};
  Vector x(n);
  lamg_solve_stats st{};
  std::vector<double> res(static_cast<std::size_t>(std::max(cfg.max_cycles, 0)) + 2);
  int rc = lamg_solve(b200::context(), h.device.get(), b.data(), x0.data(), &c, x.data(), &st, res.data(),
                      static_cast<int32_t>(res.size()));
  SolveStats s;
  s.residuals.assign(res.begin(), res.begin() + std::min<std::size_t>(res.size(), st.nresiduals));
  s.acf = st.acf;
  s.solve_work = st.solve_work;
  s.cycles = st.cycles;
  s.converged = st.converged != 0;
  s.recombinations = st.recombinations;
  s.recomb_max_growth = st.recomb_max_growth;
  if (rc == LAMG_E_DIVERGED) throw DivergedError(lamg_last_error(), std::move(s));
  b200::check(rc);
  return {std::move(x), std::move(s)};
}

// cycle.hpp:61-67 -- residual-minimizing recombination of one or two saved
// iterates (cycle.cpp:23-103) on the GPU; returns ||b - A y||
inline Real recombine(const SparseLaplacian& a, std::span<const Real> b, std::span<const Vector> saved_x,
                      std::span<const Vector> saved_r, std::span<Real> x, Real* before = nullptr) {
  const auto n = static_cast<std::size_t>(a.n);
  const std::size_t cols = saved_x.size();
  if (cols != saved_r.size() || b.size() != n || x.size() != n)
    throw DimensionMismatchError("recombine: vector lengths do not match the matrix");
  if (cols == 0) {  // nothing saved: the residual of x itself
    std::vector<Real> y(n);
    const lamg_csr v = b200::view(a);
    b200::check(lamg_k_residual(b200::context(), &v, b.data(), x.data(), y.data()));
    double s = 0.0;
    for (double r : y) s += r * r;
    if (before) *before = std::sqrt(s);
    return std::sqrt(s);
  }
  std::vector<Real> sx(cols * n), sr(cols * n);
  for (std::size_t i = 0; i < cols; ++i) {
    if (saved_x[i].size() != n || saved_r[i].size() != n)
      throw DimensionMismatchError("recombine: vector lengths do not match the matrix");
    std::copy(saved_x[i].begin(), saved_x[i].end(), sx.begin() + i * n);
    std::copy(saved_r[i].begin(), saved_r[i].end(), sr.begin() + i * n);
  }
  const lamg_csr v = b200::view(a);
  double bf = 0.0, af = 0.0;
  b200::check(lamg_k_recombine(b200::context(), &v, b.data(), static_cast<int32_t>(cols), sx.data(), sr.data(),
                               x.data(), &bf, &af));
  if (before) *before = bf;
  return af;
}

// cycle.hpp:69-74 / cycle.cpp:14-21 (host bookkeeping of the visit schedule)
struct LevelCredit {
  std::vector<double> credit;
  int take(std::size_t level, double gamma) {
    if (credit.size() <= level) credit.resize(level + 1, 0.0);
    credit[level] += gamma;
    int theta = std::max(1, static_cast<int>(std::floor(credit[level])));
    credit[level] -= theta;
    if (credit[level] < 0.0) credit[level] = 0.0;
    return theta;
  }
};

// ---- solver.hpp: whole-problem driver (components split on the host, as
// the reference's L3 driver does; every component is set up and solved on
// the GPU) --------------------------------------------------------------------
struct SolverOptions {
  SetupOptions setup;
  CycleConfig cycle;
};

struct ComponentRun {
  std::vector<Index> nodes;
  Hierarchy hierarchy;
};

struct Prepared {
  SparseLaplacian a;
  CycleConfig cycle;
  std::vector<ComponentRun> components;
  double setup_work = 0.0;
  double setup_seconds = 0.0;
  std::vector<std::string> warnings;
  // solver.cpp:23-29: the component with the most nodes (the first on ties)
  const Hierarchy& largest() const {
    std::size_t best = 0;
    for (std::size_t i = 1; i < components.size(); ++i)
      if (components[i].nodes.size() > components[best].nodes.size()) best = i;
    return components[best].hierarchy;
  }
};

struct SolveReport {
  Vector x;
  SolveStats stats;
  double solve_work = 0.0;
  double solve_seconds = 0.0;
  bool converged = false;
  double reduction = 0.0;
};

namespace b200 {
// splitmix64 draws of lamg::Rng (rng.hpp:10-41)
struct Rng {
  std::uint64_t s;
  explicit Rng(std::uint64_t seed) : s(seed ? seed : 0x9e3779b97f4a7c15ULL) {
    next_u64();
    next_u64();
  }
  std::uint64_t next_u64() {
    std::uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  double next_pm1() { return 2.0 * (static_cast<double>(next_u64() >> 11) * 0x1.0p-53) - 1.0; }
};

// components.cpp:9-56 (BFS labelling; sub-Laplacian in ascending node order)
inline std::vector<std::vector<Index>> components(const SparseLaplacian& a) {
  std::vector<Index> label(static_cast<std::size_t>(a.n), -1);
  std::vector<std::vector<Index>> out;
  std::vector<Index> q;
  for (Index s = 0; s < a.n; ++s) {
    if (label[s] >= 0) continue;
    const Index id = static_cast<Index>(out.size());
    label[s] = id;
    q.assign(1, s);
    for (std::size_t h = 0; h < q.size(); ++h)
      for (auto k = a.row_ptr[q[h]]; k < a.row_ptr[q[h] + 1]; ++k)
        if (label[a.col[k]] < 0) {
          label[a.col[k]] = id;
          q.push_back(a.col[k]);
        }
    out.emplace_back();
  }
  for (Index u = 0; u < a.n; ++u) out[label[u]].push_back(u);
  return out;
}

inline SparseLaplacian extract(const SparseLaplacian& a, const std::vector<Index>& nodes) {
  std::vector<Index> local(static_cast<std::size_t>(a.n), -1);
  for (std::size_t k = 0; k < nodes.size(); ++k) local[nodes[k]] = static_cast<Index>(k);
  SparseLaplacian s;
  s.n = static_cast<Index>(nodes.size());
  s.row_ptr.assign(1, 0);
  for (Index lu = 0; lu < s.n; ++lu) {
    const Index u = nodes[lu];
    double d = 0.0;
    for (auto k = a.row_ptr[u]; k < a.row_ptr[u + 1]; ++k) {
      s.col.push_back(local[a.col[k]]);
      s.val.push_back(a.val[k]);
      d += -a.val[k];
    }
    s.diag.push_back(d);
    s.row_ptr.push_back(static_cast<EntryCount>(s.col.size()));
  }
  s.m = static_cast<EntryCount>(s.col.size() / 2);
  return s;
}
}  // namespace b200

// solver.cpp:31-57
inline Prepared prepare(SparseLaplacian a, const SolverOptions& opts = {}) {
  Prepared p;
  p.a = std::move(a);
  p.cycle = opts.cycle;
  const auto t0 = std::chrono::steady_clock::now();
  auto comps = b200::components(p.a);
  double work_edges = 0.0;
  for (std::size_t c = 0; c < comps.size(); ++c) {
    ComponentRun run;
    run.nodes = comps[c];
    SetupOptions local = opts.setup;
    // Rng::derive(seed, c) (rng.hpp:34-37)
    local.rng_seed = lamg_rng_derive(opts.setup.rng_seed, c);
    if (run.nodes.size() > 1) {
      run.hierarchy = comps.size() == 1 ? setup(p.a, local) : setup(b200::extract(p.a, run.nodes), local);
      work_edges += run.hierarchy.setup_work * static_cast<double>(run.hierarchy.finest_m());
      for (const auto& w : run.hierarchy.warnings) p.warnings.push_back(w);
    }
    p.components.push_back(std::move(run));
  }
  p.setup_work = work_edges / static_cast<double>(std::max<EntryCount>(p.a.m, 1));
  p.setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return p;
}

// solver.cpp:59-107
inline SolveReport solve_prepared(const Prepared& p, std::span<const Real> b, std::span<const Real> x0 = {}) {
  if (static_cast<Index>(b.size()) != p.a.n)
    throw DimensionMismatchError("solve: rhs length does not match the matrix");
  SolveReport r;
  r.x.assign(static_cast<std::size_t>(p.a.n), 0.0);
  const auto t0 = std::chrono::steady_clock::now();
  std::size_t largest = 0;
  for (std::size_t i = 1; i < p.components.size(); ++i)
    if (p.components[i].nodes.size() > p.components[largest].nodes.size()) largest = i;
  b200::Rng guess(lamg_rng_derive(p.cycle.rng_seed, 0x517));
  r.converged = true;
  double work_edges = 0.0;
  for (std::size_t i = 0; i < p.components.size(); ++i) {
    const ComponentRun& run = p.components[i];
    if (run.nodes.size() == 1) {
      if (std::abs(b[run.nodes[0]]) > 0.0)
        throw IncompatibleRhsError("nonzero rhs at isolated node " + std::to_string(run.nodes[0]));
      continue;
    }
    Vector bc(run.nodes.size()), xc(run.nodes.size());
    for (std::size_t k = 0; k < run.nodes.size(); ++k) {
      bc[k] = b[run.nodes[k]];
      xc[k] = x0.empty() ? guess.next_pm1() : x0[run.nodes[k]];
    }
    auto [x, st] = solve(run.hierarchy, bc, xc, p.cycle);
    for (std::size_t k = 0; k < run.nodes.size(); ++k) r.x[run.nodes[k]] = x[k];
    r.converged = r.converged && st.converged;
    work_edges += st.solve_work * static_cast<double>(run.hierarchy.finest_m());
    if (i == largest) {
      r.stats = std::move(st);
      r.reduction = (!r.stats.residuals.empty() && r.stats.residuals.back() > 0.0)
                        ? r.stats.residuals.front() / r.stats.residuals.back()
                        : std::numeric_limits<double>::infinity();
    }
  }
  r.solve_work = work_edges / static_cast<double>(std::max<EntryCount>(p.a.m, 1));
  r.solve_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return r;
}

// solver.hpp:55-63 / solver.cpp:109-118: benchmark measures in finest-MVM
// equivalents
struct PerformanceMeasures {
  double t_setup = 0.0;
  double t_solve = 0.0;
  double t_total = 0.0;
  double setup_fraction = 0.0;
};

inline PerformanceMeasures performance_measures(double setup_work, double solve_work, double r0, double rp) {
  PerformanceMeasures m;
  m.t_setup = setup_work;
  const double digits = r0 > 0.0 && rp > 0.0 ? std::log10(r0 / rp) : 0.0;
  m.t_solve = digits > 0.0 ? solve_work / digits : 0.0;
  m.t_total = m.t_setup + 10.0 * m.t_solve;
  m.setup_fraction = m.t_total > 0.0 ? m.t_setup / m.t_total : 0.0;
  return m;
}

// ------------------------------------------------------- Matrix Market files
// matrix_market.hpp:14-52: read_matrix_market_file + assemble_problem in one
// library call (multi-threaded parse, same CSR, warnings and errors)
enum class MatrixKind { Auto, Adjacency, Laplacian };
struct MatrixMarketOptions {
  MatrixKind kind = MatrixKind::Auto;
  bool absolute_weight_policy = true;
};
struct LoadedLaplacian {  // what assemble_problem(read_matrix_market_file(path)) yields
  SparseLaplacian a;
  bool was_laplacian = false;
  std::vector<std::string> warnings;
};

inline LoadedLaplacian load_matrix_market_file(const std::string& path, const MatrixMarketOptions& opts = {}) {
  lamg_mm* mm = nullptr;
  const int kind = opts.kind == MatrixKind::Adjacency ? 1 : opts.kind == MatrixKind::Laplacian ? 2 : 0;
  b200::check(lamg_mm_read(path.c_str(), kind, opts.absolute_weight_policy ? 1 : 0, &mm));
  std::unique_ptr<lamg_mm, void (*)(lamg_mm*)> guard(mm, lamg_mm_destroy);
  int32_t n = 0, lap = 0, nw = 0;
  int64_t m = 0;
  b200::check(lamg_mm_info(mm, &n, &m, &lap, &nw));
  LoadedLaplacian out;
  out.a.n = n;
  out.a.m = m;
  out.a.row_ptr.resize((std::size_t)n + 1);
  out.a.col.resize((std::size_t)(2 * m));
  out.a.val.resize((std::size_t)(2 * m));
  out.a.diag.resize((std::size_t)n);
  b200::check(lamg_mm_csr(mm, out.a.row_ptr.data(), out.a.col.data(), out.a.val.data(), out.a.diag.data()));
  out.was_laplacian = lap != 0;
  for (int32_t i = 0; i < nw; ++i) {
    char buf[1024];
    b200::check(lamg_mm_warning(mm, i, buf, (int32_t)sizeof buf));
    out.warnings.emplace_back(buf);
  }
  return out;
}

inline void write_matrix_market_file(const std::string& path, const SparseLaplacian& a, bool as_laplacian = false) {
  const lamg_csr v = b200::view(a);
  b200::check(lamg_mm_write(path.c_str(), &v, as_laplacian ? 1 : 0));
}

}  // namespace lamg
