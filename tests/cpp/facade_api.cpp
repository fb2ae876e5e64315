// tests/cpp/facade_api.cpp -- every declaration of the reference's
// hierarchy.hpp, cycle.hpp and solver.hpp, called through the drop-in facade
// (include/lamg_b200/lamg.hpp) the way reference host code calls them. The
// inputs come from files the test writes (tests/test_cpp_facade.py); the
// outputs are written back as raw arrays plus a key/value text file, and the
// test compares them with the CPU oracle.
//
//   facade_api DIR     reads DIR/in.*, DIR/pin.* ; writes DIR/out.*, DIR/meta.txt
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include "lamg_b200/lamg.hpp"

static std::string g_dir;
static FILE* g_meta = nullptr;

template <class T>
static std::vector<T> load(const std::string& name) {
  std::ifstream f(g_dir + "/" + name, std::ios::binary);
  std::vector<char> raw((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  std::vector<T> v(raw.size() / sizeof(T));
  std::memcpy(v.data(), raw.data(), v.size() * sizeof(T));
  return v;
}
template <class V>
static void dump(const std::string& name, const V& v) {
  const auto& vec = static_cast<const std::vector<typename V::value_type>&>(v);
  std::ofstream f(g_dir + "/out." + name, std::ios::binary);
  f.write(reinterpret_cast<const char*>(vec.data()), (std::streamsize)(vec.size() * sizeof(vec[0])));
}
template <class T>
static void dump_lazy(const std::string& name, const lamg::b200::LazyArray<T>& v) {
  dump(name, v.vec());
}
static lamg::SparseLaplacian load_csr(const std::string& p) {
  lamg::SparseLaplacian a;
  a.row_ptr = load<lamg::EntryCount>(p + ".row_ptr");
  a.col = load<lamg::Index>(p + ".col");
  a.val = load<lamg::Real>(p + ".val");
  a.diag = load<lamg::Real>(p + ".diag");
  a.n = (lamg::Index)a.diag.size();
  a.m = (lamg::EntryCount)a.col.size() / 2;
  return a;
}

static const char* kind_name(lamg::LevelKind k) {
  switch (k) {
    case lamg::LevelKind::Finest: return "finest";
    case lamg::LevelKind::Elimination: return "elimination";
    case lamg::LevelKind::Aggregation: return "aggregation";
    case lamg::LevelKind::Coarsest: return "coarsest";
  }
  return "?";
}

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  g_dir = argv[1];
  g_meta = std::fopen((g_dir + "/meta.txt").c_str(), "w");
  using namespace lamg;

  // ---- hierarchy.hpp: setup, Level, Hierarchy, stats, cycle index
  const SparseLaplacian a = load_csr("in");
  SetupOptions so;
  so.gamma = 1.5;
  so.rng_seed = 1;
  so.coarsest_n = 150;
  so.tv_sweeps = 3;
  so.tv_count_finest = 4;
  so.tv_count_max = 10;
  const Hierarchy h = setup(a, so);
  std::fprintf(g_meta, "nlevels %zu\nsetup_work %.17g\nseed %llu\nwarnings %zu\n", h.levels.size(), h.setup_work,
               (unsigned long long)h.seed, h.warnings.size());
  std::fprintf(g_meta, "finest_n %d\nfinest_m %lld\ntotal_stored_edges %lld\nstorage_per_edge %.17g\nedge_ratio %.17g\n",
               h.finest_n(), (long long)h.finest_m(), (long long)h.total_stored_edges(), h.storage_per_edge(),
               h.edge_ratio());
  for (std::size_t l = 0; l < h.levels.size(); ++l) {
    const Level& L = h.levels[l];
    const std::string p = "L" + std::to_string(l) + ".";
    std::fprintf(g_meta, "%skind %s\n%sn %d\n%sm %lld\n%sgamma %.17g\n%snu_pre %d\n%snu_post %d\n%stv_count %d\n",
                 p.c_str(), kind_name(L.kind), p.c_str(), L.op.n, p.c_str(), (long long)L.op.m, p.c_str(), L.gamma,
                 p.c_str(), L.nu_pre, p.c_str(), L.nu_post, p.c_str(), L.tv_count);
    std::fprintf(g_meta, "%scoarsest %d\n%sis_elimination %d\n%sis_aggregation %d\n%scycle_index %.17g\n", p.c_str(),
                 (int)L.coarsest, p.c_str(), (int)L.is_elimination(), p.c_str(), (int)L.is_aggregation(), p.c_str(),
                 level_cycle_index(h, l, 1.5));
    dump_lazy(p + "row_ptr", L.op.row_ptr);
    dump_lazy(p + "col", L.op.col);
    dump_lazy(p + "val", L.op.val);
    dump_lazy(p + "diag", L.op.diag);
    if (std::holds_alternative<AggregationTransfer>(L.transfer)) {
      const auto& t = std::get<AggregationTransfer>(L.transfer);
      std::fprintf(g_meta, "%sfine_n %d\n%scoarse_n %d\n%sstage_used %d\n%salpha %.17g\n%sdummy_aggregate %d\n",
                   p.c_str(), t.fine_n, p.c_str(), t.coarse_n, p.c_str(), t.stage_used, p.c_str(), t.alpha, p.c_str(),
                   t.dummy_aggregate);
      dump_lazy(p + "aggregate_of", t.aggregate_of);
      dump_lazy(p + "seed_of", t.seed_of);
    } else if (std::holds_alternative<EliminationTransfer>(L.transfer)) {
      const auto& t = std::get<EliminationTransfer>(L.transfer);
      std::fprintf(g_meta, "%snstages %zu\n%scoarse_op_n %d\n", p.c_str(), t.stages.size(), p.c_str(), t.coarse_op.n);
      for (std::size_t s = 0; s < t.stages.size(); ++s) {
        const ElimStage& st = t.stages[s];
        const std::string q = p + "S" + std::to_string(s) + ".";
        std::fprintf(g_meta, "%sparent_n %d\n%scoarse_n %d\n", q.c_str(), st.parent_n, q.c_str(), st.coarse_n);
        dump_lazy(q + "f_nodes", st.f_nodes);
        dump_lazy(q + "f_diag", st.f_diag);
        dump_lazy(q + "f_ptr", st.f_ptr);
        dump_lazy(q + "f_nbr", st.f_nbr);
        dump_lazy(q + "f_val", st.f_val);
        dump_lazy(q + "coarse_of_parent", st.coarse_of_parent);
        dump_lazy(q + "parent_of_coarse", st.parent_of_coarse);
      }
    }
    if (L.coarsest_solver) {  // the level's own solver on a zero-sum right-hand side
      std::vector<Real> bc(L.op.n), xc(L.op.n, 0.0);
      for (Index i = 0; i < L.op.n; ++i) bc[i] = (i % 2 ? 1.0 : -1.0) * (1.0 + 0.001 * i);
      double s = 0.0;
      for (double v : bc) s += v;
      for (auto& v : bc) v -= s / L.op.n;
      L.coarsest_solver->solve(bc, xc);
      dump(p + "coarsest_b", bc);
      dump(p + "coarsest_x", xc);
      // the same through CoarsestSolver::make_direct / make_relaxation
      std::vector<Real> xd(L.op.n, 0.0);
      auto solver = L.coarsest == CoarsestMode::Direct ? CoarsestSolver::make_direct(L.op)
                                                       : CoarsestSolver::make_relaxation(L.op);
      solver->solve(bc, xd);
      std::fprintf(g_meta, "%scoarsest_same %d\n", p.c_str(), (int)(xd == xc));
    }
  }
  const HierarchyStats hs = hierarchy_stats(h);
  for (const LevelStats& ls : hs.levels)
    std::fprintf(g_meta, "stats%d %s %d %d %lld %.17g %d %d %d\n", ls.level, ls.kind.c_str(), (int)ls.coarsest, ls.n,
                 (long long)ls.m, ls.gamma, ls.nu_pre, ls.nu_post, ls.tv_count);
  std::fprintf(g_meta, "stats_edge_ratio %.17g\nstats_storage_per_edge %.17g\nstats_setup_work %.17g\n", hs.edge_ratio,
               hs.storage_per_edge, hs.setup_work);

  // ---- cycle.hpp: solve (flat, recombination), DivergedError, recombine,
  // LevelCredit, flat_mu
  const std::vector<Real> b = load<Real>("in.b"), x0 = load<Real>("in.x0");
  CycleConfig cfg;
  cfg.gamma = 1.5;
  cfg.correction = CorrectionMode::Flat;
  cfg.mu = flat_mu(2.0);
  cfg.max_cycles = 300;
  cfg.target_reduction = 1e10;
  cfg.divergence_factor = 1e3;
  cfg.rng_seed = 1;
  auto [x, st] = solve(h, b, x0, cfg);
  dump("x_flat", x);
  dump("res_flat", st.residuals);
  std::fprintf(g_meta, "flat_cycles %d\nflat_acf %.17g\nflat_solve_work %.17g\nflat_converged %d\n", st.cycles, st.acf,
               st.solve_work, (int)st.converged);
  CycleConfig rc = cfg;
  rc.correction = CorrectionMode::AdaptiveRecombination;
  auto [xr, sr] = solve(h, b, x0, rc);
  dump("x_recomb", xr);
  std::fprintf(g_meta, "recomb_cycles %d\nrecomb_recombinations %lld\nrecomb_growth %.17g\n", sr.cycles,
               (long long)sr.recombinations, sr.recomb_max_growth);
  CycleConfig dc = cfg;
  dc.divergence_factor = 1e-6;  // any first cycle "grows" past this: cycle.cpp:257-267
  try {
    solve(h, b, x0, dc);
    std::fprintf(g_meta, "diverged none\n");
  } catch (const DivergedError& e) {
    std::fprintf(g_meta, "diverged_message %s\ndiverged_cycles %d\ndiverged_acf %.17g\n", e.what(), e.stats.cycles,
                 e.stats.acf);
    dump("res_diverged", e.stats.residuals);
  }
  const std::vector<Vector> saved_x = {load<Real>("in.sx0"), load<Real>("in.sx1")};
  const std::vector<Vector> saved_r = {load<Real>("in.sr0"), load<Real>("in.sr1")};
  std::vector<Real> y = load<Real>("in.rx");
  Real before = 0.0;
  const Real after = recombine(a, b, saved_x, saved_r, y, &before);
  dump("recombine_x", y);
  std::fprintf(g_meta, "recombine_before %.17g\nrecombine_after %.17g\n", before, after);
  LevelCredit credit;
  std::vector<int> takes;
  for (int i = 0; i < 12; ++i) takes.push_back(credit.take(3, 1.5));
  dump("credit_takes", takes);
  std::fprintf(g_meta, "flat_mu %.17g\n", flat_mu(2.0));

  // ---- solver.hpp: prepare / solve_prepared / largest / performance_measures
  const SparseLaplacian pa = load_csr("pin");
  SolverOptions opts;
  opts.setup = so;
  opts.cycle = cfg;
  const Prepared prep = prepare(pa, opts);
  std::fprintf(g_meta, "prep_components %zu\nprep_setup_work %.17g\nprep_largest_levels %zu\n", prep.components.size(),
               prep.setup_work, prep.largest().levels.size());
  for (std::size_t c = 0; c < prep.components.size(); ++c) {
    const ComponentRun& run = prep.components[c];
    std::fprintf(g_meta, "prep_comp%zu %zu %zu\n", c, run.nodes.size(), run.hierarchy.levels.size());
  }
  const std::vector<Real> pb = load<Real>("pin.b");
  const SolveReport rep = solve_prepared(prep, pb, load<Real>("pin.x0"));
  dump("prep_x", rep.x);
  std::fprintf(g_meta, "prep_converged %d\nprep_cycles %d\nprep_solve_work %.17g\nprep_reduction %.17g\n",
               (int)rep.converged, rep.stats.cycles, rep.solve_work, rep.reduction);
  const SolveReport rep0 = solve_prepared(prep, pb);  // x0 empty: seeded random guess (solver.cpp:66-74)
  dump("prep_x_random_guess", rep0.x);
  std::vector<Real> bad = pb;
  bad.back() = 1.0;  // the last node is isolated
  try {
    solve_prepared(prep, bad);
    std::fprintf(g_meta, "prep_bad none\n");
  } catch (const IncompatibleRhsError& e) {
    std::fprintf(g_meta, "prep_bad %s\n", e.what());
  }
  const PerformanceMeasures pm =
      performance_measures(prep.setup_work, rep.solve_work, rep.stats.residuals.front(), rep.stats.residuals.back());
  std::fprintf(g_meta, "pm %.17g %.17g %.17g %.17g\n", pm.t_setup, pm.t_solve, pm.t_total, pm.setup_fraction);
  const PerformanceMeasures pk = performance_measures(200.0, 600.0, 1e5, 1e-5);  // test_cycle.cpp:336-346
  const PerformanceMeasures pd = performance_measures(10.0, 5.0, 0.0, 0.0);
  std::fprintf(g_meta, "pm_known %.17g %.17g %.17g %.17g\npm_degenerate %.17g %.17g\n", pk.t_setup, pk.t_solve,
               pk.t_total, pk.setup_fraction, pd.t_solve, pd.t_total);
  std::fclose(g_meta);
  return 0;
}
