// lamg_b200 -- command line front end over the B200 facade (SURVEY.md 8(f)
// rank 4): the `solve`, `info` and `bench` subcommands of the reference CLI
// (proj/tools/lamg.cpp:146-180 stats JSON, :197-244 info JSON, :287-357 bench
// CSV, exit codes :100-115) with the same option names, output keys, CSV
// columns and exit codes, so scripts written against the reference tool run
// unchanged. `gen` is not provided: the reference's generators are host code
// outside the hot path (tests use paper_1108_1310_b200/graphs.py).
//
//   lamg_b200 solve --matrix A.mtx [--kind auto|adjacency|laplacian] [--keep-weights]
//                   [--rhs random[:SEED]|zero|file:PATH] [--tol-reduction R] [--gamma G]
//                   [--correction flat|adaptive] [--mu M] [--max-cycles N] [--out-x PATH]
//                   [--stats PATH] [--seed S] [--mode validate|throughput]
//   lamg_b200 info  --matrix A.mtx [--kind K] [--keep-weights] [--gamma G] [--seed S] [--out PATH]
//   lamg_b200 bench --problem A.mtx [--problem B.mtx ...] [--out CSV] [--jobs N] [solve options]
//
// Build: g++ -std=c++20 -O2 -I include tools/cli/lamg_b200_cli.cpp -L paper_1108_1310_b200
//            -llamg_b200 -Wl,-rpath,$PWD/paper_1108_1310_b200 -lpthread -o tools/cli/lamg_b200
#include <atomic>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "lamg_b200/lamg.hpp"

namespace {

using namespace lamg;

// ------------------------------------------------------------ tiny JSON writer
// (objects keep insertion order; numbers print with 17 significant digits)
class Json {
 public:
  Json& num(const std::string& k, double v) {
    char buf[64];
    if (std::isfinite(v)) std::snprintf(buf, sizeof buf, "%.17g", v);
    else std::snprintf(buf, sizeof buf, "null");
    return raw(k, buf);
  }
  Json& integer(const std::string& k, long long v) { return raw(k, std::to_string(v)); }
  Json& boolean(const std::string& k, bool v) { return raw(k, v ? "true" : "false"); }
  Json& str(const std::string& k, const std::string& v) { return raw(k, quote(v)); }
  Json& strings(const std::string& k, const std::vector<std::string>& v) {
    std::string s = "[";
    for (std::size_t i = 0; i < v.size(); ++i) s += (i ? ", " : "") + quote(v[i]);
    return raw(k, s + "]");
  }
  Json& raw(const std::string& k, const std::string& text) {
    items_.emplace_back(k, text);
    return *this;
  }
  std::string dump(int indent = 2, int depth = 0) const {
    const std::string pad(static_cast<std::size_t>(indent * (depth + 1)), ' ');
    std::string s = "{\n";
    for (std::size_t i = 0; i < items_.size(); ++i)
      s += pad + quote(items_[i].first) + ": " + items_[i].second + (i + 1 < items_.size() ? ",\n" : "\n");
    return s + std::string(static_cast<std::size_t>(indent * depth), ' ') + "}";
  }
  static std::string quote(const std::string& v) {
    std::string s = "\"";
    for (char ch : v) {
      if (ch == '"' || ch == '\\') s += '\\', s += ch;
      else if (ch == '\n') s += "\\n";
      else if (static_cast<unsigned char>(ch) < 0x20) s += ' ';
      else s += ch;
    }
    return s + "\"";
  }

 private:
  std::vector<std::pair<std::string, std::string>> items_;
};

// ---------------------------------------------------------------- arguments
struct Args {
  std::map<std::string, std::vector<std::string>> opt;  // --name value (repeatable)
  std::map<std::string, bool> flag;
  std::string get(const std::string& k, const std::string& dflt = {}) const {
    auto it = opt.find(k);
    return it == opt.end() || it->second.empty() ? dflt : it->second.back();
  }
  double real(const std::string& k, double dflt) const {
    const std::string v = get(k);
    return v.empty() ? dflt : std::strtod(v.c_str(), nullptr);
  }
  std::uint64_t u64(const std::string& k, std::uint64_t dflt) const {
    const std::string v = get(k);
    return v.empty() ? dflt : std::strtoull(v.c_str(), nullptr, 10);
  }
  bool has(const std::string& k) const { return flag.count(k) || opt.count(k); }
};

Args parse_args(int argc, char** argv, int first, const std::vector<std::string>& flags) {
  Args a;
  for (int i = first; i < argc; ++i) {
    std::string t = argv[i];
    if (t.rfind("--", 0) != 0) throw Error("unexpected argument '" + t + "'");
    std::string name = t.substr(2), value;
    const auto eq = name.find('=');
    bool has_value = false;
    if (eq != std::string::npos) value = name.substr(eq + 1), name = name.substr(0, eq), has_value = true;
    bool is_flag = false;
    for (const auto& f : flags) is_flag = is_flag || f == name;
    if (is_flag) {
      a.flag[name] = true;
      continue;
    }
    if (!has_value) {
      if (i + 1 >= argc) throw Error("option --" + name + " needs a value");
      value = argv[++i];
    }
    a.opt[name].push_back(value);
  }
  return a;
}

int fail(const std::string& message, int code, const std::string& stats_path = {}) {
  Json j;
  j.str("error", message).integer("exit_code", code);
  std::cout << j.dump() << "\n";
  if (!stats_path.empty()) {
    std::ofstream out(stats_path);
    if (out) out << j.dump() << "\n";
  }
  return code;
}

int code_of(const std::exception& e) { return dynamic_cast<const IoError*>(&e) ? 2 : 1; }

// ------------------------------------------------------------------ inputs
LoadedLaplacian load(const Args& a, const std::string& path) {
  MatrixMarketOptions o;
  const std::string kind = a.get("kind", "auto");
  o.kind = kind == "adjacency" ? MatrixKind::Adjacency : kind == "laplacian" ? MatrixKind::Laplacian : MatrixKind::Auto;
  o.absolute_weight_policy = !a.has("keep-weights");
  return load_matrix_market_file(path, o);
}

SolverOptions options_of(const Args& a) {
  SolverOptions o;
  const double gamma = a.real("gamma", 1.5);
  const std::uint64_t seed = a.u64("seed", 1);
  o.setup.gamma = gamma;
  o.setup.rng_seed = seed;
  o.cycle.gamma = gamma;
  o.cycle.correction = a.get("correction", "flat") == "adaptive" ? CorrectionMode::AdaptiveRecombination
                                                                 : CorrectionMode::Flat;
  o.cycle.mu = a.real("mu", 4.0 / 3.0);
  o.cycle.max_cycles = static_cast<int>(a.real("max-cycles", 300));
  o.cycle.target_reduction = a.real("tol-reduction", 1e10);
  o.cycle.rng_seed = seed;
  return o;
}

// sequential mean subtraction, as subtract_mean (sparse_laplacian.cpp:242-252)
void subtract_mean(Vector& v, const std::vector<Index>* nodes = nullptr) {
  double s = 0.0;
  if (nodes) {
    for (Index u : *nodes) s += v[u];
    const double mean = s / static_cast<double>(nodes->size());
    for (Index u : *nodes) v[u] -= mean;
  } else {
    for (double x : v) s += x;
    const double mean = s / static_cast<double>(v.size());
    for (double& x : v) x -= mean;
  }
}

Vector read_vector(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw IoError("cannot open: " + path);
  Vector out;
  std::string line;
  bool array_header = false, sized = false;
  std::size_t lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    if (line.empty()) continue;
    if (line[0] == '%') {
      if (lineno == 1 && line.rfind("%%MatrixMarket", 0) == 0) {
        std::string low = line;
        for (char& ch : low) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
        if (low.find("array") == std::string::npos) throw ParseError("vector file must use array format, line 1");
        array_header = true;
      }
      continue;
    }
    std::istringstream row(line);
    if (array_header && !sized) {
      long long r = 0, c = 0;
      if (!(row >> r >> c) || c != 1)
        throw ParseError("vector array size line malformed at line " + std::to_string(lineno));
      sized = true;
      continue;
    }
    double v = 0.0;
    if (!(row >> v)) throw ParseError("bad vector value at line " + std::to_string(lineno));
    out.push_back(v);
  }
  return out;
}

// make_rhs (matrix_market.cpp:229-290): zero | random[:SEED] | file:PATH
Vector make_rhs(const SparseLaplacian& a, const std::string& spec, std::uint64_t default_seed) {
  const std::size_t n = static_cast<std::size_t>(a.n);
  if (spec == "zero") return Vector(n, 0.0);
  if (spec == "random" || spec.rfind("random:", 0) == 0) {
    std::uint64_t seed = spec.size() > 7 ? std::strtoull(spec.c_str() + 7, nullptr, 10) : 1;
    if (seed == 1) seed = default_seed;
    b200::Rng rng(lamg_rng_derive(seed, 0xb));
    Vector b(n);
    for (double& v : b) v = rng.next_pm1();
    subtract_mean(b);
    const auto comps = b200::components(a);
    if (comps.size() > 1)
      for (const auto& nodes : comps) subtract_mean(b, &nodes);
    return b;
  }
  if (spec.rfind("file:", 0) == 0) {
    Vector b = read_vector(spec.substr(5));
    if (b.size() != n)
      throw DimensionMismatchError("rhs file has " + std::to_string(b.size()) + " values, expected " +
                                   std::to_string(n));
    double inf = 0.0, sum = 0.0;
    for (double v : b) inf = std::max(inf, std::abs(v)), sum += v;
    if (std::abs(sum) > 1e-10 * inf) throw IncompatibleRhsError("rhs file sum is not zero");
    return b;
  }
  throw Error("unknown rhs spec '" + spec + "', expected zero|random[:SEED]|file:PATH");
}

void write_vector(const std::string& path, const Vector& x) {
  std::ofstream out(path);
  if (!out) throw IoError("cannot open for writing: " + path);
  char buf[64];
  for (double v : x) {
    std::snprintf(buf, sizeof buf, "%.17g", v);
    out << buf << "\n";
  }
}

void select_mode(const Args& a) {
  const std::string m = a.get("mode", "validate");
  b200::set_mode(m == "throughput" ? LAMG_MODE_THROUGHPUT : LAMG_MODE_VALIDATE);
}

// ------------------------------------------------------------------- solve
int cmd_solve(const Args& a) {
  const std::string stats_path = a.get("stats");
  try {
    if (!a.has("matrix")) throw Error("--matrix is required");
    LoadedLaplacian in = load(a, a.get("matrix"));
    select_mode(a);
    const SolverOptions opts = options_of(a);
    Prepared prep = prepare(std::move(in.a), opts);
    prep.warnings.insert(prep.warnings.begin(), in.warnings.begin(), in.warnings.end());
    const Vector b = make_rhs(prep.a, a.get("rhs", "random:1"), a.u64("seed", 1));
    const SolveReport rep = solve_prepared(prep, b);
    if (a.has("out-x")) write_vector(a.get("out-x"), rep.x);
    const Hierarchy& h = prep.largest();
    const PerformanceMeasures pm =
        performance_measures(prep.setup_work, rep.solve_work, rep.stats.residuals.front(), rep.stats.residuals.back());
    Json j;
    j.integer("n", prep.a.n).integer("m", prep.a.m).integer("components", (long long)prep.components.size());
    j.integer("levels", (long long)h.levels.size()).num("acf", rep.stats.acf).integer("cycles", rep.stats.cycles);
    j.boolean("converged", rep.converged).num("residual_initial", rep.stats.residuals.front());
    j.num("residual_final", rep.stats.residuals.back()).num("reduction", rep.reduction);
    j.num("setup_mvm", prep.setup_work).num("solve_mvm", rep.solve_work);
    j.num("total_mvm", prep.setup_work + rep.solve_work).num("t_setup", pm.t_setup).num("t_solve", pm.t_solve);
    j.num("t_total", pm.t_total).num("setup_fraction", pm.setup_fraction);
    j.num("storage_per_edge", h.storage_per_edge()).num("edge_ratio", h.edge_ratio());
    j.integer("recombinations", rep.stats.recombinations).num("recomb_max_growth", rep.stats.recomb_max_growth);
    j.num("wall_setup_seconds", prep.setup_seconds).num("wall_solve_seconds", rep.solve_seconds);
    j.integer("seed", (long long)a.u64("seed", 1)).num("gamma", a.real("gamma", 1.5));
    j.str("correction", a.get("correction", "flat")).num("mu", a.real("mu", 4.0 / 3.0));
    j.strings("warnings", prep.warnings);
    std::cout << j.dump() << "\n";
    if (!stats_path.empty()) {
      std::ofstream out(stats_path);
      if (!out) return fail("cannot open for writing: " + stats_path, 2);
      out << j.dump() << "\n";
    }
    return rep.converged ? 0 : 3;
  } catch (const DivergedError& e) {
    return fail(std::string("solve diverged: ") + e.what(), 4, stats_path);
  } catch (const std::exception& e) {
    return fail(e.what(), code_of(e), stats_path);
  }
}

// -------------------------------------------------------------------- info
int cmd_info(const Args& a) {
  try {
    if (!a.has("matrix")) throw Error("--matrix is required");
    LoadedLaplacian in = load(a, a.get("matrix"));
    select_mode(a);
    SolverOptions opts;
    opts.setup.gamma = a.real("gamma", 1.5);
    opts.setup.rng_seed = a.u64("seed", 1);
    Prepared prep = prepare(std::move(in.a), opts);
    prep.warnings.insert(prep.warnings.begin(), in.warnings.begin(), in.warnings.end());
    const HierarchyStats st = hierarchy_stats(prep.largest());
    std::string levels = "[";
    for (std::size_t i = 0; i < st.levels.size(); ++i) {
      const LevelStats& ls = st.levels[i];
      Json l;
      l.integer("level", (long long)ls.level).str("kind", ls.kind).boolean("coarsest", ls.coarsest);
      l.integer("n", ls.n).integer("m", ls.m).num("gamma", ls.gamma).integer("nu_pre", ls.nu_pre);
      l.integer("nu_post", ls.nu_post).integer("tvs", ls.tv_count);
      levels += (i ? ",\n    " : "\n    ") + l.dump(2, 2);
    }
    levels += st.levels.empty() ? "]" : "\n  ]";
    Json j;
    j.integer("n", prep.a.n).integer("m", prep.a.m).integer("components", (long long)prep.components.size());
    j.num("setup_mvm", prep.setup_work).num("edge_ratio", st.edge_ratio).num("storage_per_edge", st.storage_per_edge);
    j.num("wall_setup_seconds", prep.setup_seconds).strings("warnings", prep.warnings).raw("levels", levels);
    std::cout << j.dump() << "\n";
    if (a.has("out")) {
      std::ofstream out(a.get("out"));
      if (!out) return fail("cannot open for writing: " + a.get("out"), 2);
      out << j.dump() << "\n";
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e.what(), code_of(e));
  }
}

// ------------------------------------------------------------------- bench
struct Row {
  std::string name, error;
  bool ok = false;
  long long n = 0, m = 0;
  std::size_t levels = 0;
  PerformanceMeasures pm;
  double acf = 0.0, storage_per_edge = 0.0;
};

Row bench_one(const Args& a, const std::string& path) {
  Row r;
  r.name = path;
  try {
    Args plain = a;  // bench problems load with the default matrix options
    plain.opt.erase("kind");
    plain.flag.erase("keep-weights");
    LoadedLaplacian in = load(plain, path);
    select_mode(a);  // per worker thread: the facade's device context is thread-local
    const SolverOptions opts = options_of(a);
    const Prepared prep = prepare(std::move(in.a), opts);
    const Vector b = make_rhs(prep.a, "random:" + std::to_string(a.u64("seed", 1)), a.u64("seed", 1));
    const SolveReport rep = solve_prepared(prep, b);
    r.ok = true;
    r.n = prep.a.n;
    r.m = prep.a.m;
    r.levels = prep.largest().levels.size();
    r.pm = performance_measures(prep.setup_work, rep.solve_work, rep.stats.residuals.front(),
                                rep.stats.residuals.back());
    r.acf = rep.stats.acf;
    r.storage_per_edge = prep.largest().storage_per_edge();
  } catch (const std::exception& e) {
    r.error = e.what();
  }
  return r;
}

int cmd_bench(const Args& a) {
  auto it = a.opt.find("problem");
  if (it == a.opt.end() || it->second.empty()) return fail("--problem is required", 1);
  const std::vector<std::string>& problems = it->second;
  std::vector<Row> rows(problems.size());
  const int jobs = std::max(1, static_cast<int>(a.real("jobs", 1)));
  std::atomic<std::size_t> next{0};
  auto worker = [&] {  // the facade's device context is per thread: one stream per worker
    for (std::size_t i = next.fetch_add(1); i < problems.size(); i = next.fetch_add(1)) rows[i] = bench_one(a, problems[i]);
  };
  if (jobs == 1) {
    worker();
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < std::min<int>(jobs, (int)problems.size()); ++t) pool.emplace_back(worker);
    for (auto& t : pool) t.join();
  }
  std::ostringstream csv;
  csv << "name,n,m,L,t_setup,t_solve,t_total,acf,storage_per_edge,setup_pct\n";
  bool failed = false;
  for (const Row& r : rows) {
    if (!r.ok) {
      failed = true;
      std::cerr << "bench: " << r.name << " failed: " << r.error << "\n";
      continue;
    }
    char line[512];
    std::snprintf(line, sizeof line, "%s,%lld,%lld,%zu,%.4g,%.4g,%.4g,%.4g,%.4g,%.4g\n", r.name.c_str(), r.n, r.m,
                  r.levels, r.pm.t_setup, r.pm.t_solve, r.pm.t_total, r.acf, r.storage_per_edge,
                  100.0 * r.pm.setup_fraction);
    csv << line;
  }
  const std::string out_path = a.get("out");
  if (out_path.empty() || out_path == "-") {
    std::cout << csv.str();
  } else {
    std::ofstream out(out_path);
    if (!out) return fail("cannot open for writing: " + out_path, 2);
    out << csv.str();
  }
  return failed ? 1 : 0;
}

const char* kUsage =
    "usage: lamg_b200 <solve|info|bench> [options]\n"
    "  solve --matrix A.mtx [--kind auto|adjacency|laplacian] [--keep-weights] [--rhs random[:SEED]|zero|file:PATH]\n"
    "        [--tol-reduction R] [--gamma G] [--correction flat|adaptive] [--mu M] [--max-cycles N]\n"
    "        [--out-x PATH] [--stats PATH] [--seed S] [--mode validate|throughput]\n"
    "  info  --matrix A.mtx [--kind K] [--keep-weights] [--gamma G] [--seed S] [--out PATH]\n"
    "  bench --problem A.mtx [--problem B.mtx ...] [--out CSV] [--jobs N] [solve options]\n";

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2 || std::string(argv[1]) == "--help" || std::string(argv[1]) == "-h") {
    std::cout << kUsage;
    return argc < 2 ? 1 : 0;
  }
  const std::string cmd = argv[1];
  try {
    const Args a = parse_args(argc, argv, 2, {"keep-weights", "help"});
    if (a.has("help")) {
      std::cout << kUsage;
      return 0;
    }
    if (cmd == "solve") return cmd_solve(a);
    if (cmd == "info") return cmd_info(a);
    if (cmd == "bench") return cmd_bench(a);
    return fail("unknown subcommand '" + cmd + "' (solve, info, bench)", 1);
  } catch (const std::exception& e) {
    return fail(e.what(), 1);
  }
}
