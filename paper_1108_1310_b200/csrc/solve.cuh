// solve.cuh -- solve-phase driver declarations.
#pragma once

#include <string>
#include <vector>

#include "tail.cuh"

namespace lamgb {

// lamg::CycleConfig (cycle.hpp:28-36)
struct CycleCfg {
  int correction = 0;  // 0 Flat, 1 AdaptiveRecombination
  double mu = 4.0 / 3.0;
  int max_cycles = 300;
  double target_reduction = 1e10;
  double divergence_factor = 1e3;
};

// lamg::SolveStats (cycle.hpp:38-46)
struct SolveResult {
  std::vector<double> residuals;
  double acf = 0.0;
  double solve_work = 0.0;
  int cycles = 0;
  bool converged = false;
  int64_t recombinations = 0;
  double recomb_max_growth = 0.0;
  int relax_sweeps = 0;
  std::string message;
};

// LevelCredit (cycle.cpp:14-21)
struct LevelCredits {
  std::vector<double> credit;
  int take(size_t l, double gamma);
};

struct LevelWS {
  DVec<double> b, x, r;
  std::vector<DVec<double>> stage_rhs, stage_x;  // index s >= 1
  DVec<double> saved_x[2], saved_r[2], tmp;
  DVec<int32_t> xctl;  // bgs_exact ticket + per-front done counters (K > 1)
};

// per-context solve workspace, sized for the last hierarchy solved
struct Workspace {
  uint64_t owner = 0;  // DHier::uid
  int K = 1;           // right-hand sides per block: every vector is n x K, node-major
  std::vector<LevelWS> lv;
  DVec<double> direct_scratch;
  bool top_rhs_valid = false;
  TailPlan tail;          // throughput mode: on-device coarse tail
  bool tail_built = false;
  // throughput mode: one CUDA graph per host-level credit state; a cycle's
  // kernel schedule depends only on the credits at its start
  struct CycleGraph {
    std::vector<double> key, credits_after;
    cudaGraphExec_t exec = nullptr;
    double work = 0.0;
    long long launches = 0;  // kernels in the graph (counted on every replay)
  };
  std::vector<CycleGraph> graphs;
  void clear_graphs();
  ~Workspace() { clear_graphs(); }
  void ensure(Ctx& c, const DHier& h, int K = 1);
  void ensure_adaptive(Ctx& c, const DHier& h);
};

// recombine (cycle.cpp:23-103); dots land in c.dscal[120..126]
void recombine_api(Ctx& c, const CSRv& a, const double* b, int cols, LevelWS& w, double* x, bool exact,
                   double* growth);

int solve_device(Ctx& c, const DHier& h, const double* b, const double* x0, const CycleCfg& cfg,
                 double* x, SolveResult& res);

// THROUGHPUT mode, K right-hand sides in one block (batch.cuh). B and X0 are
// device RHS-major [nrhs][n]; X (device, RHS-major) receives every column at
// the cycle it converged (or stopped); res[j] are the per-column stats.
int solve_batch_device(Ctx& c, const DHier& h, int nrhs, const double* B, const double* X0, const CycleCfg& cfg,
                       double* X, std::vector<SolveResult>& res);

}  // namespace lamgb
