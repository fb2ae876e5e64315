// hier.cuh -- device-resident hierarchy (lamg::Hierarchy, hierarchy.hpp:24-50).
#pragma once

#include <atomic>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "core.cuh"

namespace lamgb {

enum LevelKind { KIND_FINEST = 0, KIND_ELIM = 1, KIND_AGG = 2, KIND_COARSEST = 3 };
enum CoarsestMode { CM_NONE = 0, CM_DIRECT = 1, CM_RELAX = 2 };

// lamg::ElimStage (elimination.hpp:16-26) + solve-time transpose lists
struct DStage {
  int32_t parent_n = 0, coarse_n = 0, nf = 0;
  int64_t nnzf = 0;
  DVec<int32_t> f_nodes;
  DVec<double> f_diag;
  DVec<int64_t> f_ptr;
  DVec<int32_t> f_nbr;
  DVec<double> f_val;
  DVec<int32_t> cop, poc;
  DVec<int64_t> t_ptr, t_p;
  DVec<int32_t> f_of_p;
  DVec<int32_t> tlong;  // coarse nodes with long contribution lists
  int32_t ntlong = 0;
  StageV view(bool exact = true) const {
    return StageV{parent_n, coarse_n, nf, f_nodes.p, f_diag.p, f_ptr.p, f_nbr.p, f_val.p,
                  cop.p, poc.p, t_ptr.p, t_p.p, f_of_p.p, tlong.p, ntlong, exact};
  }
};

// lamg::AggregationTransfer (aggregation.hpp:36-44) + member lists
struct DAgg {
  int32_t fine_n = 0, coarse_n = 0;
  int stage_used = 1;
  double alpha = 1.0;
  int32_t dummy_aggregate = -1;
  DVec<int32_t> aggregate_of, seed_of;
  DVec<int64_t> mem_ptr;
  DVec<int32_t> mem;
};

// Coarsest direct solver: bordered [[A,1],[1^T,0]] LU per connected component
// (coarse_solver.cpp:14-45), factored on the device at setup.
struct DDirect {
  int32_t n = 0, ncomp = 0, maxN = 0;
  int64_t m = 0;
  std::vector<int32_t> comp_size;  // host copy
  DVec<int32_t> comp_start;        // [ncomp+1] offsets into nodes
  DVec<int32_t> nodes;             // nodes of each component, ascending
  DVec<int64_t> lu_off;            // [ncomp] offsets into lu
  DVec<double> lu;                 // (cn+1)^2 row-major per component
  DVec<int32_t> perm;              // (cn+1) per component, offsets comp_start[c]+c
  DVec<double> inv;                // throughput: rows/cols [0,cn) of each bordered inverse
  DVec<int64_t> inv_off;           // [ncomp] offsets into inv
};

// Long rows (power-law hubs and their elimination fill): rows longer than
// kLongRow are reduced by a whole CTA (K columns: 32 strided slices); rows
// longer than `chunk` entries are split into chunks of `chunk` entries, one
// CTA each, whose sums combine in chunk order (a fixed order that depends on
// the row only: never on K, never on which CTA finishes last).
struct LongRows {
  int64_t chunk = 1024;                // entries per chunk of a super-long row
  DVec<int32_t> rows;                  // long rows (> kLongRow entries, <= chunk)
  std::vector<int32_t> ptr_h;          // per colour (stored order) or [0, count] (natural)
  DVec<int32_t> item_row, item_chunk;  // super-long rows: (row, chunk) work items
  DVec<int32_t> item_srow;             // super-long row index of each item
  std::vector<int32_t> iptr_h;
  DVec<int32_t> srows, sitem0;         // super-long rows and their first item
  std::vector<int32_t> sptr_h;
  DVec<int32_t> ptr_d, iptr_d;         // device copies of ptr_h / iptr_h (persistent kernels)
};
// lists over the row ranges `bounds` of a CSR with host row pointers rp
void build_long_rows(Ctx& c, const std::vector<int64_t>& rp, const std::vector<int32_t>& bounds, LongRows& L);

// Throughput-mode smoother data: a greedy first-fit colouring in index order
// (computed over the exact-order wavefronts, so it is the sequential greedy
// colouring) and a copy of the operator whose rows are stored colour by
// colour. A coloured sweep is a sequential sweep in colour-permuted order:
// same hierarchy, different smoother.
inline uint64_t next_object_uid() {
  static std::atomic<uint64_t> c{1};
  return c++;
}

struct DColor {
  uint64_t uid = next_object_uid();  // keys cached sweep graphs (addresses get reused)
  int32_t ncolors = 0;
  int group = 1;                // lanes per row in the throughput kernels (1, 4 or 8)
  std::vector<int32_t> cptr_h;  // [ncolors+1] row ranges of each colour
  DVec<int32_t> row_ids;        // natural row of each stored row
  DVec<int64_t> rp;             // [n+1] permuted row pointers
  DVec<int32_t> col;            // natural column indices
  DVec<double> val;
  DVec<double> diag;            // diag of each stored row
  // heavy rows (hubs: more than kHeavyRow entries) are reduced by a whole CTA
  DVec<int32_t> heavy;          // stored positions of heavy rows, ascending
  std::vector<int32_t> hptr_h;  // [ncolors+1] ranges of `heavy` per colour
  DVec<int32_t> hptr;
  DVec<int32_t> heavy_nat;      // natural rows with more than kHeavyRow entries
  int32_t nheavy_nat = 0;
  LongRows blong;  // stored (colour) order, ranges per colour
};
constexpr int64_t kLongRow = 64;

constexpr int64_t kHeavyRow = 2048;

// Exact-order sweep of a K-column block without a grid barrier (bgs_exact,
// batch.cu): the wavefronts of the level's schedule cut into work items of at
// most kExactItemRows rows, numbered in front order. Items are claimed by a
// ticket; an item of front f starts once every item of front f-1 is done.
// An item is one 256-thread CTA pass: 256 / (K/4) rows (32 rows for K <= 32,
// 16 for K = 64, 8 for K = 128).
constexpr int kMaxExactSweeps = 4;  // sweeps per launch (the counters cover them)
struct ExactItems {
  int32_t rows = 0;  // rows per item
  int32_t nitems = 0, nfronts = 0;
  DVec<int32_t> front, r0, r1;  // per item: its front and row range in sched.rows
  DVec<int32_t> count;          // items per front
};
constexpr int kExactTables = 3;  // item tables of 32, 16 and 8 rows
inline int exact_table_for(int K) { return K <= 32 ? 0 : K == 64 ? 1 : 2; }
void build_exact_items(Ctx& c, const Schedule& sch, int32_t rows, ExactItems& out);

struct DLevel {
  int kind = KIND_FINEST;
  DCSR op;
  std::vector<std::unique_ptr<DStage>> stages;  // elimination transfer
  std::unique_ptr<DAgg> agg;                    // aggregation transfer
  double gamma = 1.0;
  int nu_pre = 0, nu_post = 0, tv_count = 0;
  int coarsest = CM_NONE;
  std::unique_ptr<DDirect> direct;
  Schedule sched;          // exact-order GS wavefronts of this level's operator
  std::unique_ptr<DColor> color;  // throughput-mode coloured operator (on demand)
  std::unique_ptr<DColor> fcolor;  // front-modulo colouring of the finest smoothing level (LAMG_FRONT_MOD)
  ExactItems xitems[kExactTables];  // throughput mode: exact-order K-column sweep items (per item size)
  LongRows blong_nat;             // throughput mode: long rows in natural order (K-column residuals)
  UpperIndex upper;        // energy / relaxation helpers
};

struct DHier {
  std::vector<std::unique_ptr<DLevel>> levels;
  double setup_work = 0.0;
  double setup_seconds = 0.0;
  uint64_t seed = 0;
  std::vector<std::string> warnings;
  int device = 0;
  // recorded on the setup context's stream when setup returns: host reads of
  // the hierarchy wait on it (the event outlives the context and its stream)
  cudaEvent_t ready = nullptr;
  void mark_ready(cudaStream_t s) {
    if (!ready) CK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    CK(cudaEventRecord(ready, s));
  }
  void wait_ready() const {
    if (ready) CK(cudaEventSynchronize(ready));
  }
  ~DHier() {
    if (ready) cudaEventDestroy(ready);
  }
  // throughput mode (colour-permuted copies), built on demand
  std::atomic<bool> throughput_ready{false};
  std::mutex prep_mu;  // concurrent solves on one hierarchy (one context each) build it once
  // builds the throughput-mode data once, whichever context gets here first
  template <class F>
  void ensure_throughput(F&& build) {
    if (throughput_ready.load(std::memory_order_acquire)) return;
    std::lock_guard<std::mutex> g(prep_mu);
    if (throughput_ready.load(std::memory_order_relaxed)) return;
    build();
    throughput_ready.store(true, std::memory_order_release);
  }
  uint64_t uid = next_object_uid();  // workspaces key on this, not on the address
};

// assemble_canonical (sparse_laplacian.cpp:60-104) of a sorted, merged u<v
// edge list on the device (setup.cu)
void assemble_canonical_dev(Ctx& c, int32_t n, int64_t E, const int32_t* eu, const int32_t* ev, const double* ew,
                            DCSR& out);

struct SetupOpts {
  double gamma = 1.5;
  uint64_t seed = 1;
  int32_t coarsest_n = 150;
  int tv_sweeps = 3, tv_count_finest = 4, tv_count_max = 10;
};

// hierarchy.cpp:59-138
std::unique_ptr<DHier> setup_device(Ctx& c, const CSRv& a, const SetupOpts& o);
// hierarchy.cpp:31-40
double level_cycle_index(const DHier& h, size_t l, double gamma);

// ---- building blocks exposed for the per-kernel API -----------------------
struct SelectResult {
  int32_t nf = 0, nc = 0;
  DVec<int32_t> f, c;
};
void select_low_degree(Ctx& c, const CSRv& a, int32_t max_degree, SelectResult& out);
// schur_reduce: fills stage arrays and the coarse operator; throws like the reference
void schur_reduce(Ctx& c, const CSRv& a, const int32_t* f, int32_t nf, const int32_t* cset,
                  int32_t nc, DStage& st, DCSR& coarse, bool check_inputs);
// eliminate_rounds: false when the first round already selects too few nodes
bool eliminate_rounds(Ctx& c, const CSRv& a, std::vector<std::unique_ptr<DStage>>& stages,
                      DCSR& coarse);
double probe_relaxation(Ctx& c, const CSRv& a, const Schedule& sch, const UpperIndex& up,
                        int sweeps, uint64_t seed);
// the factor itself with the reference's sequential folds (parity harness)
double probe_factor(Ctx& c, const CSRv& a, const Schedule& sch, const UpperIndex& up, int sweeps, uint64_t seed,
                    bool exact);
void generate_tvs(Ctx& c, const CSRv& a, const Schedule& sch, int K, int sweeps, uint64_t seed,
                  DVec<double>& X /* n*K node-major */);
void compute_affinities(Ctx& c, const CSRv& a, int K, const double* X, double* aff, double* nn);
int32_t detect_hubs(Ctx& c, const CSRv& a, DVec<int32_t>& hubs);
void aggregate(Ctx& c, const CSRv& a, int K, const double* X, double gamma, const int32_t* hubs,
               int32_t nhubs, DAgg& out, int* stages_run);
void galerkin(Ctx& c, const CSRv& a, const int32_t* agg, int32_t coarse_n, DCSR& out);
void make_direct(Ctx& c, const CSRv& a, DDirect& d);
// scratch: 2*maxN + 2 doubles
void direct_solve(Ctx& c, const DDirect& d, const double* b, double* x, bool exact, double* scratch);
// col/nat: the THROUGHPUT colouring and natural-order long-row lists (nullptr: VALIDATE path)
void relax_solve(Ctx& c, const CSRv& a, const Schedule& sch, const DColor* col, const LongRows* nat,
                 const double* b, double* x, DVec<double>& r, int* sweeps_out, bool exact);

// throughput mode (throughput.cu)
void build_coloring(Ctx& c, const CSRv& a, const Schedule& sch, DColor& out);
void gs_colored(Ctx& c, const DColor& col, int32_t n, const double* b, double* x, int sweeps);
void gs_colored_one(Ctx& c, const DColor& col, const double* b, double* x, int32_t colour);
// throughput residual r = b - A x with `group` lanes per row (tree-folded rows)
void residual_tp(Ctx& c, const CSRv& a, const double* b, const double* x, double* r, const DColor& cl);
inline int row_group_for(int64_t n, int64_t m) {
  const double deg = n ? 2.0 * (double)m / (double)n : 0.0;
  return deg < 8.0 ? 1 : 8;
}
void build_direct_inverse(Ctx& c, DDirect& d);
// whole relaxation-coarsest solve in one cooperative launch; returns sweeps
int relax_colored_coop(Ctx& c, const CSRv& a, const DColor& cl, const LongRows& nat, const double* b, double* x,
                       double* r);
// THROUGHPUT residual for operators with long rows (hubs chunked over CTAs)
// group: lanes per short row (1 or 8; <= 0: residual_tasks_group(a, nat))
void residual_tasks(Ctx& c, const CSRv& a, const LongRows& nat, const double* b, const double* x, double* r,
                    int group = 0);
int residual_tasks_group(const CSRv& a, const LongRows& nat);
inline bool has_long_rows(const LongRows& L) { return !L.ptr_h.empty() && (L.ptr_h.back() > 0 || L.iptr_h.back() > 0); }
// the same as a per-sweep CUDA graph of task launches (large levels)
int relax_colored_graph(Ctx& c, const CSRv& a, const DColor& cl, const LongRows& nat, const double* b, double* x,
                        double* r);
void prepare_throughput(Ctx& c, DHier& h);
// THROUGHPUT smoother data of one operator (colouring + colour-permuted copy)
std::unique_ptr<DColor> make_color(Ctx& c, const CSRv& a, const Schedule& sch);
void build_natural_long_rows(Ctx& c, const CSRv& a, LongRows& out);

}  // namespace lamgb
