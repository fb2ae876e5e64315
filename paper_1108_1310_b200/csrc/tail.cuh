// tail.cuh -- device descriptors for the single-CTA coarse-tail kernel.
#pragma once

#include <type_traits>

#include "hier.cuh"

namespace lamgb {

constexpr int kMaxLevels = 64;
constexpr int kMaxStages = 8;
constexpr int kTailSmemMax = 200 * 1024;  // dynamic shared memory of the tail CTA (upper bound)

struct TailCounters {
  double work;          // edge units (exact integers: order-free)
  long long relax_sweeps;
  long long phases;     // diagnostics: colour phases, total cycles, GS cycles
  long long cyc_total, cyc_gs;
  long long smem_calls, smem_phases, cyc_stage, cyc_phases, cyc_global_gs, global_phases;
  long long ph_fold, ph_extra, ph_prefetch, ph_barrier;
  long long lvl_gs_cyc[kMaxLevels], lvl_gs_calls[kMaxLevels];  // per level (CTA 0, thread 0)
  long long lvl_ph[kMaxLevels][4];  // batched sweeps: first row, extra rows, prefetch, barrier
  // K > 1: cycles and calls per operation (gs, residual, restrict, interp, coarsen, inject,
  // backsub, direct), cluster scope [0..8) and slice scope [8..16) (leader thread)
  long long op_cyc[16], op_calls[16];
};

// one level as the tail kernel sees it: operator (natural + colour-permuted),
// the transfer to its child, and its workspace vectors
struct TLevel {
  int id;
  int32_t n;
  int64_t m;
  const int64_t* rp;
  const int32_t* col;
  const double* val;
  const double* diag;
  // coloured copy (GS)
  int32_t ncolors;
  const int32_t* cptr;
  const int32_t* row_ids;
  const int64_t* prp;
  const int32_t* pcol;
  const double* pval;
  const double* pdiag;
  int group;    // lanes per row (1, 4, 8)
  int smem_ok;  // the coloured operator + x + b fit the tail CTA's shared memory
  int smem_cs;  // K > 1: the operator + this CTA's column slice of x and b fit
  int gs_cta;   // K > 1 cluster tail: this level's sweeps run in CTA 0 alone (a
                // __syncthreads per colour instead of a cluster barrier)
  int sl_ok;    // K > 1 slice scope: x (n x 32 B) and two colour buffers of sl_cap
  int32_t sl_cap;  // entries fit the tail CTA's dynamic shared memory (sl_rows)
  int sl_nbuf;     // colour buffers (3: two colours in flight ahead of the fold)
  const int32_t* sl_tab;  // [2 (ncolors + 1)] colour row ranges, then their first entries
  // workspace
  double* b;
  double* x;
  double* r;
  double* nm_b;  // subtree root (K > 1): the host's node-major b and x
  double* nm_x;
  // solve parameters the parent uses when visiting this level
  double gamma;
  int nu_pre, nu_post;
  int coarsest;
  // coarsest direct (throughput inverse)
  int32_t ncomp;
  const int32_t* comp_start;
  const int32_t* nodes;
  const double* inv;
  const int64_t* inv_off;
  int whole;
  // transfer to the child level
  int child_kind;
  const int32_t* agg;
  const int64_t* mem_ptr;
  const int32_t* mem;
  int nstages;
  int64_t elim_nnz;
  StageV stages[kMaxStages];
  double* stage_rhs[kMaxStages];
  double* stage_x[kMaxStages];
};

struct Workspace;

struct TailPlan {
  int first = 1 << 30;  // first level handled on-device (>= nlevels: none)
  int32_t small_rows = 4096;  // levels this small run in CTA 0 alone
  int ctas = 64;
  int smem = kTailSmemMax;  // bytes of dynamic shared memory per tail CTA
  int32_t xs_rows = 0;      // CTA-scope sweeps keep x and b of levels this small in shared memory
                            // (K > 1 cluster tail: subtrees rooted at levels of at most this many
                            // rows are handed to the CTAs as 4-column slices, see SliceScope)
  bool occ2 = true;         // two tail CTAs per SM (64-register variant)
  int K = 1;                // right-hand sides per block (batch.cuh)
  int threads = 512;        // per tail CTA
  bool subtree = false;     // K > 1: plain launch, one column slice per CTA, CTA scope only
  bool slice = false;       // K > 1 (default): K/4 independent CTAs on node-major 4-column slices
  const void* kernel = nullptr;
  DVec<TLevel> dlevels;
  DVec<double> credits;
  DVec<double> part;
  DVec<double> root_b, root_x;  // K > 1: column-major root vectors
  DVec<int32_t> sl_tabs;        // per-level colour tables of the slice sweeps
  DVec<TailCounters> ctr;
  void build(Ctx& c, const DHier& h, Workspace& ws, int32_t max_rows);
  void reset(Ctx& c);
  void run(Ctx& c, int l, int theta, double mu, int nlevels);
  void print_debug(const TailCounters& h) const;
  void collect(Ctx& c, double* work, int* relax_sweeps);
};

}  // namespace lamgb
