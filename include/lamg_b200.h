/* include/lamg_b200.h -- C-ABI of the B200-native LAMG hot path.
 *
 * liblamg_b200.so (paper_1108_1310_b200/liblamg_b200.so) implements the
 * data-parallel kernels of Lean Algebraic Multigrid for graph Laplacians
 * (setup: elimination, test vectors, affinity, aggregation, Galerkin; solve:
 * residual, Gauss-Seidel, transfers, energy-corrected cycle) as hand-written
 * sm_100a CUDA. The reference has no plugin/FFI layer: its boundary is the
 * C++ API in /root/reference/proj/core/include/lamg/ (*.hpp). Each entry point
 * below names the reference interface it replaces; include/lamg_b200/lamg.hpp
 * re-exposes them with the reference's exact C++ signatures.
 *
 * Conventions:
 *  - plain pointers and sizes only; CSR arrays follow lamg::SparseLaplacian
 *    (sparse_laplacian.hpp:18-39): int64 row_ptr[n+1], int32 col[2m],
 *    f64 val[2m] (= -w), f64 diag[n];
 *  - every call returns a status (LAMG_OK or one code per reference exception
 *    type, errors.hpp:13-42 / cycle.hpp:50-53); lamg_last_error() returns the
 *    reference's message text for the failure (thread-local);
 *  - a lamg_ctx is one device + one CUDA stream, used by one host thread at a
 *    time; a lamg_hier is device-resident, library-owned and immutable after
 *    setup, so concurrent solves over one hierarchy are allowed from distinct
 *    contexts on the same device;
 *  - "host" arrays may be pageable or pinned; lamg_solve_dev takes device
 *    pointers for callers that keep vectors resident in HBM.
 */
#ifndef LAMG_B200_H
#define LAMG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (one per reference exception type) */
enum {
  LAMG_OK = 0,
  LAMG_E_ERROR = 1,              /* lamg::Error */
  LAMG_E_EMPTY_GRAPH = 2,        /* lamg::EmptyGraphError */
  LAMG_E_SINGULAR_DIAGONAL = 3,  /* lamg::SingularDiagonalError */
  LAMG_E_INVALID_LAPLACIAN = 4,  /* lamg::InvalidLaplacianError */
  LAMG_E_DIMENSION_MISMATCH = 5, /* lamg::DimensionMismatchError */
  LAMG_E_INCOMPATIBLE_RHS = 6,   /* lamg::IncompatibleRhsError */
  LAMG_E_DIVERGED = 7,           /* lamg::DivergedError (stats still filled) */
  LAMG_E_PARSE = 8,              /* lamg::ParseError */
  LAMG_E_IO = 9,                 /* lamg::IoError */
  LAMG_E_CUDA = 10,
  LAMG_E_NCCL = 11,
  LAMG_E_ARGUMENT = 12
};

/* execution modes */
enum {
  /* exact-order Gauss-Seidel, sequential folds, LU substitution: the solve is
   * bit-identical to the reference */
  LAMG_MODE_VALIDATE = 0,
  /* graph-coloured Gauss-Seidel on colour-permuted levels, fixed-order tree
   * reductions, fused transfers: a different smoother, same hierarchy */
  LAMG_MODE_THROUGHPUT = 1
};

typedef struct lamg_ctx lamg_ctx;
typedef struct lamg_hier lamg_hier;
typedef struct lamg_graph lamg_graph; /* a device-resident CSR Laplacian (graph ingest) */

typedef struct {
  int32_t n;
  int64_t m;
  const int64_t *row_ptr;
  const int32_t *col;
  const double *val;
  const double *diag;
} lamg_csr;

/* == lamg::SetupOptions (hierarchy.hpp:52-59) */
typedef struct {
  double gamma;
  uint64_t rng_seed;
  int32_t coarsest_n;
  int32_t tv_sweeps;
  int32_t tv_count_finest;
  int32_t tv_count_max;
} lamg_setup_opts;

/* == lamg::CycleConfig (cycle.hpp:28-36); correction 0 Flat, 1 AdaptiveRecombination */
typedef struct {
  double gamma; /* unused by the cycle, as in the reference */
  int32_t correction;
  double mu;
  int32_t max_cycles;
  double target_reduction;
  double divergence_factor;
  uint64_t rng_seed;
} lamg_cycle_cfg;

/* == lamg::SolveStats (cycle.hpp:38-46); residuals go to a caller buffer */
typedef struct {
  double acf;
  double solve_work;
  int32_t cycles;
  int32_t converged;
  int64_t recombinations;
  double recomb_max_growth;
  int32_t nresiduals; /* r_0..r_p count (may exceed the caller's capacity) */
  int32_t relax_sweeps; /* total relaxation-coarsest sweeps (diagnostic) */
} lamg_solve_stats;

/* == lamg::Level metadata (hierarchy.hpp:24-37) plus transfer summaries */
typedef struct {
  int32_t kind; /* 0 finest, 1 elimination, 2 aggregation, 3 coarsest */
  int32_t n;
  int64_t m;
  double gamma;
  int32_t nu_pre, nu_post, tv_count;
  int32_t coarsest; /* 0 none, 1 direct, 2 relaxation */
  int32_t nstages;  /* elimination stages (kind 1) */
  int32_t coarse_n; /* aggregation: coarse_n (kind 2) */
  double alpha;
  int32_t stage_used;
  int32_t dummy_aggregate;
  int32_t gs_fronts; /* exact-order Gauss-Seidel wavefronts of this level */
  int32_t colors;    /* throughput-mode colours (0 if not built) */
} lamg_level_info;

/* ---- context ---------------------------------------------------------- */
int lamg_ctx_create(int device, int mode, lamg_ctx **out);
int lamg_ctx_set_mode(lamg_ctx *ctx, int mode);
/* THROUGHPUT solves: how many of the finest SMOOTHING levels keep the
 * reference's Gauss-Seidel row order (default 1; 0 = every level greedy-
 * coloured). The first smoothing level's order decides the cycle count
 * (config 2: 129 = the reference's, greedy-coloured 141; RGG 2^20: 13 vs 15).
 * Those levels are swept with colours = wavefront mod 32 (the reference's
 * order except at the wrap; environment LAMG_FRONT_MOD, 0 = exact order:
 * wavefront kernel for one column, ticketed wavefront items for blocks), and
 * in exact order where that is not a proper colouring. Partitioned solves
 * sweep greedy-coloured. */
int lamg_ctx_set_exact_levels(lamg_ctx *ctx, int32_t levels);
void lamg_ctx_destroy(lamg_ctx *ctx);
const char *lamg_last_error(void);
const char *lamg_version(void);
/* kernels this library has launched so far (all contexts, monotone) */
int64_t lamg_launch_count(void);
/* LAMG_GUARD=1 (debugging aid): device buffers carry 256-byte guard bands checked at
 * release; buffers checked so far and overruns found (also reported on stderr) */
void lamg_guard_report(int64_t *checked, int64_t *overruns);
/* the context's cudaStream_t, for callers that time or order work with it */
void *lamg_ctx_stream(lamg_ctx *ctx);

/* ---- setup: replaces lamg::setup (hierarchy.hpp:65; hierarchy.cpp:59-138) */
int lamg_setup(lamg_ctx *ctx, const lamg_csr *a, int on_device, const lamg_setup_opts *opts,
               lamg_hier **out);
void lamg_hier_destroy(lamg_hier *h);
/* Hierarchy/HierarchyStats fields (hierarchy.hpp:39-50, 67-86) */
int lamg_hier_info(const lamg_hier *h, int32_t *nlevels, double *setup_work, int32_t *nwarnings,
                   double *setup_seconds);
int lamg_hier_warning(const lamg_hier *h, int32_t i, char *buf, int32_t cap);
int lamg_hier_level_info(const lamg_hier *h, int32_t level, lamg_level_info *out);
/* level_cycle_index (hierarchy.hpp:91; hierarchy.cpp:31-40) */
int lamg_level_cycle_index(const lamg_hier *h, int32_t level, double gamma, double *out);
/* parity downloads of the integer and value artefacts */
int lamg_hier_download_op(const lamg_hier *h, int32_t level, int64_t *row_ptr, int32_t *col,
                          double *val, double *diag);
int lamg_hier_download_agg(const lamg_hier *h, int32_t level, int32_t *aggregate_of,
                           int32_t *seed_of);
int lamg_hier_stage_info(const lamg_hier *h, int32_t level, int32_t stage, int32_t *parent_n,
                         int32_t *coarse_n, int32_t *nf, int64_t *nnz_f);
int lamg_hier_download_stage(const lamg_hier *h, int32_t level, int32_t stage, int32_t *f_nodes,
                             double *f_diag, int64_t *f_ptr, int32_t *f_nbr, double *f_val,
                             int32_t *coarse_of_parent, int32_t *parent_of_coarse);

/* ---- solve: replaces lamg::solve (cycle.hpp:58-59; cycle.cpp:221-273) ---- */
int lamg_solve(lamg_ctx *ctx, const lamg_hier *h, const double *b, const double *x0,
               const lamg_cycle_cfg *cfg, double *x, lamg_solve_stats *stats, double *residuals,
               int32_t residuals_cap);
/* same with device-resident b, x0, x (inputs already in HBM) */
int lamg_solve_dev(lamg_ctx *ctx, const lamg_hier *h, const double *d_b, const double *d_x0,
                   const lamg_cycle_cfg *cfg, double *d_x, lamg_solve_stats *stats,
                   double *residuals, int32_t residuals_cap);
/* nrhs independent right-hand sides (cycle.cpp:221-273 per column; the
 * reference runs one solve per RHS). b, x0, x are
 * RHS-major [nrhs][n]; stats[nrhs]; residuals [nrhs][residuals_cap].
 * THROUGHPUT mode + flat cycle: blocks of up to 32 columns share every
 * kernel of the cycle (node-major n x K vectors on the device); each column
 * is returned at the cycle its own convergence test fires. Otherwise: one
 * solve per column (VALIDATE: each bit-identical to the reference). */
int lamg_solve_batch(lamg_ctx *ctx, const lamg_hier *h, int32_t nrhs, const double *b,
                     const double *x0, const lamg_cycle_cfg *cfg, double *x,
                     lamg_solve_stats *stats, double *residuals, int32_t residuals_cap);
int lamg_solve_batch_dev(lamg_ctx *ctx, const lamg_hier *h, int32_t nrhs, const double *d_b,
                         const double *d_x0, const lamg_cycle_cfg *cfg, double *d_x,
                         lamg_solve_stats *stats, double *residuals, int32_t residuals_cap);
/* ---- graph ingest on the device -----------------
 * R-MAT of BASELINE.json config 5: 2^scale nodes,
 * edge_factor*2^scale samples, quadrant per bit by draw t*S+i of the
 * counter-form lamg::Rng(seed) (rng.hpp:10-41) against a, a+b, a+b+c;
 * self-loops dropped, duplicates summed into integer weights; keep_lcc keeps
 * the largest component in ascending node order (components.cpp:35-56).
 * lamg_graph_lcc does the component step alone for any CSR Laplacian.
 * lamg_graph_csr gives device pointers for lamg_setup(..., on_device=1, ...). */
int lamg_gen_rmat(lamg_ctx *ctx, int32_t scale, int32_t edge_factor, double a, double b, double c,
                  uint64_t seed, int32_t keep_lcc, lamg_graph **out);
/* BASELINE config 4 (Chung-Lu): cdf[n] = normalised cumulative expected
 * degrees (host-computed, as graphs.chung_lu); `pairs` endpoint pairs drawn
 * on the device by inverse CDF, self-loops dropped, duplicates merged to
 * unit weight, largest component kept */
int lamg_gen_chung_lu(lamg_ctx *ctx, int32_t n, const double *cdf, int64_t pairs, uint64_t seed,
                      int32_t keep_lcc, lamg_graph **out);
int lamg_graph_lcc(lamg_ctx *ctx, const lamg_csr *a, int on_device, lamg_graph **out);
int lamg_graph_csr(const lamg_graph *g, lamg_csr *out_device_view);
int lamg_graph_download(const lamg_graph *g, int64_t *row_ptr, int32_t *col, double *val, double *diag);
void lamg_graph_destroy(lamg_graph *g);

/* builds (once) the throughput-mode colour-permuted copies of the hierarchy */
int lamg_hier_prepare_throughput(lamg_ctx *ctx, lamg_hier *h);

/* THROUGHPUT smoother of one hierarchy level, for parity tests: the colour
 * order (row_ids[n]: natural row of each stored row; color_ptr[ncolors+1])
 * and `sweeps` coloured Gauss-Seidel sweeps on host vectors. nrhs == 1: b, x
 * are [n]; nrhs in {4,8,16,32}: node-major [n][nrhs]. A coloured sweep is
 * gauss_seidel_sweep (smoothing.cpp:13-40) in colour-permuted row order. */
int lamg_hier_color_count(const lamg_hier *h, int32_t level, int32_t *ncolors);
int lamg_hier_download_colors(const lamg_hier *h, int32_t level, int32_t *row_ids, int32_t *color_ptr);
int lamg_hier_smooth(lamg_ctx *ctx, const lamg_hier *h, int32_t level, int32_t nrhs, const double *b,
                     double *x, int32_t sweeps);
/* the same in the reference's exact row order (gauss_seidel_sweep,
 * smoothing.cpp:29-40, per column): nrhs == 1 the wavefront kernel; nrhs in
 * {4,8,16,32} the ticketed K-column sweep the THROUGHPUT block solve uses on
 * its exact levels. Bit-identical per column to the reference sweep. */
int lamg_hier_smooth_exact(lamg_ctx *ctx, const lamg_hier *h, int32_t level, int32_t nrhs, const double *b,
                           double *x, int32_t sweeps);

/* ---- fine-level node-block partition with halo exchange (SURVEY 8(e)
 * mode 2). A level operator split into `nparts` contiguous row blocks
 * (bounds[nparts+1], balanced by rows + entries); block p is a local CSR over
 * [owned rows | ghost columns]. A coloured sweep exchanges ghosts after every
 * colour (NCCL send/recv between ranks, or -- comm == NULL -- every part
 * owned by this process on its device). Results are bit-identical to the
 * single-device THROUGHPUT smoother and residual. ---------------------- */
typedef struct lamg_comm lamg_comm;
typedef struct lamg_part_level lamg_part_level;
int lamg_comm_unique_id(char id[128]);                           /* ncclGetUniqueId */
int lamg_comm_create(lamg_ctx *ctx, int32_t nranks, int32_t rank, const char id[128], lamg_comm **out);
void lamg_comm_destroy(lamg_comm *comm);
/* host-only (no GPU): the partition plan */
int lamg_part_bounds(int32_t n, const int64_t *row_ptr, int32_t nparts, int32_t *bounds);
int lamg_part_plan_sizes(const lamg_csr *a, const int32_t *bounds, int32_t nparts, int32_t part, int32_t *nloc,
                         int32_t *nghost, int64_t *nnz, int32_t *nsend);
int lamg_part_plan(const lamg_csr *a, const int32_t *bounds, int32_t nparts, int32_t part, int64_t *row_ptr,
                   int32_t *col, int32_t *ghost_gid, int32_t *recv_ptr, int32_t *send_ptr, int32_t *send_idx);
/* device: a (host CSR, the whole level) is partitioned by bounds; this
 * process owns parts [first_part, first_part + nown). The communicator (if
 * any) must outlive the partition. */
int lamg_part_level_create(lamg_ctx *ctx, const lamg_csr *a, const int32_t *bounds, int32_t nparts,
                           int32_t first_part, int32_t nown, lamg_comm *comm, lamg_part_level **out);
/* the first smoothing level of a hierarchy, partitioned (bounds by
 * lamg_part_bounds): level 0 when its child is an aggregation level, level 1
 * when the finest level is reduced by elimination first (cycle.cpp:131-164);
 * lamg_part_level_n gives its size */
int lamg_part_level_from_hier(lamg_ctx *ctx, const lamg_hier *h, int32_t nparts, int32_t first_part,
                              int32_t nown, lamg_comm *comm, lamg_part_level **out);
void lamg_part_level_destroy(lamg_part_level *pl);
int32_t lamg_part_level_n(const lamg_part_level *pl);
/* lamg_solve with that level partitioned (THROUGHPUT, flat cycle): its
 * sweeps/residuals run on the parts, its residual is allgathered, the levels
 * below are replicated on every rank, and a finest level above it does its
 * RHS coarsening / injection / back-substitution replicated. A partitioned
 * relaxation-coarsest level (coarse_solver.cpp:82-93; configs 4 and 5) relaxes
 * on the parts. With an aggregation child the result is bit-identical to
 * lamg_solve on a context with lamg_ctx_set_exact_levels(ctx, 0) (the parts
 * sweep coloured); the relaxation form is bit-identical across part counts
 * and within rounding of lamg_solve. pl must have been built on ctx (and,
 * from a hierarchy, from h): LAMG_E_ARGUMENT otherwise. b, x0, x: full host
 * vectors of the finest level (every rank passes all of b). */
int lamg_part_solve(lamg_ctx *ctx, const lamg_hier *h, lamg_part_level *pl, const double *b, const double *x0,
                    const lamg_cycle_cfg *cfg, double *x, lamg_solve_stats *stats, double *residuals,
                    int32_t cap);
/* global host vectors [n]: owned rows are read (b, x) and written (x, r) */
int lamg_part_smooth(lamg_part_level *pl, const double *b, double *x, int32_t sweeps);
int lamg_part_residual(lamg_part_level *pl, const double *b, const double *x, double *r);
/* device-resident timing of `sweeps` partitioned sweeps (+ one residual) */
int lamg_part_time(lamg_part_level *pl, int32_t sweeps, float *ms);

/* ---- Matrix Market files (matrix_market.hpp:34-52): read_matrix_market_file
 * + assemble_problem -> a host CSR Laplacian, and write_matrix_market_file.
 * kind: 0 auto, 1 adjacency, 2 laplacian. Lines are parsed by all host
 * threads; the assembled CSR and warnings equal the reference's. ----------- */
typedef struct lamg_mm lamg_mm;
int lamg_mm_read(const char *path, int32_t kind, int32_t absolute_weight_policy, lamg_mm **out);
int lamg_mm_info(const lamg_mm *mm, int32_t *n, int64_t *m, int32_t *was_laplacian, int32_t *nwarnings);
int lamg_mm_warning(const lamg_mm *mm, int32_t i, char *buf, int32_t cap);
int lamg_mm_csr(const lamg_mm *mm, int64_t *row_ptr, int32_t *col, double *val, double *diag);
void lamg_mm_destroy(lamg_mm *mm);
int lamg_mm_write(const char *path, const lamg_csr *a, int32_t as_laplacian);

/* ---- kernel timing (bench roofline): CUDA events around the finest-level
 * residual and Gauss-Seidel launches of the solves issued on ctx ---------- */
int lamg_ctx_profile(lamg_ctx *ctx, int enable);
int lamg_ctx_profile_read(lamg_ctx *ctx, int kernel /*0 gs, 1 residual*/, int64_t *launches,
                          double *total_ms, double *bytes_per_launch);

/* ---- per-kernel entry points (parity harness; host pointers in and out).
 * Each replaces the named reference function on one operator. ------------- */
int lamg_k_validate(lamg_ctx *ctx, const lamg_csr *a);                      /* validate_laplacian */
int lamg_k_mvm(lamg_ctx *ctx, const lamg_csr *a, const double *x, double *y); /* mvm */
int lamg_k_residual(lamg_ctx *ctx, const lamg_csr *a, const double *b, const double *x,
                    double *r);                                              /* residual */
int lamg_k_energy(lamg_ctx *ctx, const lamg_csr *a, const double *x, double *e); /* energy */
int lamg_k_gs_sweep(lamg_ctx *ctx, const lamg_csr *a, const double *b /*nullable*/, double *x,
                    int backward);                                            /* gauss_seidel_sweep */
int lamg_k_generate_tvs(lamg_ctx *ctx, const lamg_csr *a, int32_t count, int32_t sweeps,
                        uint64_t seed, double *out /*count*n, column k at out+k*n*/);
int lamg_k_probe(lamg_ctx *ctx, const lamg_csr *a, int32_t sweeps, uint64_t seed, double *factor);
int lamg_k_affinities(lamg_ctx *ctx, const lamg_csr *a, int32_t K, const double *tvs,
                      double *edge_affinity, double *node_norm, int32_t *degenerate,
                      int32_t *ndegenerate);                                   /* compute_affinities */
int lamg_k_detect_hubs(lamg_ctx *ctx, const lamg_csr *a, int32_t *hubs, int32_t *nhubs);
int lamg_k_aggregate(lamg_ctx *ctx, const lamg_csr *a, int32_t K, const double *tvs, double gamma,
                     const int32_t *hubs, int32_t nhubs, int32_t *aggregate_of, int32_t *seed_of,
                     int32_t *coarse_n, double *alpha, int32_t *stage_used,
                     int32_t *dummy_aggregate);                                /* aggregate */
/* galerkin_coarse_operator / schur_reduce produce a CSR held by the context
 * until lamg_k_take_csr copies it out (sizes via lamg_k_result_dims) */
int lamg_k_galerkin(lamg_ctx *ctx, const lamg_csr *a, const int32_t *aggregate_of,
                    int32_t coarse_n);
int lamg_k_select_low_degree(lamg_ctx *ctx, const lamg_csr *a, int32_t max_degree, int32_t *f,
                             int32_t *nf, int32_t *c, int32_t *nc);
int lamg_k_schur(lamg_ctx *ctx, const lamg_csr *a, const int32_t *f, int32_t nf, const int32_t *c,
                 int32_t nc, int32_t *f_diag_ok /*unused, may be NULL*/);
int lamg_k_result_dims(lamg_ctx *ctx, int32_t *n, int64_t *m, int64_t *nnz_f);
int lamg_k_take_csr(lamg_ctx *ctx, int64_t *row_ptr, int32_t *col, double *val, double *diag);
int lamg_k_take_stage(lamg_ctx *ctx, double *f_diag, int64_t *f_ptr, int32_t *f_nbr,
                      double *f_val, int32_t *coarse_of_parent);
int lamg_k_restrict(lamg_ctx *ctx, const int32_t *aggregate_of, int32_t fine_n, int32_t coarse_n,
                    const double *r, double *rc);                             /* restrict_residual */
int lamg_k_interpolate(lamg_ctx *ctx, const int32_t *aggregate_of, int32_t fine_n,
                       int32_t coarse_n, const double *ec, double *x);        /* add_interpolated */
int lamg_k_coarsen_rhs(lamg_ctx *ctx, int32_t parent_n, int32_t coarse_n, int32_t nf,
                       const int32_t *f_nodes, const double *f_diag, const int64_t *f_ptr,
                       const int32_t *f_nbr, const double *f_val, const int32_t *coarse_of_parent,
                       const int32_t *parent_of_coarse, const double *b, double *bc);
int lamg_k_backsub(lamg_ctx *ctx, int32_t parent_n, int32_t coarse_n, int32_t nf,
                   const int32_t *f_nodes, const double *f_diag, const int64_t *f_ptr,
                   const int32_t *f_nbr, const double *f_val, const int32_t *coarse_of_parent,
                   const int32_t *parent_of_coarse, const double *xc, const double *b, double *x);
int lamg_k_coarsest_direct(lamg_ctx *ctx, const lamg_csr *a, const double *b, double *x);
int lamg_k_coarsest_relax(lamg_ctx *ctx, const lamg_csr *a, const double *b, double *x);
int lamg_k_recombine(lamg_ctx *ctx, const lamg_csr *a, const double *b, int32_t cols,
                     const double *saved_x, const double *saved_r, double *x, double *before,
                     double *after);                                          /* recombine */
/* host-side helpers (no device work): LevelCredit::take, flat_mu, Rng::derive */
int lamg_credit_takes(double gamma, int32_t count, int32_t *out);
double lamg_flat_mu(double q);
uint64_t lamg_rng_derive(uint64_t seed, uint64_t stream);

#ifdef __cplusplus
}
#endif

#endif /* LAMG_B200_H */
