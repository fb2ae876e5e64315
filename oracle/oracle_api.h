/* oracle/oracle_api.h -- TEST INFRASTRUCTURE ONLY (the parity checker).
 *
 * The flat C API shared by both CPU oracles:
 *   - liblamg_oracle.so  (prefix orc_): oracle/lamg_oracle.c, a plain-C
 *     restatement of the reference algorithms, and
 *   - _ref/liblamg_ref.so (prefix ref_): oracle/ref_capi.cpp, a thin wrapper
 *     over the UNMODIFIED reference sources under /root/reference/proj/core
 *     compiled with -Dlamg=lamg_ref (recipe: oracle/Makefile).
 * Identical signatures let the Python harness (oracle/oracle.py) drive either
 * one and cross-check them. Nothing on the product path links this.
 *
 * CSR arguments follow lamg::SparseLaplacian
 * (/root/reference/proj/core/include/lamg/sparse_laplacian.hpp:18-39):
 * int64 row_ptr[n+1], int32 col[2m], f64 val[2m] (= -w), f64 diag[n].
 */
#ifndef LAMG_ORACLE_API_H
#define LAMG_ORACLE_API_H

#include <stdint.h>

#include "bag.h"

#ifndef ORACLE_PREFIX
#error "define ORACLE_PREFIX (orc_ or ref_)"
#endif
#define ORACLE_CAT2(a, b) a##b
#define ORACLE_CAT(a, b) ORACLE_CAT2(a, b)
#define OAPI(name) ORACLE_CAT(ORACLE_PREFIX, name)

#define CSR_ARGS \
  int32_t n, int64_t m, const int64_t *rp, const int32_t *col, const double *val, const double *diag

/* status codes, shared with include/lamg_b200.h */
enum {
  ORC_OK = 0,
  ORC_E_ERROR = 1,
  ORC_E_EMPTY_GRAPH = 2,
  ORC_E_SINGULAR_DIAGONAL = 3,
  ORC_E_INVALID_LAPLACIAN = 4,
  ORC_E_DIMENSION_MISMATCH = 5,
  ORC_E_INCOMPATIBLE_RHS = 6,
  ORC_E_DIVERGED = 7,
};

#ifdef __cplusplus
extern "C" {
#endif

/* bag access (bag.h) re-exported under the prefix */
int64_t OAPI(bag_len)(const bag *b, const char *name);
int OAPI(bag_type)(const bag *b, const char *name);
int OAPI(bag_get)(const bag *b, const char *name, void *dst);
int OAPI(bag_count)(const bag *b);
const char *OAPI(bag_name)(const bag *b, int i);
void OAPI(bag_free)(bag *b);

const char *OAPI(last_error)(void);

/* rng.hpp:10-41 */
uint64_t OAPI(rng_derive)(uint64_t seed, uint64_t stream);
void OAPI(rng_draws)(uint64_t seed, int64_t count, int kind /*0 u64, 1 unit, 2 pm1*/, void *out);

/* sparse_laplacian.cpp */
int OAPI(validate)(CSR_ARGS);
int OAPI(mvm)(CSR_ARGS, const double *x, double *y);
int OAPI(residual)(CSR_ARGS, const double *b, const double *x, double *r);
int OAPI(energy)(CSR_ARGS, const double *x, double *e);
int OAPI(vec_stats)(int64_t len, const double *x, double *sum, double *norm2);
int OAPI(subtract_mean)(int64_t len, double *x);

/* smoothing.cpp */
int OAPI(gs_sweep)(CSR_ARGS, const double *b /*nullable*/, double *x, int backward);
int OAPI(generate_tvs)(CSR_ARGS, int count, int sweeps, uint64_t seed, double *out /*count*n, col-major*/);
int OAPI(probe)(CSR_ARGS, int sweeps, uint64_t seed, double *factor);

/* aggregation.cpp */
int OAPI(affinities)(CSR_ARGS, int K, const double *tvs, bag **out);
int OAPI(detect_hubs)(CSR_ARGS, bag **out);
int OAPI(energy_ratio_qus)(CSR_ARGS, int K, const double *tvs, int32_t u, int32_t s, double *q);
int OAPI(aggregate)(CSR_ARGS, int K, const double *tvs, double gamma, const int32_t *hubs,
                    int32_t nhubs, bag **out);
int OAPI(galerkin)(CSR_ARGS, const int32_t *aggregate_of, int32_t coarse_n, bag **out);
int OAPI(restrict_residual)(const int32_t *aggregate_of, int32_t fine_n, int32_t coarse_n,
                            const double *r, double *rc);
int OAPI(add_interpolated)(const int32_t *aggregate_of, int32_t fine_n, const double *ec,
                           double *x);

/* elimination.cpp */
int OAPI(select_low_degree)(CSR_ARGS, int32_t max_degree, bag **out);
int OAPI(schur)(CSR_ARGS, const int32_t *f, int32_t nf, const int32_t *c, int32_t nc, bag **out);
int OAPI(eliminate_rounds)(CSR_ARGS, bag **out);
#define STAGE_ARGS                                                                               \
  int32_t parent_n, int32_t coarse_n, int32_t nf, const int32_t *f_nodes, const double *f_diag, \
      const int64_t *f_ptr, const int32_t *f_nbr, const double *f_val,                          \
      const int32_t *coarse_of_parent, const int32_t *parent_of_coarse
int OAPI(coarsen_rhs_stage)(STAGE_ARGS, const double *b, double *bc);
int OAPI(backsub_stage)(STAGE_ARGS, const double *xc, const double *b, double *x);

/* coarse_solver.cpp */
int OAPI(coarsest_direct)(CSR_ARGS, const double *b, double *x);
int OAPI(coarsest_relax)(CSR_ARGS, const double *b, double *x);

/* cycle.cpp */
double OAPI(flat_mu)(double q);
int OAPI(credit_takes)(double gamma, int count, int32_t *out);
int OAPI(recombine)(CSR_ARGS, const double *b, int cols, const double *saved_x,
                    const double *saved_r, double *x, double *before, double *after);

/* hierarchy.cpp / cycle.cpp drivers */
void *OAPI(setup)(CSR_ARGS, double gamma, uint64_t seed, int32_t coarsest_n, int tv_sweeps,
                  int tv_count_finest, int tv_count_max);
int OAPI(setup_status)(void); /* status of the last setup() call */
int OAPI(hier_export)(void *h, bag **out);
double OAPI(level_cycle_index)(void *h, int32_t l, double gamma);
int OAPI(solve)(void *h, const double *b, const double *x0, int correction, double mu,
                int max_cycles, double target_reduction, double divergence_factor, double gamma,
                uint64_t seed, double *x, bag **stats);
void OAPI(hier_free)(void *h);

/* solver.cpp whole-problem driver */
void *OAPI(prepare)(CSR_ARGS, double gamma, uint64_t seed, int32_t coarsest_n, int tv_sweeps,
                    int tv_count_finest, int tv_count_max, int correction, double mu,
                    int max_cycles, double target_reduction, double divergence_factor,
                    double cycle_gamma, uint64_t cycle_seed);
int OAPI(prepared_export)(void *p, bag **out);
int OAPI(solve_prepared)(void *p, const double *b, const double *x0 /*nullable*/, double *x,
                         bag **report);
void OAPI(prepared_free)(void *p);

/* CPU-baseline helper: solves nrhs independent right-hand sides over one const
 * hierarchy with nthreads host threads (solve is reentrant);
 * returns wall seconds and per-RHS cycle counts. */
int OAPI(solve_batch)(void *h, int nrhs, const double *B, const double *X0, int correction,
                      double mu, int max_cycles, double target_reduction,
                      double divergence_factor, double gamma, uint64_t seed, int nthreads,
                      double *seconds, int32_t *cycles);

#ifdef __cplusplus
}
#endif

#endif
