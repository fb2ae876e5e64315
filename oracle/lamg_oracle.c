/* oracle/lamg_oracle.c -- TEST INFRASTRUCTURE ONLY: the CPU parity oracle.
 *
 * A plain-C restatement of the LAMG reference algorithms on the north_star
 * hot path (setup + solve of a connected graph Laplacian), written from the
 * reference's behaviour, each function citing the reference file:line it
 * follows (paths relative to /root/reference/proj/core/). It is pinned
 * bit-for-bit against the compiled reference (oracle/_ref, see Makefile) and
 * against the golden fixtures in tests/golden/ by tests/test_oracle_pin.py.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
 * load it. The product (paper_1108_1310_b200/) never links or calls it.
 *
 * Floating-point rules mirrored from the reference build (SURVEY.md facts
 * 7-8): every expression is evaluated in source order with no FMA contraction
 * (ISO C mode => -ffp-contract=off), every reduction is a left-to-right fold,
 * and the hash-map accumulations of the reference (Schur, Galerkin) are
 * restated as stable sort by key + in-order fold, which is the same
 * per-key sequence of additions.
 */
#define _POSIX_C_SOURCE 200809L
#define ORACLE_PREFIX orc_
#include "oracle_api.h"

#include <math.h>
#include <pthread.h>
#include <setjmp.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------------ */
/* errors: the reference throws typed exceptions (include/lamg/errors.hpp);  */
/* here an error longjmps to the API entry, which returns the status code.  */

static _Thread_local char g_err[512];
static _Thread_local jmp_buf *g_jb;

static void throwf(int code, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  longjmp(*g_jb, code);
}

#define API_BEGIN            \
  jmp_buf jb_;               \
  jmp_buf *prev_jb_ = g_jb;  \
  g_jb = &jb_;               \
  int code_ = setjmp(jb_);   \
  if (code_ == 0) {
#define API_END              \
  g_err[0] = 0;              \
  }                          \
  g_jb = prev_jb_;           \
  return code_;

static void *xmalloc(size_t bytes) {
  void *p = malloc(bytes ? bytes : 1);
  if (!p) throwf(ORC_E_ERROR, "out of memory");
  return p;
}
static void *xcalloc(size_t count, size_t size) {
  void *p = calloc(count ? count : 1, size ? size : 1);
  if (!p) throwf(ORC_E_ERROR, "out of memory");
  return p;
}
#define NEW(T, count) ((T *)xmalloc(sizeof(T) * (size_t)(count)))
#define ZNEW(T, count) ((T *)xcalloc((size_t)(count), sizeof(T)))

/* ------------------------------------------------------------------------ */
/* work accounting: work.cpp:6-11 (thread-local edge units)                  */

static _Thread_local double g_work;
static void work_add(double units) { g_work += units; }

/* ------------------------------------------------------------------------ */
/* Rng: include/lamg/rng.hpp:10-41 (splitmix64 with two warm-up draws)        */

#define GOLDEN 0x9e3779b97f4a7c15ULL
typedef struct { uint64_t state; } rng_t;

static uint64_t rng_next_u64(rng_t *r) {
  uint64_t z = (r->state += GOLDEN);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static rng_t rng_make(uint64_t seed) {
  rng_t r = {seed ? seed : GOLDEN};
  rng_next_u64(&r);
  rng_next_u64(&r);
  return r;
}
static double rng_unit(rng_t *r) { return (double)(rng_next_u64(r) >> 11) * 0x1.0p-53; }
static double rng_pm1(rng_t *r) { return 2.0 * rng_unit(r) - 1.0; }
static uint64_t rng_derive(uint64_t seed, uint64_t stream) {
  rng_t r = rng_make(seed ^ (0xd1342543de82ef95ULL * (stream + 1)));
  return rng_next_u64(&r);
}

/* ------------------------------------------------------------------------ */
/* CSR Laplacian: include/lamg/sparse_laplacian.hpp:18-39                     */

typedef struct {
  int32_t n;
  int64_t m;
  int64_t *rp;
  int32_t *col;
  double *val;
  double *diag;
  int owned;
} csr_t;

static csr_t csr_view(CSR_ARGS) {
  csr_t a = {n, m, (int64_t *)rp, (int32_t *)col, (double *)val, (double *)diag, 0};
  return a;
}
static void csr_free(csr_t *a) {
  if (a->owned) {
    free(a->rp);
    free(a->col);
    free(a->val);
    free(a->diag);
  }
  memset(a, 0, sizeof *a);
}
static csr_t csr_clone(const csr_t *a) {
  csr_t c = *a;
  c.rp = NEW(int64_t, a->n + 1);
  c.col = NEW(int32_t, 2 * a->m);
  c.val = NEW(double, 2 * a->m);
  c.diag = NEW(double, a->n);
  memcpy(c.rp, a->rp, sizeof(int64_t) * (size_t)(a->n + 1));
  memcpy(c.col, a->col, sizeof(int32_t) * (size_t)(2 * a->m));
  memcpy(c.val, a->val, sizeof(double) * (size_t)(2 * a->m));
  memcpy(c.diag, a->diag, sizeof(double) * (size_t)a->n);
  c.owned = 1;
  return c;
}
static int32_t degree(const csr_t *a, int32_t u) { return (int32_t)(a->rp[u + 1] - a->rp[u]); }

/* sparse_laplacian.cpp:47-51 */
static double max_diag(const csr_t *a) {
  double md = 0.0;
  for (int32_t u = 0; u < a->n; ++u) {
    double d = fabs(a->diag[u]);
    if (md < d) md = d;
  }
  return md;
}

typedef struct {
  int32_t u, v;
  double w;
} wedge_t;

/* sparse_laplacian.cpp:60-104 -- CSR from a canonical (u<v, sorted, merged)
 * edge list; diag[x] accumulates w in edge order, i.e. ascending column. */
static int cmp_colval(const void *pa, const void *pb) {
  const int32_t ca = *(const int32_t *)pa, cb = *(const int32_t *)pb;
  if (ca != cb) return ca < cb ? -1 : 1;
  const double va = *(const double *)((const char *)pa + 8), vb = *(const double *)((const char *)pb + 8);
  return va < vb ? -1 : (vb < va ? 1 : 0);
}
static csr_t assemble_canonical(int32_t n, const wedge_t *e, int64_t ne) {
  if (n <= 0) throwf(ORC_E_EMPTY_GRAPH, "cannot assemble a Laplacian with n = 0");
  csr_t a;
  a.n = n;
  a.m = ne;
  a.owned = 1;
  a.rp = ZNEW(int64_t, n + 1);
  for (int64_t i = 0; i < ne; ++i) {
    ++a.rp[e[i].u + 1];
    ++a.rp[e[i].v + 1];
  }
  for (int32_t u = 0; u < n; ++u) a.rp[u + 1] += a.rp[u];
  a.col = NEW(int32_t, 2 * ne);
  a.val = NEW(double, 2 * ne);
  a.diag = ZNEW(double, n);
  int64_t *fill = NEW(int64_t, n);
  memcpy(fill, a.rp, sizeof(int64_t) * (size_t)n);
  for (int64_t i = 0; i < ne; ++i) {
    a.col[fill[e[i].u]] = e[i].v;
    a.val[fill[e[i].u]++] = -e[i].w;
    a.col[fill[e[i].v]] = e[i].u;
    a.val[fill[e[i].v]++] = -e[i].w;
    a.diag[e[i].u] += e[i].w;
    a.diag[e[i].v] += e[i].w;
  }
  free(fill);
  for (int32_t u = 0; u < n; ++u) {
    int64_t b = a.rp[u], en = a.rp[u + 1];
    int sorted = 1;
    for (int64_t k = b + 1; k < en; ++k)
      if (a.col[k - 1] >= a.col[k]) {
        sorted = 0;
        break;
      }
    if (sorted) continue;
    struct { int32_t c; int32_t pad; double v; } *row = xmalloc(16 * (size_t)(en - b));
    for (int64_t k = b; k < en; ++k) {
      row[k - b].c = a.col[k];
      row[k - b].v = a.val[k];
    }
    qsort(row, (size_t)(en - b), 16, cmp_colval);
    for (int64_t k = b; k < en; ++k) {
      a.col[k] = row[k - b].c;
      a.val[k] = row[k - b].v;
    }
    free(row);
  }
  return a;
}

/* sparse_laplacian.cpp:151-162 */
static void mvm(const csr_t *a, const double *x, double *y) {
  for (int32_t u = 0; u < a->n; ++u) {
    double s = a->diag[u] * x[u];
    for (int64_t k = a->rp[u]; k < a->rp[u + 1]; ++k) s += a->val[k] * x[a->col[k]];
    y[u] = s;
  }
  work_add((double)a->m);
}

/* sparse_laplacian.cpp:170-175 */
static void residual(const csr_t *a, const double *b, const double *x, double *r) {
  mvm(a, x, r);
  for (int32_t u = 0; u < a->n; ++u) r[u] = b[u] - r[u];
}

/* sparse_laplacian.cpp:177-192 */
static double energy(const csr_t *a, const double *x) {
  double e = 0.0;
  for (int32_t u = 0; u < a->n; ++u)
    for (int64_t k = a->rp[u]; k < a->rp[u + 1]; ++k) {
      int32_t v = a->col[k];
      if (v <= u) continue;
      double d = x[u] - x[v];
      e += -a->val[k] * d * d;
    }
  work_add((double)a->m);
  return e;
}

/* sparse_laplacian.cpp:236-252 */
static double norm2(const double *x, int64_t len) {
  double s = 0.0;
  for (int64_t i = 0; i < len; ++i) s += x[i] * x[i];
  return sqrt(s);
}
static double vec_sum(const double *x, int64_t len) {
  double s = 0.0;
  for (int64_t i = 0; i < len; ++i) s += x[i];
  return s;
}
static void subtract_mean(double *x, int64_t len) {
  if (len == 0) return;
  double mean = vec_sum(x, len) / (double)len;
  for (int64_t i = 0; i < len; ++i) x[i] -= mean;
}

/* sparse_laplacian.cpp:194-234 (same checks, same order, same messages) */
static void validate_laplacian(const csr_t *a) {
  if (a->n <= 0) throwf(ORC_E_INVALID_LAPLACIAN, "empty matrix");
  double md = max_diag(a);
  const double tol = 1e-10 * (md < 1e-300 ? 1e-300 : md);
  for (int32_t u = 0; u < a->n; ++u) {
    double row_sum = a->diag[u];
    for (int64_t k = a->rp[u]; k < a->rp[u + 1]; ++k) {
      int32_t v = a->col[k];
      if (v == u) throwf(ORC_E_INVALID_LAPLACIAN, "self entry stored in row %d", u);
      if (v < 0 || v >= a->n) throwf(ORC_E_INVALID_LAPLACIAN, "column out of range");
      if (k > a->rp[u] && a->col[k - 1] >= v)
        throwf(ORC_E_INVALID_LAPLACIAN, "row %d not strictly sorted", u);
      int64_t lo = a->rp[v], hi = a->rp[v + 1];
      while (lo < hi) { /* lower_bound of u in row v */
        int64_t mid = lo + (hi - lo) / 2;
        if (a->col[mid] < u) lo = mid + 1;
        else hi = mid;
      }
      if (lo == a->rp[v + 1] || a->col[lo] != u)
        throwf(ORC_E_INVALID_LAPLACIAN, "structural asymmetry at (%d,%d)", u, v);
      if (a->val[lo] != a->val[k]) throwf(ORC_E_INVALID_LAPLACIAN, "value asymmetry at (%d,%d)", u, v);
      row_sum += a->val[k];
    }
    if (fabs(row_sum) > tol)
      throwf(ORC_E_INVALID_LAPLACIAN, "row %d sum %f exceeds tolerance", u, row_sum);
    if (degree(a, u) > 0 && a->diag[u] <= 0.0)
      throwf(ORC_E_INVALID_LAPLACIAN, "non-positive diagonal at non-isolated node %d", u);
  }
}

/* ------------------------------------------------------------------------ */
/* smoothing.cpp                                                             */

/* smoothing.cpp:13-25 */
static void gs_update(const csr_t *a, const double *b, double *x, int32_t u) {
  double s = b ? b[u] : 0.0;
  for (int64_t k = a->rp[u]; k < a->rp[u + 1]; ++k) s -= a->val[k] * x[a->col[k]];
  if (a->diag[u] == 0.0) {
    if (degree(a, u) == 0) return;
    throwf(ORC_E_SINGULAR_DIAGONAL, "zero diagonal at node %d", u);
  }
  x[u] = s / a->diag[u];
}

/* smoothing.cpp:29-40 */
static void gs_sweep(const csr_t *a, const double *b, double *x, int backward) {
  if (!backward)
    for (int32_t u = 0; u < a->n; ++u) gs_update(a, b, x, u);
  else
    for (int32_t u = a->n; u-- > 0;) gs_update(a, b, x, u);
  work_add((double)a->m);
}

/* smoothing.cpp:42-57; columns stored back to back (column k at out + k*n) */
static void generate_tvs(const csr_t *a, int count, int sweeps, uint64_t seed, double *out) {
  for (int k = 0; k < count; ++k) {
    rng_t r = rng_make(rng_derive(seed, (uint64_t)k));
    double *x = out + (int64_t)k * a->n;
    for (int32_t u = 0; u < a->n; ++u) x[u] = rng_pm1(&r);
    for (int s = 0; s < sweeps; ++s) gs_sweep(a, NULL, x, 0);
    subtract_mean(x, a->n);
  }
}

/* smoothing.cpp:59-89 */
static double a_norm(const csr_t *a, const double *x) {
  double e = energy(a, x);
  return e > 0.0 ? sqrt(e) : 0.0;
}
static double probe_relaxation(const csr_t *a, int sweeps, uint64_t seed) {
  rng_t r = rng_make(rng_derive(seed, 0x9));
  double *x = NEW(double, a->n);
  for (int32_t u = 0; u < a->n; ++u) x[u] = rng_pm1(&r);
  subtract_mean(x, a->n);
  int half = sweeps / 2;
  double norm_mid = 0.0;
  for (int s = 0; s < sweeps; ++s) {
    gs_sweep(a, NULL, x, 0);
    subtract_mean(x, a->n);
    if (s + 1 == half) norm_mid = a_norm(a, x);
  }
  double norm_end = a_norm(a, x);
  free(x);
  if (half == 0) norm_mid = 0.0;
  if (norm_end == 0.0 || norm_mid == 0.0) return 0.0;
  return pow(norm_end / norm_mid, 1.0 / (double)(sweeps - half));
}

/* ------------------------------------------------------------------------ */
/* aggregation.cpp                                                           */

/* aggregation.cpp:83-116 */
static void compute_affinities(const csr_t *a, int K, const double *tvs, double *aff,
                               double *nn_out, int32_t *degen, int32_t *ndegen) {
  int32_t nd = 0;
  for (int32_t u = 0; u < a->n; ++u) {
    double nn = 0.0;
    for (int k = 0; k < K; ++k) {
      double x = tvs[(int64_t)k * a->n + u];
      nn += x * x;
    }
    nn_out[u] = nn;
    if (nn == 0.0) {
      if (degen) degen[nd] = u;
      ++nd;
    }
  }
  if (ndegen) *ndegen = nd;
  for (int32_t u = 0; u < a->n; ++u)
    for (int64_t k = a->rp[u]; k < a->rp[u + 1]; ++k) {
      int32_t v = a->col[k];
      if (v <= u) continue;
      double c;
      if (nn_out[u] == 0.0 || nn_out[v] == 0.0) {
        c = 1.0;
      } else {
        double dot = 0.0;
        for (int q = 0; q < K; ++q) dot += tvs[(int64_t)q * a->n + u] * tvs[(int64_t)q * a->n + v];
        c = 1.0 - (dot * dot) / (nn_out[u] * nn_out[v]);
        c = c < 0.0 ? 0.0 : (1.0 < c ? 1.0 : c); /* std::clamp */
      }
      aff[k] = c;
      int64_t lo = a->rp[v], hi = a->rp[v + 1]; /* mirror_entry, aggregation.cpp:18-22 */
      while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (a->col[mid] < u) lo = mid + 1;
        else hi = mid;
      }
      aff[lo] = c;
    }
  work_add((double)K * (double)a->m);
}

/* aggregation.cpp:118-134 */
static int32_t detect_hubs(const csr_t *a, int32_t *hubs) {
  int32_t nh = 0;
  for (int32_t u = 0; u < a->n; ++u) {
    if (degree(a, u) == 0) continue;
    double num = 0.0, den = 0.0;
    for (int64_t k = a->rp[u]; k < a->rp[u + 1]; ++k) {
      double aw = fabs(a->val[k]);
      num += aw * (double)degree(a, a->col[k]);
      den += aw;
    }
    if (den == 0.0) continue;
    if ((double)degree(a, u) >= 8.0 * num / den) hubs[nh++] = u;
  }
  return nh;
}

/* NodalQuadratic, aggregation.cpp:26-79 */
typedef struct {
  double a_uu;
  double *b, *c, *relaxed_min;
} quad_t;

static void quad_build(quad_t *q, const csr_t *a, int K, const double *tvs, int32_t u) {
  q->a_uu = a->diag[u];
  for (int k = 0; k < K; ++k) q->b[k] = q->c[k] = q->relaxed_min[k] = 0.0;
  for (int64_t j = a->rp[u]; j < a->rp[u + 1]; ++j) {
    double w = -a->val[j];
    int32_t v = a->col[j];
    for (int k = 0; k < K; ++k) {
      double xv = tvs[(int64_t)k * a->n + v];
      q->b[k] += w * xv;
      q->c[k] += 0.5 * w * xv * xv;
    }
  }
  for (int k = 0; k < K; ++k)
    q->relaxed_min[k] = q->a_uu > 0.0 ? q->c[k] - q->b[k] * q->b[k] / (2.0 * q->a_uu) : q->c[k];
}
static double quad_at(const quad_t *q, double y, int k) {
  return 0.5 * q->a_uu * y * y - q->b[k] * y + q->c[k];
}
static double quad_ratio_vs(const quad_t *q, const csr_t *a, int K, const double *tvs, int32_t s) {
  double r = -INFINITY;
  for (int k = 0; k < K; ++k) {
    double den = quad_at(q, tvs[(int64_t)k * a->n + s], k);
    if (den <= 0.0) return INFINITY;
    double v = q->relaxed_min[k] / den;
    if (r < v) r = v;
  }
  return r;
}
static double quad_inflation_vs(const quad_t *q, const csr_t *a, int K, const double *tvs, int32_t s) {
  double r = -INFINITY;
  for (int k = 0; k < K; ++k) {
    double relaxed = q->relaxed_min[k];
    if (relaxed <= 0.0) continue;
    double v = quad_at(q, tvs[(int64_t)k * a->n + s], k) / relaxed;
    if (r < v) r = v;
  }
  return r == -INFINITY ? 1.0 : r;
}

typedef struct {
  int32_t fine_n, coarse_n;
  int32_t *aggregate_of;
  int32_t *seed_of;
  int stage_used;
  double alpha;
  int32_t dummy_aggregate;
} aggt_t;

typedef struct {
  double key;
  int32_t u;
} order_t;
static int cmp_order(const void *pa, const void *pb) {
  const order_t *x = pa, *y = pb;
  if (x->key < y->key) return -1;
  if (y->key < x->key) return 1;
  return (x->u > y->u) - (x->u < y->u);
}

enum { UNDECIDED = 0, SEED = 1, ASSOCIATE = 2 };

/* aggregation.cpp:142-278 (both stages run exactly as the reference does) */
static aggt_t aggregate(const csr_t *a, int K, const double *tvs, double gamma,
                        const int32_t *hubs, int32_t nhubs) {
  const int32_t n = a->n;
  double *aff = NEW(double, 2 * a->m + 1);
  double *nn = NEW(double, n);
  compute_affinities(a, K, tvs, aff, nn, NULL, NULL);
  double *strongest = ZNEW(double, n);
  for (int32_t u = 0; u < n; ++u)
    for (int64_t k = a->rp[u]; k < a->rp[u + 1]; ++k) {
      double e = fabs(a->val[k]);
      if (strongest[u] < e) strongest[u] = e;
    }
#define USABLE(u, v, entry)                                                             \
  (fabs(entry) >= 1e-3 * (strongest[(v)] < strongest[(u)] ? strongest[(v)] : strongest[(u)]))
  char *dummy = ZNEW(char, n);
  int32_t dummy_count = 0;
  for (int32_t u = 0; u < n; ++u) {
    int any = 0;
    for (int64_t k = a->rp[u]; k < a->rp[u + 1] && !any; ++k) any = USABLE(u, a->col[k], a->val[k]);
    dummy[u] = any ? 0 : 1;
    dummy_count += dummy[u];
  }
  char *status = ZNEW(char, n);
  int32_t *seed_ref = NEW(int32_t, n);
  for (int32_t u = 0; u < n; ++u) seed_ref[u] = -1;
  for (int32_t i = 0; i < nhubs; ++i)
    if (!dummy[hubs[i]]) status[hubs[i]] = SEED;

  const double alpha_max = 0.7 / gamma;
  char *res_status[2] = {NULL, NULL};
  int32_t *res_seed[2] = {NULL, NULL};
  double res_alpha[2] = {0, 0};
  int nres = 0;
  order_t *order = NEW(order_t, n);
  quad_t q;
  q.b = NEW(double, K);
  q.c = NEW(double, K);
  q.relaxed_min = NEW(double, K);
  for (int stage = 1; stage <= 2; ++stage) {
    int32_t no = 0;
    for (int32_t u = 0; u < n; ++u) {
      if (dummy[u] || status[u] != UNDECIDED) continue;
      double best = INFINITY;
      for (int64_t j = a->rp[u]; j < a->rp[u + 1]; ++j) {
        if (!USABLE(u, a->col[j], a->val[j]) || dummy[a->col[j]]) continue;
        if (aff[j] < best) best = aff[j];
      }
      if (best < INFINITY) {
        order[no].key = best;
        order[no].u = u;
        ++no;
      }
    }
    qsort(order, (size_t)no, sizeof(order_t), cmp_order);
    for (int32_t i = 0; i < no; ++i) {
      int32_t u = order[i].u;
      if (status[u] != UNDECIDED) continue;
      quad_build(&q, a, K, tvs, u);
      int32_t best_s = -1;
      double best_c = INFINITY;
      for (int64_t j = a->rp[u]; j < a->rp[u + 1]; ++j) {
        int32_t s = a->col[j];
        if (dummy[s] || status[s] == ASSOCIATE) continue;
        if (!USABLE(u, s, a->val[j])) continue;
        double c = aff[j];
        if (c < best_c || (c == best_c && s < best_s)) {
          if (quad_inflation_vs(&q, a, K, tvs, s) <= 2.5) {
            best_c = c;
            best_s = s;
          }
        }
      }
      if (best_s >= 0) {
        if (status[best_s] == UNDECIDED) status[best_s] = SEED;
        status[u] = ASSOCIATE;
        seed_ref[u] = best_s;
      }
    }
    int32_t count = dummy_count > 0 ? 1 : 0;
    for (int32_t u = 0; u < n; ++u)
      if (!dummy[u] && status[u] != ASSOCIATE) ++count;
    double alpha = n > 0 ? (double)count / (double)n : 1.0;
    res_status[nres] = NEW(char, n);
    memcpy(res_status[nres], status, (size_t)n);
    res_seed[nres] = NEW(int32_t, n);
    memcpy(res_seed[nres], seed_ref, sizeof(int32_t) * (size_t)n);
    res_alpha[nres] = alpha;
    ++nres;
    if (alpha <= alpha_max) break;
  }
  work_add((double)K * (double)a->m * (double)nres);
  int pick = 0;
  for (int i = 1; i < nres; ++i)
    if (fabs(res_alpha[i] - alpha_max) < fabs(res_alpha[pick] - alpha_max)) pick = i;
  memcpy(status, res_status[pick], (size_t)n);
  memcpy(seed_ref, res_seed[pick], sizeof(int32_t) * (size_t)n);

  aggt_t t;
  t.fine_n = n;
  t.stage_used = pick + 1;
  t.dummy_aggregate = -1;
  t.aggregate_of = NEW(int32_t, n);
  t.seed_of = NEW(int32_t, n + 1);
  for (int32_t u = 0; u < n; ++u) t.aggregate_of[u] = -1;
  int32_t next = 0;
  for (int32_t u = 0; u < n; ++u) {
    if (dummy[u]) {
      if (t.dummy_aggregate < 0) {
        t.dummy_aggregate = next++;
        t.seed_of[t.dummy_aggregate] = -1;
      }
      t.aggregate_of[u] = t.dummy_aggregate;
    } else if (status[u] != ASSOCIATE) {
      t.aggregate_of[u] = next;
      t.seed_of[next] = u;
      ++next;
    }
  }
  for (int32_t u = 0; u < n; ++u)
    if (!dummy[u] && status[u] == ASSOCIATE) {
      int32_t s = seed_ref[u];
      if (s < 0 || t.aggregate_of[s] < 0) throwf(ORC_E_ERROR, "aggregate: associate without a seed");
      t.aggregate_of[u] = t.aggregate_of[s];
    }
  t.coarse_n = next;
  t.alpha = n > 0 ? (double)next / (double)n : 1.0;
#undef USABLE
  for (int i = 0; i < nres; ++i) {
    free(res_status[i]);
    free(res_seed[i]);
  }
  free(order);
  free(q.b);
  free(q.c);
  free(q.relaxed_min);
  free(status);
  free(seed_ref);
  free(dummy);
  free(strongest);
  free(aff);
  free(nn);
  return t;
}

/* keyed contribution for the hash-map restatements: sorting by (key, seq)
 * reproduces "per key, in emission order" (unordered_map += semantics). */
typedef struct {
  uint64_t key;
  int64_t seq;
  double w;
} contrib_t;
static int cmp_contrib(const void *pa, const void *pb) {
  const contrib_t *x = pa, *y = pb;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return (x->seq > y->seq) - (x->seq < y->seq);
}
static uint64_t pair_key(int32_t u, int32_t v) {
  if (u > v) {
    int32_t t = u;
    u = v;
    v = t;
  }
  return ((uint64_t)(uint32_t)u << 32) | (uint32_t)v;
}
/* folds sorted contributions per key from 0.0, drops exact zeros, emits the
 * canonical edge list sorted by (u,v): elimination.cpp:93-101, aggregation.cpp:293-501 */
static wedge_t *fold_contribs(contrib_t *cb, int64_t nc, int64_t *ne_out) {
  qsort(cb, (size_t)nc, sizeof(contrib_t), cmp_contrib);
  wedge_t *e = NEW(wedge_t, nc);
  int64_t ne = 0;
  for (int64_t i = 0; i < nc;) {
    int64_t j = i;
    double w = 0.0;
    while (j < nc && cb[j].key == cb[i].key) w += cb[j++].w;
    if (w != 0.0) {
      e[ne].u = (int32_t)(cb[i].key >> 32);
      e[ne].v = (int32_t)(cb[i].key & 0xffffffffu);
      e[ne].w = w;
      ++ne;
    }
    i = j;
  }
  *ne_out = ne;
  return e;
}

/* aggregation.cpp:280-313 */
static csr_t galerkin(const csr_t *a, const int32_t *agg, int32_t coarse_n) {
  contrib_t *cb = NEW(contrib_t, a->m + 1);
  int64_t nc = 0;
  for (int32_t u = 0; u < a->n; ++u)
    for (int64_t j = a->rp[u]; j < a->rp[u + 1]; ++j) {
      int32_t v = a->col[j];
      if (v <= u) continue;
      int32_t cu = agg[u], cv = agg[v];
      if (cu == cv) continue;
      cb[nc].key = pair_key(cu, cv);
      cb[nc].seq = nc;
      cb[nc].w = -a->val[j];
      ++nc;
    }
  int64_t ne;
  wedge_t *e = fold_contribs(cb, nc, &ne);
  free(cb);
  csr_t c = assemble_canonical(coarse_n, e, ne);
  free(e);
  work_add((double)a->m);
  return c;
}

/* aggregation.cpp:333-342 */
static void add_interpolated(const int32_t *agg, int32_t fine_n, const double *ec, double *x) {
  for (int32_t u = 0; u < fine_n; ++u) x[u] += ec[agg[u]];
}
static void restrict_residual(const int32_t *agg, int32_t fine_n, int32_t coarse_n, const double *r,
                              double *rc) {
  for (int32_t i = 0; i < coarse_n; ++i) rc[i] = 0.0;
  for (int32_t u = 0; u < fine_n; ++u) rc[agg[u]] += r[u];
}

/* ------------------------------------------------------------------------ */
/* elimination.cpp                                                           */

typedef struct {
  int32_t parent_n, coarse_n, nf;
  int32_t *f_nodes;
  double *f_diag;
  int64_t *f_ptr;
  int32_t *f_nbr;
  double *f_val;
  int32_t *coarse_of_parent;
  int32_t *parent_of_coarse;
} stage_t;

static void stage_free(stage_t *s) {
  free(s->f_nodes);
  free(s->f_diag);
  free(s->f_ptr);
  free(s->f_nbr);
  free(s->f_val);
  free(s->coarse_of_parent);
  free(s->parent_of_coarse);
}

/* elimination.cpp:11-27 */
static void select_low_degree(const csr_t *a, int32_t max_degree, int32_t *f, int32_t *nf,
                              int32_t *c, int32_t *nc) {
  char *eligible = NEW(char, a->n);
  char *in_f = ZNEW(char, a->n);
  memset(eligible, 1, (size_t)a->n);
  *nf = *nc = 0;
  for (int32_t u = 0; u < a->n; ++u) {
    int32_t deg = degree(a, u);
    if (!eligible[u] || deg == 0 || deg > max_degree || a->diag[u] <= 0.0) continue;
    in_f[u] = 1;
    f[(*nf)++] = u;
    for (int64_t k = a->rp[u]; k < a->rp[u + 1]; ++k) eligible[a->col[k]] = 0;
  }
  for (int32_t u = 0; u < a->n; ++u)
    if (!in_f[u]) c[(*nc)++] = u;
  free(eligible);
  free(in_f);
}

/* elimination.cpp:29-105 */
static csr_t schur_reduce(const csr_t *a, const int32_t *f, int32_t nf, const int32_t *c, int32_t nc,
                          stage_t *st) {
  st->parent_n = a->n;
  st->coarse_n = nc;
  st->nf = nf;
  st->coarse_of_parent = NEW(int32_t, a->n);
  for (int32_t u = 0; u < a->n; ++u) st->coarse_of_parent[u] = -1;
  st->parent_of_coarse = NEW(int32_t, nc);
  memcpy(st->parent_of_coarse, c, sizeof(int32_t) * (size_t)nc);
  for (int32_t k = 0; k < nc; ++k) st->coarse_of_parent[c[k]] = k;
  st->f_nodes = NEW(int32_t, nf);
  memcpy(st->f_nodes, f, sizeof(int32_t) * (size_t)nf);
  st->f_diag = NEW(double, nf);
  st->f_ptr = NEW(int64_t, nf + 1);
  int64_t cap = 0;
  for (int32_t i = 0; i < nf; ++i) cap += degree(a, f[i]);
  st->f_nbr = NEW(int32_t, cap);
  st->f_val = NEW(double, cap);
  st->f_ptr[0] = 0;
  int64_t nn = 0;
  for (int32_t i = 0; i < nf; ++i) {
    int32_t fu = f[i];
    if (st->coarse_of_parent[fu] >= 0) throwf(ORC_E_ERROR, "schur_reduce: F and C overlap at node %d", fu);
    if (a->diag[fu] <= 0.0)
      throwf(ORC_E_SINGULAR_DIAGONAL, "schur_reduce: non-positive pivot at node %d", fu);
    st->f_diag[i] = a->diag[fu];
    for (int64_t k = a->rp[fu]; k < a->rp[fu + 1]; ++k) {
      if (st->coarse_of_parent[a->col[k]] < 0)
        throwf(ORC_E_ERROR, "schur_reduce: F is not independent, edge (%d,%d)", fu, a->col[k]);
      st->f_nbr[nn] = a->col[k];
      st->f_val[nn] = a->val[k];
      ++nn;
    }
    st->f_ptr[i + 1] = nn;
  }
  int64_t ncap = a->m;
  for (int32_t i = 0; i < nf; ++i) {
    int64_t d = st->f_ptr[i + 1] - st->f_ptr[i];
    ncap += d * (d - 1) / 2;
  }
  contrib_t *cb = NEW(contrib_t, ncap + 1);
  int64_t ncb = 0;
  for (int32_t i = 0; i < nc; ++i) { /* retained C-C edges, elimination.cpp:72-80 */
    int32_t cu = c[i];
    for (int64_t k = a->rp[cu]; k < a->rp[cu + 1]; ++k) {
      int32_t v = a->col[k];
      if (st->coarse_of_parent[v] < 0) continue;
      if (v > cu) {
        cb[ncb].key = pair_key(st->coarse_of_parent[cu], st->coarse_of_parent[v]);
        cb[ncb].seq = ncb;
        cb[ncb].w = -a->val[k];
        ++ncb;
      }
    }
  }
  for (int32_t i = 0; i < nf; ++i) { /* fill cliques, elimination.cpp:81-91 */
    double aff = st->f_diag[i];
    for (int64_t p = st->f_ptr[i]; p < st->f_ptr[i + 1]; ++p)
      for (int64_t q = p + 1; q < st->f_ptr[i + 1]; ++q) {
        int32_t cu = st->coarse_of_parent[st->f_nbr[p]];
        int32_t cv = st->coarse_of_parent[st->f_nbr[q]];
        cb[ncb].key = pair_key(cu, cv);
        cb[ncb].seq = ncb;
        cb[ncb].w = (st->f_val[p] * st->f_val[q]) / aff;
        ++ncb;
      }
  }
  int64_t ne;
  wedge_t *e = fold_contribs(cb, ncb, &ne);
  free(cb);
  csr_t coarse = assemble_canonical(nc, e, ne);
  free(e);
  work_add((double)(a->m + coarse.m));
  return coarse;
}

/* elimination.cpp:107-124 */
typedef struct {
  stage_t *stages;
  int nstages;
  csr_t coarse;
} elimt_t;

static int eliminate_rounds(const csr_t *a, elimt_t *t) {
  t->stages = NULL;
  t->nstages = 0;
  memset(&t->coarse, 0, sizeof t->coarse);
  const csr_t *cur = a;
  int32_t *f = NEW(int32_t, a->n), *c = NEW(int32_t, a->n);
  while (cur->n > 1) {
    int32_t nf, nc;
    select_low_degree(cur, 4, f, &nf, c, &nc);
    if ((double)nf < 0.01 * cur->n || nf == 0 || nc == 0) break;
    t->stages = realloc(t->stages, sizeof(stage_t) * (size_t)(t->nstages + 1));
    csr_t next = schur_reduce(cur, f, nf, c, nc, &t->stages[t->nstages]);
    ++t->nstages;
    if (t->coarse.owned) csr_free(&t->coarse);
    t->coarse = next;
    cur = &t->coarse;
  }
  free(f);
  free(c);
  return t->nstages > 0;
}

/* elimination.cpp:126-140 */
static void coarsen_rhs_stage(const stage_t *s, const double *b, double *bc) {
  for (int32_t k = 0; k < s->coarse_n; ++k) bc[k] = b[s->parent_of_coarse[k]];
  for (int32_t i = 0; i < s->nf; ++i) {
    double scaled = b[s->f_nodes[i]] / s->f_diag[i];
    for (int64_t p = s->f_ptr[i]; p < s->f_ptr[i + 1]; ++p)
      bc[s->coarse_of_parent[s->f_nbr[p]]] -= s->f_val[p] * scaled;
  }
  work_add((double)s->f_ptr[s->nf]);
}

/* elimination.cpp:158-173 */
static void backsub_stage(const stage_t *s, const double *xc, const double *b, double *x) {
  for (int32_t u = 0; u < s->parent_n; ++u) x[u] = 0.0;
  for (int32_t k = 0; k < s->coarse_n; ++k) x[s->parent_of_coarse[k]] = xc[k];
  for (int32_t i = 0; i < s->nf; ++i) {
    double sum = b[s->f_nodes[i]];
    for (int64_t p = s->f_ptr[i]; p < s->f_ptr[i + 1]; ++p) sum -= s->f_val[p] * x[s->f_nbr[p]];
    x[s->f_nodes[i]] = sum / s->f_diag[i];
  }
  work_add((double)s->f_ptr[s->nf]);
}

/* ------------------------------------------------------------------------ */
/* components.cpp (needed by the coarsest direct solver and the driver)     */

typedef struct {
  int32_t count;
  int32_t *label;
  int32_t *start; /* nodes of component c are nodes[start[c] .. start[c+1]) ascending */
  int32_t *nodes;
} split_t;

/* components.cpp:9-33 */
static split_t connected_components(const csr_t *a) {
  split_t s;
  s.count = 0;
  s.label = NEW(int32_t, a->n);
  for (int32_t u = 0; u < a->n; ++u) s.label[u] = -1;
  int32_t *queue = NEW(int32_t, a->n);
  for (int32_t st = 0; st < a->n; ++st) {
    if (s.label[st] >= 0) continue;
    int32_t id = s.count++;
    s.label[st] = id;
    int32_t qn = 0;
    queue[qn++] = st;
    for (int32_t h = 0; h < qn; ++h) {
      int32_t u = queue[h];
      for (int64_t k = a->rp[u]; k < a->rp[u + 1]; ++k)
        if (s.label[a->col[k]] < 0) {
          s.label[a->col[k]] = id;
          queue[qn++] = a->col[k];
        }
    }
  }
  free(queue);
  s.start = ZNEW(int32_t, s.count + 1);
  for (int32_t u = 0; u < a->n; ++u) ++s.start[s.label[u] + 1];
  for (int32_t c = 0; c < s.count; ++c) s.start[c + 1] += s.start[c];
  s.nodes = NEW(int32_t, a->n);
  int32_t *fill = NEW(int32_t, s.count + 1);
  memcpy(fill, s.start, sizeof(int32_t) * (size_t)(s.count + 1));
  for (int32_t u = 0; u < a->n; ++u) s.nodes[fill[s.label[u]]++] = u;
  free(fill);
  return s;
}
static void split_free(split_t *s) {
  free(s->label);
  free(s->start);
  free(s->nodes);
}

static int cmp_wedge(const void *pa, const void *pb) {
  const wedge_t *x = pa, *y = pb;
  if (x->u != y->u) return x->u < y->u ? -1 : 1;
  return (x->v > y->v) - (x->v < y->v);
}

/* components.cpp:35-56 */
static csr_t extract_component(const csr_t *a, const int32_t *nodes, int32_t nn) {
  int32_t *local = NEW(int32_t, a->n);
  for (int32_t u = 0; u < a->n; ++u) local[u] = -1;
  for (int32_t k = 0; k < nn; ++k) local[nodes[k]] = k;
  int64_t cap = 0;
  for (int32_t k = 0; k < nn; ++k) cap += degree(a, nodes[k]);
  wedge_t *e = NEW(wedge_t, cap + 1);
  int64_t ne = 0;
  for (int32_t lu = 0; lu < nn; ++lu) {
    int32_t u = nodes[lu];
    for (int64_t k = a->rp[u]; k < a->rp[u + 1]; ++k) {
      int32_t lv = local[a->col[k]];
      if (lv < 0) throwf(ORC_E_ERROR, "extract_component: node set is not closed under adjacency");
      if (lv > lu) {
        e[ne].u = lu;
        e[ne].v = lv;
        e[ne].w = -a->val[k];
        ++ne;
      }
    }
  }
  qsort(e, (size_t)ne, sizeof(wedge_t), cmp_wedge);
  csr_t s = assemble_canonical(nn, e, ne);
  free(e);
  free(local);
  return s;
}

/* ------------------------------------------------------------------------ */
/* coarse_solver.cpp                                                         */

typedef struct {
  int32_t cn;      /* component size */
  int32_t *nodes;  /* NULL means "all nodes" */
  double *lu;      /* (cn+1)^2 row-major, unblocked partial-pivot LU (eigen_shim) */
  int32_t *perm;
} dcomp_t;

typedef struct {
  int mode; /* 1 direct, 2 relaxation */
  int32_t n;
  int64_t m;
  dcomp_t *comps;
  int32_t ncomps;
  csr_t relax_op; /* relaxation keeps its own copy (coarse_solver.cpp:94) */
} coarsest_t;

/* coarse_solver.cpp:14-24 + the shim's PartialPivLU (oracle/eigen_shim/Eigen/Dense) */
static void bordered_lu(const csr_t *a, dcomp_t *dc) {
  const int32_t N = a->n + 1;
  double *M = ZNEW(double, (int64_t)N * N);
  for (int32_t u = 0; u < a->n; ++u) {
    M[(int64_t)u * N + u] = a->diag[u];
    for (int64_t k = a->rp[u]; k < a->rp[u + 1]; ++k) M[(int64_t)u * N + a->col[k]] = a->val[k];
    M[(int64_t)u * N + a->n] = 1.0;
    M[(int64_t)a->n * N + u] = 1.0;
  }
  int32_t *perm = NEW(int32_t, N);
  for (int32_t i = 0; i < N; ++i) perm[i] = i;
  for (int32_t k = 0; k < N; ++k) {
    int32_t p = k;
    double best = fabs(M[(int64_t)k * N + k]);
    for (int32_t i = k + 1; i < N; ++i) {
      double v = fabs(M[(int64_t)i * N + k]);
      if (v > best) {
        best = v;
        p = i;
      }
    }
    if (p != k) {
      for (int32_t j = 0; j < N; ++j) {
        double t = M[(int64_t)k * N + j];
        M[(int64_t)k * N + j] = M[(int64_t)p * N + j];
        M[(int64_t)p * N + j] = t;
      }
      int32_t t = perm[k];
      perm[k] = perm[p];
      perm[p] = t;
    }
    double piv = M[(int64_t)k * N + k];
    if (piv == 0.0) continue;
    for (int32_t i = k + 1; i < N; ++i) {
      double l = M[(int64_t)i * N + k] / piv;
      M[(int64_t)i * N + k] = l;
      for (int32_t j = k + 1; j < N; ++j) M[(int64_t)i * N + j] -= l * M[(int64_t)k * N + j];
    }
  }
  dc->lu = M;
  dc->perm = perm;
}
static void lu_solve(const dcomp_t *dc, const double *rhs, double *y) {
  const int32_t N = dc->cn + 1;
  const double *M = dc->lu;
  for (int32_t i = 0; i < N; ++i) {
    double s = rhs[dc->perm[i]];
    for (int32_t j = 0; j < i; ++j) s -= M[(int64_t)i * N + j] * y[j];
    y[i] = s;
  }
  for (int32_t i = N; i-- > 0;) {
    double s = y[i];
    for (int32_t j = i + 1; j < N; ++j) s -= M[(int64_t)i * N + j] * y[j];
    y[i] = s / M[(int64_t)i * N + i];
  }
}

/* coarse_solver.cpp:26-76 */
static coarsest_t *make_direct(const csr_t *a) {
  coarsest_t *cs = ZNEW(coarsest_t, 1);
  cs->mode = 1;
  cs->n = a->n;
  cs->m = a->m;
  split_t sp = connected_components(a);
  if (sp.count == 1) {
    cs->ncomps = 1;
    cs->comps = ZNEW(dcomp_t, 1);
    cs->comps[0].cn = a->n;
    cs->comps[0].nodes = NULL;
    bordered_lu(a, &cs->comps[0]);
  } else {
    cs->ncomps = sp.count;
    cs->comps = ZNEW(dcomp_t, sp.count);
    for (int32_t c = 0; c < sp.count; ++c) {
      int32_t cn = sp.start[c + 1] - sp.start[c];
      csr_t sub = extract_component(a, sp.nodes + sp.start[c], cn);
      cs->comps[c].cn = cn;
      cs->comps[c].nodes = NEW(int32_t, cn);
      memcpy(cs->comps[c].nodes, sp.nodes + sp.start[c], sizeof(int32_t) * (size_t)cn);
      bordered_lu(&sub, &cs->comps[c]);
      csr_free(&sub);
    }
  }
  split_free(&sp);
  double nn = (double)cs->n + 1.0;
  work_add(nn * nn * nn / 3.0);
  return cs;
}

/* coarse_solver.cpp:78-98 */
static coarsest_t *make_relaxation(const csr_t *a) {
  coarsest_t *cs = ZNEW(coarsest_t, 1);
  cs->mode = 2;
  cs->n = a->n;
  cs->m = a->m;
  cs->relax_op = csr_clone(a);
  return cs;
}

static void coarsest_solve(const coarsest_t *cs, const double *b, double *x) {
  if (cs->mode == 1) { /* coarse_solver.cpp:47-66 */
    for (int32_t c = 0; c < cs->ncomps; ++c) {
      const dcomp_t *dc = &cs->comps[c];
      double *rhs = NEW(double, dc->cn + 1), *sol = NEW(double, dc->cn + 1);
      for (int32_t k = 0; k < dc->cn; ++k) rhs[k] = dc->nodes ? b[dc->nodes[k]] : b[k];
      rhs[dc->cn] = 0.0;
      lu_solve(dc, rhs, sol);
      for (int32_t k = 0; k < dc->cn; ++k) {
        if (dc->nodes) x[dc->nodes[k]] = sol[k];
        else x[k] = sol[k];
      }
      free(rhs);
      free(sol);
    }
    work_add((double)cs->m);
  } else { /* coarse_solver.cpp:82-93 */
    const csr_t *a = &cs->relax_op;
    double *r = NEW(double, a->n);
    residual(a, b, x, r);
    double r0 = norm2(r, a->n);
    if (r0 != 0.0) {
      const double target = 1e-12 * r0;
      for (int sweep = 0; sweep < 400; ++sweep) {
        gs_sweep(a, b, x, 0);
        subtract_mean(x, a->n);
        residual(a, b, x, r);
        if (norm2(r, a->n) <= target) break;
      }
    }
    free(r);
  }
}

static void coarsest_free(coarsest_t *cs) {
  if (!cs) return;
  for (int32_t c = 0; c < cs->ncomps; ++c) {
    free(cs->comps[c].nodes);
    free(cs->comps[c].lu);
    free(cs->comps[c].perm);
  }
  free(cs->comps);
  csr_free(&cs->relax_op);
  free(cs);
}

/* ------------------------------------------------------------------------ */
/* hierarchy.hpp:24-50 / hierarchy.cpp                                       */

enum { K_FINEST = 0, K_ELIM = 1, K_AGG = 2, K_COARSEST = 3 };

typedef struct {
  int kind;
  csr_t op;
  int has_elim, has_agg;
  elimt_t elim; /* elim.coarse unused: the operator lives on the level */
  aggt_t agg;
  double gamma;
  int nu_pre, nu_post, tv_count;
  int coarsest; /* 0 none, 1 direct, 2 relaxation */
  coarsest_t *solver;
} level_t;

typedef struct {
  level_t *levels;
  int nlevels;
  double setup_work;
  uint64_t seed;
  int nwarnings;
} hier_t;

static level_t *push_level(hier_t *h) {
  h->levels = realloc(h->levels, sizeof(level_t) * (size_t)(h->nlevels + 1));
  level_t *L = &h->levels[h->nlevels++];
  memset(L, 0, sizeof *L);
  L->gamma = 1.0;
  return L;
}

/* hierarchy.cpp:31-40 */
static double level_cycle_index(const hier_t *h, int l, double gamma) {
  if (l + 1 >= h->nlevels) return 1.0;
  if (h->levels[l + 1].kind == K_ELIM) return 1.0;
  const double m1 = (double)h->levels[0].op.m;
  const double ml = (double)h->levels[l].op.m;
  const double mc = (double)h->levels[l + 1].op.m;
  if (ml > 0.1 * m1) return gamma;
  if (mc <= 0.0) return 1.0;
  double g = 0.7 * ml / mc;
  return 2.0 < g ? 2.0 : g;
}

/* hierarchy.cpp:49-55 */
static void mark_coarsest(hier_t *h, int mode) {
  level_t *L = &h->levels[h->nlevels - 1];
  L->coarsest = mode;
  L->solver = mode == 1 ? make_direct(&L->op) : make_relaxation(&L->op);
}

typedef struct {
  double gamma;
  uint64_t seed;
  int32_t coarsest_n;
  int tv_sweeps, tv_count_finest, tv_count_max;
} setup_opts_t;

/* hierarchy.cpp:59-138 */
static hier_t *setup(const csr_t *a, const setup_opts_t *o) {
  validate_laplacian(a);
  double w0 = g_work;
  hier_t *h = ZNEW(hier_t, 1);
  h->seed = o->seed;
  level_t *L0 = push_level(h);
  L0->kind = K_FINEST;
  L0->op = csr_clone(a);
  int stagnant_rounds = 0;
  while (h->nlevels < 100) {
    const csr_t *cur = &h->levels[h->nlevels - 1].op;
    if (cur->n <= o->coarsest_n) {
      mark_coarsest(h, 1);
      break;
    }
    elimt_t et;
    if (eliminate_rounds(cur, &et)) {
      level_t *L = push_level(h);
      L->kind = K_ELIM;
      L->op = et.coarse;
      validate_laplacian(&L->op);
      memset(&et.coarse, 0, sizeof et.coarse);
      L->has_elim = 1;
      L->elim = et;
      L->gamma = 1.0;
      continue;
    }
    uint64_t level_seed = rng_derive(o->seed, (uint64_t)h->nlevels);
    double factor = probe_relaxation(cur, 8, level_seed);
    if (factor <= 0.7) {
      mark_coarsest(h, 2);
      break;
    }
    int k = o->tv_count_finest + 2 * (h->nlevels - 1);
    if (k > o->tv_count_max) k = o->tv_count_max;
    double *tvs = NEW(double, (int64_t)k * cur->n);
    generate_tvs(cur, k, o->tv_sweeps, level_seed, tvs);
    int32_t *hubs = NEW(int32_t, cur->n);
    int32_t nh = detect_hubs(cur, hubs);
    aggt_t agg = aggregate(cur, k, tvs, o->gamma, hubs, nh);
    free(tvs);
    free(hubs);
    if (agg.coarse_n >= cur->n) {
      ++h->nwarnings;
      free(agg.aggregate_of);
      free(agg.seed_of);
      mark_coarsest(h, 1);
      break;
    }
    csr_t coarse = galerkin(cur, agg.aggregate_of, agg.coarse_n);
    level_t *L = push_level(h); /* may move `cur` */
    L->kind = K_AGG;
    L->op = coarse;
    validate_laplacian(&L->op);
    L->gamma = 1.0;
    L->nu_pre = 1;
    L->nu_post = 2;
    L->tv_count = k;
    int stagnant = agg.alpha > 0.95;
    L->has_agg = 1;
    L->agg = agg;
    if (stagnant && ++stagnant_rounds >= 2) {
      ++h->nwarnings;
      mark_coarsest(h, 1);
      break;
    }
  }
  if (h->levels[h->nlevels - 1].coarsest == 0) {
    ++h->nwarnings;
    mark_coarsest(h, 1);
  }
  for (int l = 0; l + 1 < h->nlevels; ++l) h->levels[l + 1].gamma = level_cycle_index(h, l, o->gamma);
  h->setup_work = (g_work - w0) / (double)h->levels[0].op.m;
  return h;
}

static void hier_free(hier_t *h) {
  if (!h) return;
  for (int l = 0; l < h->nlevels; ++l) {
    level_t *L = &h->levels[l];
    csr_free(&L->op);
    if (L->has_elim) {
      for (int s = 0; s < L->elim.nstages; ++s) stage_free(&L->elim.stages[s]);
      free(L->elim.stages);
    }
    if (L->has_agg) {
      free(L->agg.aggregate_of);
      free(L->agg.seed_of);
    }
    coarsest_free(L->solver);
  }
  free(h->levels);
  free(h);
}

/* ------------------------------------------------------------------------ */
/* cycle.cpp                                                                 */

typedef struct {
  int correction; /* 0 flat, 1 adaptive recombination */
  double mu;
  int max_cycles;
  double target_reduction, divergence_factor, gamma;
  uint64_t seed;
} cycle_cfg_t;

typedef struct {
  double *residuals;
  int nres, cap;
  double acf, solve_work;
  int cycles, converged;
  int64_t recombinations;
  double recomb_max_growth;
} stats_t;

static void stats_push(stats_t *s, double r) {
  if (s->nres == s->cap) {
    s->cap = s->cap ? 2 * s->cap : 64;
    s->residuals = realloc(s->residuals, sizeof(double) * (size_t)s->cap);
  }
  s->residuals[s->nres++] = r;
}

/* cycle.cpp:14-21 */
static int credit_take(double *credit, double gamma) {
  *credit += gamma;
  int theta = (int)floor(*credit);
  if (theta < 1) theta = 1;
  *credit -= theta;
  if (*credit < 0.0) *credit = 0.0;
  return theta;
}

/* cycle.cpp:23-103 */
static double recombine(const csr_t *a, const double *b, int cols, double *const *saved_x,
                        double *const *saved_r, double *x, double *before) {
  const int32_t n = a->n;
  double *r = NEW(double, n);
  residual(a, b, x, r);
  double r_norm2 = 0.0;
  for (int32_t k = 0; k < n; ++k) r_norm2 += r[k] * r[k];
  if (before) *before = sqrt(r_norm2);
  double *ad[2] = {NULL, NULL};
  for (int i = 0; i < cols; ++i) {
    ad[i] = NEW(double, n);
    for (int32_t k = 0; k < n; ++k) ad[i][k] = r[k] - saved_r[i][k];
  }
  double alpha[2] = {0.0, 0.0}, g[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, c[2] = {0.0, 0.0};
  for (int i = 0; i < cols; ++i) {
    double s = 0.0;
    for (int32_t k = 0; k < n; ++k) s += r[k] * ad[i][k];
    c[i] = s;
    for (int j = 0; j <= i; ++j) {
      double t = 0.0;
      for (int32_t k = 0; k < n; ++k) t += ad[i][k] * ad[j][k];
      g[i][j] = g[j][i] = t;
    }
  }
  if (cols == 1) {
    if (g[0][0] > 0.0) alpha[0] = c[0] / g[0][0];
  } else if (cols == 2) {
    double det = g[0][0] * g[1][1] - g[0][1] * g[0][1];
    double gg = g[0][0] * g[1][1];
    if (det > 1e-14 * (gg < 1e-300 ? 1e-300 : gg)) {
      alpha[0] = (c[0] * g[1][1] - c[1] * g[0][1]) / det;
      alpha[1] = (c[1] * g[0][0] - c[0] * g[0][1]) / det;
    } else {
      double gain0 = g[0][0] > 0.0 ? c[0] * c[0] / g[0][0] : 0.0;
      double gain1 = g[1][1] > 0.0 ? c[1] * c[1] / g[1][1] : 0.0;
      if (gain0 >= gain1 && g[0][0] > 0.0) alpha[0] = c[0] / g[0][0];
      else if (g[1][1] > 0.0) alpha[1] = c[1] / g[1][1];
    }
  }
  for (int i = 0; i < cols; ++i) alpha[i] = alpha[i] < -2.0 ? -2.0 : (2.0 < alpha[i] ? 2.0 : alpha[i]);
  double predicted = r_norm2;
  for (int i = 0; i < cols; ++i) {
    predicted -= 2.0 * alpha[i] * c[i];
    for (int j = 0; j < cols; ++j) predicted += alpha[i] * g[i][j] * alpha[j];
  }
  if (predicted > r_norm2) alpha[0] = alpha[1] = 0.0;
  double new_norm2 = 0.0;
  for (int32_t k = 0; k < n; ++k) {
    double rk = r[k], xk = x[k], delta = 0.0;
    for (int i = 0; i < cols; ++i) {
      rk -= alpha[i] * ad[i][k];
      delta += alpha[i] * (saved_x[i][k] - xk);
    }
    new_norm2 += rk * rk;
    x[k] = xk + delta;
  }
  work_add((double)cols * (double)n);
  for (int i = 0; i < cols; ++i) free(ad[i]);
  free(r);
  return sqrt(new_norm2 < 0.0 ? 0.0 : new_norm2);
}

typedef struct {
  const hier_t *h;
  const cycle_cfg_t *cfg;
  stats_t *stats;
  double *credit;
  double **top_stage_rhs; /* per-solve cache, cycle.cpp:139-148, 385-386 */
  double *top_coarse_rhs;
  int top_cached;
} driver_t;

static void visit(driver_t *d, int l, const double *b, double *x, int theta);

/* cycle.cpp:166-174: stage_rhs[s] = rhs entering stage s; returns the coarse rhs */
static double *coarsen_stages(const elimt_t *t, const double *b, int32_t n0, double **stage_rhs) {
  double *rhs = NEW(double, n0);
  memcpy(rhs, b, sizeof(double) * (size_t)n0);
  for (int s = 0; s < t->nstages; ++s) {
    stage_rhs[s] = rhs;
    double *next = NEW(double, t->stages[s].coarse_n);
    coarsen_rhs_stage(&t->stages[s], rhs, next);
    rhs = next;
  }
  return rhs;
}

/* cycle.cpp:131-164 */
static void visit_elimination(driver_t *d, int l, const double *b, double *x, int theta) {
  const level_t *level = &d->h->levels[l];
  const level_t *child = &d->h->levels[l + 1];
  const elimt_t *t = &child->elim;
  double **stage_rhs;
  double *coarse_rhs;
  double **local = NULL;
  if (l == 0) {
    if (!d->top_cached) {
      d->top_stage_rhs = NEW(double *, t->nstages);
      d->top_coarse_rhs = coarsen_stages(t, b, level->op.n, d->top_stage_rhs);
      d->top_cached = 1;
    }
    stage_rhs = d->top_stage_rhs;
    coarse_rhs = d->top_coarse_rhs;
  } else {
    local = NEW(double *, t->nstages);
    coarse_rhs = coarsen_stages(t, b, level->op.n, local);
    stage_rhs = local;
  }
  for (int i = 0; i < theta; ++i) {
    double *xc = NEW(double, level->op.n);
    memcpy(xc, x, sizeof(double) * (size_t)level->op.n);
    for (int s = 0; s < t->nstages; ++s) {
      double *next = NEW(double, t->stages[s].coarse_n);
      for (int32_t k = 0; k < t->stages[s].coarse_n; ++k) next[k] = xc[t->stages[s].parent_of_coarse[k]];
      free(xc);
      xc = next;
    }
    int theta_child = credit_take(&d->credit[l + 1], child->gamma);
    visit(d, l + 1, coarse_rhs, xc, theta_child);
    for (int s = t->nstages; s-- > 0;) {
      double *up = NEW(double, t->stages[s].parent_n);
      backsub_stage(&t->stages[s], xc, stage_rhs[s], up);
      free(xc);
      xc = up;
    }
    memcpy(x, xc, sizeof(double) * (size_t)level->op.n);
    free(xc);
  }
  if (local) {
    for (int s = 0; s < t->nstages; ++s) free(local[s]);
    free(local);
    free(coarse_rhs);
  }
}

/* cycle.cpp:176-209 */
static void visit_aggregation(driver_t *d, int l, const double *b, double *x, int theta) {
  const level_t *level = &d->h->levels[l];
  const level_t *child = &d->h->levels[l + 1];
  const aggt_t *t = &child->agg;
  const int adaptive = d->cfg->correction == 1;
  const double mu = d->cfg->mu;
  const int32_t n = level->op.n;
  double *saved_x[64], *saved_r[64];
  int nsaved = 0;
  for (int i = 0; i < theta; ++i) {
    for (int s = 0; s < child->nu_pre; ++s) gs_sweep(&level->op, b, x, 0);
    double *r = NEW(double, n);
    residual(&level->op, b, x, r);
    if (adaptive) {
      if (nsaved >= 2) throwf(ORC_E_ERROR, "recombination supports at most two saved iterates");
      saved_x[nsaved] = NEW(double, n);
      memcpy(saved_x[nsaved], x, sizeof(double) * (size_t)n);
      saved_r[nsaved] = NEW(double, n);
      memcpy(saved_r[nsaved], r, sizeof(double) * (size_t)n);
      ++nsaved;
    }
    double *bc = NEW(double, t->coarse_n);
    restrict_residual(t->aggregate_of, n, t->coarse_n, r, bc);
    free(r);
    if (mu != 1.0)
      for (int32_t k = 0; k < t->coarse_n; ++k) bc[k] *= mu;
    double *ec = ZNEW(double, child->op.n);
    int theta_child = credit_take(&d->credit[l + 1], child->gamma);
    visit(d, l + 1, bc, ec, theta_child);
    add_interpolated(t->aggregate_of, n, ec, x);
    for (int s = 0; s < child->nu_post; ++s) gs_sweep(&level->op, b, x, 0);
    free(bc);
    free(ec);
  }
  if (adaptive && nsaved > 0) {
    double before = 0.0;
    double after = recombine(&level->op, b, nsaved, saved_x, saved_r, x, &before);
    ++d->stats->recombinations;
    if (before > 0.0) {
      double g = after / before;
      if (d->stats->recomb_max_growth < g) d->stats->recomb_max_growth = g;
    }
  }
  for (int i = 0; i < nsaved; ++i) {
    free(saved_x[i]);
    free(saved_r[i]);
  }
}

/* cycle.cpp:115-128 */
static void visit(driver_t *d, int l, const double *b, double *x, int theta) {
  const level_t *level = &d->h->levels[l];
  if (level->coarsest != 0) {
    coarsest_solve(level->solver, b, x);
    return;
  }
  if (d->h->levels[l + 1].kind == K_ELIM) visit_elimination(d, l, b, x, theta);
  else visit_aggregation(d, l, b, x, theta);
}

static void driver_free(driver_t *d) {
  if (d->top_cached) {
    for (int s = 0; s < d->h->levels[1].elim.nstages; ++s) free(d->top_stage_rhs[s]);
    free(d->top_stage_rhs);
    free(d->top_coarse_rhs);
  }
  free(d->credit);
}

/* cycle.cpp:221-273. Returns ORC_OK or ORC_E_DIVERGED (stats filled either way);
 * other errors longjmp. */
static int solve(const hier_t *h, const double *b, const double *x0, const cycle_cfg_t *cfg,
                 double *x, stats_t *stats) {
  const csr_t *a = &h->levels[0].op;
  const int32_t n = a->n;
  double b_inf = 0.0;
  for (int32_t u = 0; u < n; ++u) {
    double v = fabs(b[u]);
    if (b_inf < v) b_inf = v;
  }
  if (fabs(vec_sum(b, n)) > 1e-10 * b_inf)
    throwf(ORC_E_INCOMPATIBLE_RHS, "right-hand side sum %f is not zero", vec_sum(b, n));
  double w0 = g_work;
  memset(stats, 0, sizeof *stats);
  memcpy(x, x0, sizeof(double) * (size_t)n);
  double *r = NEW(double, n);
  residual(a, b, x, r);
  double r0 = norm2(r, n);
  stats_push(stats, r0);
  if (r0 == 0.0) {
    subtract_mean(x, n);
    stats->converged = 1;
    stats->acf = 0.0;
    stats->solve_work = (g_work - w0) / (double)a->m;
    free(r);
    return ORC_OK;
  }
  driver_t d;
  memset(&d, 0, sizeof d);
  d.h = h;
  d.cfg = cfg;
  d.stats = stats;
  d.credit = ZNEW(double, h->nlevels);
  const double target = r0 / cfg->target_reduction;
  int rc = ORC_OK;
  for (int cycle = 1; cycle <= cfg->max_cycles; ++cycle) {
    visit(&d, 0, b, x, 1);
    subtract_mean(x, n);
    residual(a, b, x, r);
    double rn = norm2(r, n);
    stats_push(stats, rn);
    stats->cycles = cycle;
    if (rn <= target) {
      stats->converged = 1;
      break;
    }
    if (rn > cfg->divergence_factor * r0 || !isfinite(rn)) {
      stats->acf = pow(rn / r0, 1.0 / cycle);
      stats->solve_work = (g_work - w0) / (double)a->m;
      snprintf(g_err, sizeof g_err, "solve diverged: residual grew from %f to %f", r0, rn);
      rc = ORC_E_DIVERGED;
      break;
    }
  }
  if (rc == ORC_OK) {
    double rp = stats->residuals[stats->nres - 1];
    stats->acf = pow(rp / r0, 1.0 / (double)stats->cycles);
    stats->solve_work = (g_work - w0) / (double)a->m;
  }
  driver_free(&d);
  free(r);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* solver.cpp whole-problem driver                                           */

typedef struct {
  int32_t nn;
  int32_t *nodes;
  hier_t *h;
} comp_run_t;

typedef struct {
  csr_t a;
  cycle_cfg_t cycle;
  comp_run_t *comps;
  int32_t ncomps;
  double setup_work;
} prepared_t;

/* solver.cpp:31-57 */
static prepared_t *prepare(const csr_t *a, const setup_opts_t *so, const cycle_cfg_t *cc) {
  prepared_t *p = ZNEW(prepared_t, 1);
  p->a = csr_clone(a);
  p->cycle = *cc;
  double w0 = g_work;
  split_t sp = connected_components(&p->a);
  p->ncomps = sp.count;
  p->comps = ZNEW(comp_run_t, sp.count);
  setup_opts_t local = *so;
  for (int32_t c = 0; c < sp.count; ++c) {
    comp_run_t *run = &p->comps[c];
    run->nn = sp.start[c + 1] - sp.start[c];
    run->nodes = NEW(int32_t, run->nn);
    memcpy(run->nodes, sp.nodes + sp.start[c], sizeof(int32_t) * (size_t)run->nn);
    local.seed = rng_derive(so->seed, (uint64_t)c);
    if (run->nn == 1) continue;
    if (sp.count == 1) {
      run->h = setup(&p->a, &local);
    } else {
      csr_t sub = extract_component(&p->a, run->nodes, run->nn);
      run->h = setup(&sub, &local);
      csr_free(&sub);
    }
  }
  split_free(&sp);
  p->setup_work = (g_work - w0) / (double)(p->a.m > 1 ? p->a.m : 1);
  return p;
}

/* ------------------------------------------------------------------------ */
/* exported API                                                              */

int64_t orc_bag_len(const bag *b, const char *name) { return bag_len(b, name); }
int orc_bag_type(const bag *b, const char *name) { return bag_type(b, name); }
int orc_bag_get(const bag *b, const char *name, void *dst) { return bag_get(b, name, dst); }
int orc_bag_count(const bag *b) { return bag_count(b); }
const char *orc_bag_name(const bag *b, int i) { return bag_name(b, i); }
void orc_bag_free(bag *b) { bag_free(b); }
const char *orc_last_error(void) { return g_err; }

uint64_t orc_rng_derive(uint64_t seed, uint64_t stream) { return rng_derive(seed, stream); }

void orc_rng_draws(uint64_t seed, int64_t count, int kind, void *out) {
  rng_t r = rng_make(seed);
  for (int64_t i = 0; i < count; ++i) {
    if (kind == 0) ((uint64_t *)out)[i] = rng_next_u64(&r);
    else if (kind == 1) ((double *)out)[i] = rng_unit(&r);
    else ((double *)out)[i] = rng_pm1(&r);
  }
}

#define CSR_IN csr_t A = csr_view(n, m, rp, col, val, diag)

int orc_validate(CSR_ARGS) {
  CSR_IN;
  API_BEGIN validate_laplacian(&A);
  API_END
}

int orc_mvm(CSR_ARGS, const double *x, double *y) {
  CSR_IN;
  API_BEGIN mvm(&A, x, y);
  API_END
}

int orc_residual(CSR_ARGS, const double *b, const double *x, double *r) {
  CSR_IN;
  API_BEGIN residual(&A, b, x, r);
  API_END
}

int orc_energy(CSR_ARGS, const double *x, double *e) {
  CSR_IN;
  API_BEGIN *e = energy(&A, x);
  API_END
}

int orc_vec_stats(int64_t len, const double *x, double *sum, double *nrm) {
  *sum = vec_sum(x, len);
  *nrm = norm2(x, len);
  return ORC_OK;
}

int orc_subtract_mean(int64_t len, double *x) {
  subtract_mean(x, len);
  return ORC_OK;
}

int orc_gs_sweep(CSR_ARGS, const double *b, double *x, int backward) {
  CSR_IN;
  API_BEGIN gs_sweep(&A, b, x, backward);
  API_END
}

int orc_generate_tvs(CSR_ARGS, int count, int sweeps, uint64_t seed, double *out) {
  CSR_IN;
  API_BEGIN generate_tvs(&A, count, sweeps, seed, out);
  API_END
}

int orc_probe(CSR_ARGS, int sweeps, uint64_t seed, double *factor) {
  CSR_IN;
  API_BEGIN *factor = probe_relaxation(&A, sweeps, seed);
  API_END
}

int orc_affinities(CSR_ARGS, int K, const double *tvs, bag **out) {
  CSR_IN;
  *out = NULL;
  API_BEGIN
  double *aff = NEW(double, 2 * m + 1), *nn = NEW(double, n);
  int32_t *deg = NEW(int32_t, n), nd = 0;
  compute_affinities(&A, K, tvs, aff, nn, deg, &nd);
  bag *b = bag_new();
  bag_put(b, "edge_affinity", BAG_F64, aff, 2 * m);
  bag_put(b, "node_norm", BAG_F64, nn, n);
  bag_put(b, "degenerate", BAG_I32, deg, nd);
  free(aff);
  free(nn);
  free(deg);
  *out = b;
  API_END
}

int orc_detect_hubs(CSR_ARGS, bag **out) {
  CSR_IN;
  *out = NULL;
  API_BEGIN
  int32_t *hubs = NEW(int32_t, n);
  int32_t nh = detect_hubs(&A, hubs);
  bag *b = bag_new();
  bag_put(b, "hubs", BAG_I32, hubs, nh);
  free(hubs);
  *out = b;
  API_END
}

int orc_energy_ratio_qus(CSR_ARGS, int K, const double *tvs, int32_t u, int32_t s, double *qout) {
  CSR_IN;
  API_BEGIN
  quad_t q;
  q.b = NEW(double, K);
  q.c = NEW(double, K);
  q.relaxed_min = NEW(double, K);
  quad_build(&q, &A, K, tvs, u);
  *qout = quad_ratio_vs(&q, &A, K, tvs, s);
  free(q.b);
  free(q.c);
  free(q.relaxed_min);
  API_END
}

static void put_agg(bag *b, const char *p, const aggt_t *t) {
  char k[256];
  snprintf(k, sizeof k, "%saggregate_of", p);
  bag_put(b, k, BAG_I32, t->aggregate_of, t->fine_n);
  snprintf(k, sizeof k, "%sseed_of", p);
  bag_put(b, k, BAG_I32, t->seed_of, t->coarse_n);
  snprintf(k, sizeof k, "%scoarse_n", p);
  bag_put_i32(b, k, t->coarse_n);
  snprintf(k, sizeof k, "%salpha", p);
  bag_put_f64(b, k, t->alpha);
  snprintf(k, sizeof k, "%sstage_used", p);
  bag_put_i32(b, k, t->stage_used);
  snprintf(k, sizeof k, "%sdummy_aggregate", p);
  bag_put_i32(b, k, t->dummy_aggregate);
}

static void put_csr(bag *b, const char *p, const csr_t *a) {
  char k[256];
  snprintf(k, sizeof k, "%sn", p);
  bag_put_i32(b, k, a->n);
  snprintf(k, sizeof k, "%sm", p);
  bag_put_i64(b, k, a->m);
  snprintf(k, sizeof k, "%srow_ptr", p);
  bag_put(b, k, BAG_I64, a->rp, a->n + 1);
  snprintf(k, sizeof k, "%scol", p);
  bag_put(b, k, BAG_I32, a->col, 2 * a->m);
  snprintf(k, sizeof k, "%sval", p);
  bag_put(b, k, BAG_F64, a->val, 2 * a->m);
  snprintf(k, sizeof k, "%sdiag", p);
  bag_put(b, k, BAG_F64, a->diag, a->n);
}

static void put_stage(bag *b, const char *p, const stage_t *s) {
  char k[256];
#define PUT(name, type, ptr, len)            \
  snprintf(k, sizeof k, "%s" name, p);       \
  bag_put(b, k, type, ptr, len);
  snprintf(k, sizeof k, "%sparent_n", p);
  bag_put_i32(b, k, s->parent_n);
  snprintf(k, sizeof k, "%scoarse_n", p);
  bag_put_i32(b, k, s->coarse_n);
  PUT("f_nodes", BAG_I32, s->f_nodes, s->nf);
  PUT("f_diag", BAG_F64, s->f_diag, s->nf);
  PUT("f_ptr", BAG_I64, s->f_ptr, s->nf + 1);
  PUT("f_nbr", BAG_I32, s->f_nbr, s->f_ptr[s->nf]);
  PUT("f_val", BAG_F64, s->f_val, s->f_ptr[s->nf]);
  PUT("coarse_of_parent", BAG_I32, s->coarse_of_parent, s->parent_n);
  PUT("parent_of_coarse", BAG_I32, s->parent_of_coarse, s->coarse_n);
#undef PUT
}

int orc_aggregate(CSR_ARGS, int K, const double *tvs, double gamma, const int32_t *hubs,
                  int32_t nhubs, bag **out) {
  CSR_IN;
  *out = NULL;
  API_BEGIN
  aggt_t t = aggregate(&A, K, tvs, gamma, hubs, nhubs);
  bag *b = bag_new();
  put_agg(b, "", &t);
  free(t.aggregate_of);
  free(t.seed_of);
  *out = b;
  API_END
}

int orc_galerkin(CSR_ARGS, const int32_t *aggregate_of, int32_t coarse_n, bag **out) {
  CSR_IN;
  *out = NULL;
  API_BEGIN
  csr_t c = galerkin(&A, aggregate_of, coarse_n);
  bag *b = bag_new();
  put_csr(b, "", &c);
  csr_free(&c);
  *out = b;
  API_END
}

int orc_restrict_residual(const int32_t *aggregate_of, int32_t fine_n, int32_t coarse_n,
                          const double *r, double *rc) {
  restrict_residual(aggregate_of, fine_n, coarse_n, r, rc);
  return ORC_OK;
}

int orc_add_interpolated(const int32_t *aggregate_of, int32_t fine_n, const double *ec, double *x) {
  add_interpolated(aggregate_of, fine_n, ec, x);
  return ORC_OK;
}

int orc_select_low_degree(CSR_ARGS, int32_t max_degree, bag **out) {
  CSR_IN;
  *out = NULL;
  API_BEGIN
  int32_t *f = NEW(int32_t, n), *c = NEW(int32_t, n), nf, nc;
  select_low_degree(&A, max_degree, f, &nf, c, &nc);
  bag *b = bag_new();
  bag_put(b, "f", BAG_I32, f, nf);
  bag_put(b, "c", BAG_I32, c, nc);
  free(f);
  free(c);
  *out = b;
  API_END
}

int orc_schur(CSR_ARGS, const int32_t *f, int32_t nf, const int32_t *c, int32_t nc, bag **out) {
  CSR_IN;
  *out = NULL;
  API_BEGIN
  stage_t st;
  csr_t coarse = schur_reduce(&A, f, nf, c, nc, &st);
  bag *b = bag_new();
  put_csr(b, "", &coarse);
  put_stage(b, "S.", &st);
  csr_free(&coarse);
  stage_free(&st);
  *out = b;
  API_END
}

int orc_eliminate_rounds(CSR_ARGS, bag **out) {
  CSR_IN;
  *out = NULL;
  API_BEGIN
  elimt_t t;
  int ok = eliminate_rounds(&A, &t);
  bag *b = bag_new();
  bag_put_i32(b, "nstages", t.nstages);
  if (ok) {
    put_csr(b, "", &t.coarse);
    for (int s = 0; s < t.nstages; ++s) {
      char p[64];
      snprintf(p, sizeof p, "S%d.", s);
      put_stage(b, p, &t.stages[s]);
    }
  }
  for (int s = 0; s < t.nstages; ++s) stage_free(&t.stages[s]);
  free(t.stages);
  csr_free(&t.coarse);
  *out = b;
  API_END
}

static stage_t stage_view(STAGE_ARGS) {
  stage_t s = {parent_n,        coarse_n,        nf,
               (int32_t *)f_nodes, (double *)f_diag, (int64_t *)f_ptr,
               (int32_t *)f_nbr, (double *)f_val, (int32_t *)coarse_of_parent,
               (int32_t *)parent_of_coarse};
  return s;
}

int orc_coarsen_rhs_stage(STAGE_ARGS, const double *b, double *bc) {
  stage_t s = stage_view(parent_n, coarse_n, nf, f_nodes, f_diag, f_ptr, f_nbr, f_val,
                         coarse_of_parent, parent_of_coarse);
  coarsen_rhs_stage(&s, b, bc);
  return ORC_OK;
}

int orc_backsub_stage(STAGE_ARGS, const double *xc, const double *b, double *x) {
  stage_t s = stage_view(parent_n, coarse_n, nf, f_nodes, f_diag, f_ptr, f_nbr, f_val,
                         coarse_of_parent, parent_of_coarse);
  backsub_stage(&s, xc, b, x);
  return ORC_OK;
}

int orc_coarsest_direct(CSR_ARGS, const double *b, double *x) {
  CSR_IN;
  API_BEGIN
  coarsest_t *cs = make_direct(&A);
  coarsest_solve(cs, b, x);
  coarsest_free(cs);
  API_END
}

int orc_coarsest_relax(CSR_ARGS, const double *b, double *x) {
  CSR_IN;
  API_BEGIN
  coarsest_t *cs = make_relaxation(&A);
  coarsest_solve(cs, b, x);
  coarsest_free(cs);
  API_END
}

double orc_flat_mu(double q) { return 2.0 * q / (q + 1.0); } /* cycle.cpp:12 */

int orc_credit_takes(double gamma, int count, int32_t *out) {
  double credit = 0.0;
  for (int i = 0; i < count; ++i) out[i] = credit_take(&credit, gamma);
  return ORC_OK;
}

int orc_recombine(CSR_ARGS, const double *b, int cols, const double *saved_x, const double *saved_r,
                  double *x, double *before, double *after) {
  CSR_IN;
  API_BEGIN
  double *sx[2], *sr[2];
  for (int i = 0; i < cols && i < 2; ++i) {
    sx[i] = (double *)saved_x + (int64_t)i * n;
    sr[i] = (double *)saved_r + (int64_t)i * n;
  }
  if (cols > 2) throwf(ORC_E_ERROR, "recombine supports at most two columns");
  *after = recombine(&A, b, cols, sx, sr, x, before);
  API_END
}

static _Thread_local int g_setup_status;

void *orc_setup(CSR_ARGS, double gamma, uint64_t seed, int32_t coarsest_n, int tv_sweeps,
                int tv_count_finest, int tv_count_max) {
  CSR_IN;
  setup_opts_t o = {gamma, seed, coarsest_n, tv_sweeps, tv_count_finest, tv_count_max};
  hier_t *volatile h = NULL;
  jmp_buf jb;
  jmp_buf *prev = g_jb;
  g_jb = &jb;
  int code = setjmp(jb);
  if (code == 0) {
    g_work = 0.0; /* the work total is a running thread-local: start each driver at 0 */
    h = setup(&A, &o);
    g_err[0] = 0;
  }
  g_jb = prev;
  g_setup_status = code;
  return code == 0 ? h : NULL;
}

int orc_setup_status(void) { return g_setup_status; }

static void export_hier(bag *b, const char *pfx, const hier_t *h) {
  char k[640], p[320];
  snprintf(k, sizeof k, "%snlevels", pfx);
  bag_put_i32(b, k, h->nlevels);
  snprintf(k, sizeof k, "%ssetup_work", pfx);
  bag_put_f64(b, k, h->setup_work);
  snprintf(k, sizeof k, "%snwarnings", pfx);
  bag_put_i32(b, k, h->nwarnings);
  for (int l = 0; l < h->nlevels; ++l) {
    const level_t *L = &h->levels[l];
    snprintf(p, sizeof p, "%sL%d.", pfx, l);
#define PUTI(name, v)                       \
  snprintf(k, sizeof k, "%s" name, p);      \
  bag_put_i32(b, k, v);
    PUTI("kind", L->kind);
    put_csr(b, p, &L->op);
    snprintf(k, sizeof k, "%sgamma", p);
    bag_put_f64(b, k, L->gamma);
    PUTI("nu_pre", L->nu_pre);
    PUTI("nu_post", L->nu_post);
    PUTI("tv_count", L->tv_count);
    PUTI("coarsest", L->coarsest);
    if (L->has_agg) put_agg(b, p, &L->agg);
    if (L->has_elim) {
      PUTI("nstages", L->elim.nstages);
      for (int s = 0; s < L->elim.nstages; ++s) {
        char ps[300];
        snprintf(ps, sizeof ps, "%sS%d.", p, s);
        put_stage(b, ps, &L->elim.stages[s]);
      }
    }
#undef PUTI
  }
}

int orc_hier_export(void *h, bag **out) {
  bag *b = bag_new();
  export_hier(b, "", (hier_t *)h);
  *out = b;
  return ORC_OK;
}

double orc_level_cycle_index(void *h, int32_t l, double gamma) {
  return level_cycle_index((hier_t *)h, l, gamma);
}

static void put_stats(bag *b, const stats_t *s) {
  bag_put(b, "residuals", BAG_F64, s->residuals, s->nres);
  bag_put_f64(b, "acf", s->acf);
  bag_put_f64(b, "solve_work", s->solve_work);
  bag_put_i32(b, "cycles", s->cycles);
  bag_put_i32(b, "converged", s->converged);
  bag_put_i64(b, "recombinations", s->recombinations);
  bag_put_f64(b, "recomb_max_growth", s->recomb_max_growth);
}

int orc_solve(void *hv, const double *b, const double *x0, int correction, double mu, int max_cycles,
              double target_reduction, double divergence_factor, double gamma, uint64_t seed,
              double *x, bag **stats) {
  const hier_t *h = hv;
  cycle_cfg_t cfg = {correction, mu, max_cycles, target_reduction, divergence_factor, gamma, seed};
  bag *sb = bag_new();
  *stats = sb;
  stats_t st;
  memset(&st, 0, sizeof st);
  int rc = ORC_OK;
  API_BEGIN
  g_work = 0.0;
  rc = solve(h, b, x0, &cfg, x, &st);
  put_stats(sb, &st);
  free(st.residuals);
  if (rc != ORC_OK) {
    g_jb = prev_jb_;
    return rc;
  }
  API_END
}

void orc_hier_free(void *h) { hier_free((hier_t *)h); }

void *orc_prepare(CSR_ARGS, double gamma, uint64_t seed, int32_t coarsest_n, int tv_sweeps,
                  int tv_count_finest, int tv_count_max, int correction, double mu, int max_cycles,
                  double target_reduction, double divergence_factor, double cycle_gamma,
                  uint64_t cycle_seed) {
  CSR_IN;
  setup_opts_t so = {gamma, seed, coarsest_n, tv_sweeps, tv_count_finest, tv_count_max};
  cycle_cfg_t cc = {correction, mu, max_cycles, target_reduction, divergence_factor, cycle_gamma, cycle_seed};
  prepared_t *volatile p = NULL;
  jmp_buf jb;
  jmp_buf *prev = g_jb;
  g_jb = &jb;
  int code = setjmp(jb);
  if (code == 0) {
    g_work = 0.0;
    p = prepare(&A, &so, &cc);
    g_err[0] = 0;
  }
  g_jb = prev;
  g_setup_status = code;
  return code == 0 ? p : NULL;
}

int orc_prepared_export(void *pv, bag **out) {
  prepared_t *p = pv;
  bag *b = bag_new();
  bag_put_i32(b, "ncomponents", p->ncomps);
  bag_put_f64(b, "setup_work", p->setup_work);
  for (int32_t c = 0; c < p->ncomps; ++c) {
    char k[64];
    snprintf(k, sizeof k, "C%d.nodes", c);
    bag_put(b, k, BAG_I32, p->comps[c].nodes, p->comps[c].nn);
    if (p->comps[c].h) {
      snprintf(k, sizeof k, "C%d.", c);
      export_hier(b, k, p->comps[c].h);
    }
  }
  *out = b;
  return ORC_OK;
}

/* solver.cpp:59-107 */
int orc_solve_prepared(void *pv, const double *b, const double *x0, double *x, bag **report) {
  prepared_t *p = pv;
  bag *rb = bag_new();
  *report = rb;
  API_BEGIN
  const int32_t n = p->a.n;
  g_work = 0.0;
  double w0 = g_work;
  for (int32_t u = 0; u < n; ++u) x[u] = 0.0;
  int32_t largest = 0;
  for (int32_t i = 1; i < p->ncomps; ++i)
    if (p->comps[i].nn > p->comps[largest].nn) largest = i;
  rng_t guess = rng_make(rng_derive(p->cycle.seed, 0x517));
  int all_conv = 1;
  for (int32_t i = 0; i < p->ncomps; ++i) {
    const comp_run_t *run = &p->comps[i];
    if (run->nn == 1) {
      if (fabs(b[run->nodes[0]]) > 0.0)
        throwf(ORC_E_INCOMPATIBLE_RHS, "nonzero rhs at isolated node %d", run->nodes[0]);
      x[run->nodes[0]] = 0.0;
      continue;
    }
    double *bc = NEW(double, run->nn), *xc = NEW(double, run->nn), *xs = NEW(double, run->nn);
    for (int32_t k = 0; k < run->nn; ++k) {
      bc[k] = b[run->nodes[k]];
      xc[k] = x0 ? x0[run->nodes[k]] : rng_pm1(&guess);
    }
    stats_t st;
    int rc = solve(run->h, bc, xc, &p->cycle, xs, &st);
    if (rc != ORC_OK) {
      put_stats(rb, &st);
      throwf(rc, "%s", g_err);
    }
    for (int32_t k = 0; k < run->nn; ++k) x[run->nodes[k]] = xs[k];
    all_conv = all_conv && st.converged;
    if (i == largest) {
      put_stats(rb, &st);
      double red = (st.nres > 0 && st.residuals[st.nres - 1] > 0.0)
                       ? st.residuals[0] / st.residuals[st.nres - 1]
                       : INFINITY;
      bag_put_f64(rb, "reduction", red);
    }
    free(st.residuals);
    free(bc);
    free(xc);
    free(xs);
  }
  bag_put_f64(rb, "total_solve_work", (g_work - w0) / (double)(p->a.m > 1 ? p->a.m : 1));
  bag_put_i32(rb, "all_converged", all_conv);
  API_END
}

void orc_prepared_free(void *pv) {
  prepared_t *p = pv;
  if (!p) return;
  for (int32_t c = 0; c < p->ncomps; ++c) {
    free(p->comps[c].nodes);
    hier_free(p->comps[c].h);
  }
  free(p->comps);
  csr_free(&p->a);
  free(p);
}

typedef struct {
  const hier_t *h;
  const double *B, *X0;
  cycle_cfg_t cfg;
  int nrhs, t, nthreads;
  int32_t *cycles;
  int failed;
} batch_arg_t;

static int solve_guarded(const hier_t *h, const double *b, const double *x0, const cycle_cfg_t *cfg,
                         double *x, stats_t *st) {
  memset(st, 0, sizeof *st);
  jmp_buf jb;
  g_jb = &jb;
  int code = setjmp(jb);
  if (code == 0) code = solve(h, b, x0, cfg, x, st);
  g_jb = NULL;
  return code;
}

static void *batch_worker(void *pv) {
  batch_arg_t *ba = pv;
  const int64_t n = ba->h->levels[0].op.n;
  double *x = malloc(sizeof(double) * (size_t)n);
  for (int i = ba->t; i < ba->nrhs; i += ba->nthreads) {
    stats_t st;
    int code = solve_guarded(ba->h, ba->B + i * n, ba->X0 + i * n, &ba->cfg, x, &st);
    ba->cycles[i] = code == 0 ? st.cycles : -1;
    if (code) ba->failed = 1;
    free(st.residuals);
  }
  free(x);
  return NULL;
}

int orc_solve_batch(void *h, int nrhs, const double *B, const double *X0, int correction, double mu,
                    int max_cycles, double target_reduction, double divergence_factor, double gamma,
                    uint64_t seed, int nthreads, double *seconds, int32_t *cycles) {
  cycle_cfg_t cfg = {correction, mu, max_cycles, target_reduction, divergence_factor, gamma, seed};
  if (nthreads < 1) nthreads = 1;
  batch_arg_t *args = calloc((size_t)nthreads, sizeof(batch_arg_t));
  pthread_t *th = calloc((size_t)nthreads, sizeof(pthread_t));
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  for (int t = 0; t < nthreads; ++t) {
    args[t] = (batch_arg_t){(hier_t *)h, B, X0, cfg, nrhs, t, nthreads, cycles, 0};
    pthread_create(&th[t], NULL, batch_worker, &args[t]);
  }
  int failed = 0;
  for (int t = 0; t < nthreads; ++t) {
    pthread_join(th[t], NULL);
    failed |= args[t].failed;
  }
  clock_gettime(CLOCK_MONOTONIC, &t1);
  *seconds = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
  free(args);
  free(th);
  if (failed) {
    snprintf(g_err, sizeof g_err, "solve_batch: a solve failed");
    return ORC_E_ERROR;
  }
  return ORC_OK;
}
