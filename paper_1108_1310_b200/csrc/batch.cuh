// batch.cuh -- THROUGHPUT-mode kernels over a block of K right-hand sides.
//
// The reference solves one b at a time (cycle.cpp:221-273); SURVEY.md §8(e)
// shards independent right-hand sides. On the device the K systems share
// the hierarchy, and LevelCredit (cycle.cpp:14-21) does not depend on the
// data, so all K follow one visit sequence: every kernel of the cycle runs
// once for the whole block. Vectors are node-major, X[u*K + k]; a group of
// K lanes owns a row and lane k folds column k in the row's entry order, so
// the operator is read once per block and the x gathers are K*8-byte
// coalesced segments.
#pragma once

#include <vector>

#include "hier.cuh"

namespace lamgb {

// s (-|+)= val[e] * X[col[e]*K + k] for e in [b, e1), entry order; the
// entries of a round are loaded ahead of the gathers
template <int K, bool SUB, int U = 4>
__device__ __forceinline__ double col_fold(double s, const int32_t* __restrict__ col, const double* __restrict__ val,
                                           const double* X, int64_t b, int64_t e1, int k) {
  for (int64_t e0 = b; e0 < e1; e0 += U) {
    int32_t c[U];
    double v[U], xv[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const bool ok = e0 + j < e1;
      c[j] = ok ? __ldg(col + e0 + j) : 0;
      v[j] = ok ? __ldg(val + e0 + j) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < U; ++j) xv[j] = e0 + j < e1 ? X[(int64_t)c[j] * K + k] : 0.0;
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (e0 + j < e1) s = SUB ? s - v[j] * xv[j] : s + v[j] * xv[j];
  }
  return s;
}

// a thread's four columns of one node-major row: ONE 256-bit access on
// sm_100 (LDG.E.ENL2.256 / STG.E.ENL2.256) instead of two 128-bit ones --
// half the L1TEX requests of the gathers, which the block sweep is bound by
// V = 4 columns per thread, K/V threads per row: the row's entries are loaded
// once per K/V threads instead of once per lane, so the instruction count per
// row drops ~V-fold; each column is still folded in entry order (same
// arithmetic as one thread per column).
constexpr int kV = 4;
struct d4 {
  double x, y, z, w;
};
__device__ __forceinline__ d4 ld4(const double* p) {
  d4 r;
  asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void st4(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}
// x of other CTAs' rows: read through L2 (a line this SM cached before the
// owner's update must not be hit)
__device__ __forceinline__ d4 ld4_cg(const double* p) {
  d4 r;
  asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
  return r;
}

constexpr int kColChunks = 4096;  // per-column reduction chunks (c.dbpart holds kMaxBlock x this)
constexpr int kMaxBlock = 128;    // widest block of right-hand sides (node-major n x K)

// supported block widths: powers of two from 4 (one thread's 256-bit group)
inline bool batch_width_ok(int K) { return K == 4 || K == 8 || K == 16 || K == 32 || K == 64 || K == 128; }

void bgs_colored(Ctx& c, const DColor& cl, int32_t n, const double* B, double* X, int sweeps, int K,
                 const int32_t* done = nullptr);
// exact-order (reference row order) sweeps of a K-column block; ctl holds
// 1 + kMaxExactSweeps * it.nfronts ints of scratch (per context)
void bgs_exact(Ctx& c, const CSRv& a, const Schedule& sch, const ExactItems& it, const double* B, double* X,
               int sweeps, int K, int32_t* ctl);
void bresidual(Ctx& c, const CSRv& a, const LongRows& L, const double* B, const double* X, double* R, int K);
// residual + restriction in one pass (bit-identical to bresidual then brestrict);
// false when the level has long rows (the caller runs the two kernels)
bool bresidual_restrict(Ctx& c, const CSRv& a, const LongRows& L, int32_t coarse_n, const int64_t* mem_ptr,
                        const int32_t* mem, const double* B, const double* X, double mu, double* Bc, double* Xc,
                        int K);
void brestrict(Ctx& c, int32_t coarse_n, const int64_t* mem_ptr, const int32_t* mem, const double* R, double mu,
               double* Bc, double* Xc, int K);
void binterpolate(Ctx& c, int32_t fine_n, const int32_t* agg, const double* Xc, double* X, int K);
void bcoarsen_rhs(Ctx& c, const StageV& s, const double* B, double* Bc, int K);
void binject(Ctx& c, const StageV& s, const double* X, double* Xc, int K);
void bbacksub(Ctx& c, const StageV& s, const double* Xc, const double* B, double* X, int K);
void bdirect(Ctx& c, const DDirect& d, const double* B, double* X, int K);
// per-column sums (SQ: sums of squares) of an n x K block into out[K], fixed order
void bcolsum(Ctx& c, const double* X, int64_t n, int K, bool sq, double* out);
void bsub_mean(Ctx& c, double* X, int64_t n, int K, const double* sums, const int32_t* done = nullptr);
void bcolabsmax(Ctx& c, const double* X, int64_t n, int K, unsigned long long* out);
// RHS-major [nrhs][n] <-> node-major [n][K] (columns >= nrhs are zero-filled)
void to_node_major(Ctx& c, const double* src, int64_t n, int nrhs, int K, double* dst);
// dst = column k of X (minus sums[k]/n when sums is given)
void column_out(Ctx& c, const double* X, int64_t n, int K, int k, double* dst, const double* sums = nullptr);
inline int batch_width_for(int nrhs) {
  int k = 4;
  while (k < nrhs && k < kMaxBlock) k *= 2;
  return k;
}
// RelaxationSolver::solve (coarse_solver.cpp:82-93) per column; returns the
// sweeps of every column in sweeps[K]
void brelax(Ctx& c, const CSRv& a, const DColor& cl, const LongRows& nat, const double* B, double* X, double* R,
            int K, std::vector<int>& sweeps);

}  // namespace lamgb
