// core.cuh -- solve-phase and shared kernels (host wrappers).
#pragma once

#include "common.cuh"

namespace lamgb {

// Exact-order Gauss-Seidel schedule: rows grouped into wavefronts of the
// lower-triangular dependency DAG (longest-path levels). A front holds rows
// with no edges between them; every lower neighbour of a row lies in an
// earlier front and every upper neighbour in a later one, so sweeping the
// fronts in order reproduces the sequential forward sweep exactly
// (SURVEY.md Appendix B.3).
struct Schedule {
  int32_t nfronts = 0;
  int32_t max_width = 0;
  int64_t max_len = 0;       // longest row (entries)
  DVec<int32_t> front_ptr;  // [nfronts+1]
  DVec<int32_t> rows;       // [n] rows, ascending within a front
  // heavy rows (hubs) are swept by a whole CTA: positions into `rows`,
  // grouped by front, with per-front ranges
  DVec<int32_t> heavy;
  DVec<int32_t> heavy_ptr;  // [nfronts+1]
  int32_t nheavy = 0;
  DVec<int32_t> heavy_nat;  // the same rows in natural order (residuals)
  int32_t nheavy_nat = 0;
};

void build_schedule(Ctx& c, const CSRv& a, bool backward, Schedule& out);

// r = b - A x (residual, sparse_laplacian.cpp:170-175); b == nullptr gives y = A x
// (mvm, :151-162). Per-row fold in column order: bit-exact.
void residual_exact(Ctx& c, const CSRv& a, const double* b, const double* x, double* r,
                    const int32_t* heavy = nullptr, int32_t nheavy = 0);
// natural rows with more than kHeavyRow entries (ascending)
int32_t heavy_rows(Ctx& c, const CSRv& a, DVec<int32_t>& out);

// Gauss-Seidel sweep(s) over the schedule (smoothing.cpp:13-40). x is n*K
// node-major (K independent right-hand sides / test vectors); b may be null
// (homogeneous) and is n*K when present. With check, syncs and throws
// SingularDiagonalError like the reference; validated levels (diag > 0 on
// every non-isolated row) cannot fail, so the solve runs unchecked.
void gs_exact(Ctx& c, const CSRv& a, const Schedule& sch, const double* b, double* x, int K,
              int sweeps, bool backward = false, bool check = false);

// energy x^T A x as sum over (u,v), v>u, of -a_uv (x_u - x_v)^2 in (u asc,
// k asc) order with the reference's sequential fold (sparse_laplacian.cpp:177-192)
struct UpperIndex {  // entries with col > row, in CSR order
  int64_t count = 0;
  DVec<int64_t> entry;
  DVec<int32_t> row;
};
void build_upper_index(Ctx& c, const CSRv& a, UpperIndex& out);
constexpr int64_t kHeavyRowExact = 2048;
void energy_seq(Ctx& c, const CSRv& a, const UpperIndex& up, const double* x, double* d_out,
                DVec<double>& scratch);
void energy_tree(Ctx& c, const CSRv& a, const UpperIndex& up, const double* x, double* d_out,
                DVec<double>& scratch);

// x[i] = Rng(seed) draw i in [-1,1) (rng.hpp:31), counter form; stride/offset
// place it into a node-major block
void fill_pm1(Ctx& c, double* x, int64_t n, uint64_t seed, int stride = 1, int offset = 0);

// subtract_mean with the sequential fold (sparse_laplacian.cpp:248-252);
// K node-major columns at once (each column folded independently)
void subtract_mean_seq(Ctx& c, double* x, int64_t n, int K = 1);
// fixed-order tree variant (throughput mode)
void subtract_mean_tree(Ctx& c, double* x, int64_t n);

// validate_laplacian (sparse_laplacian.cpp:194-234): same checks, same first
// failure, same message
void validate_exact(Ctx& c, const CSRv& a);

// restrict_residual (+ mu scaling, cycle.cpp:191-194): member-ordered fold
void restrict_exact(Ctx& c, int32_t coarse_n, const int64_t* mem_ptr, const int32_t* mem,
                    const double* r, double mu, double* rc);
// add_interpolated: x[u] += ec[agg[u]]
void interpolate(Ctx& c, int32_t fine_n, const int32_t* agg, const double* ec, double* x);

// elimination transfers (elimination.cpp:126-190)
struct StageV {
  int32_t parent_n, coarse_n, nf;
  const int32_t* f_nodes;
  const double* f_diag;
  const int64_t* f_ptr;
  const int32_t* f_nbr;
  const double* f_val;
  const int32_t* cop;  // coarse_of_parent
  const int32_t* poc;  // parent_of_coarse
  const int64_t* t_ptr;  // per coarse node: contributions (f asc, p asc)
  const int64_t* t_p;
  const int32_t* f_of_p;
  const int32_t* tlong = nullptr;  // coarse nodes with more than kLongT contributions (a CTA each)
  int32_t ntlong = 0;
  bool exact = true;               // VALIDATE: long lists folded in (f, p) order by one thread
};
constexpr int64_t kLongT = 64;
// coarse nodes of a stage whose contribution lists exceed kLongT entries
int32_t stage_long_lists(Ctx& c, int32_t coarse_n, const int64_t* t_ptr, DVec<int32_t>& out);
void coarsen_rhs(Ctx& c, const StageV& s, const double* b, double* bc);
void inject(Ctx& c, const StageV& s, const double* x, double* xc);
void backsub(Ctx& c, const StageV& s, const double* xc, const double* b, double* x);
// builds the transpose lists (t_ptr, t_p, f_of_p) of a stage
void build_stage_transpose(Ctx& c, int32_t coarse_n, int32_t nf, const int64_t* f_ptr,
                           const int32_t* f_nbr, const int32_t* cop, int64_t nnzf,
                           DVec<int64_t>& t_ptr, DVec<int64_t>& t_p, DVec<int32_t>& f_of_p);
// member lists of an aggregation (ascending fine node per aggregate)
void build_members(Ctx& c, int32_t fine_n, int32_t coarse_n, const int32_t* agg,
                   DVec<int64_t>& mem_ptr, DVec<int32_t>& mem);

// small vector ops
void copy_d(Ctx& c, double* dst, const double* src, int64_t n);
void gather_d(Ctx& c, double* dst, const double* src, const int32_t* idx, int64_t n);
void scatter_d(Ctx& c, double* dst, const double* src, const int32_t* idx, int64_t n);

}  // namespace lamgb
