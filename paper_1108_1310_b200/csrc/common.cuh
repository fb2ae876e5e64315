// common.cuh -- shared host/device infrastructure of liblamg_b200.
//
// Everything is compiled with --fmad=false: every fp64 multiply and add is
// rounded separately, in source order, exactly as the reference's x86-64
// build evaluates them, so kernels that keep the
// reference's fold order are bit-identical to it.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "lamg_b200.h"

namespace lamgb {

namespace cg = cooperative_groups;

// kernels launched by this library (all contexts); lamg_launch_count()
extern std::atomic<long long> g_launches;
extern thread_local long long t_launches;  // this thread's share (graph capture accounting)
inline void count_launch() {
  ++g_launches;
  ++t_launches;
}

// ----------------------------------------------------------------- errors
struct LamgError : std::runtime_error {
  int code;
  LamgError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void cuda_fail(cudaError_t e, const char* what, const char* file, int line);

#define CK(x)                                                    \
  do {                                                           \
    cudaError_t e_ = (x);                                        \
    if (e_ != cudaSuccess) ::lamgb::cuda_fail(e_, #x, __FILE__, __LINE__); \
  } while (0)
#define CK_LAUNCH() CK(cudaGetLastError())

// ------------------------------------------------------ device error slot
// Kernels that can fail record the FIRST failure in the reference's
// sequential order as a 64-bit ordering key (atomicMin). A failing kernel is
// then re-run in "payload" phase, where only the thread(s) holding the
// winning key write the payload (node ids, row sum) used to format the
// reference's message. Kernels that report errors are therefore re-runnable
// (read-only, or their output is discarded on error).
struct DevErr {
  unsigned long long key;  // ULLONG_MAX = none
  int phase;               // 0 = find min key, 1 = write payload
  int code;                // device error kind (errors.cu)
  int a, b;
  double v;
};

__device__ inline void dev_report(DevErr* e, unsigned long long key, int code, int a, int b,
                                  double v = 0.0) {
  if (e->phase == 0) {
    atomicMin(&e->key, key);
  } else if (key == e->key) {
    e->code = code;
    e->a = a;
    e->b = b;
    e->v = v;
  }
}

// device error kinds -> (status, message) in errors.cu
enum DevErrKind {
  DE_GS_SINGULAR = 1,  // smoothing.cpp:17-23
  DE_VAL_SELF,         // sparse_laplacian.cpp:206
  DE_VAL_RANGE,        // :207
  DE_VAL_SORT,         // :208-210
  DE_VAL_STRUCT,       // :214-217
  DE_VAL_VALUE,        // :219-222
  DE_VAL_ROWSUM,       // :225-228
  DE_VAL_DIAG,         // :229-232
  DE_SCHUR_OVERLAP,    // elimination.cpp:42-44
  DE_SCHUR_PIVOT,      // :45-48
  DE_SCHUR_DEPENDENT,  // :53-56
};

// ------------------------------------------------------------ device memory
// When set (lamg_hier_destroy), buffers are freed synchronously: the stream
// that allocated them may belong to a context destroyed in the meantime.
extern thread_local bool g_free_sync;

inline bool poison_enabled() {
  static const bool on = getenv("LAMG_POISON") && atoi(getenv("LAMG_POISON")) == 1;
  return on;
}

// LAMG_GUARD=1 (debugging aid; compute-sanitizer is not available on the GPU
// pool): every device buffer is allocated with a 256-byte band of a known
// pattern before and after it, and the bands are checked when the buffer is
// released -- an out-of-bounds write next to any buffer is reported on stderr
// (buffer size, which band, first bad offset) and counted
// (lamg_guard_report: buffers checked / overruns).
inline bool guard_enabled() {
  static const bool on = getenv("LAMG_GUARD") && atoi(getenv("LAMG_GUARD")) == 1;
  return on;
}
constexpr size_t kGuardBytes = 256;
void guard_fill(void* base, size_t payload, cudaStream_t s);          // common.cu
void guard_check(const void* base, size_t payload, cudaStream_t s, bool sync_free);  // common.cu
void guard_report(long long* checked, long long* overruns);

template <typename T>
struct DVec {
  T* p = nullptr;
  int64_t n = 0;
  cudaStream_t s = 0;
  DVec() = default;
  DVec(int64_t count, cudaStream_t st) { alloc(count, st); }
  DVec(const DVec&) = delete;
  DVec& operator=(const DVec&) = delete;
  DVec(DVec&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
  DVec& operator=(DVec&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; n = o.n; s = o.s;
      o.p = nullptr; o.n = 0;
    }
    return *this;
  }
  ~DVec() { release(); }
  void alloc(int64_t count, cudaStream_t st) {
    release();
    s = st;
    n = count;
    if (count > 0 && guard_enabled()) {
      unsigned char* base = nullptr;
      CK(cudaMallocAsync((void**)&base, sizeof(T) * (size_t)count + 2 * kGuardBytes, s));
      guard_fill(base, sizeof(T) * (size_t)count, s);
      p = (T*)(base + kGuardBytes);
    } else if (count > 0) {
      CK(cudaMallocAsync((void**)&p, sizeof(T) * (size_t)count, s));
    }
    // LAMG_POISON=1 (debugging aid): fresh floating-point buffers start as NaN,
    // so a read of never-written memory shows up in the results
    if constexpr (std::is_floating_point<T>::value)
      if (count > 0 && poison_enabled()) CK(cudaMemsetAsync(p, 0xff, sizeof(T) * (size_t)count, s));
  }
  void release() {
    if (p && guard_enabled()) {
      unsigned char* base = (unsigned char*)p - kGuardBytes;
      guard_check(base, sizeof(T) * (size_t)n, s, g_free_sync);
      if (g_free_sync) cudaFree(base);
      else cudaFreeAsync(base, s);
    } else if (p) {
      if (g_free_sync) cudaFree(p);
      else cudaFreeAsync(p, s);
    }
    p = nullptr;
    n = 0;
  }
  void zero() { if (n) CK(cudaMemsetAsync(p, 0, sizeof(T) * (size_t)n, s)); }
  void fill_bytes(int byte) { if (n) CK(cudaMemsetAsync(p, byte, sizeof(T) * (size_t)n, s)); }
  void upload(const T* h, int64_t count) {
    if (count) CK(cudaMemcpyAsync(p, h, sizeof(T) * (size_t)count, cudaMemcpyHostToDevice, s));
  }
  void download(T* h, int64_t count) const {
    if (count) CK(cudaMemcpyAsync(h, p, sizeof(T) * (size_t)count, cudaMemcpyDeviceToHost, s));
  }
  std::vector<T> to_host() const {
    std::vector<T> v((size_t)n);
    download(v.data(), n);
    CK(cudaStreamSynchronize(s));
    return v;
  }
  T* get() const { return p; }
};

// -------------------------------------------------------------- CSR views
struct CSRv {  // device view of a lamg::SparseLaplacian
  int32_t n = 0;
  int64_t m = 0;
  const int64_t* rp = nullptr;
  const int32_t* col = nullptr;
  const double* val = nullptr;
  const double* diag = nullptr;
};

struct DCSR {  // owning device CSR
  int32_t n = 0;
  int64_t m = 0;
  DVec<int64_t> rp;
  DVec<int32_t> col;
  DVec<double> val;
  DVec<double> diag;
  CSRv view() const { return CSRv{n, m, rp.p, col.p, val.p, diag.p}; }
  void alloc(int32_t nn, int64_t mm, cudaStream_t s) {
    n = nn;
    m = mm;
    rp.alloc(nn + 1, s);
    col.alloc(2 * mm, s);
    val.alloc(2 * mm, s);
    diag.alloc(nn, s);
  }
};

// ---------------------------------------------------------------- context
struct Workspace;  // solve.cuh

// lamg_ctx_profile: CUDA events around kernel groups of a solve (graphs off).
// Class 0 / 1: the finest level's Gauss-Seidel / residual launches (the
// bench's roofline kernels); class 2 + 4 l + {0,1,2,3}: level l's sweeps,
// residuals, transfers (restriction, interpolation, elimination stages) and
// on-device tail visits rooted at l (a per-level time breakdown).
constexpr int kProfClasses = 2 + 4 * 64;
struct Profile {
  bool enabled = false;
  std::vector<cudaEvent_t> ev[kProfClasses];  // start/stop pairs per kernel class
  int64_t used[kProfClasses] = {};
  double bytes[kProfClasses] = {};
};

struct Ctx {
  int device = 0;
  int mode = LAMG_MODE_VALIDATE;
  // THROUGHPUT one-column solves sweep this many finest levels in the
  // reference's exact order (the rest coloured); see lamg_ctx_set_exact_levels
  int exact_levels = 1;
  int sms = 148;
  cudaStream_t s = nullptr;
  DevErr* derr = nullptr;       // device error slot
  DevErr* herr = nullptr;       // pinned mirror
  double* hscal = nullptr;      // pinned scalar readback area (64 doubles)
  int* dflag = nullptr;         // scratch device ints (64)
  double* dscal = nullptr;      // scratch device scalars (256 doubles)
  double* dpart = nullptr;      // tree-reduction partials (256 doubles)
  double work = 0.0;            // thread-local work::total() equivalent (edge units)
  Profile prof;
  Workspace* ws = nullptr;      // solve workspace (owned; solve.cu)
  Workspace* bws = nullptr;     // batched (K right-hand sides) solve workspace
  double* dbpart = nullptr;     // batched reductions: per-column chunk partials (32 x kColChunks)
  double* dbscal = nullptr;     // batched scalars (256 doubles)
  int32_t* dbdone = nullptr;    // batched per-column masks (64 ints)
  DVec<double> bscratch;        // batched long-row chunk sums (grown on demand)
  // relaxation / task residual scratch, per context so concurrent solves over
  // one hierarchy never share it; rgen changes whenever a buffer moves (it
  // keys the cached sweep graph)
  DVec<double> rpart, ripart;   // cooperative relaxation: block partials, chunk partials
  DVec<uint32_t> rcnt;          // chunk counters of super-long rows (return to 0 after each row)
  int64_t rgen = 0;
  struct RelaxGraph {
    uint64_t key = 0;  // DColor::uid (monotonic: never reused, unlike an address)
    const void *op = nullptr, *b = nullptr, *x = nullptr, *r = nullptr;  // natural operator values, vectors
    int64_t gen = -1;
    cudaGraphExec_t exec = nullptr;
    long long launches = 0;
  } relax_graph;
  DVec<int32_t> rcptr;          // cooperative relaxation: natural-order range {0, n}
  DVec<double> rtpart;          // residual_tasks: chunk partials
  DVec<int32_t> rtcptr;         // residual_tasks: {0, n} of the last operator
  int32_t rtcptr_n = -1;
  // per-kernel API results kept until taken
  DCSR res_csr;
  struct {
    int32_t nf = 0;
    DVec<double> f_diag;
    DVec<int64_t> f_ptr;
    DVec<int32_t> f_nbr;
    DVec<double> f_val;
    DVec<int32_t> cop;
  } res_stage;
  int max_coop_blocks(const void* kernel, int threads, size_t smem = 0) const;
  void clear_err();
  // syncs; if a kernel recorded a failure, re-runs `launch` in payload phase
  // and throws the reference's exception for it
  template <typename F>
  void checked(F&& launch) {
    clear_err();
    launch();
    sync();
    if (herr_key() != ~0ull) {
      set_err_phase(1);
      launch();
      sync();
      fetch_err_and_throw();
    }
  }
  unsigned long long herr_key();
  void set_err_phase(int ph);
  [[noreturn]] void fetch_err_and_throw();
  void sync() { CK(cudaStreamSynchronize(s)); }
};


// ---------------------------------------------------------- launch helpers
constexpr int kThreads = 256;
inline int blocks_for(int64_t n, int threads = kThreads) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > (1 << 30)) b = 1 << 30;
  return (int)b;
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// grid barrier usable from cooperative kernels; one block uses __syncthreads
__device__ inline void grid_barrier() {
  if (gridDim.x == 1) {
    __syncthreads();
  } else {
    cg::this_grid().sync();
  }
}

// Row fold s (-|+)= val[k] * x[col[k]] for k in [b, e), in k order (bit-exact
// with the reference's sequential loop). Loads are issued in predicated
// batches of U so a row costs ~2 memory latencies per batch instead of 2 per
// nonzero: small colour phases and coarse levels are latency-bound.
template <int U, bool SUB, bool STREAM = false>
__device__ __forceinline__ double row_fold(double s, const int32_t* __restrict__ col,
                                           const double* __restrict__ val, const double* x,
                                           int64_t b, int64_t e) {
  for (int64_t k = b; k < e; k += U) {
    int32_t c[U];
    double v[U], xv[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const bool ok = k + j < e;
      // STREAM: operator entries of big levels are read once per sweep; the
      // evict-first hint keeps them from displacing the L2-resident coarse levels
      c[j] = ok ? (STREAM ? __ldcs(col + k + j) : col[k + j]) : 0;
      v[j] = ok ? (STREAM ? __ldcs(val + k + j) : val[k + j]) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < U; ++j) xv[j] = (k + j < e) ? x[c[j]] : 0.0;
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (k + j < e) s = SUB ? s - v[j] * xv[j] : s + v[j] * xv[j];
  }
  return s;
}

// THROUGHPUT-mode row dot product sum_k val[k] * x[col[k]] by a group of G
// lanes: lane j takes k = b + j, b + j + G, ...; the partials meet in a
// fixed xor-shuffle tree, so the result is deterministic (not the
// sequential fold of VALIDATE mode). All lanes of the warp must call it;
// lanes of invalid rows pass b == e. Every lane of the group gets the sum.
template <int G, bool STREAM = false>
__device__ __forceinline__ double group_dot(const int32_t* __restrict__ col, const double* __restrict__ val,
                                            const double* x, int64_t b, int64_t e) {
  constexpr int U = 4;  // entries per lane per round, loads batched ahead of use
  const int lane = threadIdx.x & (G - 1);
  double p = 0.0;
  for (int64_t k0 = b + lane; k0 < e; k0 += (int64_t)G * U) {
    int32_t c[U];
    double v[U], xv[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int64_t k = k0 + (int64_t)j * G;
      const bool ok = k < e;
      c[j] = ok ? (STREAM ? __ldcs(col + k) : col[k]) : 0;
      v[j] = ok ? (STREAM ? __ldcs(val + k) : val[k]) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < U; ++j) xv[j] = (k0 + (int64_t)j * G < e) ? x[c[j]] : 0.0;
#pragma unroll
    for (int j = 0; j < U; ++j) p += v[j] * xv[j];
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o, G);
  return p;
}

// Heavy-row dot product by a whole CTA (hub rows of power-law graphs):
// strided partials, fixed-order block tree. Every thread gets the sum.
__device__ __forceinline__ double block_dot(const int32_t* __restrict__ col, const double* __restrict__ val,
                                            const double* x, int64_t b, int64_t e) {
  __shared__ double sh_bd[33];
  constexpr int U = 4;  // loads batched ahead of use: U gathers in flight per thread
  double p = 0.0;
  for (int64_t k0 = b + threadIdx.x; k0 < e; k0 += (int64_t)blockDim.x * U) {
    int32_t c[U];
    double v[U], xv[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int64_t k = k0 + (int64_t)j * blockDim.x;
      c[j] = k < e ? __ldcs(col + k) : 0;
      v[j] = k < e ? __ldcs(val + k) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < U; ++j) xv[j] = (k0 + (int64_t)j * blockDim.x < e) ? x[c[j]] : 0.0;
#pragma unroll
    for (int j = 0; j < U; ++j) p += v[j] * xv[j];
  }
  for (int o = 16; o > 0; o >>= 1) p += __shfl_down_sync(0xffffffffu, p, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh_bd[threadIdx.x >> 5] = p;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh_bd[w];
    sh_bd[32] = t;
  }
  __syncthreads();
  return sh_bd[32];
}

// VALIDATE-mode long row by one warp: s (-|+)= val[k]*x[col[k]] for k in
// [b,e) in k order, bit-identical to the sequential loop. Lanes form 32
// products at a time (each rounded exactly as in the loop); every lane then
// runs the same add chain over the shuffled products, so all lanes hold s.
// The next 32 products are loaded before the current chain runs.
template <bool SUB>
__device__ __forceinline__ double warp_seq_fold(double s, const int32_t* __restrict__ col,
                                                const double* __restrict__ val, const double* x, int64_t b,
                                                int64_t e, int xs = 1, int xk = 0) {
  const int lane = threadIdx.x & 31;
  int64_t k = b + lane;
  double p = k < e ? val[k] * x[(int64_t)col[k] * xs + xk] : 0.0;
  for (int64_t c0 = b; c0 < e; c0 += 32) {
    const int64_t kn = c0 + 32 + lane;
    const double pn = kn < e ? val[kn] * x[(int64_t)col[kn] * xs + xk] : 0.0;
    const int cnt = e - c0 < 32 ? (int)(e - c0) : 32;
    if (cnt == 32) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const double pj = __shfl_sync(0xffffffffu, p, j);
        s = SUB ? s - pj : s + pj;
      }
    } else {
      for (int j = 0; j < cnt; ++j) {
        const double pj = __shfl_sync(0xffffffffu, p, j);
        s = SUB ? s - pj : s + pj;
      }
    }
    p = pn;
  }
  return s;
}
constexpr int64_t kWarpRowExact = 64;  // exact folds of longer rows take a warp

// VALIDATE-mode heavy row: s (-|+)= val[k]*x[col[k]] for k in [b,e) in k
// order, bit-identical to the sequential loop. The CTA computes the products
// (each rounded exactly as in the loop) in parallel chunks through shared
// memory; thread 0 runs the dependent add chain. Every thread gets s.
// x == nullptr folds val[k] itself.
// `xs`/`xk` select column k of a node-major block (x[col*xs + xk]).
template <bool SUB>
__device__ __forceinline__ double block_seq_fold(double s, const int32_t* __restrict__ col,
                                                 const double* __restrict__ val, const double* x, int64_t b,
                                                 int64_t e, int xs = 1, int xk = 0) {
  // double-buffered: while thread 0 runs the add chain over chunk q, the CTA
  // forms the products of chunk q + 1, so an iteration costs the longer of
  // the two instead of their sum (1024-entry chunks: the chain dominates)
  constexpr int C = 1024;
  __shared__ double sh_prod[2][C];
  __shared__ double sh_s;
  if (threadIdx.x == 0) sh_s = s;
  auto fill = [&](int buf, int64_t c0) {
    for (int j = threadIdx.x; j < C; j += blockDim.x) {
      const int64_t k = c0 + j;
      sh_prod[buf][j] = k < e ? (x ? val[k] * x[(int64_t)col[k] * xs + xk] : val[k]) : 0.0;
    }
  };
  __syncthreads();
  if (b < e) fill(0, b);
  int buf = 0;
  for (int64_t c0 = b; c0 < e; c0 += C) {
    __syncthreads();  // chunk c0 is in sh_prod[buf]; the other buffer is free
    if (c0 + C < e) fill(buf ^ 1, c0 + C);
    if (threadIdx.x == 0) {
      const int cnt = e - c0 < C ? (int)(e - c0) : C;
      double t = sh_s;
      for (int j = 0; j < cnt; ++j) t = SUB ? t - sh_prod[buf][j] : t + sh_prod[buf][j];
      sh_s = t;
    }
    buf ^= 1;
  }
  __syncthreads();
  const double r = sh_s;
  __syncthreads();
  return r;
}

// launches a kernel cooperatively (all blocks co-resident)
void coop_launch(Ctx& c, const void* kernel, int blocks, int threads, void** args, size_t smem = 0);

// ------------------------------------------------------------- CUB wrappers
// stable LSD radix sort of (key, value) pairs on the low `bits` key bits
void sort_pairs_u64(Ctx& c, const uint64_t* kin, uint64_t* kout, const int64_t* vin,
                    int64_t* vout, int64_t n, int bits);
void sort_keys_u64(Ctx& c, const uint64_t* kin, uint64_t* kout, int64_t n, int bits);
void sort_pairs_u64_d(Ctx& c, const uint64_t* kin, uint64_t* kout, const double* vin,
                      double* vout, int64_t n, int bits);
void sort_pairs_u32_i32(Ctx& c, const uint32_t* kin, uint32_t* kout, const int32_t* vin,
                        int32_t* vout, int64_t n, int bits);
void sort_pairs_u64_i32(Ctx& c, const uint64_t* kin, uint64_t* kout, const int32_t* vin,
                        int32_t* vout, int64_t n, int bits);
void exclusive_scan_i64(Ctx& c, const int64_t* in, int64_t* out, int64_t n);
void exclusive_scan_i32(Ctx& c, const int32_t* in, int32_t* out, int64_t n);
// stable compaction of [0, n) indices where flag != 0; returns the count
int64_t select_flagged_index(Ctx& c, const uint8_t* flags, int32_t* out, int64_t n);
int64_t select_flagged_index64(Ctx& c, const uint8_t* flags, int64_t* out, int64_t n);
double reduce_max_d(Ctx& c, const double* in, int64_t n);   // exact (max)
int64_t reduce_sum_i64(Ctx& c, const int64_t* in, int64_t n);
int32_t reduce_max_i32(Ctx& c, const int32_t* in, int64_t n);

// --------------------------------------------------------- bit-exact folds
// out = ((0 + x0) + x1) + ... (the reference's left-to-right fold); device result
void seq_sum(Ctx& c, const double* x, int64_t n, double* d_out);
// out = sqrt(sum x_i^2) with the same fold order (norm2, sparse_laplacian.cpp:236-240)
void seq_norm2(Ctx& c, const double* x, int64_t n, double* d_out);
// sums of the K <= 32 columns of a node-major [n][K] block, each in row order (bit-exact)
void seq_col_sums(Ctx& c, const double* x, int64_t n, int K, double* d_out);
// fixed-order tree reductions (throughput mode)
void tree_sum(Ctx& c, const double* x, int64_t n, double* d_out);
void tree_norm2(Ctx& c, const double* x, int64_t n, double* d_out);

// rounded-to-host scalar read (syncs)
double read_scalar(Ctx& c, const double* d);
int64_t read_i64(Ctx& c, const int64_t* d);
int32_t read_i32(Ctx& c, const int32_t* d);

}  // namespace lamgb
