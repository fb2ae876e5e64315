// common.cu -- context, error mapping, CUB wrappers and the bit-exact folds.
#include <cub/cub.cuh>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <string>

#include "common.cuh"

namespace lamgb {

std::atomic<long long> g_launches{0};
thread_local long long t_launches = 0;
thread_local bool g_free_sync = false;

void cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
  char buf[512];
  snprintf(buf, sizeof buf, "CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e),
           cudaGetErrorString(e), file, line, what);
  throw LamgError(LAMG_E_CUDA, buf);
}

int Ctx::max_coop_blocks(const void* kernel, int threads, size_t smem) const {
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem));
  if (per_sm < 1) per_sm = 1;
  return per_sm * sms;
}

void Ctx::clear_err() {
  DevErr e{~0ull, 0, 0, 0, 0, 0.0};
  CK(cudaMemcpyAsync(derr, &e, sizeof e, cudaMemcpyHostToDevice, s));
}

unsigned long long Ctx::herr_key() {
  CK(cudaMemcpyAsync(herr, derr, sizeof(DevErr), cudaMemcpyDeviceToHost, s));
  sync();
  return herr->key;
}

void Ctx::set_err_phase(int ph) {
  CK(cudaMemcpyAsync(&derr->phase, &ph, sizeof(int), cudaMemcpyHostToDevice, s));
  sync();
}

// The reference's exception type and message for each device error kind.
void Ctx::fetch_err_and_throw() {
  CK(cudaMemcpyAsync(herr, derr, sizeof(DevErr), cudaMemcpyDeviceToHost, s));
  sync();
  const DevErr& e = *herr;
  char buf[256];
  int code = LAMG_E_ERROR;
  switch (e.code) {
    case DE_GS_SINGULAR:
      code = LAMG_E_SINGULAR_DIAGONAL;
      snprintf(buf, sizeof buf, "zero diagonal at node %d", e.a);
      break;
    case DE_VAL_SELF:
      code = LAMG_E_INVALID_LAPLACIAN;
      snprintf(buf, sizeof buf, "self entry stored in row %d", e.a);
      break;
    case DE_VAL_RANGE:
      code = LAMG_E_INVALID_LAPLACIAN;
      snprintf(buf, sizeof buf, "column out of range");
      break;
    case DE_VAL_SORT:
      code = LAMG_E_INVALID_LAPLACIAN;
      snprintf(buf, sizeof buf, "row %d not strictly sorted", e.a);
      break;
    case DE_VAL_STRUCT:
      code = LAMG_E_INVALID_LAPLACIAN;
      snprintf(buf, sizeof buf, "structural asymmetry at (%d,%d)", e.a, e.b);
      break;
    case DE_VAL_VALUE:
      code = LAMG_E_INVALID_LAPLACIAN;
      snprintf(buf, sizeof buf, "value asymmetry at (%d,%d)", e.a, e.b);
      break;
    case DE_VAL_ROWSUM:
      code = LAMG_E_INVALID_LAPLACIAN;
      snprintf(buf, sizeof buf, "row %d sum %f exceeds tolerance", e.a, e.v);
      break;
    case DE_VAL_DIAG:
      code = LAMG_E_INVALID_LAPLACIAN;
      snprintf(buf, sizeof buf, "non-positive diagonal at non-isolated node %d", e.a);
      break;
    case DE_SCHUR_OVERLAP:
      snprintf(buf, sizeof buf, "schur_reduce: F and C overlap at node %d", e.a);
      break;
    case DE_SCHUR_PIVOT:
      code = LAMG_E_SINGULAR_DIAGONAL;
      snprintf(buf, sizeof buf, "schur_reduce: non-positive pivot at node %d", e.a);
      break;
    case DE_SCHUR_DEPENDENT:
      snprintf(buf, sizeof buf, "schur_reduce: F is not independent, edge (%d,%d)", e.a, e.b);
      break;
    default:
      snprintf(buf, sizeof buf, "device error kind %d", e.code);
  }
  throw LamgError(code, buf);
}

void coop_launch(Ctx& c, const void* kernel, int blocks, int threads, void** args, size_t smem) {
  if (blocks < 1) blocks = 1;
  count_launch();
  CK(cudaLaunchCooperativeKernel(kernel, dim3(blocks), dim3(threads), args, smem, c.s));
}

// ------------------------------------------------------------- CUB wrappers
namespace {
struct Temp {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t s;
  explicit Temp(cudaStream_t st) : s(st) {}
  void* get(size_t b) {
    bytes = b;
    if (b) CK(cudaMallocAsync(&p, b, s));
    return p;
  }
  ~Temp() {
    if (p) cudaFreeAsync(p, s);
  }
};
}  // namespace

#define CUB_TWICE(call)                 \
  do {                                  \
    size_t bytes_ = 0;                  \
    void* tmp_ = nullptr;               \
    CK(call);                           \
    Temp t_(c.s);                       \
    tmp_ = t_.get(bytes_);              \
    CK(call);                           \
  } while (0)

void sort_pairs_u64(Ctx& c, const uint64_t* kin, uint64_t* kout, const int64_t* vin, int64_t* vout,
                    int64_t n, int bits) {
  if (n <= 0) return;
  CUB_TWICE(cub::DeviceRadixSort::SortPairs(tmp_, bytes_, kin, kout, vin, vout, (size_t)n, 0, bits, c.s));
}
void sort_keys_u64(Ctx& c, const uint64_t* kin, uint64_t* kout, int64_t n, int bits) {
  if (n <= 0) return;
  CUB_TWICE(cub::DeviceRadixSort::SortKeys(tmp_, bytes_, kin, kout, (size_t)n, 0, bits, c.s));
}
void sort_pairs_u64_d(Ctx& c, const uint64_t* kin, uint64_t* kout, const double* vin, double* vout,
                      int64_t n, int bits) {
  if (n <= 0) return;
  CUB_TWICE(cub::DeviceRadixSort::SortPairs(tmp_, bytes_, kin, kout, vin, vout, (size_t)n, 0, bits, c.s));
}
void sort_pairs_u32_i32(Ctx& c, const uint32_t* kin, uint32_t* kout, const int32_t* vin,
                        int32_t* vout, int64_t n, int bits) {
  if (n <= 0) return;
  CUB_TWICE(cub::DeviceRadixSort::SortPairs(tmp_, bytes_, kin, kout, vin, vout, (size_t)n, 0, bits, c.s));
}
void sort_pairs_u64_i32(Ctx& c, const uint64_t* kin, uint64_t* kout, const int32_t* vin,
                        int32_t* vout, int64_t n, int bits) {
  if (n <= 0) return;
  CUB_TWICE(cub::DeviceRadixSort::SortPairs(tmp_, bytes_, kin, kout, vin, vout, (size_t)n, 0, bits, c.s));
}
void exclusive_scan_i64(Ctx& c, const int64_t* in, int64_t* out, int64_t n) {
  if (n <= 0) return;
  CUB_TWICE(cub::DeviceScan::ExclusiveSum(tmp_, bytes_, in, out, n, c.s));
}
void exclusive_scan_i32(Ctx& c, const int32_t* in, int32_t* out, int64_t n) {
  if (n <= 0) return;
  CUB_TWICE(cub::DeviceScan::ExclusiveSum(tmp_, bytes_, in, out, n, c.s));
}

int64_t select_flagged_index(Ctx& c, const uint8_t* flags, int32_t* out, int64_t n) {
  if (n <= 0) return 0;
  int64_t* dcount = (int64_t*)c.dflag;
  cub::CountingInputIterator<int32_t> it(0);
  CUB_TWICE(cub::DeviceSelect::Flagged(tmp_, bytes_, it, flags, out, dcount, n, c.s));
  return read_i64(c, dcount);
}
int64_t select_flagged_index64(Ctx& c, const uint8_t* flags, int64_t* out, int64_t n) {
  if (n <= 0) return 0;
  int64_t* dcount = (int64_t*)c.dflag;
  cub::CountingInputIterator<int64_t> it(0);
  CUB_TWICE(cub::DeviceSelect::Flagged(tmp_, bytes_, it, flags, out, dcount, n, c.s));
  return read_i64(c, dcount);
}

double reduce_max_d(Ctx& c, const double* in, int64_t n) {
  if (n <= 0) return 0.0;
  double* d = c.dscal + 200;
  CUB_TWICE(cub::DeviceReduce::Max(tmp_, bytes_, in, d, n, c.s));
  return read_scalar(c, d);
}
int64_t reduce_sum_i64(Ctx& c, const int64_t* in, int64_t n) {
  if (n <= 0) return 0;
  int64_t* d = (int64_t*)(c.dscal + 201);
  CUB_TWICE(cub::DeviceReduce::Sum(tmp_, bytes_, in, d, n, c.s));
  return read_i64(c, d);
}
int32_t reduce_max_i32(Ctx& c, const int32_t* in, int64_t n) {
  if (n <= 0) return 0;
  int32_t* d = (int32_t*)(c.dscal + 202);
  CUB_TWICE(cub::DeviceReduce::Max(tmp_, bytes_, in, d, n, c.s));
  return read_i32(c, d);
}

double read_scalar(Ctx& c, const double* d) {
  CK(cudaMemcpyAsync(c.hscal, d, sizeof(double), cudaMemcpyDeviceToHost, c.s));
  c.sync();
  return c.hscal[0];
}
int64_t read_i64(Ctx& c, const int64_t* d) {
  CK(cudaMemcpyAsync(c.hscal, d, sizeof(int64_t), cudaMemcpyDeviceToHost, c.s));
  c.sync();
  int64_t v;
  memcpy(&v, c.hscal, sizeof v);
  return v;
}
int32_t read_i32(Ctx& c, const int32_t* d) {
  CK(cudaMemcpyAsync(c.hscal, d, sizeof(int32_t), cudaMemcpyDeviceToHost, c.s));
  c.sync();
  int32_t v;
  memcpy(&v, c.hscal, sizeof v);
  return v;
}

// ------------------------------------------------------- bit-exact folds
// A left-to-right fold is one dependent chain of fp64 adds. One thread runs
// it; loads are issued 32 at a time ahead of the chain (double-buffered) so
// the chain, not memory latency, sets the pace.
// Sequential folds of K <= 32 node-major columns (the reference's left-to-
// right sums; bit-exact): three producer warps stream chunks of the input
// into a shared-memory ring while lane k of warp 0 folds column k in row
// order from shared memory. The dependent add chain, not the load latency,
// sets the pace (the former single-thread loop waited ~0.6 us per 32 loads).
constexpr int kFoldSlots = 4, kFoldSlot = 1024, kFoldThreads = 128;
template <bool SQUARE>
__global__ void __launch_bounds__(kFoldThreads) seq_cols_kernel(const double* __restrict__ x, int64_t n, int K,
                                                                double* out, bool root, bool debug = false) {
  __shared__ double ring[kFoldSlots][kFoldSlot];
  __shared__ int produced, consumed;
  const int64_t rows_per = kFoldSlot / K;
  const int64_t nchunks = (n + rows_per - 1) / rows_per;
  if (threadIdx.x == 0) produced = consumed = 0;
  __syncthreads();
  volatile int* vp = &produced;
  volatile int* vc = &consumed;
  if (threadIdx.x >= 32) {
    const int pt = threadIdx.x - 32, np = kFoldThreads - 32;
    for (int64_t k = 0; k < nchunks; ++k) {
      // one producer polls the ring (96 spinning threads would steal the
      // consumer's shared-memory bandwidth), the others wait at the barrier
      if (pt == 0)
        while (k - *vc >= kFoldSlots) {
        }
      asm volatile("bar.sync 1, %0;" ::"r"(np) : "memory");
      const int64_t r0 = k * rows_per;
      const int64_t cnt = (n - r0 < rows_per ? n - r0 : rows_per) * K;
      double* slot = ring[k % kFoldSlots];
      const double* src = x + r0 * K;
      for (int64_t j = pt; j < cnt; j += np) slot[j] = __ldcs(src + j);
      __threadfence_block();
      asm volatile("bar.sync 1, %0;" ::"r"(np) : "memory");
      if (pt == 0) *vp = (int)(k + 1);
    }
    return;
  }
  const int lane = threadIdx.x;
  double s = 0.0;
  long long t_wait = 0, t_all = clock64();
  for (int64_t k = 0; k < nchunks; ++k) {
    const long long tw = clock64();
    while (*vp <= k) {
    }
    t_wait += clock64() - tw;
    __threadfence_block();
    const int64_t r0 = k * rows_per;
    const int rows = (int)(n - r0 < rows_per ? n - r0 : rows_per);
    if (lane < K) {
      const double* slot = ring[k % kFoldSlots] + lane;
      int i = 0;
      for (; i + 16 <= rows; i += 16) {
        double v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = slot[(i + j) * K];
#pragma unroll
        for (int j = 0; j < 16; ++j) s = s + (SQUARE ? v[j] * v[j] : v[j]);
      }
      for (; i < rows; ++i) {
        const double v = slot[i * K];
        s = s + (SQUARE ? v * v : v);
      }
    }
    __syncwarp();
    __threadfence_block();
    if (lane == 0) *vc = (int)(k + 1);
  }
  if (lane < K) out[lane] = root ? sqrt(s) : s;
  if (debug && lane == 0) printf("[fold] n %lld K %d cycles %lld waiting %lld\n", (long long)n, K, clock64() - t_all, t_wait);
}

void seq_sum(Ctx& c, const double* x, int64_t n, double* d_out) {
  static const bool dbg = getenv("LAMG_FOLD_DEBUG") != nullptr;
  count_launch(), seq_cols_kernel<false><<<1, kFoldThreads, 0, c.s>>>(x, n, 1, d_out, false, dbg);
  CK_LAUNCH();
}
void seq_norm2(Ctx& c, const double* x, int64_t n, double* d_out) {
  count_launch(), seq_cols_kernel<true><<<1, kFoldThreads, 0, c.s>>>(x, n, 1, d_out, true);
  CK_LAUNCH();
}
void seq_col_sums(Ctx& c, const double* x, int64_t n, int K, double* d_out) {
  if (K < 1 || K > 32) throw LamgError(LAMG_E_ARGUMENT, "sequential column sums take 1..32 columns");
  count_launch(), seq_cols_kernel<false><<<1, kFoldThreads, 0, c.s>>>(x, n, K, d_out, false);
  CK_LAUNCH();
}

// fixed-order two-level tree reduction: deterministic for a given n
template <bool SQUARE>
__global__ void tree_partial_kernel(const double* __restrict__ x, int64_t n, double* part) {
  __shared__ double sh[kThreads];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double v = x[i];
    s += SQUARE ? v * v : v;
  }
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}
template <bool SQUARE>
__global__ void tree_final_kernel(const double* part, int np, double* out) {
  __shared__ double sh[512];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s += part[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = SQUARE ? sqrt(sh[0]) : sh[0];
}

void tree_sum(Ctx& c, const double* x, int64_t n, double* d_out) {
  double* part = c.dpart;
  int nb = (int)std::min<int64_t>(256, blocks_for(n));
  count_launch(), tree_partial_kernel<false><<<nb, kThreads, 0, c.s>>>(x, n, part);
  count_launch(), tree_final_kernel<false><<<1, 256, 0, c.s>>>(part, nb, d_out);
  CK_LAUNCH();
}
void tree_norm2(Ctx& c, const double* x, int64_t n, double* d_out) {
  double* part = c.dpart;
  int nb = (int)std::min<int64_t>(256, blocks_for(n));
  count_launch(), tree_partial_kernel<true><<<nb, kThreads, 0, c.s>>>(x, n, part);
  count_launch(), tree_final_kernel<true><<<1, 256, 0, c.s>>>(part, nb, d_out);
  CK_LAUNCH();
}

// ------------------------------------------------------- guard bands (LAMG_GUARD=1)
namespace {
__global__ void guard_fill_kernel(unsigned char* base, size_t payload) {
  const size_t t = threadIdx.x;  // kGuardBytes threads
  base[t] = (unsigned char)(0xA5 ^ t);
  base[kGuardBytes + payload + t] = (unsigned char)(0x5A ^ t);
}
__global__ void guard_check_kernel(const unsigned char* base, size_t payload, unsigned long long* bad) {
  const size_t t = threadIdx.x;
  if (base[t] != (unsigned char)(0xA5 ^ t)) atomicMin(bad, (unsigned long long)t);
  if (base[kGuardBytes + payload + t] != (unsigned char)(0x5A ^ t)) atomicMin(bad + 1, (unsigned long long)t);
}
std::atomic<long long> g_guard_checked{0}, g_guard_overruns{0};
}  // namespace

void guard_fill(void* base, size_t payload, cudaStream_t s) {
  guard_fill_kernel<<<1, (unsigned)kGuardBytes, 0, s>>>((unsigned char*)base, payload);
}

void guard_check(const void* base, size_t payload, cudaStream_t s, bool sync_free) {
  // a small synchronous check: debugging mode only
  unsigned long long* bad = nullptr;
  if (cudaMalloc((void**)&bad, 2 * sizeof(unsigned long long)) != cudaSuccess) return;
  cudaMemset(bad, 0xff, 2 * sizeof(unsigned long long));
  cudaStream_t st = sync_free ? 0 : s;
  if (sync_free) cudaDeviceSynchronize();
  guard_check_kernel<<<1, (unsigned)kGuardBytes, 0, st>>>((const unsigned char*)base, payload, bad);
  unsigned long long h[2] = {~0ull, ~0ull};
  cudaMemcpyAsync(h, bad, sizeof h, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  cudaFree(bad);
  ++g_guard_checked;
  for (int k = 0; k < 2; ++k)
    if (h[k] != ~0ull) {
      ++g_guard_overruns;
      fprintf(stderr, "[lamg guard] buffer of %zu bytes: %s band overwritten (first bad byte at offset %llu)\n", payload,
              k ? "trailing" : "leading", h[k]);
    }
}

void guard_report(long long* checked, long long* overruns) {
  *checked = g_guard_checked.load();
  *overruns = g_guard_overruns.load();
}

}  // namespace lamgb
