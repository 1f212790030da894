// Shared definitions of libqcpgrad (B200 / sm_100a).
//
// Layout of a prepared batch in HBM:
//   embedding vectors: [X: sum n | Y: sum m | T: nprob]   fp64
//   CSR(P)  over X rows, columns global X indices          int32 / fp64
//   CSR(A)  over Y rows, columns global X indices          int32 / fp64
//   CSR(A') over X rows, columns global Y indices          (= CSC(A))
//   cone blocks: table + per-class work units; DPi parameters per block.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include <algorithm>
#include <string>
#include <thread>
#include <vector>

#include "../../include/qcpgrad.h"

namespace qg {

// ---------------------------------------------------------------- errors --
struct Error {
  int code;
  std::string msg;
};

void set_error(int code, const std::string &msg);
void trace_point(const char *what, cudaStream_t st);  // QG_TRACE diagnostics (api.cu)
int fail(int code, const std::string &msg);
void count_launch(int n = 1);
// cudaFuncAttributeMaxDynamicSharedMemorySize, raised monotonically and
// thread-safely per kernel (operator.cu)
void raise_dynamic_smem(const void *kern, size_t bytes);

#define QG_CUDA(expr)                                                              \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess)                                                         \
      throw qg::Error{QG_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)}; \
  } while (0)

#define QG_LAUNCHED()                                                              \
  do {                                                                             \
    qg::count_launch();                                                            \
    cudaError_t _e = cudaGetLastError();                                           \
    if (_e != cudaSuccess)                                                         \
      throw qg::Error{QG_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(_e)}; \
  } while (0)

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kSlots = 4;  // partial-sum doubles per work unit

// Block classes of the fused Y-side work units.
enum UnitClass : int32_t { CLS_ELEM = 0, CLS_SOC = 1, CLS_PSD = 2, CLS_TRI = 3 };

// Per-block parameter record (one per cone block of the batch).
struct BlockInfo {
  int32_t kind;     // qg_cone_kind
  int32_t row;      // first global Y row
  int32_t dim;
  int32_t order;    // psd order
  double alpha;     // pow exponent
  int64_t param;    // soc index / tri index / psd storage offset (V then B)
  int32_t prob;     // problem index
  int32_t local;    // block index within its problem
};

// Prepared derivative data of the blockwise projection.
//   elem (zero/nonneg):  weight derived from zmid on the fly
//   soc:   soc_nu[blk], soc_code[blk] (0 zero map, 1 identity, 2 half, 3 formula)
//   psd:   V (order^2, column major) and B (order^2) at BlockInfo::psd_off
//   tri:   tri_D[9*blk] dense 3x3 and tri_flip[blk] (1 -> d - D d)
struct DpiView {
  const BlockInfo *blk;
  const double *zmid;     // the point (Y layout)
  const double *soc_nu;
  const int32_t *soc_code;
  const double *psd;
  const double *tri_D;
  const int32_t *tri_flip;
  int32_t dual;           // derivative of the dual projection (else primal)
};

// A unit of work: a contiguous row range of one problem; Y-units also cover
// whole cone blocks [blk0, blk1) of one class.
struct Unit {
  int32_t prob;
  int32_t row0, row1;
  int32_t blk0, blk1;
  int32_t cls;
  int32_t mode;    // MODE_SELL: thread-per-row over SELL slices [s0, s1); MODE_LONG: G lanes per CSR
                   // row; MODE_WIDE: the whole CTA per CSR row (rows of thousands of entries)
  int32_t s0, s1;
  int32_t group;   // SOC units: 1 = thread-per-block fused epilogue (dims <= 32); 0 = generic CTA path
  int32_t lanes;   // CSR lanes per row for this unit's rows (power of two <= 32, from its mean row length)
};

enum UnitMode : int32_t { MODE_SELL = 0, MODE_LONG = 1, MODE_WIDE = 2 };
constexpr int kWideRow = 512;   // mean entries per row from which a CSR unit goes CTA-per-row

// SELL-C-sigma storage (C = 32 = warp width, sigma = the work unit): the rows
// of a unit are sorted by length (descending) and cut into slices of 32; in
// slice s entry k of lane l sits at off[s] + 32 k + l, so a warp reads 32
// consecutive values per step (fully coalesced) and each thread owns one row.
struct SellView {
  const int64_t *off;   // [nslices] first entry of the slice
  const int32_t *w;     // [nslices] slice width (longest row)
  const int32_t *col;   // padded entries: col 0, val 0 (global column index)
  const double *val;
};

// ------------------------------------------------------------ host utils --
// fn(lo, hi) over [0, n) split across up to 16 host threads, at least
// min_chunk items each (batch preparation loops over rows / blocks of
// independent problems).  fn must not throw.
template <class F>
void host_parallel(int64_t n, int64_t min_chunk, F fn) {
  const int64_t hw = std::max<int64_t>(1, (int64_t)std::thread::hardware_concurrency());
  const int64_t T = std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(hw, 16), n / std::max<int64_t>(min_chunk, 1)));
  if (T <= 1) {
    fn((int64_t)0, n);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(T - 1);
  for (int64_t t = 1; t < T; ++t) th.emplace_back(fn, n * t / T, n * (t + 1) / T);
  fn((int64_t)0, n / T);
  for (auto &x : th) x.join();
}

// Page-locked staging buffer of this host thread (grow-only): large
// device<->host copies of batch preparation run at DMA speed.
void *pinned_staging(size_t bytes, int slot);

// ---------------------------------------------------------- device utils --
// Programmatic dependent launch (sm_90+): the LSMR loop's kernels are
// launched with programmatic stream serialization, so the next kernel's
// launch and CTA scheduling overlap this one's tail.  Every such kernel
// waits (pdl_wait) before its first read of data produced by the previous
// kernel, and lets the next one start (pdl_trigger) once its main work is
// issued.  Both are no-ops for ordinary launches.
// Device-side invariant checks of a QG_CHECKS=1 build (index bounds of the
// gathers, slice rows, resident plans, block tables): a violated check traps
// (the kernel fails with an error the host reports), so the GPU test suite
// run against that build is a bounds / consistency sanitizer.  Compiled out
// of the production library.  (compute-sanitizer is not available on the
// GPU pool.)
#if defined(QG_CHECKS) && QG_CHECKS
#define QG_CHECK(cond)         \
  do {                         \
    if (!(cond)) __trap();     \
  } while (0)
#else
#define QG_CHECK(cond) \
  do {                 \
  } while (0)
#endif

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic CTA reduction of kSlots values (fixed tree order); result in
// out[] on thread 0.
__device__ __forceinline__ void cta_sum_slots(double (&v)[kSlots], double *smem_red, double *out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < kSlots; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < kSlots; ++k) smem_red[warp * kSlots + k] = v[k];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < kSlots; ++k) {
      double s = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += smem_red[w * kSlots + k];
      out[k] = s;
    }
  }
  __syncthreads();
}

// NVTX range for the phases of an API call (preparation, LSMR solve,
// assembly); visible in nsys / ncu --nvtx.  Header-only NVTX v3.
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};

// Stream-ordered allocation from the device's default memory pool (kept
// resident between handles: no cudaMalloc/cudaFree synchronisation on the
// per-batch path).  The stream is the calling API entry's stream.
cudaStream_t &alloc_stream();
void init_pool();

template <class T>
inline T *dev_alloc(size_t count) {
  if (count == 0) count = 1;
  init_pool();
  T *p = nullptr;
  QG_CUDA(cudaMallocAsync((void **)&p, count * sizeof(T), alloc_stream()));
  return p;
}

inline void dev_free(void *p) {
  if (p) cudaFreeAsync(p, alloc_stream());
}

// Sets the allocation stream for the duration of an API call.
struct StreamScope {
  cudaStream_t prev;
  explicit StreamScope(cudaStream_t s) : prev(alloc_stream()) { alloc_stream() = s; }
  ~StreamScope() { alloc_stream() = prev; }
};

}  // namespace qg
