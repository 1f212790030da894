// SELL-C-sigma construction for the fused operator kernels (one-time work
// at batch preparation).
//
// Rows of every work unit are sorted by length (descending, ties by row
// index -- deterministic), cut into slices of 32 and stored slice-major /
// lane-minor so that in the hot kernels each thread owns one row and every
// warp load is 32 consecutive words.  Row sums then run in storage order
// (columns ascending), which is the reference's accumulation order for
// both A x (CSC scatter) and A' y (CSC gather) (_csc.pyx:17-50).
// Units with rows longer than kSellMaxRow keep the warp-per-row CSR path.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <cstdlib>

#include "handle.h"

namespace qg {

constexpr int kSellMaxRow = 256;
constexpr int64_t kMinSellSlices = 148 * 16;  // ~16 warps of slices per SM

void SellMat::release() {
  dev_free(off);
  dev_free(w);
  dev_free(col);
  dev_free(val);
  off = nullptr;
  w = nullptr;
  col = nullptr;
  val = nullptr;
}

namespace {

struct Lens {
  const int32_t *rp1, *rp2;  // row pointers (rp2 may be null)
  __device__ __forceinline__ int len1(int r) const { return rp1[r + 1] - rp1[r]; }
  __device__ __forceinline__ int len2(int r) const { return rp2 ? rp2[r + 1] - rp2[r] : 0; }
};

// key = unit << 32 | ~(len1 + len2): unit-major, longest first
__global__ void k_row_keys(const Unit *units, int nunits, Lens L, unsigned long long *keys, int32_t *rows) {
  const int u = blockIdx.x;
  if (u >= nunits) return;
  const Unit un = units[u];
  for (int r = un.row0 + threadIdx.x; r < un.row1; r += blockDim.x) {
    const unsigned len = (unsigned)(L.len1(r) + L.len2(r));
    keys[r] = ((unsigned long long)u << 32) | (unsigned long long)(0xffffffffu - len);
    rows[r] = r;
  }
}

// per slice: row of every lane, widths of the (one or two) matrices
__global__ void k_slice_meta(const int32_t *slice_pos, const int32_t *slice_n, int64_t nslices,
                             const int32_t *sorted_rows, Lens L, int32_t *rowof, int32_t *w1, int32_t *w2) {
  const int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= nslices) return;
  const int n = slice_n[s];
  const int r = lane < n ? sorted_rows[slice_pos[s] + lane] : -1;
  int a = r >= 0 ? L.len1(r) : 0, b = r >= 0 ? L.len2(r) : 0;
  rowof[s * 32 + lane] = r;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a = max(a, __shfl_xor_sync(0xffffffffu, a, o));
    b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
  }
  if (lane == 0) {
    w1[s] = a;
    if (w2) w2[s] = b;
  }
}

__global__ void k_width32(const int32_t *w, int64_t n, int64_t *out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = 32LL * w[i];
}

// warp per slice: scatter the CSR rows into the slice layout
__global__ void k_sell_fill(int64_t nslices, const int32_t *rowof, const int32_t *rp, const int32_t *csr_col,
                            const double *csr_val, const int64_t *off, const int32_t *w, int32_t *col, double *val,
                            const int32_t *cbase) {
  const int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= nslices) return;
  const int r = rowof[s * 32 + lane];
  const int k0 = r >= 0 ? rp[r] : 0, len = r >= 0 ? rp[r + 1] - k0 : 0;
  const int64_t o = off[s];
  const int width = w[s];
  // padding: value 0 at the problem's first column (a valid local index 0,
  // also for kernels that gather from a staged per-problem vector)
  const int base = cbase ? cbase[s] : 0;
  for (int k = 0; k < width; ++k) {
    const int64_t pos = o + 32LL * k + lane;
    const bool in = k < len;
    val[pos] = in ? csr_val[k0 + k] : 0.0;
    col[pos] = in ? csr_col[k0 + k] : base;
  }
}

inline unsigned nb(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

void fill_matrix(SellMat &M, int64_t nslices, const int32_t *rowof, const int32_t *wsrc, const DevCsr &csr,
                 const int32_t *d_cbase, cudaStream_t st) {
  M.w = dev_alloc<int32_t>(nslices);
  QG_CUDA(cudaMemcpyAsync(M.w, wsrc, sizeof(int32_t) * nslices, cudaMemcpyDeviceToDevice, st));
  int64_t *w32 = dev_alloc<int64_t>(nslices);
  M.off = dev_alloc<int64_t>(nslices + 1);
  k_width32<<<nb(nslices), 256, 0, st>>>(M.w, nslices, w32);
  QG_LAUNCHED();
  size_t tmp_bytes = 0;
  QG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, w32, M.off, (int)(nslices + 1), st));
  // the scan over nslices+1 items reads one past w32's end: give it a zero
  int64_t *w32x = dev_alloc<int64_t>(nslices + 1);
  QG_CUDA(cudaMemcpyAsync(w32x, w32, sizeof(int64_t) * nslices, cudaMemcpyDeviceToDevice, st));
  QG_CUDA(cudaMemsetAsync(w32x + nslices, 0, sizeof(int64_t), st));
  void *tmp = dev_alloc<char>(tmp_bytes);
  QG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, w32x, M.off, (int)(nslices + 1), st));
  count_launch(2);
  int64_t total = 0;
  QG_CUDA(cudaMemcpyAsync(&total, M.off + nslices, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  QG_CUDA(cudaStreamSynchronize(st));
  M.entries = total;
  M.col = dev_alloc<int32_t>(total);
  M.val = dev_alloc<double>(total);
  if (total > 0) {
    k_sell_fill<<<nb(nslices * 32), 256, 0, st>>>(nslices, rowof, csr.rp, csr.col, csr.val, M.off, M.w, M.col,
                                                  M.val, d_cbase);
    QG_LAUNCHED();
  }
  dev_free(tmp);
  dev_free(w32);
  dev_free(w32x);
}

// Decide modes and slice ranges on the host, sort rows on the device, build
// the slice metadata and the padded matrices.  Returns the number of slices.
// cb1 / cb2: per-problem column base of matrix 1 / 2 (X or Y offsets): the
// padding column (a valid index of the problem's own vector).
int64_t build_side(std::vector<Unit> &units, Unit *d_units, int64_t nrows, const int32_t *rp1, const int32_t *rp2,
                   const DevCsr &m1, const DevCsr *m2, SellMat &s1, SellMat *s2, int32_t **rowof_out,
                   bool allow_sell, const std::vector<int64_t> *cb1, const std::vector<int64_t> *cb2,
                   cudaStream_t st) {
  std::vector<int32_t> slice_pos, slice_n, slice_b1, slice_b2;
  int64_t ns = 0;
  const int max_row = allow_sell ? kSellMaxRow : -1;
  static const char *env_wide = std::getenv("QG_WIDE_ROW");  // A/B: mean row length for MODE_WIDE
  const int wide_row = env_wide ? std::atoi(env_wide) : kWideRow;
  // per-unit row statistics (units in parallel host chunks)
  host_parallel((int64_t)units.size(), 1024, [&](int64_t lo, int64_t hi) {
    for (int64_t ui = lo; ui < hi; ++ui) {
      Unit &u = units[ui];
      int maxlen = 0;
      int64_t total = 0, both = 0;
      for (int r = u.row0; r < u.row1; ++r) {
        const int l1 = rp1[r + 1] - rp1[r], l2 = rp2 ? rp2[r + 1] - rp2[r] : 0;
        const int len = std::max(l1, l2);
        maxlen = std::max(maxlen, len);
        total += len;
        both += l1 + l2;
      }
      // lanes per CSR row from THIS unit's mean row length: a side mixing a
      // few dense rows with many short ones (C5b) must not run the short rows
      // a warp each (measured 6x slower than per-unit lanes)
      u.lanes = 1;
      if (u.row1 > u.row0) {
        const double avg = (double)both / (double)(u.row1 - u.row0);
        while (u.lanes < 32 && u.lanes < avg * 0.75) u.lanes <<= 1;
      }
      u.mode = maxlen > max_row ? MODE_LONG : MODE_SELL;
      // rows of thousands of entries (dense feature blocks, C5b): the whole
      // CTA streams one row at a time instead of one warp per row
      if (u.mode == MODE_LONG && u.row1 > u.row0 && total >= (int64_t)wide_row * (u.row1 - u.row0))
        u.mode = MODE_WIDE;
    }
  });
  for (auto &u : units) {
    u.s0 = u.s1 = (int32_t)ns;
    if (u.mode == MODE_SELL) {
      for (int r = u.row0; r < u.row1; r += 32) {
        slice_pos.push_back(r);
        slice_n.push_back(std::min(32, u.row1 - r));
        if (cb1) slice_b1.push_back((int32_t)(*cb1)[u.prob]);
        if (cb2) slice_b2.push_back((int32_t)(*cb2)[u.prob]);
      }
      ns += (u.row1 - u.row0 + 31) / 32;
      u.s1 = (int32_t)ns;
    }
  }
  QG_CUDA(cudaMemcpyAsync(d_units, units.data(), sizeof(Unit) * units.size(), cudaMemcpyHostToDevice, st));
  trace_point("  sell side: unit modes + upload", st);
  *rowof_out = dev_alloc<int32_t>(32 * std::max<int64_t>(ns, 1));
  if (ns == 0 || nrows == 0) return ns;

  // sort rows by (unit, length desc); rows outside SELL units keep their key too
  unsigned long long *keys = dev_alloc<unsigned long long>(nrows), *keys_s = dev_alloc<unsigned long long>(nrows);
  int32_t *rows = dev_alloc<int32_t>(nrows), *rows_s = dev_alloc<int32_t>(nrows);
  Lens L{m1.rp, m2 ? m2->rp : nullptr};
  k_row_keys<<<(unsigned)units.size(), 256, 0, st>>>(d_units, (int)units.size(), L, keys, rows);
  QG_LAUNCHED();
  int end_bit = 32;
  while (end_bit < 64 && (1ULL << (end_bit - 32)) <= units.size()) ++end_bit;
  size_t tmp_bytes = 0;
  QG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys_s, rows, rows_s, (int)nrows, 0, end_bit, st));
  void *tmp = dev_alloc<char>(tmp_bytes);
  QG_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys_s, rows, rows_s, (int)nrows, 0, end_bit, st));
  count_launch(4);

  int32_t *d_pos = dev_alloc<int32_t>(ns), *d_n = dev_alloc<int32_t>(ns);
  QG_CUDA(cudaMemcpyAsync(d_pos, slice_pos.data(), sizeof(int32_t) * ns, cudaMemcpyHostToDevice, st));
  QG_CUDA(cudaMemcpyAsync(d_n, slice_n.data(), sizeof(int32_t) * ns, cudaMemcpyHostToDevice, st));
  int32_t *w1 = dev_alloc<int32_t>(ns), *w2 = m2 ? dev_alloc<int32_t>(ns) : nullptr;
  Lens L1{m1.rp, m2 ? m2->rp : nullptr};
  k_slice_meta<<<nb(ns * 32), 256, 0, st>>>(d_pos, d_n, ns, rows_s, L1, *rowof_out, w1, w2);
  QG_LAUNCHED();
  int32_t *d_b1 = nullptr, *d_b2 = nullptr;
  if (cb1) {
    d_b1 = dev_alloc<int32_t>(ns);
    QG_CUDA(cudaMemcpyAsync(d_b1, slice_b1.data(), sizeof(int32_t) * ns, cudaMemcpyHostToDevice, st));
  }
  if (cb2) {
    d_b2 = dev_alloc<int32_t>(ns);
    QG_CUDA(cudaMemcpyAsync(d_b2, slice_b2.data(), sizeof(int32_t) * ns, cudaMemcpyHostToDevice, st));
  }
  trace_point("  sell side: sort + slice meta", st);
  fill_matrix(s1, ns, *rowof_out, w1, m1, d_b1, st);
  if (m2) fill_matrix(*s2, ns, *rowof_out, w2, *m2, d_b2, st);
  QG_CUDA(cudaStreamSynchronize(st));
  trace_point("  sell side: fill", st);
  dev_free(keys); dev_free(keys_s); dev_free(rows); dev_free(rows_s); dev_free(tmp);
  dev_free(d_pos); dev_free(d_n); dev_free(w1); dev_free(w2); dev_free(d_b1); dev_free(d_b2);
  return ns;
}

}  // namespace

void build_sell(Handle &H, const int32_t *rpP, const int32_t *rpAT, const int32_t *rpA, bool force_sell,
                cudaStream_t st) {
  // Thread-per-row SELL pays off when a side has many short rows: enough
  // slices to fill the GPU with warps and rows short enough that a thread's
  // serial chain stays short.  Otherwise the side keeps G-lanes-per-row CSR
  // (small single problems, long rows).  QG_SELL=0/1 forces (A/B testing).
  const char *force = std::getenv("QG_SELL");
  auto sell_ok = [&](int64_t rows, int64_t nnz) {
    if (force) return std::atoi(force) != 0;
    if (force_sell) return true;
    const double avg = rows ? (double)nnz / rows : 0.0;
    return rows / 32 >= kMinSellSlices && avg <= 64.0;
  };
  const bool sx = sell_ok(H.NX, (int64_t)rpP[H.NX] + rpAT[H.NX]);
  const bool sy = sell_ok(H.NY, (int64_t)rpA[H.NY]);
  H.nslice_x = build_side(H.xunits, H.d_xunits, H.NX, rpP, rpAT, H.P, &H.AT, H.sP, &H.sAT, &H.x_rowof, sx,
                          &H.xoff, &H.yoff, st);
  H.nslice_y = build_side(H.cones.units, H.cones.d_units, H.NY, rpA, nullptr, H.A, nullptr, H.sA, nullptr,
                          &H.y_rowof, sy, &H.xoff, nullptr, st);
  H.has_wide = false;
  for (const auto *us : {&H.xunits, &H.cones.units})
    for (const Unit &u : *us) H.has_wide = H.has_wide || u.mode == MODE_WIDE;
  // Measured and removed: shared-memory staging of each
  // problem's gathered vectors (c5a F 0.457 -> 0.494 ms, F' 0.58 -> 0.88 ms)
  // and a shared-memory t for the F' Y side (neutral).
}

}  // namespace qg
