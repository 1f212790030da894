// CSC -> CSR conversion on the device (one-time preparation work).
//
// The reference stores matrices in CSC with int64 indices (sparse.py:19-73)
// and computes A x by a storage-order scatter (_csc.pyx:17-32).  The GPU
// path needs row-major access for deterministic gathers, so the batch is
// transposed once: a warp per column emits (global row key, global column)
// per entry, a stable CUB radix sort on the row key yields the CSR order
// (columns stay ascending inside a row because the input is column-major),
// and row pointers come from a binary search over the sorted keys.
#include <cub/device/device_radix_sort.cuh>

#include "handle.h"

namespace qg {

void DevCsr::release() {
  dev_free(rp);
  dev_free(col);
  dev_free(val);
  dev_free(perm);
  rp = col = perm = nullptr;
  val = nullptr;
}

namespace {

struct Offsets {
  const int64_t *coff;   // [B+1] global column offsets
  const int64_t *roff;   // [B+1] global row offsets
  const int64_t *noff;   // [B+1] global entry offsets
  const int64_t *cpoff;  // [B] start of problem p's colptr in the concatenated colptr
  int B;
};

__device__ __forceinline__ int find_prob(const int64_t *off, int B, int64_t v) {
  int lo = 0, hi = B;  // off[lo] <= v < off[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (off[mid] <= v) lo = mid; else hi = mid;
  }
  return lo;
}

// One warp per global column: write row keys and entry columns; also the
// CSC-as-rows pointer array.
__global__ void k_emit_keys(const int64_t *colptr, const int64_t *rowidx, Offsets o, int64_t ncols_total,
                            int32_t *keys, int32_t *ecol, int32_t *csc_rp) {
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= ncols_total) return;
  const int p = find_prob(o.coff, o.B, c);
  const int64_t j = c - o.coff[p];
  const int64_t *cp = colptr + o.cpoff[p];
  const int64_t k0 = cp[j], k1 = cp[j + 1];
  const int64_t base = o.noff[p];
  if (lane == 0 && csc_rp) {
    csc_rp[c] = (int32_t)(base + k0);
    if (c == ncols_total - 1) csc_rp[c + 1] = (int32_t)(base + k1);
  }
  for (int64_t k = k0 + lane; k < k1; k += 32) {
    keys[base + k] = (int32_t)(o.roff[p] + rowidx[base + k]);
    ecol[base + k] = (int32_t)c;
  }
}

__global__ void k_iota(int32_t *v, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = (int32_t)i;
}

__global__ void k_rowptr(const int32_t *sorted_keys, int64_t nnz, int64_t nrows, int32_t *rp) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r > nrows) return;
  int64_t lo = 0, hi = nnz;  // first position with key >= r
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (sorted_keys[mid] < r) lo = mid + 1; else hi = mid;
  }
  rp[r] = (int32_t)lo;
}

__global__ void k_gather(const int32_t *perm, const int32_t *ecol, const double *vals, int64_t nnz,
                         int32_t *col, double *val) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nnz) return;
  const int32_t s = perm[k];
  col[k] = ecol[s];
  val[k] = vals[s];
}

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

void csc_to_csr(const CscBatch &in, DevCsr &out, DevCsr *csc_as_rows, bool keep_perm, cudaStream_t st) {
  const int B = (int)in.nnz.size();
  std::vector<int64_t> coff(B + 1, 0), roff(B + 1, 0), noff(B + 1, 0), cpoff(B, 0);
  for (int p = 0; p < B; ++p) {
    coff[p + 1] = coff[p] + in.ncols[p];
    roff[p + 1] = roff[p] + in.nrows[p];
    noff[p + 1] = noff[p] + in.nnz[p];
    cpoff[p] = (p == 0) ? 0 : cpoff[p - 1] + in.ncols[p - 1] + 1;
  }
  const int64_t nnz = noff[B], ncols = coff[B], nrows = roff[B];
  if (nnz >= (int64_t)INT32_MAX || nrows >= (int64_t)INT32_MAX || ncols >= (int64_t)INT32_MAX)
    throw Error{QG_ERR_UNSUPPORTED, "matrix too large for 32-bit indices"};
  int64_t *d_off = dev_alloc<int64_t>(4 * (size_t)B + 3);
  std::vector<int64_t> hoff;
  hoff.insert(hoff.end(), coff.begin(), coff.end());
  hoff.insert(hoff.end(), roff.begin(), roff.end());
  hoff.insert(hoff.end(), noff.begin(), noff.end());
  hoff.insert(hoff.end(), cpoff.begin(), cpoff.end());
  QG_CUDA(cudaMemcpyAsync(d_off, hoff.data(), sizeof(int64_t) * hoff.size(), cudaMemcpyHostToDevice, st));
  Offsets o{d_off, d_off + (B + 1), d_off + 2 * (B + 1), d_off + 3 * (B + 1), B};

  int32_t *keys = dev_alloc<int32_t>(nnz), *ecol = dev_alloc<int32_t>(nnz);
  int32_t *keys_sorted = dev_alloc<int32_t>(nnz), *iota = dev_alloc<int32_t>(nnz);
  int32_t *perm = dev_alloc<int32_t>(nnz);
  int32_t *csc_rp = nullptr;
  if (csc_as_rows) csc_rp = dev_alloc<int32_t>(ncols + 1);
  if (ncols > 0) {
    k_emit_keys<<<blocks_for(ncols * 32, 256), 256, 0, st>>>(in.colptr, in.rowidx, o, ncols, keys, ecol, csc_rp);
    QG_LAUNCHED();
  } else if (csc_rp) {
    QG_CUDA(cudaMemsetAsync(csc_rp, 0, sizeof(int32_t), st));
  }
  out.nrows = nrows;
  out.nnz = nnz;
  out.rp = dev_alloc<int32_t>(nrows + 1);
  out.col = dev_alloc<int32_t>(nnz);
  out.val = dev_alloc<double>(nnz);
  if (nnz > 0) {
    k_iota<<<blocks_for(nnz, 256), 256, 0, st>>>(iota, nnz);
    QG_LAUNCHED();
    int end_bit = 1;
    while (end_bit < 31 && (1LL << end_bit) <= nrows) ++end_bit;
    size_t tmp_bytes = 0;
    QG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys_sorted, iota, perm, (int)nnz, 0,
                                            end_bit, st));
    void *tmp = dev_alloc<char>(tmp_bytes);
    QG_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys_sorted, iota, perm, (int)nnz, 0, end_bit,
                                            st));
    count_launch(4);
    k_gather<<<blocks_for(nnz, 256), 256, 0, st>>>(perm, ecol, in.vals, nnz, out.col, out.val);
    QG_LAUNCHED();
    QG_CUDA(cudaStreamSynchronize(st));
    dev_free(tmp);
  }
  k_rowptr<<<blocks_for(nrows + 1, 256), 256, 0, st>>>(keys_sorted, nnz, nrows, out.rp);
  QG_LAUNCHED();
  if (csc_as_rows) {
    csc_as_rows->nrows = ncols;
    csc_as_rows->nnz = nnz;
    csc_as_rows->rp = csc_rp;
    csc_as_rows->col = keys;  // global row of every CSC entry, storage order
    keys = nullptr;
    csc_as_rows->val = nullptr;
  }
  QG_CUDA(cudaStreamSynchronize(st));
  if (keep_perm) out.perm = perm; else dev_free(perm);
  dev_free(keys);
  dev_free(ecol);
  dev_free(keys_sorted);
  dev_free(iota);
  dev_free(d_off);
}

}  // namespace qg
