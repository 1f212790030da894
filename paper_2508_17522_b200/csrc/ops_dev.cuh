// Device-side argument bundles shared by the operator, LSMR and assembly
// kernels.
#pragma once

#include "handle.h"

namespace qg {

struct Mats {
  const int32_t *P_rp, *P_col; const double *P_val;
  const int32_t *AT_rp, *AT_col; const double *AT_val;
  const int32_t *A_rp, *A_col; const double *A_val;
  const Unit *xu, *yu;
  int nxu, nyu;
  const int64_t *xu_ptr, *yu_ptr;  // [B+1] unit ranges per problem
  const double *q, *b, *Pxbar, *xbar, *ybar, *sbar;
  const Embed *emb;
  int64_t NX, NY;
  DpiView dpi;
  SellView sP, sAT, sA;                 // SELL copies (MODE_SELL units)
  const int32_t *x_rowof, *y_rowof;     // lane -> row per slice (-1 = padding)
  const int64_t *xoff, *yoff;           // [B+1] problem offsets in X / Y
  int x_owner;                          // 0: X rows are replicated and counted by rank 0 only
  const int32_t *ft_order;              // F' launch order of the units (PSD first), or null
};

// Row-partitioned mode, X side of an operator step / rhs assembly:
//   X_FULL    normal fused X rows (whole problems)
//   X_PARTIAL X units write this rank's A' partial product to xred (no row
//             update); Y units run as usual
//   X_FINISH  X units only: row update with the summed A' product from xred
enum XMode : int { X_FULL = 0, X_PARTIAL = 1, X_FINISH = 2 };

// Streamed matrix loads (each stored entry is read once per step):
// read-only and not allocated in L1, so the gathered vectors keep the L1 to
// themselves (c5a: F 0.462 -> 0.454 ms, F' 0.584 -> 0.574 ms vs __ldcs).
// (Measured and dropped: an L2 evict-first policy on these loads, within
// 0.3% on c5a, c5b and c3.)
__device__ __forceinline__ double ld_stream(const double *p) {
  double v;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ld_stream(const int *p) {
  int v;
  asm("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// Two slices of one matrix at once (independent load streams -> twice the
// memory-level parallelism per warp); slice b may be absent (sb < 0).  Each
// lane's sums stay in storage order.
// UNR: unroll of the entry loop.  Measured on c5a (ms, F / F'): 2 -> 0.520 /
// 0.527, 4 -> 0.454 / 0.574, 8 -> 0.563 / 0.588: the F step wants 4, the F'
// step (which also carries the epilogue at 40 registers) wants 2.
// (Measured and dropped: 16-bit problem-local column indices -- the gathers
// are latency-, not byte-bound, and the local base costs an add per entry.)
template <int UNR>
__device__ __forceinline__ void sell_dot2(const SellView &S, int64_t sa, int64_t sb, int lane, const double *vec,
                                          double &acc_a, double &acc_b) {
  const int64_t oa = S.off[sa] + lane, ob = sb >= 0 ? S.off[sb] + lane : 0;
  const int wa = S.w[sa], wb = sb >= 0 ? S.w[sb] : 0;
  const int wm = wa < wb ? wa : wb;
  const int32_t *colp = S.col;
  double a = 0.0, b = 0.0;
  int k = 0;
#pragma unroll UNR
  for (; k < wm; ++k) {
    const int64_t pa = oa + 32LL * k, pb = ob + 32LL * k;
    const double va = ld_stream(S.val + pa), vb = ld_stream(S.val + pb);
    const int ca = ld_stream(colp + pa), cb = ld_stream(colp + pb);
    QG_CHECK(ca >= 0 && cb >= 0);
    a += va * vec[ca];
    b += vb * vec[cb];
  }
#pragma unroll 4
  for (int j = k; j < wa; ++j) {
    const int64_t pa = oa + 32LL * j;
    a += ld_stream(S.val + pa) * vec[ld_stream(colp + pa)];
  }
#pragma unroll 4
  for (int j = k; j < wb; ++j) {
    const int64_t pb = ob + 32LL * j;
    b += ld_stream(S.val + pb) * vec[ld_stream(colp + pb)];
  }
  acc_a = a;
  acc_b = b;
}

// CTA-strided dot of one long CSR row (MODE_WIDE): thread t takes entries
// t, t + blockDim, ... into 4 rotating partial sums, combined pairwise.
__device__ __forceinline__ double wide_dot(const int32_t *rp, const int32_t *col, const double *val,
                                           const double *vec, int r) {
  const int k1 = rp[r + 1], step = (int)blockDim.x;
  double a = 0.0, b = 0.0, c = 0.0, d = 0.0;
  int k = rp[r] + (int)threadIdx.x;
  for (; k + 3 * step < k1; k += 4 * step) {
    a += ld_stream(val + k) * vec[ld_stream(col + k)];
    b += ld_stream(val + k + step) * vec[ld_stream(col + k + step)];
    c += ld_stream(val + k + 2 * step) * vec[ld_stream(col + k + 2 * step)];
    d += ld_stream(val + k + 3 * step) * vec[ld_stream(col + k + 3 * step)];
  }
  for (; k < k1; k += step) a += ld_stream(val + k) * vec[ld_stream(col + k)];
  return (a + b) + (c + d);
}

// Warp-per-row dot (G = 32), lane-strided in storage order per lane.
__device__ __forceinline__ double row_dot32(const int32_t *rp, const int32_t *col, const double *val,
                                            const double *vec, int r, int lane) {
  double s = 0.0;
  const int k1 = rp[r + 1];
#pragma unroll 4
  for (int k = rp[r] + lane; k < k1; k += 32) s += val[k] * vec[col[k]];
  return s;
}

// R rows per warp at once (rows r0, r0 + stride, ...; valid ones only): one
// loop walks all R rows together, so the R rows' column / value loads and
// vector gathers are in flight at the same time instead of R serial
// load -> gather chains.  Each row still sums its lane's entries k, k + 32,
// ... in the same order as row_dot32, so the row sums are bit-identical.
template <int R>
__device__ __forceinline__ void row_dot32_multi(const int32_t *rp, const int32_t *col, const double *val,
                                                const double *vec, int r0, int stride, int r_end, int lane,
                                                double (&s)[R]) {
  int k[R], ke[R];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const int r = r0 + j * stride;
    const bool ok = r < r_end;
    k[j] = ok ? rp[r] + lane : 0;
    ke[j] = ok ? rp[r + 1] : 0;
    s[j] = 0.0;
  }
  for (;;) {
    bool any = false;
#pragma unroll
    for (int j = 0; j < R; ++j)
      if (k[j] < ke[j]) {
        s[j] += val[k[j]] * vec[col[k[j]]];
        k[j] += 32;
        any = true;
      }
    if (!any) break;
  }
}

// Group-of-G sum inside a warp (G power of two, runtime).
__device__ __forceinline__ double gsum(double v, int G) {
  for (int o = G >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// R rows per lane group at once (rows r0, r0 + stride, ...; rows >= r_end
// give 0), each summed in row_dot's order (bit-identical row sums).
template <int R>
__device__ __forceinline__ void row_dot_multi(const int32_t *rp, const int32_t *col, const double *val,
                                              const double *vec, int r0, int stride, int r_end, int lane_g, int G,
                                              double (&s)[R]) {
  int k[R], ke[R];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const int r = r0 + j * stride;
    const bool ok = r < r_end;
    k[j] = ok ? rp[r] + lane_g : 0;
    ke[j] = ok ? rp[r + 1] : 0;
    s[j] = 0.0;
  }
  for (;;) {
    bool any = false;
#pragma unroll
    for (int j = 0; j < R; ++j)
      if (k[j] < ke[j]) {
        s[j] += val[k[j]] * vec[col[k[j]]];
        k[j] += G;
        any = true;
      }
    if (!any) break;
  }
}

// Row dot product by a group of G lanes: sum_k val[k] * vec[col[k]].
__device__ __forceinline__ double row_dot(const int32_t *rp, const int32_t *col, const double *val,
                                          const double *vec, int r, int lane_g, int G) {
  double s = 0.0;
  const int k1 = rp[r + 1];
  for (int k = rp[r] + lane_g; k < k1; k += G) s += val[k] * vec[col[k]];
  return s;
}

}  // namespace qg
