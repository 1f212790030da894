// The hot path: one LSMR iteration on the implicit-function operator
//   F w  = ((D_uQ - I) D Pi + I) w / z_N        (embedding.py:399-427)
// and its transpose, for a whole batch of problems at once.
//
// Per iteration:
//   k_step<F>   u <- s_in * F v  - c_out * u   fused CSR SpMV (P, A', A) + epilogue
//   k_fin       per problem: T component, ||u||, scalars          (lsmr.py:115-118)
//   k_step<FT>  v <- s_in * F' u - c_out * v   SpMV + D Pi epilogue (x2) per cone block
//   k_fin       ||v||, Givens recurrences, update coefficients   (lsmr.py:119-171)
//   k_update    hbar, x, h axpys + ||x||^2 partials               (lsmr.py:142-144, 168)
//   k_fin       stopping rules                                     (lsmr.py:173-182)
// The LSMR vectors are kept unnormalised ("raw") with per-problem scale
// factors, so no kernel has to wait for a norm before writing its output.
#include <map>
#include <mutex>

#include "dpi_dev.cuh"
#include "lsmr_dev.cuh"
#include "ops_dev.cuh"
#include "operator.h"

namespace qg {

__device__ __forceinline__ bool lsmr_runs(const StepArgs &a, int p, double &s_in, double &c_out) {
  const Lsmr *st = a.st;
  const int is_v_step = a.is_v_step;
  if (!st) {
    s_in = a.fixed_s_in != 0.0 ? a.fixed_s_in : 1.0;
    c_out = a.old ? a.fixed_c_out : 0.0;
    return true;
  }
  const Lsmr &L = st[p];
  s_in = L.s_in;
  c_out = L.c_out;
  return L.active && !(is_v_step && L.skip_v);
}

// ------------------------------------------------------------- op steps --
// Iterate the rows of a unit: MODE_SELL -> one thread per row over the unit's
// SELL slices; MODE_LONG -> a group of G lanes per CSR row.  `row(r, s1, s2)`
// receives the row sums of the one or two matrices (second may be unused).
// WIDE: compile the CTA-per-row path (MODE_WIDE units exist); kept out of the
// common kernels, whose SELL loops lose ~15% to its extra shared state.
#ifndef QG_ROWS32
#define QG_ROWS32 2  // CSR rows walked together per warp on the warp-per-row path, F step (1: one at a time)
#endif
#ifndef QG_ROWS32_SELL
#define QG_ROWS32_SELL 1  // same, F step of SELL handles (8 CTAs/SM; multi-row walks cost c5a F 0.4515 -> 0.472 ms)
#endif
#ifndef QG_ROWS32_FT
#define QG_ROWS32_FT 1  // same for the F' step: c2 / c3 / c4 F 0.0086 / 0.0320 / 0.0325 -> 0.0080 / 0.0297 /
#endif                  // 0.0329 ms with 2 rows; F' c4 0.0847 -> 0.0874 (4 rows: slower everywhere)
#ifndef QG_ROWSG
#define QG_ROWSG 2  // row groups walked together per warp on the G-lanes-per-row path, F step:
#endif                // c2 / c3 F 0.0079 / 0.0298 -> 0.0076 / 0.0290 ms with 2 (4: 0.0078 / 0.0297)
#ifndef QG_ROWSG_FT
#define QG_ROWSG_FT 4  // same, F' step: c5b F' 0.2671 -> 0.2595 ms with 4 (2: 0.2676),
#endif                   // c3 0.0272 -> 0.0276, c2 / c4 neutral
#ifndef QG_SLICE_CLAIM
#define QG_SLICE_CLAIM 2  // SELL slices claimed (and streamed together) per warp: 1 or 2
#endif
// One row sum kept by a lane until its epilogue runs (for_rows' CSR paths).
struct RowKeep {
  double s1 = 0.0, s2 = 0.0;
  int r = -1;
  __device__ __forceinline__ void set(int row, double a, double b) {
    r = row;
    s1 = a;
    s2 = b;
  }
  template <class RowFn>
  __device__ __forceinline__ void flush(RowFn &row) {
    if (r >= 0) row(r, s1, s2);
    r = -1;
  }
};

template <bool WIDE, int UNR, int ROWS32, int ROWSG, class RowFn>
__device__ __forceinline__ void for_rows(const Unit &u, const SellView &S1, const SellView *S2,
                                         const int32_t *rowof, const int32_t *rp1, const int32_t *c1,
                                         const double *v1, const int32_t *rp2, const int32_t *c2,
                                         const double *v2, const double *x1, const double *x2, int G,
                                         int64_t b1, int64_t b2, RowFn row) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (u.mode == MODE_SELL) {
    // warps take pairs of slices in a fixed round-robin order: every row goes
    // to the same thread on every run, so the row callbacks' partial sums are
    // bit-reproducible (dynamic claims through a shared-memory counter made
    // them depend on warp timing)
    const int nw = (int)(blockDim.x >> 5);
    for (int s = u.s0 + warp * QG_SLICE_CLAIM; s < u.s1; s += nw * QG_SLICE_CLAIM) {
      const int sb = (QG_SLICE_CLAIM == 2 && s + 1 < u.s1) ? s + 1 : -1;
      const int ra = rowof[(int64_t)s * 32 + lane];
      const int rb = sb >= 0 ? rowof[(int64_t)sb * 32 + lane] : -1;
      double a1, b1v, a2 = 0.0, b2v = 0.0;
      sell_dot2<UNR>(S1, s, sb, lane, x1, a1, b1v);
      if (S2) sell_dot2<UNR>(*S2, s, sb, lane, x2, a2, b2v);
      if (ra >= 0) row(ra, a1, a2);
      if (rb >= 0) row(rb, b1v, b2v);
    }
  } else if (WIDE && u.mode == MODE_WIDE) {
    // the whole CTA per CSR row: 4 independent partial sums per thread keep
    // the loads in flight, then a fixed-order warp / CTA reduction
    __shared__ double wred[2 * 32];
    const int nw = (int)(blockDim.x >> 5);
    for (int r = u.row0; r < u.row1; ++r) {
      double s1 = wide_dot(rp1, c1, v1, x1, r), s2 = rp2 ? wide_dot(rp2, c2, v2, x2, r) : 0.0;
      s1 = warp_sum(s1);
      s2 = warp_sum(s2);
      if (lane == 0) {
        wred[warp] = s1;
        wred[32 + warp] = s2;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        double t1 = wred[0], t2 = wred[32];
        for (int w = 1; w < nw; ++w) {
          t1 += wred[w];
          t2 += wred[32 + w];
        }
        row(r, t1, t2);
      }
      __syncthreads();
    }
  } else if (G == 32) {
    // warp per row with a compile-time lane stride: the loop unrolls into
    // independent loads (a runtime stride measured 7x slower on C5b).
    // Row epilogues are spread over the lanes: after the xor reduction every
    // lane holds the row's sums, lane k keeps the warp's k-th row (mod 32)
    // and every 32 rows (and at the end) each lane runs row() for the row it
    // keeps -- 32 epilogues (their loads) in parallel instead of lane 0
    // running them one after another
    RowKeep keep;
    int k = 0;
    auto put = [&](int r, double a, double b) {
      if (lane == k) keep.set(r, a, b);
      if (++k == 32) {
        keep.flush(row);
        k = 0;
      }
    };
    if constexpr (ROWS32 > 1) {
      // ROWS32 rows of the warp's row sequence at once (same rows, same
      // order as the one-row loop)
      const int nw = (int)(blockDim.x >> 5);
      constexpr int R = ROWS32;
      for (int r0 = u.row0 + warp; r0 < u.row1; r0 += R * nw) {
        double s1[R], s2[R];
        row_dot32_multi<R>(rp1, c1, v1, x1, r0, nw, u.row1, lane, s1);
        if (rp2) row_dot32_multi<R>(rp2, c2, v2, x2, r0, nw, u.row1, lane, s2);
#pragma unroll
        for (int j = 0; j < R; ++j) {
          s1[j] = warp_sum(s1[j]);
          s2[j] = rp2 ? warp_sum(s2[j]) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < R; ++j)
          if (r0 + j * nw < u.row1) put(r0 + j * nw, s1[j], s2[j]);
      }
    } else {
      for (int r = u.row0 + warp; r < u.row1; r += (int)(blockDim.x >> 5)) {
        double s1 = row_dot32(rp1, c1, v1, x1, r, lane);
        double s2 = rp2 ? row_dot32(rp2, c2, v2, x2, r, lane) : 0.0;
        s1 = warp_sum(s1);
        s2 = warp_sum(s2);
        put(r, s1, s2);
      }
    }
    keep.flush(row);
  } else {
    // G lanes per CSR row (G from the average row length of the matrices),
    // loops warp-uniform so every lane reaches the shuffles; the epilogues
    // are spread over each group's G lanes as above (lane lg keeps the
    // group's k-th row mod G)
    const int lg = lane & (G - 1), gpw = 32 / G, nw = (int)(blockDim.x >> 5);
    RowKeep keep;
    int k = 0;
    auto put = [&](bool valid, int r, double a, double b) {
      if (valid && lg == k) keep.set(r, a, b);
      if (++k == G) {
        keep.flush(row);
        k = 0;
      }
    };
    if constexpr (ROWSG > 1) {
      // ROWSG row groups of the warp's sequence at once
      constexpr int R = ROWSG;
      const int stride = nw * gpw;
      for (int base = u.row0 + warp * gpw; base < u.row1; base += R * stride) {
        const int r = base + lane / G;
        double s1[R], s2[R];
        row_dot_multi<R>(rp1, c1, v1, x1, r, stride, u.row1, lg, G, s1);
        if (rp2) row_dot_multi<R>(rp2, c2, v2, x2, r, stride, u.row1, lg, G, s2);
#pragma unroll
        for (int j = 0; j < R; ++j) {
          s1[j] = gsum(s1[j], G);
          s2[j] = rp2 ? gsum(s2[j], G) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < R; ++j) put(r + j * stride < u.row1, r + j * stride, s1[j], s2[j]);
      }
    } else {
      for (int base = u.row0 + warp * gpw; base < u.row1; base += nw * gpw) {
        const int r = base + lane / G;
        const bool valid = r < u.row1;
        double s1 = valid ? row_dot(rp1, c1, v1, x1, r, lg, G) : 0.0;
        double s2 = (valid && rp2) ? row_dot(rp2, c2, v2, x2, r, lg, G) : 0.0;
        s1 = gsum(s1, G);
        s2 = gsum(s2, G);
        put(valid, r, s1, s2);
      }
    }
    keep.flush(row);
  }
}

// F'-step epilogue for a unit of SOC blocks of dim <= 32: one thread per
// block (soc_entry, dpi_dev.cuh, applied twice).  Entries stream through L1
// in three short passes with independent loads (no shuffles, no CTA barrier).
template <class Fin>
__device__ __forceinline__ void soc_epilogue(const DpiView &dv, const Unit &u, const double *t, Fin fin_row,
                                             const double *outY, double *dpout) {
  for (int k = u.blk0 + (int)threadIdx.x; k < u.blk1; k += blockDim.x) {
    const BlockInfo b = dv.blk[k];
    const int dim = b.dim, row = b.row, code = dv.soc_code[b.param];
    const double nu = dv.soc_nu[b.param];
    const double *z = dv.zmid + row, *tt = t + row;
    const double t0 = z[0], dt = tt[0];
    double udu = 0.0;
    for (int i = 1; i < dim; ++i) udu += z[i] * tt[i];
    double o0 = 0.0, udu2 = 0.0;
    for (int i = 0; i < dim; ++i) {
      const double o = fin_row(row + i, soc_entry(code, i, nu, t0, z[i], tt[i], dt, udu));
      if (i == 0) o0 = o; else udu2 += z[i] * o;
    }
    if (dpout)
      for (int i = 0; i < dim; ++i) {
        const double oi = i == 0 ? o0 : outY[row + i];
        dpout[row + i] = soc_entry(code, i, nu, t0, z[i], oi, o0, udu2);
      }
  }
}

// 128-thread CTAs: more slice pairs per warp inside a unit (smaller tail at the
// closing reduction) at the same register-limited occupancy (8 CTAs/SM).
constexpr int kStepThreads = 128;
#ifndef QG_F_UNROLL
#define QG_F_UNROLL 4
#endif
#ifndef QG_FT_UNROLL
#define QG_FT_UNROLL 2
#endif
#ifndef QG_PSD_PREFETCH
#define QG_PSD_PREFETCH 1
#endif
constexpr int kFeatDist = 1, kFeatRk1 = 2, kFeatWide = 4, kFeatDF = 8;
constexpr int kFeatAll = kFeatDist | kFeatRk1 | kFeatWide;

// Deferred finalize (kFeatDF, single-problem graph loops): CTA 0 of a step
// launch runs the previous step's finalize and publishes its coefficients
// (defined with the finalize kernels below).
__device__ void df_fin(const Mats &M, const StepArgs &a);

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned *p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// FEAT bits: kFeatWide (CTA-per-row units), kFeatDist (row-partitioned
// X_PARTIAL / X_FINISH phases), kFeatRk1 (refine rank-one term, applied when
// a.rk1 is set).
// The common variant (0) carries none of them.
// One work unit (`ui`: X units then Y units) of an operator step, by the
// whole CTA; the partial-sum slot of the unit is part[ui].
template <int KIND, int FEAT, bool SELL8 = false>
__device__ __forceinline__ void step_unit(const Mats &M, const StepArgs &a, int ui) {
  constexpr bool kDist = (FEAT & kFeatDist) != 0, kWide = (FEAT & kFeatWide) != 0;
  constexpr int kUnr = KIND == STEP_F ? QG_F_UNROLL : QG_FT_UNROLL;  // SELL entry-loop unroll
  // rows per warp, warp-per-row CSR; SELL8 = the 8-CTA/SM SELL F instantiation
  constexpr int kRows32 = KIND == STEP_F ? (SELL8 ? QG_ROWS32_SELL : QG_ROWS32) : QG_ROWS32_FT;
  // row groups per warp, G-lane CSR (the SELL F kernel: one group, as for ROWS32)
  constexpr int kRowsG = KIND == STEP_F ? (SELL8 ? 1 : QG_ROWSG) : QG_ROWSG_FT;
  const bool kRk1 = (FEAT & kFeatRk1) != 0 && a.rk1 != nullptr;
  extern __shared__ double sm[];
  __shared__ double red[kWarps * kSlots];
  const bool isx = ui < M.nxu;
  const Unit u = isx ? M.xu[ui] : M.yu[ui - M.nxu];  // preparation-time data: before the PDL wait
  const int p = u.prob;
  const Embed E = M.emb[p];                            // (also preparation-time)
  if (KIND == STEP_FT && !isx && QG_PSD_PREFETCH) psd_prefetch_v(M.dpi, u, sm);  // V behind the SpMV pass
  pdl_wait();  // the previous kernel's vectors / LSMR state are complete past this point
  const long long a_t0 = (a.prof != nullptr && threadIdx.x == 0) ? clock64() : 0;
  const double wN = a.in[M.NX + M.NY + p];             // issued with the LSMR-state loads below
  double s_in, c_out;
  if (!lsmr_runs(a, p, s_in, c_out)) {  // CTA-uniform
    if (KIND == STEP_FT && QG_PSD_PREFETCH) asm volatile("cp.async.wait_all;" ::: "memory");  // (prefetch)
    return;
  }
  const double *inX = a.in, *inY = a.in + M.NX;
  double acc[kSlots] = {0.0, 0.0, 0.0, 0.0};

  // deferred vector update of the previous iteration over the unit's own rows
  // (in = v_k on the u-step): lsmr.py:142-144, ||x||^2 partial in slot 3
  const Lsmr *L = a.st ? a.st + p : nullptr;
  if (a.upd_h && L && L->itn > 0 && !(kDist && isx && a.xmode == X_PARTIAL)) {
    const double c1 = L->c_hbar, c2 = L->c_x, c3 = L->c_h, sv = L->s_v;
    const int64_t off = isx ? 0 : M.NX;
    for (int64_t r = off + u.row0 + threadIdx.x; r < off + u.row1; r += blockDim.x) {
      const double hb = a.upd_h[r] - c1 * a.upd_hb[r];
      const double x = a.upd_x[r] + c2 * hb;
      a.upd_h[r] = a.in[r] * sv - c3 * a.upd_h[r];
      a.upd_hb[r] = hb;
      a.upd_x[r] = x;
      acc[3] += x * x;
    }
  }

  if (isx) {
    const double *x2 = KIND == STEP_F ? a.dpin : inY;
    if (kDist && a.xmode == X_PARTIAL) {
      // this rank's A_r' (D Pi w)_2 (F) or A_r' w2 (F') for the X rows
      for_rows<kWide, kUnr, kRows32, kRowsG>(u,M.sAT, nullptr, M.x_rowof, M.AT_rp, M.AT_col, M.AT_val, nullptr, nullptr, nullptr, x2, nullptr,
               u.lanes, M.yoff[p], 0, [&](int r, double s, double) { a.xred[r] = s; });
      return;  // CTA-uniform; the X slots are written by the X_FINISH launch
    }
    auto xrow = [&](int r, double s1, double s2) {
               const double w = inX[r];
               double res;
               if (KIND == STEP_F) {
                 // out1 = P w1 + A' (D Pi w)_2 + w_N q ; (out - v + w)/z_N with v1 = w1
                 const double o1 = (s1 + s2) + wN * M.q[r];
                 res = ((o1 - w) + w) / E.zN;
                 acc[0] += M.Pxbar[r] * w;
                 if (kRk1) res -= a.rk1[r] * wN;
               } else {
                 // g1 = P w1 - A' w2 - (2/tau) w_N P xbar - w_N q ; (D Pi (g - w) + w)/z_N
                 const double g = ((s1 - s2) - ((2.0 / E.tau) * wN) * M.Pxbar[r]) - wN * M.q[r];
                 res = ((g - w) + w) / E.zN;
                 if (kRk1) acc[3] += a.rk1[r] * w;
               }
               acc[1] += M.q[r] * w;
               const double o = s_in * res - (c_out != 0.0 ? c_out * a.old[r] : 0.0);
               a.out[r] = o;
               acc[2] += o * o;
             };
    if (kDist && a.xmode == X_FINISH)
      for_rows<kWide, kUnr, kRows32, kRowsG>(u,M.sP, nullptr, M.x_rowof, M.P_rp, M.P_col, M.P_val, nullptr, nullptr, nullptr, inX, nullptr, u.lanes,
               M.xoff[p], 0, [&](int r, double s1, double) { xrow(r, s1, a.xred[r]); });
    else
      for_rows<kWide, kUnr, kRows32, kRowsG>(u,M.sP, &M.sAT, M.x_rowof, M.P_rp, M.P_col, M.P_val, M.AT_rp, M.AT_col, M.AT_val, inX, x2, u.lanes,
               M.xoff[p], M.yoff[p], xrow);
    if (kDist && !M.x_owner)
#pragma unroll
      for (int k = 0; k < kSlots; ++k) acc[k] = 0.0;  // replicated rows: rank 0 counts them
  } else {
    double *outY = a.out + M.NX;
    const double *oldY = a.old ? a.old + M.NX : nullptr;
    if (KIND == STEP_F) {
      for_rows<kWide, kUnr, kRows32, kRowsG>(u,M.sA, nullptr, M.y_rowof, M.A_rp, M.A_col, M.A_val, nullptr, nullptr, nullptr, inX, nullptr, u.lanes,
               M.xoff[p], 0,
               [&](int r, double s, double) {
                 // out2 = -A w1 + w_N b ; (out - D Pi w + w)/z_N
                 const double o2 = (-s) + wN * M.b[r];
                 double res = ((o2 - a.dpin[r]) + inY[r]) / E.zN;
                 if (kRk1) res -= a.rk1[M.NX + r] * wN;
                 const double o = s_in * res - (c_out != 0.0 ? c_out * oldY[r] : 0.0);
                 outY[r] = o;
                 acc[0] += M.b[r] * a.dpin[r];
                 acc[2] += o * o;
               });
    } else {
      // pass 1: t = (A w1 - w_N b) - w2  for every row of the unit
      double *tY = a.tY;
      for_rows<kWide, kUnr, kRows32, kRowsG>(u,M.sA, nullptr, M.y_rowof, M.A_rp, M.A_col, M.A_val, nullptr, nullptr, nullptr, inX, nullptr, u.lanes,
               M.xoff[p], 0,
               [&](int r, double s, double) {
                 tY[r] = (s - wN * M.b[r]) - inY[r];
                 if (kRk1) acc[3] += a.rk1[M.NX + r] * inY[r];
               });
      __syncthreads();
      // per row: o = s_in (D Pi t + w2)/z_N - c_out old ; D Pi o for the next F step
      auto fin_row = [&](int r, double dpt) {
        const double w = inY[r];
        const double o = s_in * ((dpt + w) / E.zN) - (c_out != 0.0 ? c_out * oldY[r] : 0.0);
        outY[r] = o;
        acc[0] += M.b[r] * w;
        acc[2] += o * o;
        return o;
      };
      if (u.cls == CLS_ELEM) {
        // fused register epilogue: weight read once, both D Pi applications
        const int kind = M.dpi.blk[u.blk0].kind;
        for (int r = u.row0 + threadIdx.x; r < u.row1; r += blockDim.x) {
          const double wgt = elem_weight(kind, M.dpi.dual, M.dpi.zmid[r]);
          const double o = fin_row(r, wgt * tY[r]);
          if (a.dpout) a.dpout[r] = wgt * o;
        }
      } else if (u.cls == CLS_TRI) {
        for (int k = u.blk0 + (int)threadIdx.x; k < u.blk1; k += blockDim.x) {
          const BlockInfo b = M.dpi.blk[k];
          double D[9];
#pragma unroll
          for (int i = 0; i < 9; ++i) D[i] = M.dpi.tri_D[9 * b.param + i];
          const int flip = M.dpi.tri_flip[b.param];
          const double t3[3] = {tY[b.row], tY[b.row + 1], tY[b.row + 2]};
          double r3[3], o3[3], d3[3];
          tri_apply(D, flip, t3, r3);
#pragma unroll
          for (int i = 0; i < 3; ++i) o3[i] = fin_row(b.row + i, r3[i]);
          if (a.dpout) {
            tri_apply(D, flip, o3, d3);
#pragma unroll
            for (int i = 0; i < 3; ++i) a.dpout[b.row + i] = d3[i];
          }
        }
      } else if (u.cls == CLS_SOC && u.group > 0) {
        soc_epilogue(M.dpi, u, tY, fin_row, outY, a.dpout);
      } else {
        // generic path (PSD blocks, very large SOC blocks): CTA-wide phases
        // (a.prof: QG_PSD_PROF diagnostics -- SM cycles of a PSD unit's
        // phases: [units, SpMV pass, D Pi t, rows, D Pi o])
        const bool tp = a.prof != nullptr && threadIdx.x == 0 && u.cls == CLS_PSD;
        long long t1 = tp ? clock64() : 0;
        dpi_apply_unit(M.dpi, u, a.tY + u.row0, a.tY2 + u.row0, sm, QG_PSD_PREFETCH && u.cls == CLS_PSD);
        long long t2 = tp ? clock64() : 0;
        for (int r = u.row0 + threadIdx.x; r < u.row1; r += blockDim.x) fin_row(r, a.tY2[r]);
        __syncthreads();
        long long t3 = tp ? clock64() : 0;
        if (a.dpout) dpi_apply_unit(M.dpi, u, outY + u.row0, a.dpout + u.row0, sm, true);  // V still in sm
        if (tp) {
          const long long t4 = clock64();
          atomicAdd(a.prof + 0, 1ULL);
          atomicAdd(a.prof + 1, (unsigned long long)(t1 - a_t0));
          atomicAdd(a.prof + 2, (unsigned long long)(t2 - t1));
          atomicAdd(a.prof + 3, (unsigned long long)(t3 - t2));
          atomicAdd(a.prof + 4, (unsigned long long)(t4 - t3));
        }
      }
    }
  }
  pdl_trigger();  // the next kernel may start launching (it waits for our completion)
  double tot[kSlots];
  cta_sum_slots(acc, red, tot);
  if (threadIdx.x == 0 && a.part)
#pragma unroll
    for (int k = 0; k < kSlots; ++k) a.part[(size_t)ui * kSlots + k] = tot[k];
}

// One work unit of a kFeatDF step (single problem, no PSD / row partition /
// rank-one term): the SpMV row sums are staged in shared memory (2 doubles
// per unit row) while CTA 0 finalizes the previous step; the row epilogues
// then run from the staged sums with the published coefficients.  Same
// per-row expressions as step_unit; the unit partials are summed over a
// fixed row -> thread mapping.
template <int KIND, int FEAT>
__device__ __forceinline__ void step_unit_df(const Mats &M, const StepArgs &a, int ui) {
  constexpr bool kWide = (FEAT & kFeatWide) != 0;
  constexpr int kUnr = KIND == STEP_F ? QG_F_UNROLL : QG_FT_UNROLL;
  constexpr int kRows32 = KIND == STEP_F ? QG_ROWS32 : QG_ROWS32_FT;
  constexpr int kRowsG = KIND == STEP_F ? QG_ROWSG : QG_ROWSG_FT;
  extern __shared__ double sm[];
  __shared__ double red[kWarps * kSlots];
  __shared__ DfPub sP;
  const bool isx = ui < M.nxu;
  const Unit u = isx ? M.xu[ui] : M.yu[ui - M.nxu];
  const int p = u.prob;
  const Embed E = M.emb[p];
  pdl_wait();  // the previous step's vectors are complete past this point
  const double *inX = a.in, *inY = a.in + M.NX;
  double *stg = sm;  // staged row sums: [2 * (r - row0)] = s1, [+1] = s2
  auto stage = [&](int r, double s1, double s2) {
    stg[2 * (r - u.row0)] = s1;
    stg[2 * (r - u.row0) + 1] = s2;
  };
  if (isx)
    for_rows<kWide, kUnr, kRows32, kRowsG>(u, M.sP, &M.sAT, M.x_rowof, M.P_rp, M.P_col, M.P_val, M.AT_rp, M.AT_col,
                                            M.AT_val, inX, KIND == STEP_F ? a.dpin : inY, u.lanes, M.xoff[p],
                                            M.yoff[p], stage);
  else
    for_rows<kWide, kUnr, kRows32, kRowsG>(u, M.sA, nullptr, M.y_rowof, M.A_rp, M.A_col, M.A_val, nullptr, nullptr,
                                            nullptr, inX, nullptr, u.lanes, M.xoff[p], 0, stage);
  // the previous step's finalize (CTA 0 of this launch)
  if (threadIdx.x == 0) {
    const unsigned want = ld_acquire_u32(&a.df->flag[a.df_par ^ 1]) + 1;
    // (exponential back-off from 64 / 256 ns measured neutral to slightly
    // slower on c2 and c3: the poll does not crowd out CTA 0)
    while (ld_acquire_u32(&a.df->flag[a.df_par]) != want) __nanosleep(32);
    const DfPub *g = &a.df->pub[a.df_par];
    sP.s_in = __ldcg(&g->s_in); sP.c_out = __ldcg(&g->c_out); sP.wN = __ldcg(&g->wN);
    sP.c_hbar = __ldcg(&g->c_hbar); sP.c_x = __ldcg(&g->c_x); sP.c_h = __ldcg(&g->c_h); sP.s_v = __ldcg(&g->s_v);
    sP.runs = __ldcg(&g->runs); sP.upd = __ldcg(&g->upd);
  }
  __syncthreads();  // (also: every staged sum is in shared memory)
  if (!sP.runs) return;  // CTA-uniform
  const double wN = sP.wN, s_in = sP.s_in, c_out = sP.c_out;
  double acc[kSlots] = {0.0, 0.0, 0.0, 0.0};
  if (a.upd_h && sP.upd) {  // deferred vector update of the previous iteration (lsmr.py:142-144)
    const double c1 = sP.c_hbar, c2 = sP.c_x, c3 = sP.c_h, sv = sP.s_v;
    const int64_t off = isx ? 0 : M.NX;
    for (int64_t r = off + u.row0 + threadIdx.x; r < off + u.row1; r += blockDim.x) {
      const double hb = a.upd_h[r] - c1 * a.upd_hb[r];
      const double x = a.upd_x[r] + c2 * hb;
      a.upd_h[r] = a.in[r] * sv - c3 * a.upd_h[r];
      a.upd_hb[r] = hb;
      a.upd_x[r] = x;
      acc[3] += x * x;
    }
  }
  if (isx) {
    for (int r = u.row0 + threadIdx.x; r < u.row1; r += blockDim.x) {
      const double s1 = stg[2 * (r - u.row0)], s2 = stg[2 * (r - u.row0) + 1];
      const double w = inX[r];
      double res;
      if (KIND == STEP_F) {
        const double o1 = (s1 + s2) + wN * M.q[r];
        res = ((o1 - w) + w) / E.zN;
        acc[0] += M.Pxbar[r] * w;
      } else {
        const double g = ((s1 - s2) - ((2.0 / E.tau) * wN) * M.Pxbar[r]) - wN * M.q[r];
        res = ((g - w) + w) / E.zN;
      }
      acc[1] += M.q[r] * w;
      const double o = s_in * res - (c_out != 0.0 ? c_out * a.old[r] : 0.0);
      a.out[r] = o;
      acc[2] += o * o;
    }
  } else {
    double *outY = a.out + M.NX;
    const double *oldY = a.old ? a.old + M.NX : nullptr;
    if (KIND == STEP_F) {
      for (int r = u.row0 + threadIdx.x; r < u.row1; r += blockDim.x) {
        const double o2 = (-stg[2 * (r - u.row0)]) + wN * M.b[r];
        const double res = ((o2 - a.dpin[r]) + inY[r]) / E.zN;
        const double o = s_in * res - (c_out != 0.0 ? c_out * oldY[r] : 0.0);
        outY[r] = o;
        acc[0] += M.b[r] * a.dpin[r];
        acc[2] += o * o;
      }
    } else {
      double *tY = a.tY;
      for (int r = u.row0 + threadIdx.x; r < u.row1; r += blockDim.x)
        tY[r] = (stg[2 * (r - u.row0)] - wN * M.b[r]) - inY[r];
      __syncthreads();
      auto fin_row = [&](int r, double dpt) {
        const double w = inY[r];
        const double o = s_in * ((dpt + w) / E.zN) - (c_out != 0.0 ? c_out * oldY[r] : 0.0);
        outY[r] = o;
        acc[0] += M.b[r] * w;
        acc[2] += o * o;
        return o;
      };
      if (u.cls == CLS_ELEM) {
        const int kind = M.dpi.blk[u.blk0].kind;
        for (int r = u.row0 + threadIdx.x; r < u.row1; r += blockDim.x) {
          const double wgt = elem_weight(kind, M.dpi.dual, M.dpi.zmid[r]);
          const double o = fin_row(r, wgt * tY[r]);
          if (a.dpout) a.dpout[r] = wgt * o;
        }
      } else if (u.cls == CLS_TRI) {
        for (int k = u.blk0 + (int)threadIdx.x; k < u.blk1; k += blockDim.x) {
          const BlockInfo b = M.dpi.blk[k];
          double D[9];
#pragma unroll
          for (int i = 0; i < 9; ++i) D[i] = M.dpi.tri_D[9 * b.param + i];
          const int flip = M.dpi.tri_flip[b.param];
          const double t3[3] = {tY[b.row], tY[b.row + 1], tY[b.row + 2]};
          double r3[3], o3[3], d3[3];
          tri_apply(D, flip, t3, r3);
#pragma unroll
          for (int i = 0; i < 3; ++i) o3[i] = fin_row(b.row + i, r3[i]);
          if (a.dpout) {
            tri_apply(D, flip, o3, d3);
#pragma unroll
            for (int i = 0; i < 3; ++i) a.dpout[b.row + i] = d3[i];
          }
        }
      } else if (u.cls == CLS_SOC && u.group > 0) {
        soc_epilogue(M.dpi, u, tY, fin_row, outY, a.dpout);
      } else {  // large SOC blocks: CTA-wide phases (no PSD in kFeatDF handles)
        dpi_apply_unit(M.dpi, u, a.tY + u.row0, a.tY2 + u.row0, nullptr);
        for (int r = u.row0 + threadIdx.x; r < u.row1; r += blockDim.x) fin_row(r, a.tY2[r]);
        __syncthreads();
        if (a.dpout) dpi_apply_unit(M.dpi, u, outY + u.row0, a.dpout + u.row0, nullptr);
      }
    }
  }
  pdl_trigger();
  double tot[kSlots];
  cta_sum_slots(acc, red, tot);
  if (threadIdx.x == 0 && a.part)
#pragma unroll
    for (int k = 0; k < kSlots; ++k) a.part[(size_t)ui * kSlots + k] = tot[k];
}

// F' launches of batches with PSD blocks take their units in M.ft_order:
// the PSD units (two D Pi applications of 4 dense products each: the
// longest CTAs) first, so they start in the first wave instead of forming
// the launch's tail.
template <int KIND, int MINB, int FEAT>
__global__ void __launch_bounds__(kStepThreads, MINB) k_step(Mats M, StepArgs a) {
  // (an X_FINISH launch covers only the X units: natural order)
  if constexpr ((FEAT & kFeatDF) != 0) {  // CTA 0: the previous step's finalize; units from CTA 1
    if (blockIdx.x == 0) df_fin(M, a);
    else step_unit_df<KIND, FEAT>(M, a, (int)blockIdx.x - 1);
    return;
  }
  const int ui = (KIND == STEP_FT && M.ft_order && a.xmode != X_FINISH) ? M.ft_order[blockIdx.x] : (int)blockIdx.x;
  step_unit<KIND, FEAT, KIND == STEP_F && MINB == 8>(M, a, ui);
}

// F' step of the PSD units (one PSD block each), launched on a forked stream
// beside the k_step<F'> launch of every other unit (launch_step_one): the two
// D Pi applications of 4 dense products each make these the longest CTAs of
// the step, so they get 256 threads (half the per-warp product chain of the
// 128-thread step CTA, twice the SpMV lanes) and keep the whole epilogue in
// shared memory -- t, w and old are staged there by the SpMV pass, D Pi t and
// the row outputs never leave the CTA (the generic k_step path round-trips
// them through the global tY / tY2 scratch).  The other units' launch then
// needs no dynamic shared memory (more CTAs per SM, L1 left to the gathers).
// Same expressions as step_unit's F' Y side; the unit's partials are summed
// over a fixed row -> thread mapping (deterministic).
constexpr int kPsdThreads = 256;
template <int FEAT>
__global__ void __launch_bounds__(kPsdThreads, 4) k_step_psd(Mats M, StepArgs a) {  // 4 CTAs/SM: 64 registers
  constexpr bool kWide = (FEAT & kFeatWide) != 0;
  const bool kRk1 = (FEAT & kFeatRk1) != 0 && a.rk1 != nullptr;
  extern __shared__ double sm[];
  __shared__ double red[kWarps * kSlots];
  const int ui = M.ft_order[blockIdx.x];  // PSD units lead the F' order
  const Unit u = M.yu[ui - M.nxu];         // preparation-time data: before the PDL wait
  const int p = u.prob;
  const Embed E = M.emb[p];
  const BlockInfo blk = M.dpi.blk[u.blk0];
  const int d = blk.order, dim = u.row1 - u.row0;
  const double *Vg = M.dpi.psd + blk.param, *Bg = Vg + d * d;
  QG_CHECK(u.cls == CLS_PSD && u.blk1 == u.blk0 + 1 && blk.row == u.row0 && dim == d * (d + 1) / 2);
  psd_prefetch_v(M.dpi, u, sm);
  pdl_wait();
  const bool tp = a.prof != nullptr && threadIdx.x == 0;
  const long long t0 = tp ? clock64() : 0;
  const double wN = a.in[M.NX + M.NY + p];
  double s_in, c_out;
  if (!lsmr_runs(a, p, s_in, c_out)) {
    asm volatile("cp.async.wait_all;" ::: "memory");
    return;
  }
  double *ts = sm + psd_core_words(d), *ws = ts + dim, *os = ws + dim;  // svec-indexed staging
  const double *inX = a.in, *inY = a.in + M.NX;
  const double *oldY = a.old ? a.old + M.NX : nullptr;
  double *outY = a.out + M.NX;
  double acc[kSlots] = {0.0, 0.0, 0.0, 0.0};
  const Lsmr *L = a.st ? a.st + p : nullptr;
  if (a.upd_h && L && L->itn > 0) {  // deferred vector update (as step_unit)
    const double c1 = L->c_hbar, c2 = L->c_x, c3 = L->c_h, sv = L->s_v;
    for (int64_t r = M.NX + u.row0 + threadIdx.x; r < M.NX + u.row1; r += blockDim.x) {
      const double hb = a.upd_h[r] - c1 * a.upd_hb[r];
      const double x = a.upd_x[r] + c2 * hb;
      a.upd_h[r] = a.in[r] * sv - c3 * a.upd_h[r];
      a.upd_hb[r] = hb;
      a.upd_x[r] = x;
      acc[3] += x * x;
    }
  }
  // pass 1: t = (A w1 - w_N b) - w2, w2 and old staged by row
  for_rows<kWide, QG_FT_UNROLL, QG_ROWS32_FT, QG_ROWSG_FT>(
      u, M.sA, nullptr, M.y_rowof, M.A_rp, M.A_col, M.A_val, nullptr, nullptr, nullptr, inX, nullptr, u.lanes,
      M.xoff[p], 0, [&](int r, double s, double) {
        const int o = r - u.row0;
        const double w = inY[r];
        ts[o] = (s - wN * M.b[r]) - w;
        ws[o] = w;
        os[o] = c_out != 0.0 ? oldY[r] : 0.0;
      });
  __syncthreads();
  const long long t1 = tp ? clock64() : 0;
  // D Pi t (in place: the input is read into S before the result is written)
  psd_apply_core<2>(Vg, Bg, d, [&](int k) { return ts[k]; }, [&](int k, double v) { ts[k] = v; }, sm, true);
  const long long t2 = tp ? clock64() : 0;
  // rows: o = s_in (D Pi t + w2)/z_N - c_out old
  for (int o = threadIdx.x; o < dim; o += blockDim.x) {
    const int r = u.row0 + o;
    const double w = ws[o];
    const double v = s_in * ((ts[o] + w) / E.zN) - (c_out != 0.0 ? c_out * os[o] : 0.0);
    outY[r] = v;
    os[o] = v;
    acc[0] += M.b[r] * w;
    acc[2] += v * v;
    if (kRk1) acc[3] += a.rk1[M.NX + r] * w;
  }
  __syncthreads();
  const long long t3 = tp ? clock64() : 0;
  // D Pi o for the next F step (V still in shared memory)
  if (a.dpout) {
    double *dp = a.dpout + u.row0;
    psd_apply_core<2>(Vg, Bg, d, [&](int k) { return os[k]; }, [&](int k, double v) { dp[k] = v; }, sm, true);
  }
  if (tp) {
    const long long t4 = clock64();
    atomicAdd(a.prof + 0, 1ULL);
    atomicAdd(a.prof + 1, (unsigned long long)(t1 - t0));
    atomicAdd(a.prof + 2, (unsigned long long)(t2 - t1));
    atomicAdd(a.prof + 3, (unsigned long long)(t3 - t2));
    atomicAdd(a.prof + 4, (unsigned long long)(t4 - t3));
  }
  pdl_trigger();
  double tot[kSlots];
  cta_sum_slots(acc, red, tot);
  if (threadIdx.x == 0 && a.part)
#pragma unroll
    for (int k = 0; k < kSlots; ++k) a.part[(size_t)ui * kSlots + k] = tot[k];
}

// -------------------------------------------------------------- update --
// hbar = h - c1 hbar ; x = x + c2 hbar ; h = v s_v - c3 h   (lsmr.py:142-144)
__global__ void __launch_bounds__(kThreads) k_update(Mats M, UpdArgs a) {
  __shared__ double red[kWarps * kSlots];
  const bool isx = (int)blockIdx.x < M.nxu;
  const Unit u = isx ? M.xu[blockIdx.x] : M.yu[blockIdx.x - M.nxu];
  const Lsmr &L = a.st[u.prob];
  if (!L.active) return;
  const double c1 = L.c_hbar, c2 = L.c_x, c3 = L.c_h, sv = L.s_v;
  const int64_t off = isx ? 0 : M.NX;
  double acc[kSlots] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t r = off + u.row0 + threadIdx.x; r < off + u.row1; r += blockDim.x) {
    const double hb = a.h[r] - c1 * a.hb[r];
    const double x = a.x[r] + c2 * hb;
    a.h[r] = a.v[r] * sv - c3 * a.h[r];
    a.hb[r] = hb;
    a.x[r] = x;
    acc[0] += x * x;
  }
  if (isx && !M.x_owner) acc[0] = 0.0;
  double tot[kSlots];
  cta_sum_slots(acc, red, tot);
  if (threadIdx.x == 0)
#pragma unroll
    for (int k = 0; k < kSlots; ++k) a.part[(size_t)blockIdx.x * kSlots + k] = tot[k];
}

// Per-problem sums of the unit partials in exactly k_fin's order (row-
// partitioned mode): psum = [X sums: B x kSlots | Y sums: B x kSlots].
__global__ void k_part_reduce(const double *px, const int64_t *px_ptr, const double *py, const int64_t *py_ptr,
                              int B, double *psum) {
  const int p = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (p >= B) return;
  double sx[kSlots] = {0, 0, 0, 0}, sy[kSlots] = {0, 0, 0, 0};
  for (int64_t k = px_ptr[p] + lane; k < px_ptr[p + 1]; k += 32)
#pragma unroll
    for (int j = 0; j < kSlots; ++j) sx[j] += px[k * kSlots + j];
  for (int64_t k = py_ptr[p] + lane; k < py_ptr[p + 1]; k += 32)
#pragma unroll
    for (int j = 0; j < kSlots; ++j) sy[j] += py[k * kSlots + j];
#pragma unroll
  for (int j = 0; j < kSlots; ++j) { sx[j] = warp_sum(sx[j]); sy[j] = warp_sum(sy[j]); }
  if (lane == 0)
#pragma unroll
    for (int j = 0; j < kSlots; ++j) {
      psum[(size_t)p * kSlots + j] = sx[j];
      psum[((size_t)B + p) * kSlots + j] = sy[j];
    }
}

// Finalize of problem p by one warp (all 32 lanes call it).
__device__ __forceinline__ bool fin_skips(const FinArgs &a, int p) {
  // inactive problems have nothing to finalize (a skipped v-step still runs
  // its recurrences: skip_v problems stay active)
  return a.st && a.phase != PH_APPLY && a.phase != PH_RHS && !a.st[p].active;
}

// pre: the 2 x kSlots per-problem sums already reduced (CTA-per-problem
// finalize); else the warp reduces them (all 32 lanes call).  Lsh: a
// shared-memory copy of the problem's LSMR state to work on (the caller
// loads and stores it cooperatively), else the state in global memory.
// The scalar work is fin_core (lsmr_dev.cuh) on the T entries of the
// vectors, loaded here and stored back where fin_core wrote them.
// T entries of problem p a finalize of phase a.phase reads (lsmr_dev.cuh TVals).
__device__ __forceinline__ TVals load_tvals(const Mats &M, const FinArgs &a, int p) {
  const int64_t T = M.NX + M.NY + p;
  TVals t;
  t.in = a.in ? __ldcg(a.in + T) : 0.0;
  t.old = a.old ? __ldcg(a.old + T) : 0.0;
  t.out = t.old;
  t.h = (a.phase == PH_STEP_V) ? __ldcg(a.h + T) : 0.0;
  t.hb = (a.phase == PH_STEP_V) ? __ldcg(a.hb + T) : 0.0;
  t.x = (a.phase == PH_STEP_V || a.phase == PH_STEP_U || a.phase == PH_STEP_X) ? __ldcg(a.x + T) : 0.0;
  t.rk1 = a.rk1 ? __ldcg(a.rk1 + T) : 0.0;
  return t;
}

__device__ __forceinline__ void fin_problem(const Mats &M, const FinArgs &a, int p, int lane,
                                            const double *pre = nullptr, Lsmr *Lsh = nullptr,
                                            const TVals *tpre = nullptr) {
  Lsmr *L = Lsh ? Lsh : (a.st ? a.st + p : nullptr);
  if (fin_skips(a, p)) return;
  // deterministic per-problem sums of the producers' partials (fixed order)
  double sx[kSlots] = {0, 0, 0, 0}, sy[kSlots] = {0, 0, 0, 0};
  if (pre) {
#pragma unroll
    for (int j = 0; j < kSlots; ++j) { sx[j] = pre[j]; sy[j] = pre[kSlots + j]; }
  } else {
#pragma unroll 4
    for (int64_t k = a.px_ptr[p] + lane; k < a.px_ptr[p + 1]; k += 32)
#pragma unroll
      for (int j = 0; j < kSlots; ++j) sx[j] += __ldcg(a.px + k * kSlots + j);
#pragma unroll 4
    for (int64_t k = a.py_ptr[p] + lane; k < a.py_ptr[p + 1]; k += 32)
#pragma unroll
      for (int j = 0; j < kSlots; ++j) sy[j] += __ldcg(a.py + k * kSlots + j);
#pragma unroll
    for (int j = 0; j < kSlots; ++j) { sx[j] = warp_sum(sx[j]); sy[j] = warp_sum(sy[j]); }
  }
  if (lane != 0) return;
  const int64_t T = M.NX + M.NY + p;
  TVals t = tpre ? *tpre : load_tvals(M, a, p);
  const int w = fin_core(M.emb[p], a.phase, a.kind, L, sx, sy, t, a.rk1 != nullptr, true);
  if (w & TV_OUT) a.out[T] = t.out;
  if (w & TV_H) a.h[T] = t.h;
  if (w & TV_HB) a.hb[T] = t.hb;
  if (w & TV_X) a.x[T] = t.x;
}

__global__ void k_fin(Mats M, FinArgs a) {
  pdl_wait();
  pdl_trigger();
  const int p = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (p < a.B) fin_problem(M, a, p, threadIdx.x & 31);
}

// CTA per problem, for batches whose problems have many work units (small
// single problems cut into hundreds of units): 256 threads stride over the
// slots, fixed-order CTA reduction, thread 0 runs the scalar part.  The
// warp-per-problem version spent ~25 sequential L2 round trips per lane
// summing c2's ~800 slots.
// The per-problem finalize by one CTA (<= 256 threads), after its PDL wait:
// fixed-order sums of the unit partials, thread 0 runs the scalar part on a
// shared-memory copy of the LSMR state.  early: the state and T entries were
// loaded before the wait (into sLw / *tv).
__device__ __forceinline__ void fin_cta_run(const Mats &M, const FinArgs &a, int p, unsigned long long *sLw,
                                            bool early, TVals *tv) {
  constexpr int kLw = (int)(sizeof(Lsmr) / sizeof(unsigned long long));
  Lsmr *Lsh = a.st ? reinterpret_cast<Lsmr *>(sLw) : nullptr;
  const unsigned long long *Lg = reinterpret_cast<const unsigned long long *>(a.st + p);
  if (!early && Lsh)
    for (int w = threadIdx.x; w < kLw; w += blockDim.x) sLw[w] = Lg[w];
  if (fin_skips(a, p)) return;  // CTA-uniform
  __shared__ double red[(1024 / 32) * 2 * kSlots];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (int)(blockDim.x >> 5);
  double s[2 * kSlots] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll 4
  for (int64_t k = a.px_ptr[p] + threadIdx.x; k < a.px_ptr[p + 1]; k += blockDim.x)
#pragma unroll
    for (int j = 0; j < kSlots; ++j) s[j] += __ldcg(a.px + k * kSlots + j);
#pragma unroll 4
  for (int64_t k = a.py_ptr[p] + threadIdx.x; k < a.py_ptr[p + 1]; k += blockDim.x)
#pragma unroll
    for (int j = 0; j < kSlots; ++j) s[kSlots + j] += __ldcg(a.py + k * kSlots + j);
#pragma unroll
  for (int j = 0; j < 2 * kSlots; ++j) s[j] = warp_sum(s[j]);
  if (lane == 0)
#pragma unroll
    for (int j = 0; j < 2 * kSlots; ++j) red[warp * 2 * kSlots + j] = s[j];
  __syncthreads();
  if (threadIdx.x == 0) {
    double pre[2 * kSlots];
#pragma unroll
    for (int j = 0; j < 2 * kSlots; ++j) {
      double t = red[j];
      for (int w = 1; w < nw; ++w) t += red[w * 2 * kSlots + j];
      pre[j] = t;
    }
    fin_problem(M, a, p, 0, pre, Lsh, early ? tv : nullptr);
  }
  if (Lsh) {
    __syncthreads();
    unsigned long long *Lw = reinterpret_cast<unsigned long long *>(a.st + p);
    for (int w = threadIdx.x; w < kLw; w += blockDim.x) Lw[w] = sLw[w];
  }
}

template <int NT>
__global__ void __launch_bounds__(NT) k_fin_cta(Mats M, FinArgs a) {
  const int p = (int)blockIdx.x;
  // the LSMR state goes to shared memory in one coalesced sweep (the scalar
  // recurrence then never waits on global memory for it), and back at the end
  constexpr int kLw = (int)(sizeof(Lsmr) / sizeof(unsigned long long));
  static_assert(sizeof(Lsmr) % sizeof(unsigned long long) == 0, "Lsmr is copied as 8-byte words");
  __shared__ unsigned long long sLw[kLw];
  const unsigned long long *Lg = reinterpret_cast<const unsigned long long *>(a.st + p);
  TVals tv{};
  if (a.early) {
    // loop finalizes (FinArgs::early): state and T entries issued ahead of
    // the wait for the step kernel; L2 loads (cg): written by an earlier grid
    if (a.st)
      for (int w = threadIdx.x; w < kLw; w += blockDim.x) sLw[w] = __ldcg(Lg + w);
    if (threadIdx.x == 0) tv = load_tvals(M, a, p);
  }
  pdl_wait();
  pdl_trigger();
  fin_cta_run(M, a, p, sLw, a.early != 0, &tv);
}

// CTA 0 of a kFeatDF step launch (single problem): the finalize the previous
// step owes (a.fin, its partials in the other part buffer), then the
// coefficients of THIS step's row epilogues -> pub[par], released through
// flag[par] = flag[par ^ 1] + 1 (the unit CTAs of this launch wait on it).
// CTA 0 is the only reader / writer of the LSMR state and the T entries
// during the launch.
__device__ void df_fin(const Mats &M, const StepArgs &a) {
  constexpr int kLw = (int)(sizeof(Lsmr) / sizeof(unsigned long long));
  __shared__ unsigned long long sLw[kLw];
  __shared__ double red[kWarps * 2 * kSlots];
  DfCtl *D = a.df;
  const FinArgs &f = a.fin;
  const int par = a.df_par, p = 0;
  pdl_wait();
  pdl_trigger();
  // every load of the finalize at once (state, owed phase, T entries, unit
  // partials): one L2 round trip before the scalar recurrence
  const int pend = __ldcg(&D->pend_phase);
  const unsigned long long *Lg = reinterpret_cast<const unsigned long long *>(f.st + p);
  for (int w = threadIdx.x; w < kLw; w += blockDim.x) sLw[w] = __ldcg(Lg + w);
  TVals tv{};
  double wN0 = 0.0;
  if (threadIdx.x == 0) {
    tv = load_tvals(M, f, p);
    wN0 = __ldcg(a.in + M.NX + M.NY + p);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (int)(blockDim.x >> 5);
  double s[2 * kSlots] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (pend) {
#pragma unroll 8
    for (int64_t k = f.px_ptr[p] + threadIdx.x; k < f.px_ptr[p + 1]; k += blockDim.x)
#pragma unroll
      for (int j = 0; j < kSlots; ++j) s[j] += __ldcg(f.px + k * kSlots + j);
#pragma unroll 8
    for (int64_t k = f.py_ptr[p] + threadIdx.x; k < f.py_ptr[p + 1]; k += blockDim.x)
#pragma unroll
      for (int j = 0; j < kSlots; ++j) s[kSlots + j] += __ldcg(f.py + k * kSlots + j);
  }
#pragma unroll
  for (int j = 0; j < 2 * kSlots; ++j) s[j] = warp_sum(s[j]);
  if (lane == 0)
#pragma unroll
    for (int j = 0; j < 2 * kSlots; ++j) red[warp * 2 * kSlots + j] = s[j];
  __syncthreads();
  Lsmr *L = reinterpret_cast<Lsmr *>(sLw);
  if (threadIdx.x == 0) {
    double wN = wN0;
    // the owed finalize (fin_problem's work on the shared copy; an inactive
    // problem has nothing to finalize, as fin_skips)
    if (pend && L->active) {
      double pre[2 * kSlots];
#pragma unroll
      for (int j = 0; j < 2 * kSlots; ++j) {
        double t = red[j];
        for (int w = 1; w < nw; ++w) t += red[w * 2 * kSlots + j];
        pre[j] = t;
      }
      const int64_t T = M.NX + M.NY + p;
      const int w = fin_core(M.emb[p], f.phase, f.kind, L, pre, pre + kSlots, tv, false, true);
      if (w & TV_OUT) { f.out[T] = tv.out; wN = tv.out; }  // (f.out is this step's input)
      if (w & TV_H) f.h[T] = tv.h;
      if (w & TV_HB) f.hb[T] = tv.hb;
      if (w & TV_X) f.x[T] = tv.x;
    }
    DfPub P;
    P.runs = (L->active && !(a.is_v_step && L->skip_v)) ? 1 : 0;
    P.s_in = L->s_in;
    P.c_out = L->c_out;
    P.wN = wN;
    P.upd = L->itn > 0 ? 1 : 0;
    P.c_hbar = L->c_hbar; P.c_x = L->c_x; P.c_h = L->c_h; P.s_v = L->s_v;
    D->pub[par] = P;
    D->pend_phase = a.df_next;  // the finalize owed to the next kFeatDF step
    __threadfence();
    st_release_u32(&D->flag[par], __ldcg(&D->flag[par ^ 1]) + 1);
  }
  __syncthreads();
  if (pend) {  // the finalized state back to global memory (read by the next step's CTA 0)
    unsigned long long *Lw = reinterpret_cast<unsigned long long *>(f.st + p);
    for (int w = threadIdx.x; w < kLw; w += blockDim.x) Lw[w] = sLw[w];
  }
}

// The finalize the last step of a kFeatDF loop owes (after the loop).
__global__ void __launch_bounds__(256) k_df_tail(Mats M, FinArgs a, DfCtl *D) {
  constexpr int kLw = (int)(sizeof(Lsmr) / sizeof(unsigned long long));
  __shared__ unsigned long long sLw[kLw];
  if (__ldcg(&D->pend_phase) != a.phase) return;  // (no iteration ran: nothing owed)
  fin_cta_run(M, a, 0, sLw, false, nullptr);
  __syncthreads();
  if (threadIdx.x == 0) D->pend_phase = 0;
}

// (Measured and dropped: the same loop as ONE 1024-thread CTA for a single
// tiny problem with whole-problem units -- c1 8.1 -> 9.5 ms per step.)

__global__ void k_count_active(const Lsmr *st, int B, int *out) {
  __shared__ int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  int c = 0;
  for (int p = threadIdx.x; p < B; p += blockDim.x) c += st[p].active ? 1 : 0;
  atomicAdd(&cnt, c);
  __syncthreads();
  if (threadIdx.x == 0) *out = cnt;
}

// Body tail of the device-terminated LSMR loop (a CUDA-graph conditional
// WHILE node): count the still-active problems, advance the iteration
// counter by one body (chunk iterations) and let the graph repeat the body
// only while some problem is active and the cap is not reached -- the
// control decision of lsmr.py's loop without a host round trip.
// loop[0] = iterations run, loop[1] = cap.
__global__ void k_loop_cond(const Lsmr *st, int B, long long *loop, long long chunk, cudaGraphConditionalHandle h) {
  __shared__ int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  int c = 0;
  for (int p = threadIdx.x; p < B; p += blockDim.x) c += st[p].active ? 1 : 0;
  if (c) atomicAdd(&cnt, c);
  __syncthreads();
  if (threadIdx.x == 0) {
    const long long done = loop[0] + chunk;
    loop[0] = done;
    cudaGraphSetConditional(h, (cnt > 0 && done < loop[1]) ? 1u : 0u);
  }
}

void launch_loop_cond(const Handle &H, cudaGraphConditionalHandle h, long long chunk, cudaStream_t st) {
  k_loop_cond<<<1, 256, 0, st>>>(H.ws.st, H.B, H.ws.d_loop, chunk, h);
  QG_LAUNCHED();
}

// Fresh LSMR state per problem, its iteration cap computed on the device
// (no host-to-device copy: a chunked host pipeline keeps the copy engine busy
// with the next chunk's upload): opt > 0 explicit cap, opt < 0 explicit 0,
// opt == 0 the reference default 20 (n + m + 1) (lsmr.py:69-70 on the
// embedding).  Thread 0 also arms the device-terminated loop: [0, cap].
__global__ void k_init_state(Lsmr *st, int B, double atol, double btol, long long opt, const int64_t *xoff,
                             const int64_t *yoff, long long *loop, long long cap) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p == 0 && loop) {
    loop[0] = 0;
    loop[1] = cap;
  }

  if (p >= B) return;
  Lsmr L{};
  L.atol = atol;
  L.btol = btol;
  const long long N = (xoff[p + 1] - xoff[p]) + (yoff[p + 1] - yoff[p]) + 1;
  L.max_iter = opt > 0 ? opt : (opt < 0 ? 0 : 20 * N);
  L.s_u = L.s_v = 1.0;
  st[p] = L;
}

// ---------------------------------------------------------------- host --
Mats make_mats(const Handle &H) {
  Mats M{};
  M.P_rp = H.P.rp; M.P_col = H.P.col; M.P_val = H.P.val;
  M.AT_rp = H.AT.rp; M.AT_col = H.AT.col; M.AT_val = H.AT.val;
  M.A_rp = H.A.rp; M.A_col = H.A.col; M.A_val = H.A.val;
  M.xu = H.d_xunits; M.yu = H.cones.d_units;
  M.nxu = H.nxu(); M.nyu = H.nyu();
  M.xu_ptr = H.d_xunit_ptr; M.yu_ptr = H.d_yunit_ptr;
  M.q = H.q; M.b = H.b; M.Pxbar = H.Pxbar; M.xbar = H.xbar; M.ybar = H.ybar; M.sbar = H.sbar;
  M.emb = H.emb;
  M.NX = H.NX; M.NY = H.NY;
  M.dpi = H.cones.view();
  M.sP = H.sP.view(); M.sAT = H.sAT.view(); M.sA = H.sA.view();
  M.x_rowof = H.x_rowof; M.y_rowof = H.y_rowof;
  M.xoff = H.d_xoff; M.yoff = H.d_yoff;
  M.x_owner = H.x_owner() ? 1 : 0;
  M.ft_order = H.d_ft_order;
  return M;
}

// cudaFuncAttributeMaxDynamicSharedMemorySize is process-wide per function:
// only ever raised (handles on concurrent host threads must not lower it
// under each other's launches).
void raise_dynamic_smem(const void *kern, size_t bytes) {
  static std::mutex mu;
  static std::map<const void *, size_t> raised;
  std::lock_guard<std::mutex> lock(mu);
  size_t &r = raised[kern];
  if (bytes > r) {
    QG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    r = bytes;
  }
}

static size_t step_smem(const Handle &H) { return H.cones.max_psd_order ? H.cones.psd_smem_apply() : 0; }

// Launch with programmatic stream serialization (see pdl_wait / pdl_trigger
// in qg_common.cuh); QG_PDL=0 falls back to ordinary serialization (A/B).
//
// INVARIANT (pre-wait reads): k_step reads preparation-time data -- the
// work units, M.emb and (cp.async) the PSD eigenvectors V -- BEFORE its
// griddepcontrol.wait, so those reads may overlap the previous kernel.  This
// is only correct because every writer of that data (k_embed_* in
// launch_embed_consts, k_cone_prep in ConeTable::prepare, the unit / SELL
// uploads) runs in qg_create_batch* or qg_set_point, and both end with a
// cudaStreamSynchronize before any PDL chain (a jvp / vjp / apply_F) starts.
// A new writer of emb / D Pi data must keep that host fence (or launch a
// non-PDL kernel between it and the first step launch).
template <class... KArgs, class... Args>
static void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args &&...args) {
  static const char *env = std::getenv("QG_PDL");
  static const bool pdl = !env || std::atoi(env) != 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  QG_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

static void launch_step_one(const Handle &H, const Mats &M, int kind, const StepArgs &a, cudaStream_t st);

// One operator step.  Row-partitioned handles split it around the exchange:
// X_PARTIAL (Y rows + this rank's A' partials) -> sum over ranks -> X_FINISH.
void launch_step(const Handle &H, const Mats &M, int kind, const StepArgs &a0, cudaStream_t st) {
  if (!H.comm) {
    launch_step_one(H, M, kind, a0, st);
    return;
  }
  StepArgs a = a0;
  a.xred = H.xred;
  a.xmode = X_PARTIAL;
  launch_step_one(H, M, kind, a, st);
  H.comm->allreduce(H.xred, H.NX, st);
  a.xmode = X_FINISH;
  launch_step_one(H, M, kind, a, st);
}

// Kernel variant of a step: the CTA-per-row path and the rarely used
// features run as their own instantiations (12 CTAs/SM): plain wide-row
// handles get a lean variant, partitioned / rank-one steps the all-features one.
static int step_feat(const Handle &H, const StepArgs &a) {
  return (H.comm || a.rk1) ? kFeatAll : (H.has_wide ? kFeatWide : 0);
}

// Per-host-thread side stream and fork / join events of the PSD F' launch
// (thread-local: calls from different host threads never share an event).
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  SideStream() {
    QG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    QG_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    QG_CUDA(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
  }
  ~SideStream() {  // at host-thread exit (errors ignored: the context may be gone at process exit)
    if (join) cudaEventDestroy(join);
    if (fork) cudaEventDestroy(fork);
    if (s) cudaStreamDestroy(s);
    cudaGetLastError();
  }
  SideStream(const SideStream &) = delete;
  SideStream &operator=(const SideStream &) = delete;
};

bool psd_split(const Handle &H) { return H.psd_split && H.n_psd_units > 0; }

// k_step_psd's shared memory: psd_apply_core's matrices + t, w, old (svec).
static size_t psd_step_smem(const Handle &H) {
  const int d = H.cones.max_psd_order;
  return ((size_t)psd_core_words(d) + 3 * (size_t)(d * (d + 1) / 2)) * sizeof(double);
}

// k_step over `grid` units (the unit order of M), on st with PDL.
static void launch_step_main(const Handle &H, const Mats &M, int kind, const StepArgs &a, unsigned grid,
                             size_t smem, cudaStream_t st) {
  // (grid is captured by reference in `go`: kFeatDF launches add CTA 0)
  static int threads = 0;
  if (!threads) {  // QG_STEP_THREADS: A/B switch for the CTA size (32..128)
    const char *e = std::getenv("QG_STEP_THREADS");
    threads = e ? std::max(32, std::min(kStepThreads, std::atoi(e))) : kStepThreads;
  }
  // Occupancy target: the SELL F step keeps many loads in flight per thread
  // (64 registers, 8 CTAs/SM measured best: c5a 0.460 vs 0.509 ms); the F'
  // step (two-pass Y side, epilogue) and the CSR group path gain from 12
  // CTAs/SM (c5a F' 0.625 -> 0.574 ms; c3: 11.2 -> 8.7 ms per jvp).
  // QG_STEP_MINB=8|12 overrides (10 CTAs/SM, 48 registers, measured slower for
  // both steps).
  static const char *env_minb = std::getenv("QG_STEP_MINB");
  const bool sell = H.nslice_x + H.nslice_y > 0;
  const int minb = env_minb ? (std::atoi(env_minb) >= 12 ? 12 : 8) : (sell && kind == STEP_F ? 8 : 12);
  auto go = [&](auto kern, size_t sm_bytes) {
    if (sm_bytes > 48 * 1024) raise_dynamic_smem(reinterpret_cast<const void *>(kern), sm_bytes);
    launch_pdl(kern, dim3(grid), dim3(threads), sm_bytes, st, M, a);
  };
  const int feat = step_feat(H, a);
  if (a.df) {  // deferred finalize: CTA 0 + the units, row sums staged in shared memory
    grid += 1;
    const size_t stg = (size_t)2 * H.max_unit_rows * sizeof(double);
    (void)feat;  // (deferred-finalize handles have no CTA-per-row units: api.cu)
    // 8 CTAs/SM (64 registers: fewer spills) when the launch still fits in
    // one wave, else 12: unit CTAs waiting for CTA 0 must not hold back a
    // second wave (c2 30.1 -> 29.1, c4 99.8 -> 98.6 us per iteration with 8;
    // c3's 1194 CTAs at 8 per SM: 47.9 -> 62.6, so it keeps 12)
    static int nsm = 0;
    if (!nsm) {
      int dev = 0;
      QG_CUDA(cudaGetDevice(&dev));
      QG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    }
    const bool one_wave8 = grid <= 8u * (unsigned)nsm;
    if (kind == STEP_F) {
      if (one_wave8) go(k_step<STEP_F, 8, kFeatDF>, stg);
      else go(k_step<STEP_F, 12, kFeatDF>, stg);
    } else {
      if (one_wave8) go(k_step<STEP_FT, 8, kFeatDF>, stg);
      else go(k_step<STEP_FT, 12, kFeatDF>, stg);
    }
    QG_LAUNCHED();
    return;
  }
  if (kind == STEP_F) {
    if (feat == kFeatAll) go(k_step<STEP_F, 12, kFeatAll>, 0);
    else if (feat == kFeatWide) go(k_step<STEP_F, 12, kFeatWide>, 0);
    else if (minb == 12) go(k_step<STEP_F, 12, 0>, 0);
    else go(k_step<STEP_F, 8, 0>, 0);
  } else {
    if (feat == kFeatAll) go(k_step<STEP_FT, 12, kFeatAll>, smem);
    else if (feat == kFeatWide) go(k_step<STEP_FT, 12, kFeatWide>, smem);
    else if (minb == 12) go(k_step<STEP_FT, 12, 0>, smem);
    else go(k_step<STEP_FT, 8, 0>, smem);
  }
  QG_LAUNCHED();
}

void launch_step_psd(const Handle &H, const Mats &M, const StepArgs &a, cudaStream_t st) {
  const size_t psm = psd_step_smem(H);
  const int feat = step_feat(H, a);
  auto kp = feat == kFeatAll ? k_step_psd<kFeatAll> : (feat == kFeatWide ? k_step_psd<kFeatWide> : k_step_psd<0>);
  if (psm > 48 * 1024) raise_dynamic_smem(reinterpret_cast<const void *>(kp), psm);
  kp<<<(unsigned)H.n_psd_units, kPsdThreads, psm, st>>>(M, a);
  QG_LAUNCHED();
}

static void launch_step_one(const Handle &H, const Mats &M0, int kind, const StepArgs &a, cudaStream_t st) {
  const unsigned grid = (unsigned)(a.xmode == X_FINISH ? H.nxu() : H.nxu() + H.nyu());
  if (grid == 0) return;
  if (!(kind == STEP_FT && a.xmode != X_FINISH && psd_split(H))) {
    launch_step_main(H, M0, kind, a, grid, step_smem(H), st);
    return;
  }
  // F' with PSD blocks: the PSD units run as k_step_psd on a forked stream,
  // the rest of the step as k_step (no PSD unit left: no dynamic smem).
  // QG_PSD_SPLIT=0 at handle creation: every unit in k_step (A/B).
  static thread_local SideStream side;
  QG_CUDA(cudaEventRecord(side.fork, st));
  QG_CUDA(cudaStreamWaitEvent(side.s, side.fork, 0));
  launch_step_psd(H, M0, a, side.s);
  QG_CUDA(cudaEventRecord(side.join, side.s));
  Mats M = M0;
  M.ft_order = M0.ft_order + H.n_psd_units;
  const unsigned rest = grid - (unsigned)H.n_psd_units;
  if (rest) launch_step_main(H, M, kind, a, rest, 0, st);
  QG_CUDA(cudaStreamWaitEvent(st, side.join, 0));
}

void fin_ptrs(const Handle &H, FinArgs &a) {
  // every producer writes one slot per work unit: X units, then Y units, in
  // the buffer a.part (the workspace's part, or part2 for the steps of a
  // deferred-finalize loop that write there)
  const double *base = a.part ? a.part : H.ws.part;
  a.px = base;
  a.px_ptr = H.d_xunit_ptr;
  a.py = base + (size_t)H.nxu() * kSlots;
  a.py_ptr = H.d_yunit_ptr;
}

void launch_fin(const Handle &H, const Mats &M, const FinArgs &a0, cudaStream_t st) {
  FinArgs a = a0;
  fin_ptrs(H, a);
  const unsigned grid = (unsigned)((H.B * 32 + 255) / 256);
  if (H.comm) {
    // row-partitioned: per-problem sums (k_fin's order), summed over ranks,
    // then k_fin reads one reduced unit per problem
    k_part_reduce<<<grid, 256, 0, st>>>(a.px, a.px_ptr, a.py, a.py_ptr, H.B, H.psum);
    QG_LAUNCHED();
    H.comm->allreduce(H.psum, 2 * (int64_t)H.B * kSlots, st);
    a.px = H.psum;
    a.py = H.psum + (size_t)H.B * kSlots;
    a.px_ptr = a.py_ptr = H.d_iota;
  }
  // many work units per problem (>= 64 on average): a CTA per problem.
  // QG_FIN_CTA=0|1 forces (A/B).
  static const char *env = std::getenv("QG_FIN_CTA");
  const bool cta = !H.comm && (env ? std::atoi(env) != 0 : (int64_t)(H.nxu() + H.nyu()) >= 64LL * H.B);
  // (problems of >= 2048 units -- c5b, ~12k -- sum their partials with 1024
  // threads: 4x fewer dependent load batches per thread)
  if (cta && (int64_t)(H.nxu() + H.nyu()) >= 2048LL * H.B)
    launch_pdl(k_fin_cta<1024>, dim3((unsigned)H.B), dim3(1024), 0, st, M, a);
  else if (cta) launch_pdl(k_fin_cta<256>, dim3((unsigned)H.B), dim3(256), 0, st, M, a);
  else launch_pdl(k_fin, dim3(grid), dim3(256), 0, st, M, a);
  QG_LAUNCHED();
}

void launch_update(const Handle &H, const Mats &M, const UpdArgs &a, cudaStream_t st) {
  const unsigned grid = (unsigned)(H.nxu() + H.nyu());
  if (grid == 0) return;
  k_update<<<grid, kThreads, 0, st>>>(M, a);
  QG_LAUNCHED();
}

void launch_count_active(const Handle &H, cudaStream_t st) {
  k_count_active<<<1, 256, 0, st>>>(H.ws.st, H.B, H.ws.d_nactive);
  QG_LAUNCHED();
}

void launch_df_tail(const Handle &H, const Mats &M, const FinArgs &a, cudaStream_t st) {
  k_df_tail<<<1, 256, 0, st>>>(M, a, H.ws.df);  // (a carries the owing step's partial-sum buffers)
  QG_LAUNCHED();
}

__global__ void k_init_df(DfCtl *df, int pend) {
  df->flag[0] = df->flag[1] = 0;
  df->pend_phase = pend;
}

void launch_init_df(const Handle &H, int pend, cudaStream_t st) {
  k_init_df<<<1, 1, 0, st>>>(H.ws.df, pend);
  QG_LAUNCHED();
}

void launch_init_state(const Handle &H, double atol, double btol, long long opt, long long cap, cudaStream_t st) {
  k_init_state<<<(H.B + 127) / 128, 128, 0, st>>>(H.ws.st, H.B, atol, btol, opt, H.d_xoff, H.d_yoff, H.ws.d_loop, cap);
  QG_LAUNCHED();
}

}  // namespace qg
