// Problem-resident LSMR engine: batches of small problems (c5a: 4096 QCPs
// of n=1000, m=1500; c1) run their WHOLE solve inside one persistent kernel.
//
// One 1024-thread CTA per SM owns one problem at a time (claimed from a
// counter) and runs every remaining LSMR iteration of it (lsmr.py:111-184)
// without leaving the SM.  Shared memory holds
//
//   u[N] | v[N] | rs[n+m] | dp[m]        the LSMR vectors (N = n+m+1, T entry
//                                        at n+m), row sums, D Pi of the F input
//   resident matrix part                 a slice prefix of each of the
//                                        problem's SELL-32 matrices P, A, A'
//                                        (fp64 values + 16-bit local column
//                                        indices), loaded ONCE per problem by
//                                        TMA bulk copies (cp.async.bulk +
//                                        mbarrier complete_tx)
//
// and the rest of the matrix streams from HBM / L2 every operator
// application with read-only no-L1-allocate loads.  With one problem per SM
// the streamed parts of all resident problems (~150 x 160 KB at c5a) stay in
// L2 across the solve's 200 applications.
//
// Iteration (the graph path's order: the vector update of iteration k runs
// fused into the u-step epilogue of k+1, its stop test before fin U):
//
//   A_u  SpMV of v (all slices, dynamic claims)  ||  warp 0: sums + fin V(k-1)
//   B_u  u-step row epilogue + update of h, hbar, x (lsmr.py:142-144)
//   A_v  SpMV of u                               ||  warp 0: sums + stop test + fin U
//   B_v  v-step row epilogue (+ D Pi of the F' step per cone block)
//
// so the scalar finalize (thread 0: norms, Givens recurrences, stopping
// rules) overlaps the next SpMV phase instead of idling the SM; 4 CTA
// barriers per iteration, no kernel launch, no grid-wide barrier, no host
// round trip; a finished problem frees its CTA for the next claim at once.
//
// The arithmetic of every row / block / scalar is the graph path's
// (operator.cu expressions, fin_core through lsmr_dev.cuh); only the CTA
// summation trees differ (deterministic, fixed order).
#include "dpi_dev.cuh"
#include "lsmr_dev.cuh"
#include "ops_dev.cuh"
#include "operator.h"

namespace qg {

constexpr int kEngMaxWarps = 32;  // CTAs of 1024 threads (one per SM) or 512 (two per SM, QG_ENG_THREADS=512)
constexpr uint16_t kPad16 = 0xffff;
#ifndef QG_ENG_UNROLL
#define QG_ENG_UNROLL 8
#endif

struct EngArgs {
  Lsmr *st;
  double *u, *v, *h, *hb, *x;  // EVec workspace (global)
  const double *dp0;           // Y layout: D Pi of the first F step's input (jvp: dpv; vjp: unused)
  const uint16_t *c16P, *c16AT, *c16A;  // 16-bit local columns parallel to the SELL entries
  const uint16_t *r16x, *r16y;          // 16-bit local row of every slice lane (kPad16 = padding)
  int *next;                   // problem claim counter (zeroed before the launch)
  int B;
  int nmax, mmax;              // vector strides (max n+m+1, max m over the batch)
  int vec_doubles;             // 3 nmax + mmax rounded up to even (16-byte aligned resident area)
  int res_cap;                 // resident matrix capacity in entries (multiple of 8)
};

// One SELL matrix of the resident problem: slices [s0, s1); the prefix
// [s0, sres) sits in shared memory at entry offset soff.
struct Region {
  int64_t g0;        // first entry (S.off[s0])
  int s0, s1, sres;
  int soff;
};

struct EngShared {
  unsigned long long L[sizeof(Lsmr) / sizeof(unsigned long long)];
  double red[kEngMaxWarps * 2 * kSlots];
  double tvh[3];      // T entries of h, hbar, x
  unsigned long long mbar;
  Region reg[3];      // P, A' (X slices), A (Y slices)
  int p, cnt[2], rescount;
};

// ------------------------------------------------------------ TMA bulk --
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, unsigned long long *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      " @!P bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

// The streamed matrix part is re-read every operator application and must
// STAY in L2 across the solve: plain .nc / L1::no_allocate loads are tagged
// evict-first in L2 (measured: 78% of those sectors missed, 2% of normal
// ones), so these loads carry an explicit L2 evict-last policy and skip L1.
__device__ __forceinline__ uint64_t l2_keep_policy() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ double ld_keep(const double *p, uint64_t pol) {
  double v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint16_t ld_keep16(const uint16_t *p, uint64_t pol) {
  unsigned short v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u16 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(pol));
  return v;
}

// Row sum of this lane's row in slice s of region R: resident slices read
// values / columns from shared memory, the others stream them from global
// memory; the gather reads the shared-memory vector `vec` (local columns).
template <int UNR>
__device__ __forceinline__ double slice_dot(const Region &R, const SellView &S, const uint16_t *c16, int s, int lane,
                                            const double *vec, const double *sv, const uint16_t *sc) {
  const int w = S.w[s];
  const int64_t off = S.off[s];
  double a = 0.0;
  if (s < R.sres) {
    const int base = R.soff + (int)(off - R.g0) + lane;
    const double *vp = sv + base;
    const uint16_t *cp = sc + base;
#pragma unroll 4
    for (int k = 0; k < w; ++k) a += vp[32 * k] * vec[cp[32 * k]];
  } else {
    // every load of an UNR-entry group in flight at once (predicated tail:
    // no serial remainder chain); sums stay in storage order
    const double *vp = S.val + off + lane;
    const uint16_t *cp = c16 + off + lane;
    const uint64_t pol = l2_keep_policy();
    for (int k = 0; k < w; k += UNR) {
      double vv[UNR];
      uint16_t cc[UNR];
#pragma unroll
      for (int j = 0; j < UNR; ++j) {
        const bool ok = k + j < w;
        vv[j] = ok ? ld_keep(vp + 32 * (k + j), pol) : 0.0;
        cc[j] = ok ? ld_keep16(cp + 32 * (k + j), pol) : (uint16_t)0;
      }
#pragma unroll
      for (int j = 0; j < UNR; ++j)
        if (k + j < w) a += vv[j] * vec[cc[j]];
    }
  }
  return a;
}

// Phase A: the row sums of one operator application into rs (X rows: P w1
// +- A' (D Pi) w2 ; Y rows: A w1), slices claimed one at a time from cnt.
template <int KIND>
__device__ __forceinline__ void eng_spmv(const Mats &M, const EngArgs &a, const EngShared &S, int n, const double *in,
                                         const double *dp, double *rs, const double *sv, const uint16_t *sc,
                                         int *cnt) {
  const int lane = threadIdx.x & 31;
  const Region &RP = S.reg[0], &RT = S.reg[1], &RA = S.reg[2];
  const int nxs = RP.s1 - RP.s0, ntot = nxs + (RA.s1 - RA.s0);
  const double *x2 = KIND == STEP_F ? dp : in + n;  // A' gathers D Pi w_2 (F) or w_2 (F')
  while (true) {
    int q = 0;
    if (lane == 0) q = atomicAdd(cnt, 1);
    q = __shfl_sync(0xffffffffu, q, 0);
    if (q >= ntot) break;
    if (q < nxs) {
      const int s = RP.s0 + q;
      const double a1 = slice_dot<QG_ENG_UNROLL>(RP, M.sP, a.c16P, s, lane, in, sv, sc);
      const double a2 = slice_dot<QG_ENG_UNROLL>(RT, M.sAT, a.c16AT, s, lane, x2, sv, sc);
      const uint16_t r = a.r16x[(int64_t)s * 32 + lane];
      if (r != kPad16) rs[r] = KIND == STEP_F ? (a1 + a2) : (a1 - a2);
    } else {
      const int s = RA.s0 + (q - nxs);
      const double a1 = slice_dot<QG_ENG_UNROLL>(RA, M.sA, a.c16A, s, lane, in, sv, sc);
      const uint16_t r = a.r16y[(int64_t)s * 32 + lane];
      if (r != kPad16) rs[n + r] = a1;
    }
  }
}

// Warp 0: fixed-order sums of the per-warp partials (lanes 0..7 one slot
// each), returned on every lane of warp 0.
__device__ __forceinline__ void warp0_sums(const double *red, double (&s)[2 * kSlots]) {
  const int lane = threadIdx.x & 31;
  double t = 0.0;
  if (lane < 2 * kSlots)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w * 2 * kSlots + lane];
#pragma unroll
  for (int k = 0; k < 2 * kSlots; ++k) s[k] = __shfl_sync(0xffffffffu, t, k);
}

__device__ __forceinline__ void warp_partials(double (&v)[2 * kSlots], double *red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 2 * kSlots; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < 2 * kSlots; ++k) red[warp * 2 * kSlots + k] = v[k];
}

struct Geo {
  int n, m;
  int64_t xo, yo, T;
  int yu0, yu1;  // Y work units (cone-block classes)
};

// Phase B: row epilogue of one application (graph path expressions,
// operator.cu step_unit): out <- s_in OP(in) - c_out out (in place), with
// the deferred LSMR vector update fused into the u-step (upd), per-warp
// partials into red (X slots 0..3, Y slots 4..7; slot 3 / 7: ||x||^2).
template <int KIND>
__device__ __forceinline__ void eng_epilogue(const Mats &M, const EngArgs &a, const Geo &g, const Embed &E,
                                             const double *in, double *out, const double *rs, double *rsw,
                                             double *dp, double s_in, double c_out, bool upd, const Lsmr &L,
                                             double *red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = g.n, m = g.m;
  const int by = (int)g.yo;
  const double wN = in[n + m];
  double acc[2 * kSlots] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (upd) {
    // hbar = h - c1 hbar ; x = x + c2 hbar ; h = v s_v - c3 h (v = this step's input)
    const double c1 = L.c_hbar, c2 = L.c_x, c3 = L.c_h, svs = L.s_v;
    for (int i = tid; i < n + m; i += (int)blockDim.x) {
      const int64_t gi = i < n ? g.xo + i : M.NX + g.yo + (i - n);
      const double hv = __ldcg(a.h + gi), hbo = __ldcg(a.hb + gi), xo = __ldcg(a.x + gi);
      const double hbv = hv - c1 * hbo;
      const double xv = xo + c2 * hbv;
      __stcg(a.h + gi, in[i] * svs - c3 * hv);
      __stcg(a.hb + gi, hbv);
      __stcg(a.x + gi, xv);
      if (i < n) acc[3] += xv * xv; else acc[7] += xv * xv;
    }
  }
  const double izN = E.zN;
  for (int i = tid; i < n; i += (int)blockDim.x) {
    const int64_t r = g.xo + i;
    const double w = in[i];
    double res;
    if (KIND == STEP_F) {
      const double o1 = rs[i] + wN * M.q[r];
      res = ((o1 - w) + w) / izN;
      acc[0] += M.Pxbar[r] * w;
    } else {
      const double gg = (rs[i] - ((2.0 / E.tau) * wN) * M.Pxbar[r]) - wN * M.q[r];
      res = ((gg - w) + w) / izN;
    }
    acc[1] += M.q[r] * w;
    const double o = s_in * res - (c_out != 0.0 ? c_out * out[i] : 0.0);
    out[i] = o;
    acc[2] += o * o;
  }
  double *outY = out + n;
  const double *inY = in + n;
  if (KIND == STEP_F) {
    for (int j = tid; j < m; j += (int)blockDim.x) {
      const int64_t r = g.yo + j;
      const double o2 = (-rs[n + j]) + wN * M.b[r];
      const double res = ((o2 - dp[j]) + inY[j]) / izN;
      const double o = s_in * res - (c_out != 0.0 ? c_out * outY[j] : 0.0);
      outY[j] = o;
      acc[4] += M.b[r] * dp[j];
      acc[6] += o * o;
    }
  } else {
    // t = (A w1 - w_N b) - w2 (recomputed where needed), then per cone block:
    // o = s_in (D Pi t + w2)/z_N - c_out old ; dp = D Pi o
    const double *tsrc = rs + n;
    auto tval = [&](int j) { return (tsrc[j] - wN * M.b[g.yo + j]) - inY[j]; };
    auto fin_row = [&](int j, double dpt) {
      const double w = inY[j];
      const double o = s_in * ((dpt + w) / izN) - (c_out != 0.0 ? c_out * outY[j] : 0.0);
      outY[j] = o;
      acc[4] += M.b[g.yo + j] * w;
      acc[6] += o * o;
      return o;
    };
    const DpiView &dv = M.dpi;
    for (int ui = g.yu0; ui < g.yu1; ++ui) {
      const Unit u = M.yu[ui];
      if (u.cls == CLS_ELEM) {
        const int kind = dv.blk[u.blk0].kind;
        for (int r = u.row0 + tid; r < u.row1; r += (int)blockDim.x) {
          const int j = r - by;
          const double wgt = elem_weight(kind, dv.dual, dv.zmid[r]);
          const double o = fin_row(j, wgt * tval(j));
          dp[j] = wgt * o;
        }
      } else if (u.cls == CLS_TRI) {
        for (int k = u.blk0 + tid; k < u.blk1; k += (int)blockDim.x) {
          const BlockInfo b = dv.blk[k];
          const int j = b.row - by;
          double D[9];
#pragma unroll
          for (int i = 0; i < 9; ++i) D[i] = dv.tri_D[9 * b.param + i];
          const int flip = dv.tri_flip[b.param];
          const double t3[3] = {tval(j), tval(j + 1), tval(j + 2)};
          double r3[3], o3[3], d3[3];
          tri_apply(D, flip, t3, r3);
#pragma unroll
          for (int i = 0; i < 3; ++i) o3[i] = fin_row(j + i, r3[i]);
          tri_apply(D, flip, o3, d3);
#pragma unroll
          for (int i = 0; i < 3; ++i) dp[j + i] = d3[i];
        }
      } else if (u.cls == CLS_SOC && u.group > 0) {
        // G = u.group lanes per block (dims <= 32), one lane per row:
        // soc_entry twice (cones.py:740-764) with group shuffle sums
        const int G = u.group, per = 32 / G, lg = lane & (G - 1);
        const int nw = (int)(blockDim.x >> 5);
        for (int base = u.blk0 + warp * per; base < u.blk1; base += nw * per) {
          const int k = base + lane / G;
          const bool blk_ok = k < u.blk1;
          const BlockInfo b = dv.blk[blk_ok ? k : u.blk0];
          const int dim = blk_ok ? b.dim : 0, j0 = b.row - by, code = dv.soc_code[b.param];
          const double nu = dv.soc_nu[b.param];
          const bool ok = lg < dim;
          const double zi = ok ? dv.zmid[b.row + lg] : 0.0;
          const double ti = ok ? tval(j0 + lg) : 0.0;
          const double udu = gsum((ok && lg > 0) ? zi * ti : 0.0, G);
          const int src = lane & ~(G - 1);
          const double t0 = __shfl_sync(0xffffffffu, zi, src), dt = __shfl_sync(0xffffffffu, ti, src);
          const double oi = ok ? fin_row(j0 + lg, soc_entry(code, lg, nu, t0, zi, ti, dt, udu)) : 0.0;
          const double udu2 = gsum((ok && lg > 0) ? zi * oi : 0.0, G);
          const double o0 = __shfl_sync(0xffffffffu, oi, src);
          if (ok) dp[j0 + lg] = soc_entry(code, lg, nu, t0, zi, oi, o0, udu2);
        }
      } else {
        // large SOC blocks: a warp per block (soc_apply_warp), t in place in rs
        for (int k = u.blk0 + warp; k < u.blk1; k += (int)(blockDim.x >> 5)) {
          const BlockInfo b = dv.blk[k];
          const int dim = b.dim, j0 = b.row - by;
          double *tb = rsw + n + j0;
          for (int i = lane; i < dim; i += 32) tb[i] = tval(j0 + i);
          __syncwarp();
          soc_apply_warp(dv.zmid + b.row, dim, dv.soc_nu[b.param], dv.soc_code[b.param], tb, tb);
          __syncwarp();
          for (int i = lane; i < dim; i += 32) fin_row(j0 + i, tb[i]);
          __syncwarp();
          soc_apply_warp(dv.zmid + b.row, dim, dv.soc_nu[b.param], dv.soc_code[b.param], outY + j0, dp + j0);
          __syncwarp();
        }
      }
    }
  }
  warp_partials(acc, red);
}

// Resident prefix of one region: the largest slice prefix whose entries fit
// in `room` (counted by the whole CTA; S.off is monotone).
__device__ __forceinline__ void plan_region(Region &R, const SellView &S, int s0, int s1, int &room, int &soff,
                                            int *count) {
  const int64_t g0 = S.off[s0];
  int c = 0;
  for (int s = s0 + (int)threadIdx.x; s < s1; s += (int)blockDim.x) c += (S.off[s + 1] - g0 <= room) ? 1 : 0;
  if (threadIdx.x == 0) *count = 0;
  __syncthreads();
  if (c) atomicAdd(count, c);
  __syncthreads();
  const int sres = s0 + *count;
  const int ent = (int)(S.off[sres] - g0);
  if (threadIdx.x == 0) {
    R.g0 = g0;
    R.s0 = s0;
    R.s1 = s1;
    R.sres = sres;
    R.soff = soff;
  }
  room -= ent;
  soff += ent;
  __syncthreads();
}

template <int KU, int KV, int NT>
__global__ void __launch_bounds__(NT, 1024 / NT) k_engine(Mats M, EngArgs a) {
  extern __shared__ __align__(16) double sm[];
  __shared__ EngShared S;
  Lsmr &L = *reinterpret_cast<Lsmr *>(S.L);
  constexpr int kLw = (int)(sizeof(Lsmr) / sizeof(unsigned long long));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double *su = sm, *sv = sm + a.nmax, *rs = sm + 2 * a.nmax, *dp = sm + 3 * a.nmax;
  double *resv = sm + a.vec_doubles;                                  // resident values (16-byte aligned)
  uint16_t *resc = reinterpret_cast<uint16_t *>(resv + a.res_cap);   // resident 16-bit columns
  if (tid == 0) mbar_init(&S.mbar, 1);
  __syncthreads();
  uint32_t mphase = 0;

  while (true) {
    if (tid == 0) S.p = atomicAdd(a.next, 1);
    __syncthreads();
    const int p = S.p;
    if (p >= a.B) return;
    Geo g;
    g.xo = M.xoff[p];
    g.yo = M.yoff[p];
    g.n = (int)(M.xoff[p + 1] - g.xo);
    g.m = (int)(M.yoff[p + 1] - g.yo);
    g.T = M.NX + M.NY + p;
    const int64_t xu0 = M.xu_ptr[p], xu1 = M.xu_ptr[p + 1], yu0 = M.yu_ptr[p], yu1 = M.yu_ptr[p + 1];
    g.yu0 = (int)yu0;
    g.yu1 = (int)yu1;
    const int xs0 = xu1 > xu0 ? M.xu[xu0].s0 : 0, xs1 = xu1 > xu0 ? M.xu[xu1 - 1].s1 : 0;
    const int ys0 = yu1 > yu0 ? M.yu[yu0].s0 : 0, ys1 = yu1 > yu0 ? M.yu[yu1 - 1].s1 : 0;
    const int n = g.n, m = g.m, nm = n + m;
    const Embed E = M.emb[p];
    // resident slice prefixes: P, then A (Y), then A' with what is left
    {
      int room = a.res_cap, soff = 0;
      plan_region(S.reg[0], M.sP, xs0, xs1, room, soff, &S.rescount);
      plan_region(S.reg[2], M.sA, ys0, ys1, room, soff, &S.rescount);
      plan_region(S.reg[1], M.sAT, xs0, xs1, room, soff, &S.rescount);
    }
    if (tid == 0) {
      // one mbarrier phase per problem: every resident region by bulk copies
      // (all offsets are multiples of 32 entries: 16-byte aligned both sides)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of the area
      uint32_t bytes = 0;
      const SellView *mats[3] = {&M.sP, &M.sAT, &M.sA};
      const uint16_t *c16[3] = {a.c16P, a.c16AT, a.c16A};
      for (int r = 0; r < 3; ++r) {
        const Region &R = S.reg[r];
        bytes += (uint32_t)(mats[r]->off[R.sres] - R.g0) * 10u;
      }
      mbar_expect_tx(&S.mbar, bytes);
      for (int r = 0; r < 3; ++r) {
        const Region &R = S.reg[r];
        const uint32_t ent = (uint32_t)(mats[r]->off[R.sres] - R.g0);
        if (ent) {
          bulk_g2s(resv + R.soff, mats[r]->val + R.g0, ent * 8u, &S.mbar);
          bulk_g2s(resc + R.soff, c16[r] + R.g0, ent * 2u, &S.mbar);
        }
      }
    }
    // LSMR state, u, v (rows + T), D Pi of the F input, T entries of h / hbar / x
    const unsigned long long *Lg = reinterpret_cast<const unsigned long long *>(a.st + p);
    for (int w = tid; w < kLw; w += (int)blockDim.x) S.L[w] = Lg[w];
    for (int i = tid; i < nm; i += (int)blockDim.x) {
      const int64_t gi = i < n ? g.xo + i : M.NX + g.yo + (i - n);
      su[i] = a.u[gi];
      sv[i] = a.v[gi];
    }
    if (a.dp0)
      for (int j = tid; j < m; j += (int)blockDim.x) dp[j] = a.dp0[g.yo + j];
    if (tid == 0) {
      su[nm] = a.u[g.T];
      sv[nm] = a.v[g.T];
      S.tvh[0] = a.h[g.T];
      S.tvh[1] = a.hb[g.T];
      S.tvh[2] = a.x[g.T];
      S.cnt[0] = S.cnt[1] = 0;
    }
    mbar_wait(&S.mbar, mphase);
    mphase ^= 1;
    __syncthreads();

    bool pending_v = false;  // a v-step's partials await fin V (warp 0, during A_u)
    if (L.active) {
      while (true) {
        // ---- A_u || fin V of the previous iteration
        if (warp == 0 && pending_v) {
          double s8[2 * kSlots];
          warp0_sums(S.red, s8);
          if (lane == 0) {
            TVals t{su[nm], sv[nm], sv[nm], S.tvh[0], S.tvh[1], S.tvh[2], 0.0};
            const int w = fin_core(E, PH_STEP_V, KV, &L, s8, s8 + kSlots, t, false, false);
            if (w & TV_OUT) sv[nm] = t.out;
            if (w & TV_H) S.tvh[0] = t.h;
            if (w & TV_HB) S.tvh[1] = t.hb;
            if (w & TV_X) S.tvh[2] = t.x;
          }
          __syncwarp();
        }
        eng_spmv<KU>(M, a, S, n, sv, dp, rs, resv, resc, &S.cnt[0]);
        __syncthreads();
        if (!L.active) break;  // fin V stopped the solve (non-finite)
        // ---- B_u (+ the deferred update of the previous iteration)
        if (tid == 0) S.cnt[1] = 0;
        eng_epilogue<KU>(M, a, g, E, sv, su, rs, rs, dp, L.s_in, L.c_out, L.itn > 0, L, S.red);
        __syncthreads();
        // ---- A_v || stop test + fin U
        if (warp == 0) {
          double s8[2 * kSlots];
          warp0_sums(S.red, s8);
          if (lane == 0) {
            bool stop = L.itn > 0 && stop_test(&L, s8[3] + s8[kSlots + 3], S.tvh[2]);
            if (!stop) {
              TVals t{sv[nm], su[nm], su[nm], S.tvh[0], S.tvh[1], S.tvh[2], 0.0};
              const int w = fin_core(E, PH_STEP_U, KU, &L, s8, s8 + kSlots, t, false, false);
              if (w & TV_OUT) su[nm] = t.out;
            }
          }
          __syncwarp();
        }
        eng_spmv<KV>(M, a, S, n, su, dp, rs, resv, resc, &S.cnt[1]);
        __syncthreads();
        if (!L.active) break;  // the stop test ended the solve
        // ---- B_v (a zero beta skips the v-step: fin V keeps v)
        if (tid == 0) S.cnt[0] = 0;
        if (!L.skip_v) eng_epilogue<KV>(M, a, g, E, su, sv, rs, rs, dp, L.s_in, L.c_out, false, L, S.red);
        pending_v = true;
        __syncthreads();
      }
    }

    // write back: state, T entries, u and v (x / h / hbar rows are global)
    unsigned long long *Lw = reinterpret_cast<unsigned long long *>(a.st + p);
    for (int w = tid; w < kLw; w += (int)blockDim.x) Lw[w] = S.L[w];
    for (int i = tid; i < nm; i += (int)blockDim.x) {
      const int64_t gi = i < n ? g.xo + i : M.NX + g.yo + (i - n);
      a.u[gi] = su[i];
      a.v[gi] = sv[i];
    }
    if (tid == 0) {
      a.u[g.T] = su[nm];
      a.v[g.T] = sv[nm];
      a.h[g.T] = S.tvh[0];
      a.hb[g.T] = S.tvh[1];
      a.x[g.T] = S.tvh[2];
    }
    __syncthreads();
  }
}

// ------------------------------------------------- 16-bit local indices --
// Warp per slice: local column (col - the problem's column base) and local
// row of every entry / lane of a SELL matrix.
__global__ void k_local16(int64_t nslices, const int32_t *sprob, const int64_t *off, const int32_t *w,
                          const int32_t *col, const int64_t *cbase, uint16_t *c16, const int32_t *rowof,
                          const int64_t *rbase, uint16_t *r16) {
  const int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= nslices) return;
  const int p = sprob[s];
  const int64_t cb = cbase[p];
  const int64_t o = off[s];
  for (int k = 0; k < w[s]; ++k) c16[o + 32LL * k + lane] = (uint16_t)(col[o + 32LL * k + lane] - cb);
  if (r16) {
    const int r = rowof[s * 32 + lane];
    r16[s * 32 + lane] = r >= 0 ? (uint16_t)(r - rbase[p]) : kPad16;
  }
}

// ---------------------------------------------------------------- host --
static void engine_dims(const Handle &H, int &nmax, int &mmax) {
  nmax = mmax = 0;
  for (int p = 0; p < H.B; ++p) {
    nmax = std::max<int>(nmax, (int)(H.n[p] + H.m[p] + 1));
    mmax = std::max<int>(mmax, (int)H.m[p]);
  }
}

constexpr size_t kEngSmemMax = 227 * 1024 - sizeof(EngShared) - 256;        // one CTA per SM
constexpr size_t kEngSmemMax2 = 228 * 1024 / 2 - 1024 - sizeof(EngShared) - 256;  // two CTAs per SM
constexpr size_t kEngMinResident = 0;

static size_t engine_vec_bytes(const Handle &H) {
  int nmax, mmax;
  engine_dims(H, nmax, mmax);
  return sizeof(double) * (size_t)((3 * nmax + mmax + 1) & ~1);
}

bool engine_candidate(const Handle &H) {
  if (H.comm || H.cones.max_psd_order > 0) return false;
  const char *env = std::getenv("QG_ENGINE");
  if (env && std::atoi(env) == 0) return false;
  if (engine_vec_bytes(H) + kEngMinResident > kEngSmemMax) return false;
  for (int p = 0; p < H.B; ++p)
    if (H.n[p] >= 65535 || H.m[p] >= 65535) return false;  // 16-bit local indices
  if (env && std::atoi(env) != 0) return true;
  // resident solves win when the batch fills the GPU with problems, or the
  // single problems are small enough that launch latency dominates
  int64_t maxent = 0;
  for (int p = 0; p < H.B; ++p) maxent = std::max<int64_t>(maxent, H.nnzP[p] + 2 * H.nnzA[p]);
  return H.B >= 148 || maxent <= 16384;
}

bool engine_units_ok(const Handle &H) {
  for (const auto *us : {&H.xunits, &H.cones.units})
    for (const Unit &u : *us)
      if (u.mode != MODE_SELL) return false;
  return true;
}

static void slice_probs(const std::vector<Unit> &units, int64_t nslices, std::vector<int32_t> &out) {
  out.assign(std::max<int64_t>(nslices, 1), 0);
  for (const Unit &u : units)
    for (int s = u.s0; s < u.s1; ++s) out[s] = u.prob;
}

void build_engine_layout(Handle &H, cudaStream_t st) {
  std::vector<int32_t> spx, spy;
  slice_probs(H.xunits, H.nslice_x, spx);
  slice_probs(H.cones.units, H.nslice_y, spy);
  int32_t *d_spx = dev_alloc<int32_t>(spx.size()), *d_spy = dev_alloc<int32_t>(spy.size());
  QG_CUDA(cudaMemcpyAsync(d_spx, spx.data(), sizeof(int32_t) * spx.size(), cudaMemcpyHostToDevice, st));
  QG_CUDA(cudaMemcpyAsync(d_spy, spy.data(), sizeof(int32_t) * spy.size(), cudaMemcpyHostToDevice, st));
  H.c16P = dev_alloc<uint16_t>(H.sP.entries);
  H.c16AT = dev_alloc<uint16_t>(H.sAT.entries);
  H.c16A = dev_alloc<uint16_t>(H.sA.entries);
  H.r16x = dev_alloc<uint16_t>(32 * std::max<int64_t>(H.nslice_x, 1));
  H.r16y = dev_alloc<uint16_t>(32 * std::max<int64_t>(H.nslice_y, 1));
  const unsigned gx = (unsigned)((H.nslice_x * 32 + 255) / 256), gy = (unsigned)((H.nslice_y * 32 + 255) / 256);
  if (H.nslice_x) {
    k_local16<<<gx, 256, 0, st>>>(H.nslice_x, d_spx, H.sP.off, H.sP.w, H.sP.col, H.d_xoff, H.c16P, H.x_rowof,
                                  H.d_xoff, H.r16x);
    QG_LAUNCHED();
    k_local16<<<gx, 256, 0, st>>>(H.nslice_x, d_spx, H.sAT.off, H.sAT.w, H.sAT.col, H.d_yoff, H.c16AT, nullptr,
                                  nullptr, nullptr);
    QG_LAUNCHED();
  }
  if (H.nslice_y) {
    k_local16<<<gy, 256, 0, st>>>(H.nslice_y, d_spy, H.sA.off, H.sA.w, H.sA.col, H.d_xoff, H.c16A, H.y_rowof,
                                  H.d_yoff, H.r16y);
    QG_LAUNCHED();
  }
  QG_CUDA(cudaStreamSynchronize(st));  // host vectors spx / spy
  dev_free(d_spx);
  dev_free(d_spy);
}

void launch_engine(Handle &H, const Mats &M, bool jvp, cudaStream_t st) {
  Workspace &W = H.ws;
  EngArgs a{};
  a.st = W.st;
  a.u = W.u; a.v = W.v; a.h = W.h; a.hb = W.hb; a.x = W.x;
  a.dp0 = jvp ? W.dpv : nullptr;
  a.c16P = H.c16P; a.c16AT = H.c16AT; a.c16A = H.c16A;
  a.r16x = H.r16x; a.r16y = H.r16y;
  a.next = W.d_claim;
  a.B = H.B;
  engine_dims(H, a.nmax, a.mmax);
  a.vec_doubles = (3 * a.nmax + a.mmax + 1) & ~1;
  const size_t vec = sizeof(double) * (size_t)a.vec_doubles;
  static const char *env_nt = std::getenv("QG_ENG_THREADS");  // A/B: 512 = two CTAs (problems) per SM
  const int nt = env_nt && std::atoi(env_nt) == 512 ? 512 : 1024;
  const size_t cap = nt == 512 ? kEngSmemMax2 : kEngSmemMax;
  a.res_cap = vec < cap ? (int)(((cap - vec) / 10) & ~size_t(31)) : 0;
  if (const char *e = std::getenv("QG_ENG_RESIDENT")) a.res_cap = std::min(a.res_cap, std::atoi(e) & ~31);  // A/B
  const size_t smem = vec + (size_t)a.res_cap * 10;
  auto kern = nt == 512 ? (jvp ? k_engine<STEP_F, STEP_FT, 512> : k_engine<STEP_FT, STEP_F, 512>)
                        : (jvp ? k_engine<STEP_F, STEP_FT, 1024> : k_engine<STEP_FT, STEP_F, 1024>);
  QG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, nsm = 0;
  QG_CUDA(cudaGetDevice(&dev));
  QG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  const int grid = std::max(1, std::min(H.B, nsm * (1024 / nt)));
  QG_CUDA(cudaMemsetAsync(W.d_claim, 0, sizeof(int), st));
  kern<<<grid, nt, smem, st>>>(M, a);
  QG_LAUNCHED();
}

}  // namespace qg
