// Problem-resident LSMR engine: batches of small problems (c5a: 4096 QCPs
// of n=1000, m=1500; c1) run their WHOLE solve inside one persistent kernel.
//
// One CTA (512 threads, one per SM; QG_ENG_CFG) owns one problem at
// a time (claimed from a counter) and runs every remaining LSMR iteration of
// it (lsmr.py:111-184) without leaving the SM.  Shared memory holds
//
//   u[N] | v[N] | rs[N] | dp[m]   the LSMR vectors (N = n+m+1, T entry at
//                                 n+m), row sums, D Pi of the F input
//   meta blob                     the problem's slice table (widths, offsets,
//                                 16-bit rows), Y work units and cone blocks
//                                 (built once at preparation, k_engine_meta)
//   resident matrix part          a slice prefix of each of the problem's
//                                 SELL-32 matrices P, A, A' (fp64 values +
//                                 16-bit local columns)
//
// the blob and the resident part arrive by TMA bulk copies (cp.async.bulk +
// one mbarrier complete_tx phase per problem); the rest of the matrix
// streams from L2 every operator application with an L2 evict-last policy
// (~150 problems x 160 KB stay L2-resident across their 200 applications).
//
// Iteration (the graph path's order: the vector update of iteration k runs
// fused into the u-step epilogue of k+1, its stop test before fin U):
//
//   A_u  SpMV of v (static slice pairs per warp)  ||  warp 0: sums + fin V(k-1)
//   B_u  u-step row epilogue + update of h, hbar, x (lsmr.py:142-144)
//   A_v  SpMV of u                                ||  warp 0: sums + stop test + fin U
//   B_v  v-step row epilogue (+ D Pi of the F' step per cone block)
//
// so the scalar finalize (thread 0: norms, Givens recurrences, stopping
// rules) overlaps the next SpMV phase; 4 CTA barriers per iteration, no
// kernel launch, no grid-wide barrier, no host round trip; a finished
// problem frees its CTA for the next claim at once.
//
// The arithmetic of every row / block / scalar is the graph path's
// (operator.cu expressions, fin_core through lsmr_dev.cuh); only the CTA
// summation trees differ (deterministic, fixed order).
#include <algorithm>
#include <cstdio>
#include <mutex>
#include <vector>

#include "dpi_dev.cuh"
#include "lsmr_dev.cuh"
#include "ops_dev.cuh"
#include "operator.h"

namespace qg {

constexpr int kEngMaxWarps = 32;
constexpr uint16_t kPad16 = 0xffff;
#ifndef QG_ENG_UNROLL
#define QG_ENG_UNROLL 4
#endif

// ---------------------------------------------------------- meta blob --
// Per problem, fixed stride (the batch maximum), 16-byte aligned sections.
struct EngHead {
  int32_t nxs, nys, nyu, nblk;     // X / Y slices, Y units, cone blocks
  int32_t res[3];                  // resident slice count of P, A', A
  int32_t soff[3];                 // their smem entry offsets
  int32_t ent[3];                  // their resident entries
  int32_t pad;
  int64_t g0[3];                   // first entry of each matrix region
};
struct SliceMeta {                 // X slice: P part (off0, w0), A' part (off1, w1); Y slice: A part in (off1, w1)
  int32_t off0, off1;              // entry offsets from the region start
  uint16_t w0, w1;
};
struct EUnit {                     // a Y work unit, local rows / blocks
  int32_t cls, kind, G, row0, row1, blk0, blk1, pad;
};
struct EBlk {                      // a cone block: parameter index, local row, dim
  int32_t param;
  uint16_t j0, dim;
};
struct BlobLayout {
  int smax, umax, bmax, mmax;
  size_t o_slices, o_rows, o_units, o_blks, o_rowblk, stride;
};
static __host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~size_t(15); }
static __host__ __device__ inline BlobLayout blob_layout(int smax, int umax, int bmax, int mmax) {
  BlobLayout L{smax, umax, bmax, mmax, 0, 0, 0, 0, 0, 0};
  L.o_slices = al16(sizeof(EngHead));
  L.o_rows = al16(L.o_slices + sizeof(SliceMeta) * (size_t)smax);
  L.o_units = al16(L.o_rows + sizeof(uint16_t) * 32 * (size_t)smax);
  L.o_blks = al16(L.o_units + sizeof(EUnit) * (size_t)umax);
  L.o_rowblk = al16(L.o_blks + sizeof(EBlk) * (size_t)bmax);
  L.stride = al16(L.o_rowblk + sizeof(uint16_t) * (size_t)mmax);  // Y row -> its cone block (local)
  return L;
}

struct EngArgs {
  Lsmr *st;
  double *u, *v, *h, *hb, *x;  // EVec workspace (global)
  const double *dp0;           // Y layout: D Pi of the first F step's input (jvp: dpv; vjp: unused)
  const uint16_t *c16P, *c16AT, *c16A;  // 16-bit local columns parallel to the SELL entries
  const unsigned char *blob;   // per-problem meta blobs
  BlobLayout bl;
  int *next;                   // problem claim counter (zeroed before the launch)
  int B;
  int nmax, mmax;              // vector strides (max n+m+1, max m over the batch)
  // shared-memory byte offsets: u, v, rs (nmax each), dp (mmax), then the
  // problem's static rows q, P xbar (xmax each), b, z (mmax each), the SOC
  // parameters nu (double) / code (int) per block (bmax), blob, resident part
  int o_q, o_px, o_b, o_z, o_nu, o_code, o_scr, o_blob;
  int res_cap;                 // resident matrix capacity in entries (multiple of 32)
  unsigned long long *prof;    // QG_ENG_PROF=1: SM cycles [setup, A_u, B_u, A_v, B_v, iters, fin, spmv(warp 1)]
};

struct EngShared {
  unsigned long long L[sizeof(Lsmr) / sizeof(unsigned long long)];
  double red[kEngMaxWarps * 2 * kSlots];
  double tvh[3];      // T entries of h, hbar, x
  unsigned long long mbar;
  unsigned long long prof[10];
  int p;
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

// Per-problem views of the shared-memory blob and resident area, derived
// on demand from the kernel parameters (constant bank) so they hold no
// registers across the loop.
struct EngView {
  const Mats &M;
  const EngArgs &a;
  __device__ __forceinline__ unsigned char *blob() const {
    extern __shared__ __align__(16) double sm[];
    return reinterpret_cast<unsigned char *>(sm) + a.o_blob;
  }
  __device__ __forceinline__ const EngHead *hd() const { return reinterpret_cast<const EngHead *>(blob()); }
  __device__ __forceinline__ const SliceMeta *sl() const {
    return reinterpret_cast<const SliceMeta *>(blob() + a.bl.o_slices);
  }
  __device__ __forceinline__ const uint16_t *rows() const {
    return reinterpret_cast<const uint16_t *>(blob() + a.bl.o_rows);
  }
  __device__ __forceinline__ const EUnit *units() const { return reinterpret_cast<const EUnit *>(blob() + a.bl.o_units); }
  __device__ __forceinline__ const EBlk *blks() const { return reinterpret_cast<const EBlk *>(blob() + a.bl.o_blks); }
  __device__ __forceinline__ const uint16_t *rowblk() const {
    return reinterpret_cast<const uint16_t *>(blob() + a.bl.o_rowblk);
  }
  __device__ __forceinline__ double *resv() const { return reinterpret_cast<double *>(blob() + a.bl.stride); }
  __device__ __forceinline__ uint16_t *resc() const { return reinterpret_cast<uint16_t *>(resv() + a.res_cap); }
  __device__ __forceinline__ const double *gval(int r) const {
    return (r == 0 ? M.sP.val : r == 1 ? M.sAT.val : M.sA.val) + hd()->g0[r];
  }
  __device__ __forceinline__ const uint16_t *gcol(int r) const {
    return (r == 0 ? a.c16P : r == 1 ? a.c16AT : a.c16A) + hd()->g0[r];
  }
};

// Loads of one entry of a slice lane: shared memory (resident) or global
// with the L2 evict-last policy (streamed).
template <bool RES>
__device__ __forceinline__ double ldv(const double *p, uint64_t pol) {
  if constexpr (RES) return *p;
  else return ld_keep(p, pol);
}
template <bool RES>
__device__ __forceinline__ uint16_t ldc(const uint16_t *p, uint64_t pol) {
  if constexpr (RES) return *p;
  else return ld_keep16(p, pol);
}

// Row sums of this lane's rows in two slices (widths wa, wb; wb = 0: no
// second slice).  SELL padding (value 0, local column 0) makes every lane
// valid up to its slice width, so the loops carry no per-entry predicate:
// 4-entry groups of both slices issue all their loads before any gather.
// Each sum runs in storage order.
template <bool RA, bool RB>
__device__ __forceinline__ void dot2(const double *va, const uint16_t *ca, int wa, const double *vb,
                                     const uint16_t *cb, int wb, const double *vec, int vlen, double &sa,
                                     double &sb) {
  const uint64_t pol = (RA && RB) ? 0 : l2_keep_policy();
  double a = 0.0, b = 0.0;
  const int wm = wa < wb ? wa : wb;
  int k = 0;
  for (; k + 4 <= wm; k += 4) {
    double xa[4], xb[4];
    uint16_t ka[4], kb[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      xa[j] = ldv<RA>(va + 32 * (k + j), pol);
      ka[j] = ldc<RA>(ca + 32 * (k + j), pol);
      xb[j] = ldv<RB>(vb + 32 * (k + j), pol);
      kb[j] = ldc<RB>(cb + 32 * (k + j), pol);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      QG_CHECK(ka[j] < vlen && kb[j] < vlen);
      a += xa[j] * vec[ka[j]];
      b += xb[j] * vec[kb[j]];
    }
  }
  for (; k < wm; ++k) {
    const double x1 = ldv<RA>(va + 32 * k, pol), x2 = ldv<RB>(vb + 32 * k, pol);
    const uint16_t k1 = ldc<RA>(ca + 32 * k, pol), k2 = ldc<RB>(cb + 32 * k, pol);
    QG_CHECK(k1 < vlen && k2 < vlen);
    a += x1 * vec[k1];
    b += x2 * vec[k2];
  }
  int j = wm;
  for (; j + 4 <= wa; j += 4) {
    double xa[4];
    uint16_t ka[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      xa[i] = ldv<RA>(va + 32 * (j + i), pol);
      ka[i] = ldc<RA>(ca + 32 * (j + i), pol);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) a += xa[i] * vec[ka[i]];
  }
  for (; j < wa; ++j) a += ldv<RA>(va + 32 * j, pol) * vec[ldc<RA>(ca + 32 * j, pol)];
  for (int i = wm; i < wb; ++i) b += ldv<RB>(vb + 32 * i, pol) * vec[ldc<RB>(cb + 32 * i, pol)];
  sa = a;
  sb = b;
}

// Two slices of region r (0: P, 1: A', 2: A) at entry offsets oa / ob and
// widths wa / wb (wb = 0: none); slice a resident iff ra (b resident only if
// a is: resident slices are a prefix and qa < qb).
__device__ __forceinline__ void region_dot2(const EngView &V, int r, bool ra, int oa, int wa, bool rb, int ob, int wb,
                                            int lane, const double *vec, int vlen, double &sa, double &sb) {
  QG_CHECK(!ra || V.hd()->soff[r] + oa + 32 * wa <= V.hd()->soff[r] + V.hd()->ent[r]);
  QG_CHECK(!(ra && rb && wb > 0) || V.hd()->soff[r] + ob + 32 * wb <= V.hd()->soff[r] + V.hd()->ent[r]);
  QG_CHECK(V.hd()->soff[r] + V.hd()->ent[r] <= V.a.res_cap);
  const int so = V.hd()->soff[r] + lane;
  const double *rv = V.resv() + so;
  const uint16_t *rc = V.resc() + so;
  const double *gv = V.gval(r) + lane;
  const uint16_t *gc = V.gcol(r) + lane;
  if (ra && (rb || wb == 0))
    dot2<true, true>(rv + oa, rc + oa, wa, rv + ob, rc + ob, wb, vec, vlen, sa, sb);
  else if (ra)
    dot2<true, false>(rv + oa, rc + oa, wa, gv + ob, gc + ob, wb, vec, vlen, sa, sb);
  else
    dot2<false, false>(gv + oa, gc + oa, wa, gv + ob, gc + ob, wb, vec, vlen, sa, sb);
}

// Phase A: the row sums of one operator application into rs (X rows: P w1
// +- A' (D Pi) w2 ; Y rows: A w1).  Slot i takes slices i, i + nw, ...,
// two per round when both are on the same side (their loads overlap), so
// the last slots hold the fewest slices.  While warp 0 runs the scalar
// finalize (fin_warp) it takes the LAST slot and warp w slot w - 1: warp 0
// was the phase's critical path (c5a: finalize 5k + a full slice share 14k
// cycles of a 19.5k-cycle A_u).  Each row is summed by one lane in storage
// order whichever warp owns it, so the sums do not depend on the mapping.
template <int KIND>
__device__ __forceinline__ void eng_spmv(const EngView &V, int n, int m, const double *in, const double *dp,
                                         double *rs, bool fin_warp) {
  const int lane = threadIdx.x & 31, nw = (int)(blockDim.x >> 5);
  const int warp = fin_warp ? (int)((threadIdx.x >> 5) + nw - 1) % nw : (int)(threadIdx.x >> 5);
  const int nxs = V.hd()->nxs, ntot = nxs + V.hd()->nys;
  const double *x2 = KIND == STEP_F ? dp : in + n;  // A' gathers D Pi w_2 (F) or w_2 (F')
  for (int qa0 = warp; qa0 < ntot; qa0 += 2 * nw) {
    int qa = qa0, qb = qa0 + nw;
    if (qb < ntot && (qa < nxs) != (qb < nxs)) qb = ntot + 1;  // X / Y boundary: one at a time
    for (int rep = 0; rep < 2; ++rep) {
      const bool two = qb < ntot;
      const SliceMeta ma = V.sl()[qa], mb = two ? V.sl()[qb] : ma;
      double sa, sb;
      if (qa < nxs) {
        double ta, tb;
        region_dot2(V, 0, qa < V.hd()->res[0], ma.off0, ma.w0, !two || qb < V.hd()->res[0], mb.off0,
                                   two ? mb.w0 : 0, lane, in, n, sa, sb);
        region_dot2(V, 1, qa < V.hd()->res[1], ma.off1, ma.w1, !two || qb < V.hd()->res[1], mb.off1,
                                   two ? mb.w1 : 0, lane, x2, m, ta, tb);
        sa = KIND == STEP_F ? (sa + ta) : (sa - ta);
        sb = KIND == STEP_F ? (sb + tb) : (sb - tb);
      } else {
        region_dot2(V, 2, qa - nxs < V.hd()->res[2], ma.off1, ma.w1, !two || qb - nxs < V.hd()->res[2],
                                   mb.off1, two ? mb.w1 : 0, lane, in, n, sa, sb);
      }
      const int ya = qa < nxs ? 0 : n;
      const uint16_t ra = V.rows()[qa * 32 + lane];
      QG_CHECK(ra == kPad16 || ra < (qa < nxs ? n : m));
      if (ra != kPad16) rs[ya + ra] = sa;
      if (two) {
        const uint16_t rb = V.rows()[qb * 32 + lane];
        if (rb != kPad16) rs[ya + rb] = sb;
      }
      // the boundary case: the second slice on its own
      if (qb == ntot + 1 && qa0 + nw < ntot && rep == 0) {
        qa = qa0 + nw;
        qb = ntot;
      } else {
        break;
      }
    }
  }
}

// Slots of the step partials each application actually fills (X 0..3,
// Y 4..7): F: P xbar'w, q'w, ||o||^2 / b'D Pi w, ||o||^2 ; F': q'w,
// ||o||^2 / b'w, ||o||^2 ; slot 3 / 7: ||x||^2 of the fused update.
template <int KIND>
__device__ __forceinline__ constexpr unsigned slot_mask(bool upd) {
  return (KIND == STEP_F ? 0x57u : 0x56u) | (upd ? 0x88u : 0u);
}

__device__ __forceinline__ void warp_partials(double (&v)[2 * kSlots], double *red, unsigned mask) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 2 * kSlots; ++k)
    if (mask >> k & 1) v[k] = warp_sum(v[k]);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < 2 * kSlots; ++k) red[warp * 2 * kSlots + k] = (mask >> k & 1) ? v[k] : 0.0;
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

struct Geo {
  int n, m;
  int64_t xo, yo, T;
};

// Phase B: row epilogue of one application (graph path expressions,
// operator.cu step_unit): out <- s_in OP(in) - c_out out (in place), with
// the deferred LSMR vector update fused into the u-step (upd), per-warp
// partials into red.  z_N = 1 (every jvp / vjp) skips the divisions.
template <int KIND>
__device__ __forceinline__ void eng_epilogue(const Mats &M, const EngArgs &a, const EngView &V, const Geo &g,
                                             const Embed &E, const double *in, double *out, double *rs,
                                             double *dp, double s_in, double c_out, bool upd, const Lsmr &L,
                                             double *red, unsigned long long *prof = nullptr) {
  extern __shared__ __align__(16) double sm[];
  const bool tp = prof != nullptr && threadIdx.x == 0;  // QG_ENG_PROF: sub-phase cycles of thread 0
  long long t0c = tp ? clock64() : 0;
  const unsigned char *smb = reinterpret_cast<const unsigned char *>(sm);
  const double *sq = reinterpret_cast<const double *>(smb + a.o_q), *spx = reinterpret_cast<const double *>(smb + a.o_px);
  const double *bY = reinterpret_cast<const double *>(smb + a.o_b), *zY = reinterpret_cast<const double *>(smb + a.o_z);
  const double *snu = reinterpret_cast<const double *>(smb + a.o_nu);
  const int *scode = reinterpret_cast<const int *>(smb + a.o_code);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nt = (int)blockDim.x, nw = nt >> 5;
  const int n = g.n, m = g.m;
  const double wN = in[n + m];
  const bool zn1 = E.zN == 1.0;
  const double zN = E.zN;
  auto divz = [&](double x) { return zn1 ? x : x / zN; };
  double acc[2 * kSlots] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (upd) {
    // hbar = h - c1 hbar ; x = x + c2 hbar ; h = v s_v - c3 h (v = this step's input)
    const double c1 = L.c_hbar, c2 = L.c_x, c3 = L.c_h, svs = L.s_v;
    for (int i = tid; i < n + m; i += nt) {
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
  for (int i = tid; i < n; i += nt) {
    const double w = in[i], qr = sq[i], px = spx[i];
    double res;
    if (KIND == STEP_F) {
      const double o1 = rs[i] + wN * qr;
      res = divz((o1 - w) + w);
      acc[0] += px * w;
    } else {
      const double gg = (rs[i] - ((2.0 / E.tau) * wN) * px) - wN * qr;
      res = divz((gg - w) + w);
    }
    acc[1] += qr * w;
    const double o = s_in * res - (c_out != 0.0 ? c_out * out[i] : 0.0);
    out[i] = o;
    acc[2] += o * o;
  }
  double *outY = out + n;
  const double *inY = in + n;
  if (KIND == STEP_F) {
    for (int j = tid; j < m; j += nt) {
      const double br = bY[j];
      const double o2 = (-rs[n + j]) + wN * br;
      const double res = divz((o2 - dp[j]) + inY[j]);
      const double o = s_in * res - (c_out != 0.0 ? c_out * outY[j] : 0.0);
      outY[j] = o;
      acc[4] += br * dp[j];
      acc[6] += o * o;
    }
  } else {
    // t = (A w1 - w_N b) - w2, then per cone block:
    // o = s_in (D Pi t + w2)/z_N - c_out old ; dp = D Pi o
    auto tval = [&](int j) { return (rs[n + j] - wN * bY[j]) - inY[j]; };
    auto fin_row = [&](int j, double dpt) {
      const double w = inY[j];
      const double o = s_in * divz(dpt + w) - (c_out != 0.0 ? c_out * outY[j] : 0.0);
      outY[j] = o;
      acc[4] += bY[j] * w;
      acc[6] += o * o;
      return o;
    };
    const DpiView &dv = M.dpi;
    const int nyu = V.hd()->nyu;
    if (tp) {
      const long long t = clock64();
      prof[8] += (unsigned long long)(t - t0c);  // update + X rows
      t0c = t;
    }
    for (int ui = 0; ui < nyu; ++ui) {
      const EUnit u = V.units()[ui];
      // rows / blocks go to threads by their problem-local index (not by unit
      // offsets), so every partial sum -- and the LSMR iterates -- are the same
      // whatever batch (and hence unit cut) the problem is prepared in
      if (u.cls == CLS_ELEM) {
        for (int j = u.row0 + (tid - u.row0 % nt + nt) % nt; j < u.row1; j += nt) {
          const double wgt = elem_weight(u.kind, dv.dual, zY[j]);
          const double o = fin_row(j, wgt * tval(j));
          dp[j] = wgt * o;
        }
      } else if (u.cls == CLS_TRI) {
        for (int k = u.blk0 + (tid - u.blk0 % nt + nt) % nt; k < u.blk1; k += nt) {
          const EBlk b = V.blks()[k];
          const int j = b.j0;
          double D[9];
#pragma unroll
          for (int i = 0; i < 9; ++i) D[i] = dv.tri_D[9 * (int64_t)b.param + i];
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
      } else if (u.G > 0) {
        // SOC blocks of dim <= 32 (cones.py:740-764 applied twice) in four
        // balanced phases: per-block sums by a thread per block, per-row
        // entries by a thread per row (Y row -> block from the meta blob)
        double *sU = reinterpret_cast<double *>(const_cast<unsigned char *>(smb) + a.o_scr);
        double *sA = sU + a.bl.bmax, *sB = sA + a.bl.bmax;
        const EBlk *bl = V.blks();
        const uint16_t *rbk = V.rowblk();
        for (int k = u.blk0 + (tid - u.blk0 % nt + nt) % nt; k < u.blk1; k += nt) {   // udu = z[1:]'t[1:]
          const EBlk b = bl[k];
          double s = 0.0;
          for (int i = 1; i < b.dim; ++i) s += zY[b.j0 + i] * tval(b.j0 + i);
          sU[k] = s;
          sA[k] = tval(b.j0);  // dt
        }
        __syncthreads();
        for (int j = u.row0 + (tid - u.row0 % nt + nt) % nt; j < u.row1; j += nt) {  // o = fin_row(D Pi t)
          const int k = rbk[j];
          const int i = j - bl[k].j0;
          const double t0 = zY[bl[k].j0];
          fin_row(j, soc_entry(scode[k], i, snu[k], t0, zY[j], tval(j), sA[k], sU[k]));
        }
        __syncthreads();
        for (int k = u.blk0 + (tid - u.blk0 % nt + nt) % nt; k < u.blk1; k += nt) {   // udu2 = z[1:]'o[1:]
          const EBlk b = bl[k];
          double s = 0.0;
          for (int i = 1; i < b.dim; ++i) s += zY[b.j0 + i] * outY[b.j0 + i];
          sB[k] = s;
        }
        __syncthreads();
        for (int j = u.row0 + (tid - u.row0 % nt + nt) % nt; j < u.row1; j += nt) {  // dp = D Pi o
          const int k = rbk[j];
          const int j0 = bl[k].j0;
          dp[j] = soc_entry(scode[k], j - j0, snu[k], zY[j0], zY[j], outY[j], outY[j0], sB[k]);
        }
      } else {
        // large SOC blocks: a warp per block (soc_apply_warp), t in place in rs
        for (int k = u.blk0 + (warp - u.blk0 % nw + nw) % nw; k < u.blk1; k += nw) {
          const EBlk b = V.blks()[k];
          const int dim = b.dim, j0 = b.j0;
          const int code = scode[k];
          const double nu = snu[k];
          double *tb = rs + n + j0;
          for (int i = lane; i < dim; i += 32) tb[i] = tval(j0 + i);
          __syncwarp();
          soc_apply_warp(zY + j0, dim, nu, code, tb, tb);
          __syncwarp();
          for (int i = lane; i < dim; i += 32) fin_row(j0 + i, tb[i]);
          __syncwarp();
          soc_apply_warp(zY + j0, dim, nu, code, outY + j0, dp + j0);
          __syncwarp();
        }
      }
    }
  }
  if (tp && KIND == STEP_FT) prof[9] += (unsigned long long)(clock64() - t0c);  // Y cone blocks
  warp_partials(acc, red, slot_mask<KIND>(upd));
}

template <int KU, int KV, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_engine(Mats M, EngArgs a) {
  extern __shared__ __align__(16) double sm[];
  __shared__ EngShared S;
  Lsmr &L = *reinterpret_cast<Lsmr *>(S.L);
  constexpr int kLw = (int)(sizeof(Lsmr) / sizeof(unsigned long long));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double *su = sm, *sv = sm + a.nmax, *rs = sm + 2 * a.nmax, *dp = sm + 3 * a.nmax;
  unsigned char *smb = reinterpret_cast<unsigned char *>(sm);
  double *sq = reinterpret_cast<double *>(smb + a.o_q), *spx = reinterpret_cast<double *>(smb + a.o_px);
  double *sb = reinterpret_cast<double *>(smb + a.o_b), *sz = reinterpret_cast<double *>(smb + a.o_z);
  double *snu = reinterpret_cast<double *>(smb + a.o_nu);
  int *scode = reinterpret_cast<int *>(smb + a.o_code);
  const EngView V{M, a};
  unsigned char *blob = V.blob();  // 16-byte aligned
  double *resv = V.resv();
  uint16_t *resc = V.resc();
  if (tid == 0) {
    mbar_init(&S.mbar, 1);
    for (int k = 0; k < 10; ++k) S.prof[k] = 0;
  }
  __syncthreads();
  uint32_t mphase = 0;
  const bool prof = a.prof != nullptr && tid == 0;
  long long t_mark = 0;
  auto tick = [&](int k) {
    if (prof) {
      const long long t = clock64();
      S.prof[k] += (unsigned long long)(t - t_mark);
      t_mark = t;
    }
  };

  while (true) {
    if (tid == 0) S.p = atomicAdd(a.next, 1);
    __syncthreads();
    const int p = S.p;
    if (p >= a.B) {
      if (prof)
        for (int k = 0; k < 10; ++k) atomicAdd(a.prof + k, S.prof[k]);
      return;
    }
    if (prof) t_mark = clock64();
    Geo g;
    g.xo = M.xoff[p];
    g.yo = M.yoff[p];
    g.n = (int)(M.xoff[p + 1] - g.xo);
    g.m = (int)(M.yoff[p + 1] - g.yo);
    g.T = M.NX + M.NY + p;
    const int n = g.n, m = g.m, nm = n + m;
    const Embed E = M.emb[p];
    const unsigned char *gblob = a.blob + (size_t)p * a.bl.stride;
    const EngHead *gh = reinterpret_cast<const EngHead *>(gblob);
    const SellView *mats[3] = {&M.sP, &M.sAT, &M.sA};
    const uint16_t *c16[3] = {a.c16P, a.c16AT, a.c16A};
    if (tid == 0) {
      // one mbarrier phase per problem: the meta blob and every resident
      // region by bulk copies (all sizes / offsets multiples of 16 bytes)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of the area
      const EngHead h = *gh;
      uint32_t bytes = (uint32_t)a.bl.stride;
      for (int r = 0; r < 3; ++r) bytes += (uint32_t)h.ent[r] * 10u;
      mbar_expect_tx(&S.mbar, bytes);
      bulk_g2s(blob, gblob, (uint32_t)a.bl.stride, &S.mbar);
      for (int r = 0; r < 3; ++r)
        if (h.ent[r]) {
          bulk_g2s(resv + h.soff[r], mats[r]->val + h.g0[r], (uint32_t)h.ent[r] * 8u, &S.mbar);
          bulk_g2s(resc + h.soff[r], c16[r] + h.g0[r], (uint32_t)h.ent[r] * 2u, &S.mbar);
        }
    }
    // LSMR state, u, v (rows + T), D Pi of the F input, T entries of h / hbar / x
    const unsigned long long *Lg = reinterpret_cast<const unsigned long long *>(a.st + p);
    for (int w = tid; w < kLw; w += NT) S.L[w] = Lg[w];
    for (int i = tid; i < nm; i += NT) {
      const int64_t gi = i < n ? g.xo + i : M.NX + g.yo + (i - n);
      su[i] = a.u[gi];
      sv[i] = a.v[gi];
    }
    if (a.dp0)
      for (int j = tid; j < m; j += NT) dp[j] = a.dp0[g.yo + j];
    // the problem's static rows and SOC parameters (read every iteration by
    // the row epilogues: kept on chip, no global round trip in phase B)
    for (int i = tid; i < n; i += NT) {
      sq[i] = M.q[g.xo + i];
      spx[i] = M.Pxbar[g.xo + i];
    }
    for (int j = tid; j < m; j += NT) {
      sb[j] = M.b[g.yo + j];
      sz[j] = M.dpi.zmid[g.yo + j];
    }
    {
      const EBlk *gb = reinterpret_cast<const EBlk *>(gblob + a.bl.o_blks);
      for (int k = tid; k < gh->nblk; k += NT) {
        const int prm = gb[k].param;
        snu[k] = M.dpi.soc_nu[prm];
        scode[k] = M.dpi.soc_code[prm];
      }
    }
    if (tid == 0) {
      su[nm] = a.u[g.T];
      sv[nm] = a.v[g.T];
      S.tvh[0] = a.h[g.T];
      S.tvh[1] = a.hb[g.T];
      S.tvh[2] = a.x[g.T];
    }
    mbar_wait(&S.mbar, mphase);
    mphase ^= 1;
    __syncthreads();
    tick(0);

    bool pending_v = false;  // a v-step's partials await fin V (warp 0, during A_u)
    if (L.active) {
      while (true) {
        // ---- A_u || fin V of the previous iteration
        const bool prof1 = a.prof != nullptr && tid == 32;
        long long t_sp = prof1 ? clock64() : 0;
        if (warp == 0 && pending_v) {
          const long long t_f = prof ? clock64() : 0;
          double s8[2 * kSlots];
          warp0_sums(S.red, s8);
          if (lane == 0) {
            TVals t{su[nm], sv[nm], sv[nm], S.tvh[0], S.tvh[1], S.tvh[2], 0.0};
            const int w = fin_core(E, PH_STEP_V, KV, &L, s8, s8 + kSlots, t, false, false);
            if (w & TV_OUT) sv[nm] = t.out;
            if (w & TV_H) S.tvh[0] = t.h;
            if (w & TV_HB) S.tvh[1] = t.hb;
            if (w & TV_X) S.tvh[2] = t.x;
            if (prof) S.prof[6] += (unsigned long long)(clock64() - t_f);
          }
          __syncwarp();
        }
        eng_spmv<KU>(V, n, m, sv, dp, rs, pending_v);
        if (prof1) S.prof[7] += (unsigned long long)(clock64() - t_sp);
        __syncthreads();
        tick(1);
        if (!L.active) break;  // fin V stopped the solve (non-finite)
        // ---- B_u (+ the deferred update of the previous iteration)
        eng_epilogue<KU>(M, a, V, g, E, sv, su, rs, dp, L.s_in, L.c_out, L.itn > 0, L, S.red,
                         a.prof ? S.prof : nullptr);
        __syncthreads();
        tick(2);
        // ---- A_v || stop test + fin U
        if (prof1) t_sp = clock64();
        if (warp == 0) {
          const long long t_f = prof ? clock64() : 0;
          double s8[2 * kSlots];
          warp0_sums(S.red, s8);
          if (lane == 0) {
            const bool stop = L.itn > 0 && stop_test(&L, s8[3] + s8[kSlots + 3], S.tvh[2]);
            if (!stop) {
              TVals t{sv[nm], su[nm], su[nm], S.tvh[0], S.tvh[1], S.tvh[2], 0.0};
              const int w = fin_core(E, PH_STEP_U, KU, &L, s8, s8 + kSlots, t, false, false);
              if (w & TV_OUT) su[nm] = t.out;
            }
            if (prof) S.prof[6] += (unsigned long long)(clock64() - t_f);
          }
          __syncwarp();
        }
        eng_spmv<KV>(V, n, m, su, dp, rs, true);
        if (prof1) S.prof[7] += (unsigned long long)(clock64() - t_sp);
        __syncthreads();
        tick(3);
        if (!L.active) break;  // the stop test ended the solve
        // ---- B_v (a zero beta skips the v-step: fin V keeps v)
        if (!L.skip_v)
          eng_epilogue<KV>(M, a, V, g, E, su, sv, rs, dp, L.s_in, L.c_out, false, L, S.red, a.prof ? S.prof : nullptr);
        pending_v = true;
        __syncthreads();
        tick(4);
        if (prof) S.prof[5] += 1;
      }
    }

    // write back: state, T entries, u and v (x / h / hbar rows are global)
    unsigned long long *Lw = reinterpret_cast<unsigned long long *>(a.st + p);
    for (int w = tid; w < kLw; w += NT) Lw[w] = S.L[w];
    for (int i = tid; i < nm; i += NT) {
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

// ------------------------------------------------- engine preparation --
// Warp per slice: local column (col - the problem's column base) of every
// entry of a SELL matrix.
__global__ void k_local16(int64_t nslices, const int32_t *sprob, const int64_t *off, const int32_t *w,
                          const int32_t *col, const int64_t *cbase, uint16_t *c16) {
  const int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= nslices) return;
  const int64_t cb = cbase[sprob[s]];
  const int64_t o = off[s];
  for (int k = 0; k < w[s]; ++k) c16[o + 32LL * k + lane] = (uint16_t)(col[o + 32LL * k + lane] - cb);
}

// One CTA per problem: its meta blob (slice table, local rows, Y units,
// blocks) and the resident plan (largest slice prefix of P, then A', then A
// fitting res_cap entries).
__global__ void k_engine_meta(Mats M, BlobLayout bl, int res_cap, unsigned char *blobs) {
  const int p = blockIdx.x;
  unsigned char *b = blobs + (size_t)p * bl.stride;
  EngHead *hd = reinterpret_cast<EngHead *>(b);
  SliceMeta *sl = reinterpret_cast<SliceMeta *>(b + bl.o_slices);
  uint16_t *rows = reinterpret_cast<uint16_t *>(b + bl.o_rows);
  EUnit *un = reinterpret_cast<EUnit *>(b + bl.o_units);
  EBlk *bk = reinterpret_cast<EBlk *>(b + bl.o_blks);
  const int64_t xu0 = M.xu_ptr[p], xu1 = M.xu_ptr[p + 1], yu0 = M.yu_ptr[p], yu1 = M.yu_ptr[p + 1];
  const int xs0 = xu1 > xu0 ? M.xu[xu0].s0 : 0, xs1 = xu1 > xu0 ? M.xu[xu1 - 1].s1 : 0;
  const int ys0 = yu1 > yu0 ? M.yu[yu0].s0 : 0, ys1 = yu1 > yu0 ? M.yu[yu1 - 1].s1 : 0;
  const int kb0 = yu1 > yu0 ? M.yu[yu0].blk0 : 0, kb1 = yu1 > yu0 ? M.yu[yu1 - 1].blk1 : 0;
  const int nxs = xs1 - xs0, nys = ys1 - ys0;
  const int64_t xo = M.xoff[p], yo = M.yoff[p];
  // (a side without slices may have no SELL arrays at all)
  const int64_t g0[3] = {nxs ? M.sP.off[xs0] : 0, nxs ? M.sAT.off[xs0] : 0, nys ? M.sA.off[ys0] : 0};
  for (int q = threadIdx.x; q < nxs + nys; q += blockDim.x) {
    SliceMeta s{};
    if (q < nxs) {
      const int gs = xs0 + q;
      s.off0 = (int32_t)(M.sP.off[gs] - g0[0]);
      s.off1 = (int32_t)(M.sAT.off[gs] - g0[1]);
      s.w0 = (uint16_t)M.sP.w[gs];
      s.w1 = (uint16_t)M.sAT.w[gs];
    } else {
      const int gs = ys0 + (q - nxs);
      s.off1 = (int32_t)(M.sA.off[gs] - g0[2]);
      s.w1 = (uint16_t)M.sA.w[gs];
    }
    sl[q] = s;
  }
  for (int i = threadIdx.x; i < 32 * (nxs + nys); i += blockDim.x) {
    const int q = i / 32, lane = i % 32;
    const int r = q < nxs ? M.x_rowof[(int64_t)(xs0 + q) * 32 + lane] : M.y_rowof[(int64_t)(ys0 + q - nxs) * 32 + lane];
    rows[i] = r < 0 ? kPad16 : (uint16_t)(r - (q < nxs ? xo : yo));
  }
  for (int ui = (int)yu0 + threadIdx.x; ui < (int)yu1; ui += blockDim.x) {
    const Unit u = M.yu[ui];
    EUnit e{};
    e.cls = u.cls;
    e.kind = M.dpi.blk[u.blk0].kind;
    e.G = u.cls == CLS_SOC ? u.group : 0;
    e.row0 = (int32_t)(u.row0 - yo);
    e.row1 = (int32_t)(u.row1 - yo);
    e.blk0 = u.blk0 - kb0;
    e.blk1 = u.blk1 - kb0;
    un[ui - yu0] = e;
  }
  uint16_t *rb = reinterpret_cast<uint16_t *>(b + bl.o_rowblk);
  for (int k = kb0 + threadIdx.x; k < kb1; k += blockDim.x) {
    const BlockInfo bi = M.dpi.blk[k];
    bk[k - kb0] = EBlk{(int32_t)bi.param, (uint16_t)(bi.row - yo), (uint16_t)bi.dim};
    for (int i = 0; i < bi.dim; ++i) rb[bi.row - yo + i] = (uint16_t)(k - kb0);
  }
  if (threadIdx.x == 0) {
    EngHead h{};
    h.nxs = nxs;
    h.nys = nys;
    h.nyu = (int)(yu1 - yu0);
    h.nblk = kb1 - kb0;
    const SellView *mats[3] = {&M.sP, &M.sAT, &M.sA};
    const int sr0[3] = {xs0, xs0, ys0}, sr1[3] = {xs1, xs1, ys1};
    int room = res_cap, soff = 0;
    for (int r : {0, 1, 2}) {  // P, then A' (wide X rows), then A: the streamed rest are narrow Y slices
      int s = sr0[r];
      while (s < sr1[r] && mats[r]->off[s + 1] - g0[r] <= room) ++s;
      const int ent = s > sr0[r] ? (int)(mats[r]->off[s] - g0[r]) : 0;
      h.res[r] = s - sr0[r];
      h.soff[r] = soff;
      h.ent[r] = ent;
      h.g0[r] = g0[r];
      room -= ent;
      soff += ent;
    }
    *hd = h;
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

constexpr size_t kEngSmemMax = 227 * 1024 - sizeof(EngShared) - 256;              // one CTA per SM
constexpr size_t kEngSmemMax2 = 228 * 1024 / 2 - 1024 - sizeof(EngShared) - 256;  // two CTAs per SM

static BlobLayout engine_blob_layout(const Handle &H);

// Shared-memory byte offsets (EngArgs::o_*) of a batch; returns the bytes
// before the blob.
static size_t engine_offsets(const Handle &H, int bmax, EngArgs *a) {
  int nmax, mmax, xmax = 0;
  engine_dims(H, nmax, mmax);
  for (int p = 0; p < H.B; ++p) xmax = std::max<int>(xmax, (int)H.n[p]);
  size_t o = sizeof(double) * (size_t)(3 * nmax + mmax);
  const size_t oq = o; o += sizeof(double) * xmax;
  const size_t opx = o; o += sizeof(double) * xmax;
  const size_t ob = o; o += sizeof(double) * mmax;
  const size_t oz = o; o += sizeof(double) * mmax;
  const size_t onu = o; o += sizeof(double) * bmax;
  const size_t ocode = o; o += sizeof(int) * bmax;
  o = al16(o);
  const size_t oscr = o; o += 3 * sizeof(double) * bmax;   // per-block udu, dt, udu2 scratch
  o = al16(o);                                               // blob: cp.async.bulk destination
  if (a) {
    a->nmax = nmax;
    a->mmax = mmax;
    a->o_q = (int)oq; a->o_px = (int)opx; a->o_b = (int)ob; a->o_z = (int)oz;
    a->o_nu = (int)onu; a->o_code = (int)ocode; a->o_scr = (int)oscr; a->o_blob = (int)o;
  }
  return o;
}

static int engine_cfg() {
  static const char *env = std::getenv("QG_ENG_CFG");
  static const int c = env ? std::max(0, std::min(2, std::atoi(env))) : 1;
  return c;
}
static int engine_threads() { return engine_cfg() == 0 ? 1024 : 512; }
static int engine_ctas_per_sm() { return engine_cfg() == 2 ? 2 : 1; }

// Blob maxima from the host-side units / blocks (slices: the unit ranges).
static BlobLayout engine_blob_layout(const Handle &H) {
  int smax = 0, umax = 0, bmax = 0;
  for (int p = 0; p < H.B; ++p) {
    int ns = 0;
    for (int64_t u = H.xunit_ptr[p]; u < H.xunit_ptr[p + 1]; ++u) ns += H.xunits[u].s1 - H.xunits[u].s0;
    const int64_t y0 = H.cones.unit_ptr[p], y1 = H.cones.unit_ptr[p + 1];
    for (int64_t u = y0; u < y1; ++u) ns += H.cones.units[u].s1 - H.cones.units[u].s0;
    smax = std::max(smax, ns);
    umax = std::max(umax, (int)(y1 - y0));
    if (y1 > y0) bmax = std::max(bmax, H.cones.units[y1 - 1].blk1 - H.cones.units[y0].blk0);
  }
  int nmax, mmax;
  engine_dims(H, nmax, mmax);
  return blob_layout(smax, umax, bmax, mmax);
}

static int engine_res_cap(const Handle &H, size_t blob_stride) {
  const size_t cap = engine_ctas_per_sm() == 2 ? kEngSmemMax2 : kEngSmemMax;
  const size_t used = engine_offsets(H, engine_blob_layout(H).bmax, nullptr) + blob_stride;
  int rc = used < cap ? (int)(((cap - used) / 10) & ~size_t(31)) : 0;
  if (const char *e = std::getenv("QG_ENG_RESIDENT")) rc = std::min(rc, std::atoi(e) & ~31);  // A/B
  return rc;
}

bool engine_candidate(const Handle &H) {
  if (H.comm || H.cones.max_psd_order > 0) return false;
  const char *env = std::getenv("QG_ENGINE");
  if (env && std::atoi(env) == 0) return false;
  for (int p = 0; p < H.B; ++p)
    if (H.n[p] >= 65535 || H.m[p] >= 65535) return false;  // 16-bit local indices
  if (engine_offsets(H, engine_blob_layout(H).bmax, nullptr) + 16 * 1024 >
      (engine_ctas_per_sm() == 2 ? kEngSmemMax2 : kEngSmemMax))
    return false;
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
  const BlobLayout bl = engine_blob_layout(H);
  return engine_offsets(H, bl.bmax, nullptr) + bl.stride <= (engine_ctas_per_sm() == 2 ? kEngSmemMax2 : kEngSmemMax);
}

static void slice_probs(const std::vector<Unit> &units, int64_t nslices, std::vector<int32_t> &out) {
  out.assign(std::max<int64_t>(nslices, 1), 0);
  for (const Unit &u : units)
    for (int s = u.s0; s < u.s1; ++s) out[s] = u.prob;
}

// After build_sell (slices) and the cone table: 16-bit local columns and
// the per-problem meta blobs.
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
  const unsigned gx = (unsigned)((H.nslice_x * 32 + 255) / 256), gy = (unsigned)((H.nslice_y * 32 + 255) / 256);
  if (H.nslice_x) {
    k_local16<<<gx, 256, 0, st>>>(H.nslice_x, d_spx, H.sP.off, H.sP.w, H.sP.col, H.d_xoff, H.c16P);
    QG_LAUNCHED();
    k_local16<<<gx, 256, 0, st>>>(H.nslice_x, d_spx, H.sAT.off, H.sAT.w, H.sAT.col, H.d_yoff, H.c16AT);
    QG_LAUNCHED();
  }
  if (H.nslice_y) {
    k_local16<<<gy, 256, 0, st>>>(H.nslice_y, d_spy, H.sA.off, H.sA.w, H.sA.col, H.d_xoff, H.c16A);
    QG_LAUNCHED();
  }
  const BlobLayout bl = engine_blob_layout(H);
  H.eng_res_cap = engine_res_cap(H, bl.stride);
  H.eng_blob = dev_alloc<unsigned char>(bl.stride * (size_t)H.B);
  QG_CUDA(cudaMemsetAsync(H.eng_blob, 0, bl.stride * (size_t)H.B, st));
  Mats M = make_mats(H);
  k_engine_meta<<<H.B, 256, 0, st>>>(M, bl, H.eng_res_cap, H.eng_blob);
  QG_LAUNCHED();
  QG_CUDA(cudaStreamSynchronize(st));  // host vectors spx / spy
  dev_free(d_spx);
  dev_free(d_spy);
}

template <class K>
static void set_max_dynamic_smem(K kern) {
  static std::mutex mu;
  static std::vector<const void *> done;
  std::lock_guard<std::mutex> lock(mu);
  const void *key = reinterpret_cast<const void *>(kern);
  if (std::find(done.begin(), done.end(), key) != done.end()) return;
  int dev = 0, optin = 0;
  QG_CUDA(cudaGetDevice(&dev));
  QG_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  cudaFuncAttributes fa{};
  QG_CUDA(cudaFuncGetAttributes(&fa, kern));
  QG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes));
  done.push_back(key);
}

void launch_engine(Handle &H, const Mats &M, bool jvp, cudaStream_t st) {
  Workspace &W = H.ws;
  EngArgs a{};
  a.st = W.st;
  a.u = W.u; a.v = W.v; a.h = W.h; a.hb = W.hb; a.x = W.x;
  a.dp0 = jvp ? W.dpv : nullptr;
  a.c16P = H.c16P; a.c16AT = H.c16AT; a.c16A = H.c16A;
  a.blob = H.eng_blob;
  a.bl = engine_blob_layout(H);
  a.next = W.d_claim;
  a.B = H.B;
  engine_offsets(H, a.bl.bmax, &a);
  a.res_cap = H.eng_res_cap;
  const int nt = engine_threads();
  const size_t smem = (size_t)a.o_blob + a.bl.stride + (size_t)a.res_cap * 10;
  const int cfg = engine_cfg();
  auto kern = cfg == 2 ? (jvp ? k_engine<STEP_F, STEP_FT, 512, 2> : k_engine<STEP_FT, STEP_F, 512, 2>)
              : cfg == 1 ? (jvp ? k_engine<STEP_F, STEP_FT, 512, 1> : k_engine<STEP_FT, STEP_F, 512, 1>)
                         : (jvp ? k_engine<STEP_F, STEP_FT, 1024, 1> : k_engine<STEP_FT, STEP_F, 1024, 1>);
  // the attribute is per function and process-wide: raise it once to the
  // opt-in maximum (per-handle sizes set from concurrent host threads would
  // race each other's launches)
  set_max_dynamic_smem(kern);
  int dev = 0, nsm = 0;
  QG_CUDA(cudaGetDevice(&dev));
  QG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  const int grid = std::max(1, std::min(H.B, nsm * engine_ctas_per_sm()));
  QG_CUDA(cudaMemsetAsync(W.d_claim, 0, sizeof(int), st));
  static const bool want_prof = std::getenv("QG_ENG_PROF") != nullptr;
  if (want_prof) {
    if (!H.eng_prof) H.eng_prof = dev_alloc<unsigned long long>(10);
    QG_CUDA(cudaMemsetAsync(H.eng_prof, 0, 10 * sizeof(unsigned long long), st));
    a.prof = H.eng_prof;
  }
  kern<<<grid, nt, smem, st>>>(M, a);
  QG_LAUNCHED();
  if (want_prof) {
    unsigned long long h[10];
    QG_CUDA(cudaMemcpyAsync(h, H.eng_prof, sizeof(h), cudaMemcpyDeviceToHost, st));
    QG_CUDA(cudaStreamSynchronize(st));
    const double it = (double)std::max<unsigned long long>(h[5], 1);
    std::fprintf(stderr, "[qg engine] grid %d x %d thr, smem %zu B, res_cap %d | cycles/iter: A_u %.0f B_u %.0f "
                 "A_v %.0f B_v %.0f | fin %.0f x2, spmv(warp 1) %.0f x2 | F' epilogue rows %.0f, F' cone blocks %.0f | "
                 "setup/problem %.0f | iters %llu\n", grid, nt, smem, a.res_cap, h[1] / it, h[2] / it, h[3] / it,
                 h[4] / it, h[6] / it / 2, h[7] / it / 2, h[8] / it, h[9] / it, h[0] / (double)H.B, h[5]);
  }
}

}  // namespace qg
