// Blockwise projection-derivative application for one work unit (CTA-wide),
// and the CTA-level PSD Jacobi eigensolver used by the preparation kernels.
//
// Reference semantics: ConeDerivative.matvec (cones.py:886-906) with the
// per-kind appliers of cones.py:740-795, 837-883; svec layout cones.py:176-202.
#pragma once

#include "cones_dev.cuh"
#include "qg_common.cuh"

namespace qg {

constexpr int kMaxPsdOrder = 64;
constexpr double kSqrt2 = 1.4142135623730951;

__device__ __forceinline__ int svec_index(int i, int j, int d) {  // i >= j
  return j * d - (j * (j - 1)) / 2 + (i - j);
}

// Elementwise (zero / nonneg) derivative weight (cones.py:837-848, 867-872).
__device__ __forceinline__ double elem_weight(int kind, int dual, double z) {
  if (kind == QG_CONE_ZERO) return dual ? 1.0 : 0.0;
  return z > 0.0 ? 1.0 : (z == 0.0 ? 0.5 : 0.0);
}

// SOC applier (cones.py:740-764) executed by one warp for one block.
__device__ __forceinline__ void soc_apply_warp(const double *zb, int dim, double nu, int code,
                                               const double *in, double *out) {
  const int lane = threadIdx.x & 31;
  if (code != 3) {
    const double f = (code == 0) ? 0.0 : (code == 1 ? 1.0 : 0.5);
    for (int i = lane; i < dim; i += 32) out[i] = (code == 0) ? 0.0 : (code == 1 ? in[i] : f * in[i]);
    return;
  }
  const double t = zb[0], dt = in[0];
  double part = 0.0;
  for (int i = 1 + lane; i < dim; i += 32) part += zb[i] * in[i];
  const double udu = warp_sum(part);
  const double two_nu = 2.0 * nu;
  const double c = (t / (nu * nu)) * udu;
  const double tn = t + nu;
  for (int i = lane; i < dim; i += 32) {
    double v;
    if (i == 0) v = nu * dt + udu;
    else v = (zb[i] * dt + tn * in[i]) - c * zb[i];
    out[i] = v / two_nu;
  }
}

// Entry i of the SOC derivative applied to dt (cones.py:740-764) for a block
// with t0 = z[0], nu = ||z[1:]||, udu = z[1:]'dt[1:], di = dt[i], zi = z[i];
// code: 0 zero map, 1 identity, 2 half, 3 formula.
__device__ __forceinline__ double soc_entry(int code, int i, double nu, double t0, double zi, double di,
                                            double dt, double udu) {
  if (code == 0) return 0.0;
  if (code == 1) return di;
  if (code == 2) return 0.5 * di;
  const double two_nu = 2.0 * nu;
  if (i == 0) return (nu * dt + udu) / two_nu;
  const double c = (t0 / (nu * nu)) * udu;
  return ((zi * dt + (t0 + nu) * di) - c * zi) / two_nu;
}

// d x d product C = sum_k a(i,k) b(k,j) with TI x TJ register tiles per
// thread (TI + TJ shared-memory loads per TI*TJ FMAs); out(i, j, c) stores.
// lower = true: only tiles touching the lower triangle (j <= i) are computed
// (symmetric results / lower-triangle consumers).  a/b must return 0 for
// indices >= d (the padded operand matrices are zero-filled).
template <int TI, int TJ, class FA, class FB, class FO>
__device__ __forceinline__ void mm_tiles(int d, bool lower, FA a, FB b, FO out) {
  const int ni = (d + TI - 1) / TI, nj = (d + TJ - 1) / TJ;
  for (int t = threadIdx.x; t < ni * nj; t += blockDim.x) {
    const int i0 = TI * (t % ni), j0 = TJ * (t / ni);
    if (lower && j0 > i0 + TI - 1) continue;
    double c[TI][TJ];
#pragma unroll
    for (int x = 0; x < TI; ++x)
#pragma unroll
      for (int y = 0; y < TJ; ++y) c[x][y] = 0.0;
    for (int k = 0; k < d; ++k) {
      double av[TI], bv[TJ];
#pragma unroll
      for (int x = 0; x < TI; ++x) av[x] = a(i0 + x, k);
#pragma unroll
      for (int y = 0; y < TJ; ++y) bv[y] = b(k, j0 + y);
#pragma unroll
      for (int x = 0; x < TI; ++x)
#pragma unroll
        for (int y = 0; y < TJ; ++y) c[x][y] += av[x] * bv[y];
    }
#pragma unroll
    for (int x = 0; x < TI; ++x)
#pragma unroll
      for (int y = 0; y < TJ; ++y)
        if (i0 + x < d && j0 + y < d) out(i0 + x, j0 + y, c[x][y]);
  }
}

// d x d product on the FP64 tensor cores (mma.sync m8n8k4 f64): operands in
// shared memory, element (i, k) of A at A[i*ai + k*ak], (k, j) of B at
// B[k*bk + j*bj], zero-padded to nt*8 rows / columns.  Each warp owns up to
// four 8x8 output tiles at a time (independent accumulator chains); lower =
// only tiles with tj <= ti.  out(i, j, c) for every element of the owned
// tiles, padding included (the callers filter).  Fragment layouts (PTX ISA,
// m8n8k4 .f64): A[lane/4][lane%4], B[lane%4][lane/4], C[lane/4][2*(lane%4)+e].
__device__ __forceinline__ void dmma_8x8x4(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int TPW = 4, class FO>
__device__ __forceinline__ void mm_dmma(int nt, bool lower, const double *A, int ai, int ak, const double *B, int bk,
                                        int bj, FO out) {
  // TPW: output tiles per warp and pass (independent accumulator chains);
  // 128-thread CTAs use 4 (16 tiles of a 32 x 32 product in one pass), the
  // 256-thread PSD step 2 (one pass over 8 warps, half the chain per warp)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (int)(blockDim.x >> 5);
  const int fr = lane >> 2, fc = lane & 3;
  const int ntile = lower ? nt * (nt + 1) / 2 : nt * nt;
  for (int t0 = warp * TPW; t0 < ntile; t0 += nw * TPW) {
    int ti[TPW], tj[TPW];
    double c0[TPW], c1[TPW];
#pragma unroll
    for (int q = 0; q < TPW; ++q) {
      int t = t0 + q, i = 0;
      if (lower) {
        while (t > i) t -= ++i;  // row-major lower-triangle enumeration
      } else {
        i = t % nt;
        t /= nt;
      }
      ti[q] = t0 + q < ntile ? i : -1;
      tj[q] = t;
      c0[q] = c1[q] = 0.0;
    }
    for (int k = 0; k < nt * 8; k += 4) {
#pragma unroll
      for (int q = 0; q < TPW; ++q)
        if (ti[q] >= 0) {
          const double a = A[(ti[q] * 8 + fr) * ai + (k + fc) * ak];
          const double b = B[(k + fc) * bk + (tj[q] * 8 + fr) * bj];
          dmma_8x8x4(c0[q], c1[q], a, b);
        }
    }
#pragma unroll
    for (int q = 0; q < TPW; ++q)
      if (ti[q] >= 0) {
        out(ti[q] * 8 + fr, tj[q] * 8 + 2 * fc, c0[q]);
        out(ti[q] * 8 + fr, tj[q] * 8 + 2 * fc + 1, c1[q]);
      }
  }
}

// PSD applier (cones.py:791-793): out = svec(V (B o (V' smat(in) V)) V'),
// evaluated as V' (S V).  CTA-wide; smem holds 4 padded (d x (d+1))
// matrices (leading dimension d+1 breaks the column-stride bank conflicts).
// V, B column-major (d x d) in global.
// Matrices are padded to dp = d rounded up to 4 (zero rows / columns) so the
// register tiles (up to 4 wide) never leave the arrays; V'T V and the final product are
// symmetric, so only their lower triangles are computed (3 d^3 instead of
// 4 d^3 FMAs; c4: 512 blocks of order 32 per F' step).
// The products run on the FP64 tensor cores (mm_dmma; matrices padded to a
// multiple of 8, leading dimension dp + 4 = 4 mod 16 doubles: both fragment
// orientations hit every bank pair exactly twice).  QG_PSD_DMMA=0 builds the
// CUDA-core register-tile path instead (padding 4, leading dimension dp + 1).
// c4 F' (512 PSD(32) blocks per step): CUDA-core 2x2 tiles 0.137 ms (4x2
// 0.145, 4x4 0.325 at 40 registers).
#ifndef QG_PSD_DMMA
#define QG_PSD_DMMA 1
#endif
#if QG_PSD_DMMA
static __device__ __forceinline__ int psd_pad(int d) { return (d + 7) & ~7; }
static __device__ __forceinline__ int psd_ld(int dp) { return dp + 4; }
#else
static __device__ __forceinline__ int psd_pad(int d) { return (d + 3) & ~3; }
static __device__ __forceinline__ int psd_ld(int dp) { return dp + 1; }
#endif
#ifndef PSD_TI
#define PSD_TI 2
#endif
#ifndef PSD_TJ
#define PSD_TJ 2
#endif

// Asynchronous copy of a PSD unit's eigenvector matrix V (preparation-time
// data) into its shared-memory slot, issued at the start of the F' step so
// the load latency hides behind the unit's SpMV pass; psd_apply_cta(...,
// have_v = true) then waits for it.  No-op for other units.
static __device__ __forceinline__ void psd_prefetch_v(const DpiView &dv, const Unit &u, double *sm) {
  if (u.cls != CLS_PSD) return;
  const BlockInfo b = dv.blk[u.blk0];
  const int d = b.order, dp = psd_pad(d), ld = psd_ld(dp);
  const double *Vg = dv.psd + b.param;
  for (int idx = threadIdx.x; idx < dp * dp; idx += blockDim.x) {
    const int i = idx % dp, j = idx / dp;
    double *dst = sm + i + j * ld;
    if (i < d && j < d) {
      const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(Vg + i + j * d) : "memory");
    } else {
      *dst = 0.0;
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// Shared memory: V, S and T (W reuses S, dead after the first product:
// 3 instead of 4 matrices -> more CTAs per SM for the whole F' step).
// have_v: V is already in sm from the previous apply of the same block (the
// F' epilogue applies D Pi twice per block; no product writes V).
// Core with svec accessors: in(k) returns entry k of the input, out(k, v)
// stores entry k of the result (global or shared memory); TPW as mm_dmma.
template <int TPW, class FI, class FO>
static __device__ void psd_apply_core(const double *Vg, const double *Bg, int d, FI in, FO out, double *sm,
                                      bool have_v) {
  const int dp = psd_pad(d), ld = psd_ld(dp), sz = dp * ld;
  double *V = sm, *S = sm + sz, *T = sm + 2 * sz, *W = S;
  if (have_v) asm volatile("cp.async.wait_all;" ::: "memory");  // psd_prefetch_v (barrier below)
  for (int idx = threadIdx.x; idx < dp * dp; idx += blockDim.x) {
    const int i = idx % dp, j = idx / dp;
    const bool in_d = i < d && j < d;
    if (!have_v) V[i + j * ld] = in_d ? Vg[i + j * d] : 0.0;
    double s = 0.0;
    if (in_d) {
      const int a = i >= j ? i : j, b = i >= j ? j : i;
      const double v = in(svec_index(a, b, d));
      s = (a == b) ? v : v / kSqrt2;
    }
    S[i + j * ld] = s;
    T[i + j * ld] = 0.0;
  }
  __syncthreads();
#if QG_PSD_DMMA
  const int nt = dp >> 3;
  // T = S V ; W = (V' T) o B (lower, mirrored) ; T = V W ; out = svec(T V')
  // (padded rows / columns of every product are zero; only W and out filter)
  mm_dmma<TPW>(nt, false, S, 1, ld, V, 1, ld, [&](int i, int j, double c) { T[i + j * ld] = c; });
  __syncthreads();
  mm_dmma<TPW>(nt, true, V, ld, 1, T, 1, ld, [&](int i, int j, double c) {
    if (i >= j && i < d) {
      const double w = Bg[i + j * d] * c;
      W[i + j * ld] = w;
      W[j + i * ld] = w;
    }
  });
  __syncthreads();
  mm_dmma<TPW>(nt, false, V, 1, ld, W, 1, ld, [&](int i, int j, double c) { T[i + j * ld] = c; });
  __syncthreads();
  mm_dmma<TPW>(nt, true, T, 1, ld, V, ld, 1, [&](int i, int j, double c) {
    if (i >= j && i < d) out(svec_index(i, j, d), (i == j) ? c : c * kSqrt2);
  });
  __syncthreads();
#else
  // T = S V
  mm_tiles<PSD_TI, PSD_TJ>(d, false, [&](int i, int k) { return S[i + k * ld]; }, [&](int k, int j) { return V[k + j * ld]; },
                 [&](int i, int j, double c) { T[i + j * ld] = c; });
  __syncthreads();
  // W = (V' T) o B, symmetric: lower triangle computed, mirrored
  mm_tiles<PSD_TI, PSD_TJ>(d, true, [&](int i, int k) { return V[k + i * ld]; }, [&](int k, int j) { return T[k + j * ld]; },
                 [&](int i, int j, double c) {
                   if (i >= j) {
                     const double w = Bg[i + j * d] * c;
                     W[i + j * ld] = w;
                     W[j + i * ld] = w;
                   }
                 });
  __syncthreads();
  // T = V W
  mm_tiles<PSD_TI, PSD_TJ>(d, false, [&](int i, int k) { return V[i + k * ld]; }, [&](int k, int j) { return W[k + j * ld]; },
                 [&](int i, int j, double c) { T[i + j * ld] = c; });
  __syncthreads();
  // out = svec(T V') on the lower triangle
  mm_tiles<PSD_TI, PSD_TJ>(d, true, [&](int i, int k) { return T[i + k * ld]; }, [&](int k, int j) { return V[j + k * ld]; },
                 [&](int i, int j, double c) {
                   if (i >= j) out(svec_index(i, j, d), (i == j) ? c : c * kSqrt2);
                 });
  __syncthreads();
#endif
}

static __device__ void psd_apply_cta(const double *Vg, const double *Bg, int d, const double *in, double *out,
                                     double *sm, bool have_v = false) {
  psd_apply_core<4>(Vg, Bg, d, [&](int k) { return in[k]; }, [&](int k, double v) { out[k] = v; }, sm, have_v);
}

// Shared-memory words of psd_apply_core for order d (V, S = W, T).
static __host__ __device__ __forceinline__ int psd_core_words(int d) {
#if QG_PSD_DMMA
  const int dp = (d + 7) & ~7, ld = dp + 4;
#else
  const int dp = (d + 3) & ~3, ld = dp + 1;
#endif
  return 3 * dp * ld;
}

// Apply D Pi to the unit's rows.  in/out are indexed by (row - unit.row0);
// they may live in global memory (written by this CTA before a barrier).
static __device__ void dpi_apply_unit(const DpiView &dv, const Unit &u, const double *in, double *out, double *sm,
                                      bool have_v = false) {
  if (u.cls == CLS_ELEM) {
    const BlockInfo b = dv.blk[u.blk0];
    for (int r = u.row0 + threadIdx.x; r < u.row1; r += blockDim.x) {
      const int o = r - u.row0;
      out[o] = elem_weight(b.kind, dv.dual, dv.zmid[r]) * in[o];
    }
  } else if (u.cls == CLS_SOC) {
    const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int k = u.blk0 + warp; k < u.blk1; k += nw) {
      const BlockInfo b = dv.blk[k];
      const int o = b.row - u.row0;
      soc_apply_warp(dv.zmid + b.row, b.dim, dv.soc_nu[b.param], dv.soc_code[b.param], in + o, out + o);
    }
  } else if (u.cls == CLS_PSD) {
    const BlockInfo b = dv.blk[u.blk0];
    const double *V = dv.psd + b.param;
    const int d = b.order;
    psd_apply_cta(V, V + d * d, d, in + (b.row - u.row0), out + (b.row - u.row0), sm, have_v);
  } else {  // CLS_TRI
    for (int k = u.blk0 + (int)threadIdx.x; k < u.blk1; k += blockDim.x) {
      const BlockInfo b = dv.blk[k];
      const int o = b.row - u.row0;
      const double *D = dv.tri_D + 9 * b.param;
      double Dl[9], dd[3] = {in[o], in[o + 1], in[o + 2]}, oo[3];
#pragma unroll
      for (int i = 0; i < 9; ++i) Dl[i] = D[i];
      tri_apply(Dl, dv.tri_flip[b.param], dd, oo);
      out[o] = oo[0]; out[o + 1] = oo[1]; out[o + 2] = oo[2];
    }
  }
  __syncthreads();
}

// ------------------------------------------------ PSD Jacobi (CTA-wide) --
// Symmetric A (column major, d x d, in smem) -> eigenvalues lam[d] and
// eigenvectors V (columns) by parallel cyclic Jacobi with round-robin pair
// ordering.  Scratch: rot[2*32] doubles + pairs.
static __device__ void jacobi_eigh_cta(double *A, double *V, double *lam, int d, double *rot, int *flag) {
  const int dp = d + (d & 1);          // players (one dummy when d is odd)
  const int npair = dp / 2;
  for (int idx = threadIdx.x; idx < d * d; idx += blockDim.x) V[idx] = (idx % d == idx / d) ? 1.0 : 0.0;
  __shared__ double s_fro;
  if (threadIdx.x == 0) {
    double f = 0.0;
    for (int k = 0; k < d * d; ++k) f += A[k] * A[k];
    s_fro = sqrt(f);
  }
  __syncthreads();
  const double floor_abs = 1e-18 * s_fro;
  for (int sweep = 0; sweep < 40; ++sweep) {
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    for (int round = 0; round < dp - 1; ++round) {
      // rotation parameters, one thread per pair
      if ((int)threadIdx.x < npair) {
        const int k = threadIdx.x;
        auto player = [&](int pos) { return pos == 0 ? 0 : 1 + ((pos - 1 + round) % (dp - 1)); };
        int p = player(k), q = player(dp - 1 - k);
        if (p > q) { int t = p; p = q; q = t; }
        double c = 1.0, s = 0.0;
        if (q < d) {
          const double apq = A[p + q * d], app = A[p + p * d], aqq = A[q + q * d];
          const double thr = 2.220446049250313e-16 * sqrt(fabs(app * aqq));
          if (fabs(apq) > floor_abs && fabs(apq) > thr) {
            const double th = (aqq - app) / (2.0 * apq);
            const double t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
            c = 1.0 / sqrt(t * t + 1.0);
            s = t * c;
            *flag = 1;
          }
        }
        rot[4 * k + 0] = c; rot[4 * k + 1] = s;
        rot[4 * k + 2] = (double)p; rot[4 * k + 3] = (double)q;
      }
      __syncthreads();
      // rows: A <- J' A
      for (int idx = threadIdx.x; idx < npair * d; idx += blockDim.x) {
        const int k = idx / d, col = idx % d;
        const double c = rot[4 * k], s = rot[4 * k + 1];
        const int p = (int)rot[4 * k + 2], q = (int)rot[4 * k + 3];
        if (q >= d || s == 0.0) continue;
        const double ap = A[p + col * d], aq = A[q + col * d];
        A[p + col * d] = c * ap - s * aq;
        A[q + col * d] = s * ap + c * aq;
      }
      __syncthreads();
      // columns: A <- A J ; V <- V J
      for (int idx = threadIdx.x; idx < npair * d; idx += blockDim.x) {
        const int k = idx / d, row = idx % d;
        const double c = rot[4 * k], s = rot[4 * k + 1];
        const int p = (int)rot[4 * k + 2], q = (int)rot[4 * k + 3];
        if (q >= d || s == 0.0) continue;
        const double ap = A[row + p * d], aq = A[row + q * d];
        A[row + p * d] = c * ap - s * aq;
        A[row + q * d] = s * ap + c * aq;
        const double vp = V[row + p * d], vq = V[row + q * d];
        V[row + p * d] = c * vp - s * vq;
        V[row + q * d] = s * vp + c * vq;
      }
      __syncthreads();
    }
    const int any = *flag;
    __syncthreads();
    if (!any) break;
  }
  for (int i = threadIdx.x; i < d; i += blockDim.x) lam[i] = A[i + i * d];
  __syncthreads();
}

}  // namespace qg
