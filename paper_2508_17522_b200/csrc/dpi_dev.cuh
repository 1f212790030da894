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

// PSD applier (cones.py:791-793): out = svec(V (B o (V' smat(in) V)) V'),
// evaluated as V' (S V).  CTA-wide; smem holds 4 padded (d x (d+1))
// matrices (leading dimension d+1 breaks the column-stride bank conflicts).
// V, B column-major (d x d) in global.
// Matrices are padded to dp = d rounded up to 4 (zero rows / columns) so the
// register tiles (up to 4 wide) never leave the arrays; V'T V and the final product are
// symmetric, so only their lower triangles are computed (3 d^3 instead of
// 4 d^3 FMAs; c4: 512 blocks of order 32 per F' step).
static __device__ __forceinline__ int psd_pad(int d) { return (d + 3) & ~3; }
// Register tile of the PSD products.  c4 F' (512 PSD(32) blocks): 2x2 0.137
// ms, 4x2 0.145 ms, 4x4 0.325 ms (the F' step runs at 40 registers).
#ifndef PSD_TI
#define PSD_TI 2
#endif
#ifndef PSD_TJ
#define PSD_TJ 2
#endif

static __device__ void psd_apply_cta(const double *Vg, const double *Bg, int d, const double *in, double *out,
                                     double *sm) {
  const int dp = psd_pad(d), ld = dp + 1, sz = dp * ld;
  double *V = sm, *S = sm + sz, *T = sm + 2 * sz, *W = sm + 3 * sz;
  for (int idx = threadIdx.x; idx < dp * dp; idx += blockDim.x) {
    const int i = idx % dp, j = idx / dp;
    const bool in_d = i < d && j < d;
    V[i + j * ld] = in_d ? Vg[i + j * d] : 0.0;
    double s = 0.0;
    if (in_d) {
      const int a = i >= j ? i : j, b = i >= j ? j : i;
      const double v = in[svec_index(a, b, d)];
      s = (a == b) ? v : v / kSqrt2;
    }
    S[i + j * ld] = s;
    T[i + j * ld] = 0.0;
    W[i + j * ld] = 0.0;
  }
  __syncthreads();
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
                   if (i >= j) out[svec_index(i, j, d)] = (i == j) ? c : c * kSqrt2;
                 });
  __syncthreads();
}

// Apply D Pi to the unit's rows.  in/out are indexed by (row - unit.row0);
// they may live in global memory (written by this CTA before a barrier).
static __device__ void dpi_apply_unit(const DpiView &dv, const Unit &u, const double *in, double *out, double *sm) {
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
    psd_apply_cta(V, V + d * d, d, in + (b.row - u.row0), out + (b.row - u.row0), sm);
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
