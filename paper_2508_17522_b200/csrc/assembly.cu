// One-shot kernels around the LSMR solve: embedding preparation, the JVP
// right-hand side, the D phi / D phi' maps, the VJP data-space gradient on
// the sparsity patterns of P and A, and the KKT pre-check.
//
// References: embed (solution_map.py:170-179), dthetaq_apply
// (embedding.py:265-292), dphi_apply / dphi_adjoint (solution_map.py:206-260),
// dthetaq_adjoint + scaled (embedding.py:295-334, 151-159), check_solution
// (solution_map.py:263-288).
#include "ops_dev.cuh"
#include "operator.h"

namespace qg {

namespace {

__device__ __forceinline__ Unit unit_of(const Mats &M, bool &isx) {
  isx = (int)blockIdx.x < M.nxu;
  return isx ? M.xu[blockIdx.x] : M.yu[blockIdx.x - M.nxu];
}

__device__ __forceinline__ void write_slots(double (&acc)[kSlots], double *red, double *part) {
  double tot[kSlots];
  cta_sum_slots(acc, red, tot);
  if (threadIdx.x == 0)
#pragma unroll
    for (int k = 0; k < kSlots; ++k) part[(size_t)blockIdx.x * kSlots + k] = tot[k];
}

// rhs = -D_theta Q(u)[dtheta] / |z_N|, u = (xbar, ybar, tau).
// Row-partitioned handles run it twice around the exchange (XMode): X_PARTIAL
// writes this rank's dA_r' ybar to xred, X_FINISH completes the X rows.
__global__ void __launch_bounds__(kThreads) k_jvp_rhs(Mats M, PertDev d, double *u, double *part, int xmode,
                                                      double *xred) {
  __shared__ double red[kWarps * kSlots];
  bool isx;
  const Unit un = unit_of(M, isx);
  const Embed E = M.emb[un.prob];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int G = un.lanes, lg = lane & (G - 1), gpw = 32 / G;
  double acc[kSlots] = {0, 0, 0, 0};
  for (int base = un.row0 + warp * gpw; base < un.row1; base += kWarps * gpw) {
    const int r = base + lane / G;
    const bool valid = r < un.row1;
    if (isx && xmode == X_PARTIAL) {
      double s2 = valid ? row_dot(d.dAT_rp, d.dAT_col, d.dAT_val, M.ybar, r, lg, G) : 0.0;
      s2 = gsum(s2, G);
      if (valid && lg == 0) xred[r] = s2;
    } else if (isx) {
      double s1 = valid ? row_dot(d.dP_rp, d.dP_col, d.dP_val, M.xbar, r, lg, G) : 0.0;
      double s2 = (valid && xmode == X_FULL) ? row_dot(d.dAT_rp, d.dAT_col, d.dAT_val, M.ybar, r, lg, G) : 0.0;
      s1 = gsum(s1, G);
      s2 = gsum(s2, G);
      if (valid && xmode == X_FINISH) s2 = xred[r];
      if (valid && lg == 0) {
        const double out = (s1 + s2) + E.tau * d.dq[r];
        const double rhs = (-out) / fabs(E.zN);
        u[r] = rhs;
        acc[0] += M.xbar[r] * s1;
        acc[1] += d.dq[r] * M.xbar[r];
        acc[2] += rhs * rhs;
      }
    } else {
      double s = valid ? row_dot(d.dA_rp, d.dA_col, d.dA_val, M.xbar, r, lg, G) : 0.0;
      s = gsum(s, G);
      if (valid && lg == 0) {
        const double out = (-s) + E.tau * d.db[r];
        const double rhs = (-out) / fabs(E.zN);
        u[M.NX + r] = rhs;
        acc[0] += d.db[r] * M.ybar[r];
        acc[2] += rhs * rhs;
      }
    }
  }
  if (isx && xmode == X_PARTIAL) return;  // CTA-uniform: X slots come from X_FINISH
  if (isx && !M.x_owner)
#pragma unroll
    for (int k = 0; k < kSlots; ++k) acc[k] = 0.0;
  write_slots(acc, red, part);
}

// rhs = -dz with dz = (dx, D Pi(dy + ds) - ds, -x'dx - y'dy - s'ds).
__global__ void __launch_bounds__(kThreads) k_vjp_rhs(Mats M, const double *dx, const double *dy, const double *ds,
                                                      const double *dpi, double *u, double *part) {
  __shared__ double red[kWarps * kSlots];
  bool isx;
  const Unit un = unit_of(M, isx);
  double acc[kSlots] = {0, 0, 0, 0};
  for (int r = un.row0 + threadIdx.x; r < un.row1; r += blockDim.x) {
    if (isx) {
      const double v = -dx[r];
      u[r] = v;
      acc[0] += M.xbar[r] * dx[r];
      acc[2] += v * v;
    } else {
      const double v = -(dpi[r] - ds[r]);
      u[M.NX + r] = v;
      acc[0] += M.ybar[r] * dy[r];
      acc[1] += M.sbar[r] * ds[r];
      acc[2] += v * v;
    }
  }
  if (isx && !M.x_owner)
#pragma unroll
    for (int k = 0; k < kSlots; ++k) acc[k] = 0.0;
  write_slots(acc, red, part);
}

__global__ void k_add(const double *a, const double *b, double *out, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = a[i] + b[i];
}

__global__ void k_gather_vals(const int32_t *perm, const double *src, double *dst, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[perm[i]];
}

// dx = dz1 - dzN x ; dy = D Pi dz_mid - dzN y ; ds = (D Pi dz_mid - dz_mid) - dzN s
__global__ void __launch_bounds__(kThreads) k_dphi(Mats M, const double *dz, const double *dpi, double *dx,
                                                   double *dy, double *ds) {
  bool isx;
  const Unit un = unit_of(M, isx);
  const double dzN = dz[M.NX + M.NY + un.prob];
  for (int r = un.row0 + threadIdx.x; r < un.row1; r += blockDim.x) {
    if (isx) {
      dx[r] = dz[r] - dzN * M.xbar[r];
    } else {
      const double dm = dpi[r];
      dy[r] = dm - dzN * M.ybar[r];
      ds[r] = (dm - dz[M.NX + r]) - dzN * M.sbar[r];
    }
  }
}

// Data-space adjoint on the stored entries (embedding.py:321-333), times
// 1/|z_N| (embedding.py:151-159).  dP is emitted per column c of P's CSC
// structure; entry (r, c) and (c, r) use the same commuted products so dP
// stays exactly symmetric (no FMA contraction: __dmul_rn / __dadd_rn).
__global__ void __launch_bounds__(kThreads) k_vjp_grad(Mats M, const int32_t *Pc_rp, const int32_t *Pc_col,
                                                       const double *w, double *dP, double *dA, double *dq,
                                                       double *db) {
  bool isx;
  const Unit un = unit_of(M, isx);
  const Embed E = M.emb[un.prob];
  const double a = 1.0 / fabs(E.zN);
  const double wN = w[M.NX + M.NY + un.prob];
  const double wt = wN / E.tau;
  const double *x = M.xbar, *w1 = w, *w2 = w + M.NX;
  if (isx) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int c = un.row0 + warp; c < un.row1; c += kWarps) {
      const double xc = x[c], w1c = w1[c];
      for (int k = Pc_rp[c] + lane; k < Pc_rp[c + 1]; k += 32) {
        const int r = Pc_col[k];
        const double t1 = __dmul_rn(w1[r], xc), t2 = __dmul_rn(x[r], w1c);
        const double pv = __dsub_rn(__dmul_rn(0.5, __dadd_rn(t1, t2)), __dmul_rn(wt, __dmul_rn(x[r], xc)));
        dP[k] = __dmul_rn(a, pv);
      }
      for (int k = M.AT_rp[c] + lane; k < M.AT_rp[c + 1]; k += 32) {
        const int r = M.AT_col[k];
        const double av = __dsub_rn(__dmul_rn(M.ybar[r], w1c), __dmul_rn(w2[r], xc));
        dA[k] = __dmul_rn(a, av);
      }
      if (lane == 0) dq[c] = __dmul_rn(a, __dsub_rn(__dmul_rn(E.tau, w1c), __dmul_rn(wN, xc)));
    }
  } else {
    for (int r = un.row0 + threadIdx.x; r < un.row1; r += blockDim.x)
      db[r] = __dmul_rn(a, __dsub_rn(__dmul_rn(E.tau, w2[r]), __dmul_rn(wN, M.ybar[r])));
  }
}

__global__ void k_embed_prep(const double *y, const double *s, double *zmid, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) zmid[i] = y[i] - s[i];
}

// P xbar and the partials of xbar' P xbar (X units only).
__global__ void __launch_bounds__(kThreads) k_pxbar(Mats M, double *Pxbar, double *part) {
  __shared__ double red[kWarps * kSlots];
  const Unit un = M.xu[blockIdx.x];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int G = un.lanes, lg = lane & (G - 1), gpw = 32 / G;
  double acc[kSlots] = {0, 0, 0, 0};
  for (int base = un.row0 + warp * gpw; base < un.row1; base += kWarps * gpw) {
    const int r = base + lane / G;
    const bool valid = r < un.row1;
    double s = valid ? row_dot(M.P_rp, M.P_col, M.P_val, M.xbar, r, lg, G) : 0.0;
    s = gsum(s, G);
    if (valid && lg == 0) {
      Pxbar[r] = s;
      acc[0] += M.xbar[r] * s;
    }
  }
  write_slots(acc, red, part);
}

// zT: the points' T coordinates (B values), or null for embed()'s z_N = 1.
__global__ void k_embed_fin(Mats M, const double *part, Embed *emb, int B, const double *zT) {
  const int p = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (p >= B) return;
  double s = 0.0;
  for (int64_t k = M.xu_ptr[p] + lane; k < M.xu_ptr[p + 1]; k += 32) s += part[k * kSlots];
  s = warp_sum(s);
  if (lane == 0) {
    Embed E;
    E.zN = zT ? zT[p] : 1.0;          // embed(): last coordinate exactly 1
    E.tau = fmax(E.zN, 0.0);
    E.last = E.zN > 0.0 ? 1.0 : 0.0;
    E.xPx = s;
    emb[p] = E;
  }
}

// KKT residual partials: X: [stat^2], Y: [prim^2, s'y, sdist^2, ydist^2]
__global__ void __launch_bounds__(kThreads) k_kkt(Mats M, const double *x, const double *y, const double *s,
                                                  const double *projs, const double *projy, double *part) {
  __shared__ double red[kWarps * kSlots];
  bool isx;
  const Unit un = unit_of(M, isx);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int G = un.lanes, lg = lane & (G - 1), gpw = 32 / G;
  double acc[kSlots] = {0, 0, 0, 0};
  for (int base = un.row0 + warp * gpw; base < un.row1; base += kWarps * gpw) {
    const int r = base + lane / G;
    const bool valid = r < un.row1;
    if (isx) {
      double s1 = valid ? row_dot(M.P_rp, M.P_col, M.P_val, x, r, lg, G) : 0.0;
      double s2 = valid ? row_dot(M.AT_rp, M.AT_col, M.AT_val, y, r, lg, G) : 0.0;
      s1 = gsum(s1, G);
      s2 = gsum(s2, G);
      if (valid && lg == 0) {
        const double v = (s1 + s2) + M.q[r];
        acc[0] += v * v;
      }
    } else {
      double sa = valid ? row_dot(M.A_rp, M.A_col, M.A_val, x, r, lg, G) : 0.0;
      sa = gsum(sa, G);
      if (valid && lg == 0) {
        const double v = (sa + s[r]) - M.b[r];
        acc[0] += v * v;
        acc[1] += s[r] * y[r];
        const double ds = s[r] - projs[r], dy = y[r] - projy[r];
        acc[2] += ds * ds;
        acc[3] += dy * dy;
      }
    }
  }
  write_slots(acc, red, part);
}

__global__ void k_kkt_fin(Mats M, const double *part, double *report, int B) {
  const int p = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (p >= B) return;
  double sx = 0.0, sy[kSlots] = {0, 0, 0, 0};
  for (int64_t k = M.xu_ptr[p] + lane; k < M.xu_ptr[p + 1]; k += 32) sx += part[k * kSlots];
  for (int64_t k = M.yu_ptr[p] + lane; k < M.yu_ptr[p + 1]; k += 32)
    for (int j = 0; j < kSlots; ++j) sy[j] += part[(M.nxu + k) * kSlots + j];
  sx = warp_sum(sx);
  for (int j = 0; j < kSlots; ++j) sy[j] = warp_sum(sy[j]);
  if (lane == 0) {
    report[5 * p + 0] = sqrt(sy[0]);
    report[5 * p + 1] = sqrt(sx);
    report[5 * p + 2] = fabs(sy[1]);
    report[5 * p + 3] = sqrt(sy[2]);
    report[5 * p + 4] = sqrt(sy[3]);
  }
}

// plain CSR SpMV, one warp per row (qg_spmv_csc)
__global__ void k_csr_spmv(const int32_t *rp, const int32_t *col, const double *val, int64_t nrows,
                           const double *x, double *out) {
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= nrows) return;
  double s = 0.0;
  for (int k = rp[r] + lane; k < rp[r + 1]; k += 32) s += val[k] * x[col[k]];
  s = warp_sum(s);
  if (lane == 0) out[r] = s;
}

// Normalized residual N(z) = (Q(Pi z) - Pi z + z) / |z_N| at the handle's
// point (embedding.py:198-211, 374-396): X / Y rows here, T in k_residual_fin.
// Partials: X [.., q'x], Y [b'y].
__global__ void __launch_bounds__(kThreads) k_residual(Mats M, double *out, double *part) {
  __shared__ double red[kWarps * kSlots];
  bool isx;
  const Unit un = unit_of(M, isx);
  const Embed E = M.emb[un.prob];
  const double inv = 1.0 / fabs(E.zN);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int G = un.lanes, lg = lane & (G - 1), gpw = 32 / G;
  double acc[kSlots] = {0, 0, 0, 0};
  for (int base = un.row0 + warp * gpw; base < un.row1; base += kWarps * gpw) {
    const int r = base + lane / G;
    const bool valid = r < un.row1;
    if (isx) {
      double s = valid ? row_dot(M.AT_rp, M.AT_col, M.AT_val, M.ybar, r, lg, G) : 0.0;
      s = gsum(s, G);
      if (valid && lg == 0) {
        const double x = M.xbar[r];
        const double qx = (M.Pxbar[r] + s) + E.tau * M.q[r];
        out[r] = ((qx - x) + x) * inv;
        acc[1] += M.q[r] * x;
      }
    } else {
      double s = valid ? row_dot(M.A_rp, M.A_col, M.A_val, M.xbar, r, lg, G) : 0.0;
      s = gsum(s, G);
      if (valid && lg == 0) {
        const double qy = (-s) + E.tau * M.b[r];
        out[M.NX + r] = ((qy - M.ybar[r]) + M.dpi.zmid[r]) * inv;
        acc[0] += M.b[r] * M.ybar[r];
      }
    }
  }
  write_slots(acc, red, part);
}

__global__ void k_residual_fin(Mats M, const double *part, double *out, int B) {
  const int p = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (p >= B) return;
  double qx = 0.0, by = 0.0;
  for (int64_t k = M.xu_ptr[p] + lane; k < M.xu_ptr[p + 1]; k += 32) qx += part[k * kSlots + 1];
  for (int64_t k = M.yu_ptr[p] + lane; k < M.yu_ptr[p + 1]; k += 32) by += part[(M.nxu + k) * kSlots];
  qx = warp_sum(qx);
  by = warp_sum(by);
  if (lane == 0) {
    const Embed E = M.emb[p];
    const double qn = ((-E.xPx) / E.tau - qx) - by;
    out[M.NX + M.NY + p] = ((qn - E.tau) + E.zN) / fabs(E.zN);
  }
}

// LSMR right-hand side from a given vector (X / Y rows; T is set by the
// PH_RHS finalize): u = r, ||u_XY||^2 partials in slot 2.
__global__ void __launch_bounds__(kThreads) k_vec_rhs(Mats M, const double *r, double *u, double *part) {
  __shared__ double red[kWarps * kSlots];
  bool isx;
  const Unit un = unit_of(M, isx);
  const int64_t off = isx ? 0 : M.NX;
  double acc[kSlots] = {0, 0, 0, 0};
  for (int64_t i = off + un.row0 + threadIdx.x; i < off + un.row1; i += blockDim.x) {
    const double v = r[i];
    u[i] = v;
    acc[2] += v * v;
  }
  write_slots(acc, red, part);
}

inline unsigned nb(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

}  // namespace

static unsigned units_grid(const Handle &H) { return (unsigned)(H.nxu() + H.nyu()); }

void launch_jvp_rhs(const Handle &H, const Mats &M, const PertDev &d, double *u, double *part, cudaStream_t st) {
  if (!H.comm) {
    if (!units_grid(H)) return;
    k_jvp_rhs<<<units_grid(H), kThreads, 0, st>>>(M, d, u, part, X_FULL, nullptr);
    QG_LAUNCHED();
    return;
  }
  if (units_grid(H)) {
    k_jvp_rhs<<<units_grid(H), kThreads, 0, st>>>(M, d, u, part, X_PARTIAL, H.xred);
    QG_LAUNCHED();
  }
  H.comm->allreduce(H.xred, H.NX, st);  // every rank, even with no rows of its own
  if (H.nxu()) {
    k_jvp_rhs<<<H.nxu(), kThreads, 0, st>>>(M, d, u, part, X_FINISH, H.xred);
    QG_LAUNCHED();
  }
}

void launch_vjp_rhs(const Handle &H, const Mats &M, const double *dx, const double *dy, const double *ds,
                    const double *dpi_dyds, double *u, double *part, cudaStream_t st) {
  if (!units_grid(H)) return;
  k_vjp_rhs<<<units_grid(H), kThreads, 0, st>>>(M, dx, dy, ds, dpi_dyds, u, part);
  QG_LAUNCHED();
}

void launch_add(const Handle &, const double *a, const double *b, double *out, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  k_add<<<nb(n), 256, 0, st>>>(a, b, out, n);
  QG_LAUNCHED();
}

void launch_gather(const int32_t *perm, const double *src, double *dst, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  k_gather_vals<<<nb(n), 256, 0, st>>>(perm, src, dst, n);
  QG_LAUNCHED();
}

void launch_dphi(const Handle &H, const Mats &M, const double *dz, const double *dpi_dz, double *dx, double *dy,
                 double *ds, cudaStream_t st) {
  if (!units_grid(H)) return;
  k_dphi<<<units_grid(H), kThreads, 0, st>>>(M, dz, dpi_dz, dx, dy, ds);
  QG_LAUNCHED();
}

void launch_vjp_grad(const Handle &H, const Mats &M, const double *w, double *dP, double *dA, double *dq,
                     double *db, cudaStream_t st) {
  if (!units_grid(H)) return;
  k_vjp_grad<<<units_grid(H), kThreads, 0, st>>>(M, H.Pc.rp, H.Pc.col, w, dP, dA, dq, db);
  QG_LAUNCHED();
}

void launch_embed_prep(const Handle &H, const double *, const double *y, const double *s, double *zmid,
                       cudaStream_t st) {
  if (H.NY <= 0) return;
  k_embed_prep<<<nb(H.NY), 256, 0, st>>>(y, s, zmid, H.NY);
  QG_LAUNCHED();
}

void launch_embed_consts(const Handle &H, const Mats &M, double *part, cudaStream_t st, const double *zT) {
  if (H.nxu() > 0) {
    k_pxbar<<<H.nxu(), kThreads, 0, st>>>(M, H.Pxbar, part);
    QG_LAUNCHED();
  }
  k_embed_fin<<<nb((int64_t)H.B * 32), 256, 0, st>>>(M, part, H.emb, H.B, zT);
  QG_LAUNCHED();
}

void launch_residual(const Handle &H, const Mats &M, double *out, double *part, cudaStream_t st) {
  if (units_grid(H)) {
    k_residual<<<units_grid(H), kThreads, 0, st>>>(M, out, part);
    QG_LAUNCHED();
  }
  k_residual_fin<<<nb((int64_t)H.B * 32), 256, 0, st>>>(M, part, out, H.B);
  QG_LAUNCHED();
}

void launch_vec_rhs(const Handle &H, const Mats &M, const double *r, double *u, double *part, cudaStream_t st) {
  if (!units_grid(H)) return;
  k_vec_rhs<<<units_grid(H), kThreads, 0, st>>>(M, r, u, part);
  QG_LAUNCHED();
}

void launch_csr_spmv(const int32_t *rp, const int32_t *col, const double *val, int64_t nrows, const double *x,
                     double *out, cudaStream_t st) {
  if (nrows <= 0) return;
  k_csr_spmv<<<nb(nrows * 32), 256, 0, st>>>(rp, col, val, nrows, x, out);
  QG_LAUNCHED();
}

void launch_kkt(const Handle &H, const Mats &M, const double *x, const double *y, const double *s,
                const double *projs, const double *projy, double *part, double *report_dev, cudaStream_t st) {
  if (units_grid(H)) {
    k_kkt<<<units_grid(H), kThreads, 0, st>>>(M, x, y, s, projs, projy, part);
    QG_LAUNCHED();
  }
  k_kkt_fin<<<nb((int64_t)H.B * 32), 256, 0, st>>>(M, part, report_dev, H.B);
  QG_LAUNCHED();
}

}  // namespace qg
