// Device cone calculus for the 3-dimensional families (exp, pow and their
// duals): projection and the dense 3x3 projection derivative, one thread per
// block.  Follows the reference's root finders and fixed generalized-Jacobian
// choices (reference pkg/src/conegrad/cones.py:209-722) so results agree to
// rounding; libm exp/pow differ from glibc by <= 2 ulp.
#pragma once

#include "qg_common.cuh"

namespace qg {

constexpr double kE = 2.718281828459045;  // np.e

// ------------------------------------------------------------ exponential --
__device__ __forceinline__ bool exp_in(double x, double y, double z) {   // cones.py:213
  if (y > 0.0) return y * exp(x / y) <= z;
  return y == 0.0 && x <= 0.0 && z >= 0.0;
}

__device__ __forceinline__ bool exp_in_polar(double x, double y, double z) {   // cones.py:222
  if (x > 0.0) return x * exp(y / x) <= -kE * z;
  return x == 0.0 && y <= 0.0 && z <= 0.0;
}

// h(rho), h'(rho) of the ratio equation (cones.py:231-261).
__device__ __forceinline__ void exp_h(const double p[3], double r, double &h, double &hp) {
  const double x = p[0], y = p[1], z = p[2];
  if (r <= 0.0) {
    const double e1 = exp(r), e2 = e1 * e1;
    const double a = (e1 == 0.0) ? 0.0 : z * e1 * (r * r - r + 1.0);
    const double ad = (e1 == 0.0) ? 0.0 : z * e1 * (r * r + r);
    h = x * (-1.0 - (1.0 - r) * e2) + y * (r + e2) - a;
    hp = x * e2 * (2.0 * r - 1.0) + y * (1.0 + 2.0 * e2) - ad;
  } else {
    const double e1 = exp(-r), e2 = e1 * e1;
    const double a = (e1 == 0.0) ? 0.0 : z * e1 * (r * r - r + 1.0);
    const double ad = (e1 == 0.0) ? 0.0 : z * e1 * (r * r - 3.0 * r + 2.0);
    h = x * (r - 1.0 - e2) + y * (1.0 + r * e2) - a;
    hp = x * (1.0 + 2.0 * e2) + y * e2 * (1.0 - 2.0 * r) + ad;
  }
}

__device__ __forceinline__ double exp_h0(const double p[3], double r) {
  double h, hp;
  exp_h(p, r, h, hp);
  return h;
}

// Candidate projection for a ratio root (cones.py:264-294).
__device__ __forceinline__ void exp_candidate(const double p[3], double r, double ph[3], double &yh,
                                              double &mu, double &mue) {
  const double x = p[0], y = p[1], z = p[2];
  if (fabs(r) > 1e150) {
    yh = x / r;
    ph[0] = x; ph[1] = yh; ph[2] = 0.0;
    mu = (r < 0) ? -z : 0.0;
    mue = 0.0;
    return;
  }
  double zh;
  if (r <= 0.0) {
    const double e1 = exp(r);
    const double den = r * r + 1.0 + e1 * e1;
    yh = (r * x + y + z * e1) / den;
    zh = yh * e1;
    const double om = 1.0 - r;
    const double dden = e1 * e1 * (1.0 + om * om) + 1.0;
    mu = (x * e1 + y * (1.0 - r) * e1 - z) / dden;
    mue = mu * e1;
  } else {
    const double e1 = exp(-r), e2 = e1 * e1;
    const double den = (r * r + 1.0) * e2 + 1.0;
    yh = ((r * x + y) * e2 + z * e1) / den;
    zh = ((r * x + y) * e1 + z) / den;
    const double om = 1.0 - r;
    const double dden = 1.0 + om * om + e2;
    mu = ((x + y * (1.0 - r)) * e1 - z * e2) / dden;
    mue = ((x + y * (1.0 - r)) - z * e1) / dden;
  }
  ph[0] = r * yh; ph[1] = yh; ph[2] = zh;
}

__device__ __forceinline__ double exp_worst_res(const double p[3], double r, const double ph[3],
                                                double mu, double mue) {   // cones.py:297-308
  const double r1 = fabs(ph[0] - p[0] + mue);
  const double r2 = fabs(ph[1] - p[1] + mue * (1.0 - r));
  const double r3 = fabs(ph[2] - p[2] - mu);
  const double r4 = (fabs(r) > 700.0) ? 0.0 : fabs(ph[1] * exp(r) - ph[2]);
  return fmax(fmax(r1, r2), fmax(r3, r4));
}

static __device__ double exp_newton(const double p[3], double lo, double hi, double flo) {   // cones.py:311-331
  double r = 0.5 * (lo + hi);
  for (int it = 0; it < 200; ++it) {
    double f, fp;
    exp_h(p, r, f, fp);
    if (f == 0.0) return r;
    if ((f > 0.0) == (flo > 0.0)) { lo = r; flo = f; } else { hi = r; }
    double nx = (fp != 0.0) ? r - f / fp : 0.5 * (lo + hi);
    if (!(lo < nx && nx < hi)) nx = 0.5 * (lo + hi);
    if (fabs(nx - r) <= 1e-14 * (1.0 + fabs(r))) return nx;
    r = nx;
  }
  return r;
}

__device__ __forceinline__ double norm3(const double p[3]) {
  return sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
}

// Root-finding case (cones.py:334-378).  Returns true on success.
static __device__ bool exp_root(const double p[3], double &rho, double ph[3], double &yh, double &mu) {
  const double tol = 1e-10 * (1.0 + norm3(p));
  const double x = p[0], y = p[1];
  double lim = 4.0;
  if (y != 0.0) lim = fmax(lim, 4.0 * fabs(x / y));
  if (x != 0.0) lim = fmax(lim, 4.0 * fabs(1.0 - y / x));
  lim = fmin(lim, 1e160);
  double span = 1.0;
  while (true) {
    const double start = -span, step = (span - start) / 128.0;
    double ga = start, ha = exp_h0(p, ga);
    for (int i = 0; i < 128; ++i) {
      const double gb = (i + 1 == 128) ? span : (double)(i + 1) * step + start;
      const double hb = exp_h0(p, gb);
      double r;
      bool cand = false;
      if (ha == 0.0) { r = ga; cand = true; }
      else if (ha * hb < 0.0) { r = exp_newton(p, ga, gb, ha); cand = true; }
      if (cand) {
        double mue;
        exp_candidate(p, r, ph, yh, mu, mue);
        if (yh > 0.0 && mu >= -tol && exp_worst_res(p, r, ph, mu, mue) <= tol) { rho = r; return true; }
      }
      ga = gb; ha = hb;
    }
    if (ha == 0.0) {
      double mue;
      exp_candidate(p, span, ph, yh, mu, mue);
      if (yh > 0.0 && mu >= -tol && exp_worst_res(p, span, ph, mu, mue) <= tol) { rho = span; return true; }
    }
    if (span >= lim) return false;
    span = fmin(2.0 * span, lim);
  }
}

__device__ __forceinline__ bool exp_soft(const double p[3], double tol) {   // cones.py:396-402
  if (p[1] > tol) return p[1] * exp(p[0] / p[1]) <= p[2] + tol;
  return fabs(p[1]) <= tol && p[0] <= tol && p[2] >= -tol;
}

__device__ __forceinline__ bool exp_polar_soft(const double p[3], double tol) {   // cones.py:405-411
  if (p[0] > tol) return p[0] * exp(p[1] / p[0]) <= -kE * p[2] + tol;
  return fabs(p[0]) <= tol && p[1] <= tol && p[2] <= tol;
}

// Projection onto K_exp (cones.py:414-433).  Returns a qg_status.
static __device__ int exp_project(const double p[3], double out[3]) {
  const double x = p[0], y = p[1], z = p[2];
  if (exp_in(x, y, z)) { out[0] = x; out[1] = y; out[2] = z; return QG_OK; }
  if (exp_in_polar(x, y, z)) { out[0] = out[1] = out[2] = 0.0; return QG_OK; }
  if (x <= 0.0 && y <= 0.0) { out[0] = x; out[1] = 0.0; out[2] = fmax(z, 0.0); return QG_OK; }
  double rho, yh, mu;
  if (exp_root(p, rho, out, yh, mu)) return QG_OK;
  const double tol = 1e-9 * (1.0 + norm3(p));
  if (exp_soft(p, tol)) { out[0] = x; out[1] = y; out[2] = z; return QG_OK; }
  if (exp_polar_soft(p, tol)) { out[0] = out[1] = out[2] = 0.0; return QG_OK; }
  return QG_ERR_NUMERICAL;
}

__device__ __forceinline__ void set_diag3(double D[9], double a, double b, double c) {
  for (int i = 0; i < 9; ++i) D[i] = 0.0;
  D[0] = a; D[4] = b; D[8] = c;
}

// Solve J X = E[:, :3] for the 4x4 J by Gaussian elimination with partial
// pivoting (LAPACK dgesv's pivot rule), return X[:3,:] symmetrized.
static __device__ bool solve4_sym(double J[16], double D[9]) {
  double R[12];  // 4x3 right-hand sides
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 3; ++j) R[i * 3 + j] = (i == j) ? 1.0 : 0.0;
  for (int k = 0; k < 4; ++k) {
    int piv = k;
    double best = fabs(J[k * 4 + k]);
    for (int i = k + 1; i < 4; ++i)
      if (fabs(J[i * 4 + k]) > best) { best = fabs(J[i * 4 + k]); piv = i; }
    if (best == 0.0) return false;
    if (piv != k) {
      for (int j = 0; j < 4; ++j) { double t = J[k * 4 + j]; J[k * 4 + j] = J[piv * 4 + j]; J[piv * 4 + j] = t; }
      for (int j = 0; j < 3; ++j) { double t = R[k * 3 + j]; R[k * 3 + j] = R[piv * 3 + j]; R[piv * 3 + j] = t; }
    }
    const double inv = 1.0 / J[k * 4 + k];
    for (int i = k + 1; i < 4; ++i) {
      const double l = J[i * 4 + k] * inv;
      if (l == 0.0) continue;
      for (int j = k; j < 4; ++j) J[i * 4 + j] -= l * J[k * 4 + j];
      for (int j = 0; j < 3; ++j) R[i * 3 + j] -= l * R[k * 3 + j];
    }
  }
  for (int k = 3; k >= 0; --k)
    for (int j = 0; j < 3; ++j) {
      double s = R[k * 3 + j];
      for (int c = k + 1; c < 4; ++c) s -= J[k * 4 + c] * R[c * 3 + j];
      R[k * 3 + j] = s / J[k * 4 + k];
    }
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) D[i * 3 + j] = 0.5 * (R[i * 3 + j] + R[j * 3 + i]);
  for (int i = 0; i < 9; ++i)
    if (!isfinite(D[i])) return false;
  return true;
}

// Projection derivative at p (cones.py:436-480).
static __device__ int exp_deriv(const double p[3], double D[9]) {
  const double x = p[0], y = p[1], z = p[2];
  if (y > 0.0 && y * exp(x / y) < z) { set_diag3(D, 1.0, 1.0, 1.0); return QG_OK; }
  if (exp_in_polar(x, y, z)) { set_diag3(D, 0.0, 0.0, 0.0); return QG_OK; }
  if (x <= 0.0 && y <= 0.0) { set_diag3(D, 1.0, 0.0, z > 0.0 ? 1.0 : 0.0); return QG_OK; }
  double rho, ph[3], yh, mu;
  if (!exp_root(p, rho, ph, yh, mu)) {
    const double tol = 1e-9 * (1.0 + norm3(p));
    if (exp_soft(p, tol)) { set_diag3(D, 1.0, 1.0, 1.0); return QG_OK; }
    if (exp_polar_soft(p, tol)) { set_diag3(D, 0.0, 0.0, 0.0); return QG_OK; }
    if (x <= tol && y <= tol) { set_diag3(D, 1.0, 0.0, z > 0.0 ? 1.0 : 0.0); return QG_OK; }
    return QG_ERR_NUMERICAL;
  }
  if (fabs(rho) > 700.0) return QG_ERR_NUMERICAL;
  const double e = exp(rho), k = mu * e / yh;
  double J[16] = {1.0 + k,  -rho * k,            0.0, e,
                  -rho * k, 1.0 + rho * rho * k, 0.0, (1.0 - rho) * e,
                  0.0,      0.0,                 1.0, -1.0,
                  e,        (1.0 - rho) * e,     -1.0, 0.0};
  for (int i = 0; i < 16; ++i)
    if (!isfinite(J[i])) return QG_ERR_NUMERICAL;
  if (!solve4_sym(J, D)) return QG_ERR_NUMERICAL;
  return QG_OK;
}

// ------------------------------------------------------------------ power --
__device__ __forceinline__ bool pow_in(const double p[3], double a) {   // cones.py:490-493
  return p[0] >= 0.0 && p[1] >= 0.0 && pow(p[0], a) * pow(p[1], 1.0 - a) >= fabs(p[2]);
}

__device__ __forceinline__ bool pow_in_polar(const double p[3], double a) {   // cones.py:496-501
  if (p[0] > 0.0 || p[1] > 0.0) return false;
  return pow(-p[0] / a, a) * pow(-p[1] / (1.0 - a), 1.0 - a) >= fabs(p[2]);
}

__device__ __forceinline__ double pow_coord(double w, double c, double r, double az) {   // cones.py:504-514
  const double qq = 4.0 * c * r * (az - r);
  const double sq = sqrt(w * w + qq);
  return (w >= 0.0) ? 0.5 * (w + sq) : 0.5 * qq / (sq - w);
}

// residual and derivative (has_d = false where the reference returns None).
__device__ __forceinline__ double pow_res(const double p[3], double a, double r, double az,
                                          double *hp, bool *has_d) {   // cones.py:517-531
  const double x = p[0], y = p[1];
  const double fx = pow_coord(x, a, r, az), fy = pow_coord(y, 1.0 - a, r, az);
  const double prod = pow(fx, a) * pow(fy, 1.0 - a);
  if (hp) {
    if (fx > 0.0 && fy > 0.0) {
      const double dfx = a * (az - 2.0 * r) / sqrt(x * x + 4.0 * a * r * (az - r));
      const double dfy = (1.0 - a) * (az - 2.0 * r) / sqrt(y * y + 4.0 * (1.0 - a) * r * (az - r));
      *hp = prod * (a * dfx / fx + (1.0 - a) * dfy / fy) - 1.0;
      *has_d = true;
    } else {
      *has_d = false;
    }
  }
  return prod - r;
}

// 0 = root bracketed, 1 = cone side, 2 = polar side (cones.py:534-556).
static __device__ int pow_bracket(const double p[3], double a, double &lo, double &flo, double &hi, double &fhi) {
  const double az = fabs(p[2]);
  fhi = pow_res(p, a, az, az, nullptr, nullptr);
  hi = az;
  if (fhi >= 0.0) return 1;
  if (p[0] > 0.0 && p[1] > 0.0) {
    lo = 0.0;
    flo = pow(p[0], a) * pow(p[1], 1.0 - a);
    return 0;
  }
  lo = 0.5 * az;
  flo = pow_res(p, a, lo, az, nullptr, nullptr);
  for (int i = 0; i < 200; ++i) {
    if (flo > 0.0) return 0;
    lo *= 0.5;
    flo = pow_res(p, a, lo, az, nullptr, nullptr);
  }
  return 2;
}

static __device__ double pow_root(const double p[3], double a, double lo, double flo, double hi) {   // cones.py:559-618
  const double az = fabs(p[2]);
  const double tol = 1e-12 * (1.0 + az);
  if (flo == 0.0) return lo;
  while (hi - lo > 1e-14 * az) {
    const double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    const double fm = pow_res(p, a, mid, az, nullptr, nullptr);
    if (fm > 0.0) lo = mid;
    else if (fm < 0.0) hi = mid;
    else return mid;
  }
  double r = 0.5 * (lo + hi);
  for (int it = 0; it < 50; ++it) {
    double fp = 0.0;
    bool hd = false;
    const double f = pow_res(p, a, r, az, &fp, &hd);
    if (fabs(f) <= 0.25 * tol) break;
    if (f > 0.0) lo = r; else hi = r;
    double nx = (hd && fp != 0.0) ? r - f / fp : 0.5 * (lo + hi);
    if (!(lo < nx && nx < hi)) nx = 0.5 * (lo + hi);
    if (fabs(nx - r) <= 1e-17 * (1.0 + r)) { r = nx; break; }
    r = nx;
  }
  const double f = pow_res(p, a, r, az, nullptr, nullptr);
  if (fabs(f) <= tol) return r;
  if (f > 0.0) lo = r; else hi = r;
  for (int it = 0; it < 80; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    const double fm = pow_res(p, a, mid, az, nullptr, nullptr);
    if (fm > 0.0) lo = mid;
    else if (fm < 0.0) hi = mid;
    else return mid;
  }
  const double fl = pow_res(p, a, lo, az, nullptr, nullptr);
  const double fh = pow_res(p, a, hi, az, nullptr, nullptr);
  return (fabs(fl) <= fabs(fh)) ? lo : hi;
}

__device__ __forceinline__ double sgn(double v) { return (v > 0.0) ? 1.0 : ((v < 0.0) ? -1.0 : 0.0); }

static __device__ int pow_project(const double p[3], double a, double out[3]) {   // cones.py:647-663
  if (pow_in(p, a)) { out[0] = p[0]; out[1] = p[1]; out[2] = p[2]; return QG_OK; }
  if (pow_in_polar(p, a)) { out[0] = out[1] = out[2] = 0.0; return QG_OK; }
  const double x = p[0], y = p[1], z = p[2];
  if (z == 0.0) { out[0] = fmax(x, 0.0); out[1] = fmax(y, 0.0); out[2] = 0.0; return QG_OK; }
  const double az = fabs(z);
  double lo, flo, hi, fhi;
  const int side = pow_bracket(p, a, lo, flo, hi, fhi);
  if (side == 1) { out[0] = x; out[1] = y; out[2] = z; return QG_OK; }
  if (side == 2) { out[0] = out[1] = out[2] = 0.0; return QG_OK; }
  const double r = pow_root(p, a, lo, flo, hi);
  out[0] = pow_coord(x, a, r, az);
  out[1] = pow_coord(y, 1.0 - a, r, az);
  out[2] = sgn(z) * r;
  return QG_OK;
}

static __device__ int pow_deriv(const double p[3], double a, double D[9]) {   // cones.py:666-722
  const double x = p[0], y = p[1], z = p[2];
  if (z == 0.0 && (x == 0.0 || y == 0.0)) return QG_ERR_NOT_DIFFERENTIABLE;
  if (pow_in(p, a)) { set_diag3(D, 1.0, 1.0, 1.0); return QG_OK; }
  if (pow_in_polar(p, a)) { set_diag3(D, 0.0, 0.0, 0.0); return QG_OK; }
  if (z != 0.0) {
    const double az = fabs(z);
    double lo, flo, hi, fhi;
    const int side = pow_bracket(p, a, lo, flo, hi, fhi);
    if (side == 1) { set_diag3(D, 1.0, 1.0, 1.0); return QG_OK; }
    if (side == 2) { set_diag3(D, 0.0, 0.0, 0.0); return QG_OK; }
    const double r = pow_root(p, a, lo, flo, hi);
    const double gx = 2.0 * pow_coord(x, a, r, az) - x;
    const double gy = 2.0 * pow_coord(y, 1.0 - a, r, az) - y;
    const double ratio = a * x / gx + (1.0 - a) * y / gy;
    const double L = 2.0 * (az - r) / (az + (az - 2.0 * r) * ratio);
    const double sz = sgn(z);
    D[0] = 0.5 + x / (2.0 * gx) + (a * a) * (az - 2.0 * r) * r * L / (gx * gx);
    D[4] = 0.5 + y / (2.0 * gy) + ((1.0 - a) * (1.0 - a)) * (az - 2.0 * r) * r * L / (gy * gy);
    D[1] = D[3] = (a - a * a) * (az - 2.0 * r) * r * L / (gx * gy);
    D[2] = D[6] = sz * a * r * L / gx;
    D[5] = D[7] = sz * (1.0 - a) * r * L / gy;
    D[8] = r / az - r / az * ratio * L;
    return QG_OK;
  }
  double d;
  if (x > 0.0) d = (a > 0.5) ? 1.0 : ((a < 0.5) ? 0.0 : x / (2.0 * fabs(y) + x));
  else d = (a < 0.5) ? 1.0 : ((a > 0.5) ? 0.0 : y / (2.0 * fabs(x) + y));
  set_diag3(D, x > 0.0 ? 1.0 : 0.0, y > 0.0 ? 1.0 : 0.0, d);
  return QG_OK;
}

// ------------------------------------------------- 3-cone block dispatch --
// flip: the block is handled through the Moreau identity at -z
// (Pi(z) = z + Pi_base(-z), DPi = I - DPi_base(-z)); cones.py:803-883.
__device__ __forceinline__ bool tri_flip_of(int kind, int dual) {
  const bool dual_kind = (kind == QG_CONE_DEXP || kind == QG_CONE_DPOW);
  return dual ? !dual_kind : dual_kind;
}

__device__ __forceinline__ int tri_project(int kind, double alpha, int dual, const double z[3], double out[3]) {
  const bool flip = tri_flip_of(kind, dual);
  const bool is_exp = (kind == QG_CONE_EXP || kind == QG_CONE_DEXP);
  double p[3] = {flip ? -z[0] : z[0], flip ? -z[1] : z[1], flip ? -z[2] : z[2]};
  double pr[3];
  const int st = is_exp ? exp_project(p, pr) : pow_project(p, alpha, pr);
  if (st != QG_OK) return st;
  for (int i = 0; i < 3; ++i) out[i] = flip ? z[i] + pr[i] : pr[i];
  return QG_OK;
}

__device__ __forceinline__ int tri_deriv(int kind, double alpha, int dual, const double z[3], double D[9], int &flip) {
  flip = tri_flip_of(kind, dual) ? 1 : 0;
  const bool is_exp = (kind == QG_CONE_EXP || kind == QG_CONE_DEXP);
  double p[3] = {flip ? -z[0] : z[0], flip ? -z[1] : z[1], flip ? -z[2] : z[2]};
  return is_exp ? exp_deriv(p, D) : pow_deriv(p, alpha, D);
}

__device__ __forceinline__ void tri_apply(const double D[9], int flip, const double d[3], double o[3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double r = D[i * 3 + 0] * d[0] + D[i * 3 + 1] * d[1] + D[i * 3 + 2] * d[2];
    o[i] = flip ? d[i] - r : r;
  }
}

}  // namespace qg
