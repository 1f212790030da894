// Scalar part of the LSMR finalize (lsmr.py:57-184), shared by the graph
// path's k_fin / k_fin_cta (operator.cu) and the problem-resident engine
// (engine.cu): the T component of an operator step, the norms, Givens
// recurrences and stopping rules of one problem, on its LSMR state and the
// T entries of its vectors.
#pragma once

#include "operator.h"

namespace qg {

__device__ __forceinline__ double dsign(double v) { return (v > 0.0) ? 1.0 : ((v < 0.0) ? -1.0 : 0.0); }

__device__ __forceinline__ void sym_ortho(double a, double b, double &c, double &s, double &r) {   // lsmr.py:38-54
  if (b == 0.0) { c = dsign(a); s = 0.0; r = fabs(a); return; }
  if (a == 0.0) { c = 0.0; s = dsign(b); r = fabs(b); return; }
  if (fabs(b) > fabs(a)) {
    const double t = a / b;
    s = dsign(b) / sqrt(1.0 + t * t);
    c = s * t;
    r = b / s;
  } else {
    const double t = b / a;
    c = dsign(a) / sqrt(1.0 + t * t);
    s = c * t;
    r = a / c;
  }
}

// T component of an operator step output (embedding.py:232-237, 261 and 420-425).
__device__ __forceinline__ double t_component(int kind, const Embed &E, double wN, const double sx[kSlots],
                                              const double sy[kSlots]) {
  if (kind == STEP_F) {
    const double outN = ((-(2.0 / E.tau)) * sx[0] - sx[1] - sy[0]) + (E.xPx / (E.tau * E.tau)) * wN;
    return ((outN - E.last * wN) + wN) / E.zN;
  }
  const double gN = (sx[1] + sy[0]) + (E.xPx / (E.tau * E.tau)) * wN;
  return (E.last * (gN - wN) + wN) / E.zN;
}

// Stopping rules after iteration itn with ||x||^2 = xx + xN^2 (lsmr.py:168-184).
// Returns true when the solve ended (problem deactivated).
__device__ __forceinline__ bool stop_test(Lsmr *L, double xx, double xN) {
  const double normx = sqrt(xx + xN * xN);
  L->normx = normx;
  const double normr = L->normr, normar = L->normar, normA = L->normA, normb = L->normb;
  if (!(isfinite(normr) && isfinite(normar) && isfinite(normx))) {
    L->status = QG_ERR_NUMERICAL;
    L->active = 0;
    return true;
  }
  bool stop = false;
  if (normar == 0.0) stop = true;
  else {
    const double test1 = normr / normb;
    const double test2 = normr > 0.0 ? normar / (normA * normr) : 0.0;
    const double rtol = L->btol + L->atol * normA * normx / normb;
    const double t1 = test1 / (1.0 + normA * normx / normb);
    if (1.0 + test2 <= 1.0 || 1.0 + t1 <= 1.0) stop = true;
    else if (test2 <= L->atol || test1 <= rtol) stop = true;
  }
  if (stop) { L->active = 0; L->converged = 1; return true; }
  if (L->itn >= L->max_iter) { L->active = 0; L->converged = 0; return true; }
  return false;
}

// T entries (index N-1 of the problem's embedding vectors) that a finalize
// reads and writes.  out starts equal to old (a skipped v-step keeps v).
struct TVals {
  double in, old, out, h, hb, x, rk1;
};
enum TvWrites : int { TV_OUT = 1, TV_H = 2, TV_HB = 4, TV_X = 8 };

// One finalize phase of one problem: sx / sy are the problem's X-side and
// Y-side sums of the step's kSlots partials.  do_stop: PH_STEP_U first runs
// the stopping test of the previous iteration (the graph path defers the
// vector update into the u-step; the engine runs it before calling with
// do_stop = false).  Returns the TVals fields written (TvWrites bits).
__device__ __forceinline__ int fin_core(const Embed &E, int phase, int kind, Lsmr *L, const double sx[kSlots],
                                        const double sy[kSlots], TVals &tv, bool rk1, bool do_stop) {
  // T component of the step output, with the refine rank-one term
  // (testkit.py:446-451): F: - r_N w_N ; F': - r'w
  auto tcomp = [&](double wN) {
    double t = t_component(kind, E, wN, sx, sy);
    if (rk1) t -= (kind == STEP_F) ? tv.rk1 * wN : (sx[3] + sy[3]) + tv.rk1 * wN;
    return t;
  };

  if (phase == PH_APPLY) {
    tv.out = tcomp(tv.in);
    return TV_OUT;
  }
  if (phase == PH_RHS) {
    // rhs_N from the assembly partials; then lsmr.py:72-80
    double rN;
    if (kind == RHS_JVP) {
      const double outN = ((-sx[0]) / E.tau - sx[1]) - sy[0];   // embedding.py:291
      rN = (-outN) / fabs(E.zN);
    } else if (kind == RHS_VEC) {
      rN = tv.in;                                                // given right-hand side
    } else {
      const double dzN = ((-sx[0]) - sy[0]) - sy[1];             // solution_map.py:259
      rN = -dzN;
    }
    tv.out = rN;
    const double beta = sqrt((sx[2] + sy[2]) + rN * rN);
    L->beta = beta;
    L->normb = beta;
    L->itn = 0;
    L->status = 0;
    L->skip_v = 0;
    L->alpha = 0.0;
    L->s_v = 1.0;
    if (beta > 0.0) {
      L->s_u = 1.0 / beta;
      L->s_in = L->s_u;
      L->c_out = 0.0;
      L->active = 1;
    } else {
      L->s_u = 1.0;
      L->active = 0;
      L->converged = 1;
      L->normr = beta;
      L->normar = 0.0;
    }
    return TV_OUT;
  }
  if (phase == PH_INIT_V) {
    const double vN = tcomp(tv.in) * L->s_in;
    tv.out = vN;
    const double alpha = sqrt((sx[2] + sy[2]) + vN * vN);
    L->alpha = alpha;
    L->s_v = alpha > 0.0 ? 1.0 / alpha : 1.0;
    const double beta = L->beta;
    if (alpha * beta == 0.0) {
      L->active = 0;
      L->converged = 1;
      L->normr = beta;
      L->normar = 0.0;
      return TV_OUT;
    }
    L->zetabar = alpha * beta;
    L->alphabar = alpha;
    L->rho = L->rhobar = L->cbar = 1.0;
    L->sbar = 0.0;
    L->betadd = beta;
    L->betad = 0.0;
    L->rhodold = 1.0;
    L->tautildeold = L->thetatilde = L->zeta = L->d = 0.0;
    L->normA2 = alpha * alpha;
    L->normr = beta;
    L->normar = alpha * beta;
    L->c_hbar = L->c_x = L->c_h = 0.0;
    tv.h = vN * L->s_v;
    tv.hb = 0.0;
    tv.x = 0.0;
    L->s_in = L->s_v;
    L->c_out = alpha * L->s_u;
    if (L->max_iter <= 0) { L->active = 0; L->converged = 0; }
    return TV_OUT | TV_H | TV_HB | TV_X;
  }
  if (phase == PH_STEP_U) {
    if (do_stop && L->itn > 0 && stop_test(L, sx[3] + sy[3], tv.x)) return 0;  // iteration itn ended the solve
    L->itn += 1;
    const double uN = L->s_in * tcomp(tv.in) - L->c_out * tv.old;
    tv.out = uN;
    const double beta = sqrt((sx[2] + sy[2]) + uN * uN);
    L->beta = beta;
    if (beta > 0.0) {
      L->s_u = 1.0 / beta;
      L->skip_v = 0;
      L->s_in = L->s_u;
      L->c_out = beta * L->s_v;
    } else {
      L->s_u = 1.0;
      L->skip_v = 1;
    }
    return TV_OUT;
  }
  if (phase == PH_STEP_V) {
    double alpha = L->alpha;
    int w = 0;
    if (!L->skip_v) {
      const double vN = L->s_in * tcomp(tv.in) - L->c_out * tv.old;
      tv.out = vN;
      w = TV_OUT;
      alpha = sqrt((sx[2] + sy[2]) + vN * vN);
      L->alpha = alpha;
      L->s_v = alpha > 0.0 ? 1.0 / alpha : 1.0;
    }
    const double beta = L->beta;
    if (!(isfinite(alpha) && isfinite(beta))) {
      L->status = QG_ERR_NUMERICAL;
      L->active = 0;
      return w;
    }
    // lsmr.py:127-171
    double chat, shat, alphahat;
    sym_ortho(L->alphabar, 0.0, chat, shat, alphahat);
    const double rhoold = L->rho;
    double c, s, rho;
    sym_ortho(alphahat, beta, c, s, rho);
    const double thetanew = s * alpha;
    L->alphabar = c * alpha;
    const double rhobarold = L->rhobar;
    const double zetaold = L->zeta;
    const double thetabar = L->sbar * rho;
    const double rhotemp = L->cbar * rho;
    double cbar, sbar, rhobar;
    sym_ortho(rhotemp, thetanew, cbar, sbar, rhobar);
    const double zeta = cbar * L->zetabar;
    L->zetabar = -sbar * L->zetabar;
    L->c_hbar = thetabar * rho / (rhoold * rhobarold);
    L->c_x = zeta / (rho * rhobar);
    L->c_h = thetanew / rho;
    const double betaacute = chat * L->betadd;
    const double betacheck = -shat * L->betadd;
    const double betahat = c * betaacute;
    L->betadd = -s * betaacute;
    const double thetatildeold = L->thetatilde;
    double ctildeold, stildeold, rhotildeold;
    sym_ortho(L->rhodold, thetabar, ctildeold, stildeold, rhotildeold);
    L->thetatilde = stildeold * rhobar;
    L->rhodold = ctildeold * rhobar;
    L->betad = -stildeold * L->betad + ctildeold * betahat;
    L->tautildeold = (zetaold - thetatildeold * L->tautildeold) / rhotildeold;
    const double taud = (zeta - L->thetatilde * L->tautildeold) / L->rhodold;
    L->d = L->d + betacheck * betacheck;
    const double bt = L->betad - taud;
    L->normr = sqrt(L->d + bt * bt + L->betadd * L->betadd);
    L->normA2 = L->normA2 + beta * beta;
    L->normA = sqrt(L->normA2);
    L->normA2 = L->normA2 + alpha * alpha;
    L->normar = fabs(L->zetabar);
    L->rho = rho;
    L->rhobar = rhobar;
    L->cbar = cbar;
    L->sbar = sbar;
    L->zeta = zeta;
    // T parts of the vector updates (v = the new v, i.e. out)
    const double hb = tv.h - L->c_hbar * tv.hb;
    tv.x = tv.x + L->c_x * hb;
    tv.h = tv.out * L->s_v - L->c_h * tv.h;
    tv.hb = hb;
    L->s_in = L->s_v;
    L->c_out = alpha * L->s_u;
    return w | TV_H | TV_HB | TV_X;
  }
  if (phase == PH_STEP_X) stop_test(L, sx[0] + sy[0], tv.x);
  return 0;
}

}  // namespace qg
