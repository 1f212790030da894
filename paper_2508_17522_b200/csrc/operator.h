// Host interface of the operator / LSMR / assembly kernels.
#pragma once

#include "handle.h"
#include "ops_dev.cuh"

namespace qg {

enum StepKind { STEP_F = 0, STEP_FT = 1 };
enum FinPhase { PH_APPLY = 0, PH_RHS = 1, PH_INIT_V = 2, PH_STEP_U = 3, PH_STEP_V = 4, PH_STEP_X = 5 };
enum RhsKind { RHS_JVP = 0, RHS_VJP = 1, RHS_VEC = 2 };

struct FinArgs {
  int B;
  int phase;
  int kind;            // STEP_F / STEP_FT (or RhsKind for PH_RHS)
  Lsmr *st;
  const double *part;
  const double *in;    // EVec (T component read)
  const double *old;   // EVec
  double *out;         // EVec (T component written)
  double *h, *hb, *x, *v;
  // filled by launch_fin: partial-sum arrays and per-problem ranges of the
  // X-side and Y-side producers of this phase
  const double *px = nullptr, *py = nullptr;
  const int64_t *px_ptr = nullptr, *py_ptr = nullptr;
  const double *rk1 = nullptr;  // rank-one term (StepArgs::rk1), T entries read here
  // LSMR loop finalizes: the LSMR state and the T entries come from EARLIER
  // finalizes (the step kernel launched in between never writes them), so
  // k_fin_cta loads them before its griddepcontrol.wait
  int early = 0;
};

// Deferred finalize of single-problem graph loops (kFeatDF steps): CTA 0
// of every step launch runs the PREVIOUS step's finalize and publishes the
// coefficients this step's row epilogues need; the other CTAs stage their
// row sums in shared memory meanwhile and wait for pub[par] (flag[par] ==
// flag[par ^ 1] + 1).  pend_phase: the finalize still owed by the last step
// (0: none).
struct DfPub {
  double s_in, c_out, wN, c_hbar, c_x, c_h, s_v;
  int runs, upd;
};
struct DfCtl {
  DfPub pub[2];
  unsigned flag[2];
  int pend_phase, pad;
};

struct StepArgs {
  const double *in;    // EVec, raw
  const double *dpin;  // Y: D Pi applied to in_Y (F step)
  const double *old;   // EVec or null
  double *out;         // EVec
  double *dpout;       // Y: D Pi applied to out_Y (F' step), or null
  double *tY, *tY2;    // Y scratch (F' step)
  const Lsmr *st;      // per-problem coefficients / run flags; null = (1, 0), all run
  int is_v_step;
  double *part;
  double fixed_s_in = 0.0, fixed_c_out = 0.0;  // used when st == null (0 -> 1, 0)
  // deferred LSMR vector update of the previous iteration (u-step only):
  // hbar = h - c1 hbar ; x += c2 hbar ; h = in s_v - c3 h over the unit's own
  // rows, ||x||^2 partial in slot 3 (lsmr.py:142-144, 168)
  double *upd_h = nullptr, *upd_hb = nullptr, *upd_x = nullptr;
  int xmode = X_FULL;         // row-partitioned mode phase (ops_dev.cuh)
  double *xred = nullptr;     // [NX] A' partials (X_PARTIAL writes, X_FINISH reads)
  // rank-one term of the refine Jacobian J = F - r e_N' (testkit.py:443-451):
  // F step out -= r w_N ; F' step T out -= r'w (dot partial in slot 3)
  const double *rk1 = nullptr;
  unsigned long long *prof = nullptr;  // QG_PSD_PROF diagnostics (qg_time_kernel): PSD unit phase cycles
  // deferred finalize (kFeatDF launches: CTA 0 finalizes, units from blockIdx 1)
  DfCtl *df = nullptr;
  int df_par = 0;   // this step's publication slot (alternates between successive kFeatDF steps)
  int df_next = 0;  // the finalize owed to the next kFeatDF step after this one (its phase; 0: none)
  FinArgs fin{};    // the previous step's finalize (its partial sums in the other part buffer)
};

struct UpdArgs {
  double *h, *hb, *x;
  const double *v;
  const Lsmr *st;
  double *part;
};

Mats make_mats(const Handle &H);
void launch_step(const Handle &H, const Mats &M, int kind, const StepArgs &a, cudaStream_t st);
bool psd_split(const Handle &H);  // F' PSD units run as their own kernel (k_step_psd) beside k_step
void launch_step_psd(const Handle &H, const Mats &M, const StepArgs &a, cudaStream_t st);  // k_step_psd alone
void launch_fin(const Handle &H, const Mats &M, const FinArgs &a, cudaStream_t st);
void fin_ptrs(const Handle &H, FinArgs &a);  // partial-sum producers of a whole-problem handle
void launch_update(const Handle &H, const Mats &M, const UpdArgs &a, cudaStream_t st);
void launch_count_active(const Handle &H, cudaStream_t st);
void launch_init_state(const Handle &H, double atol, double btol, long long opt, long long cap, cudaStream_t st);
void launch_df_tail(const Handle &H, const Mats &M, const FinArgs &a, cudaStream_t st);  // owed finalize after the loop
void launch_init_df(const Handle &H, int pend, cudaStream_t st);  // arm the deferred-finalize control block
void launch_engine(Handle &H, const Mats &M, bool jvp, cudaStream_t st);
void launch_loop_cond(const Handle &H, cudaGraphConditionalHandle h, long long chunk, cudaStream_t st);

// assembly (assembly.cu)
struct PertDev {
  // dP as CSR over X rows (values in CSR order), dA as CSR over Y rows and as
  // CSC-as-rows over X rows; dq, db.
  const int32_t *dP_rp, *dP_col; const double *dP_val;
  const int32_t *dA_rp, *dA_col; const double *dA_val;
  const int32_t *dAT_rp, *dAT_col; const double *dAT_val;
  const double *dq, *db;
};
void launch_jvp_rhs(const Handle &H, const Mats &M, const PertDev &d, double *u, double *part, cudaStream_t st);
void launch_vjp_rhs(const Handle &H, const Mats &M, const double *dx, const double *dy, const double *ds,
                    const double *dpi_dyds, double *u, double *part, cudaStream_t st);
void launch_add(const Handle &H, const double *a, const double *b, double *out, int64_t n, cudaStream_t st);
void launch_gather(const int32_t *perm, const double *src, double *dst, int64_t n, cudaStream_t st);
void launch_dphi(const Handle &H, const Mats &M, const double *dz, const double *dpi_dz, double *dx, double *dy,
                 double *ds, cudaStream_t st);
void launch_vjp_grad(const Handle &H, const Mats &M, const double *w, double *dP, double *dA, double *dq,
                     double *db, cudaStream_t st);
void launch_embed_prep(const Handle &H, const double *x, const double *y, const double *s, double *zmid,
                       cudaStream_t st);
void launch_embed_consts(const Handle &H, const Mats &M, double *part, cudaStream_t st, const double *zT = nullptr);
void launch_residual(const Handle &H, const Mats &M, double *out, double *part, cudaStream_t st);
void launch_vec_rhs(const Handle &H, const Mats &M, const double *r, double *u, double *part, cudaStream_t st);
void launch_csr_spmv(const int32_t *rp, const int32_t *col, const double *val, int64_t nrows, const double *x,
                     double *out, cudaStream_t st);
void launch_kkt(const Handle &H, const Mats &M, const double *x, const double *y, const double *s,
                const double *projs, const double *projy, double *part, double *report_dev, cudaStream_t st);

}  // namespace qg
