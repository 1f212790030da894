// The prepared batch ("QCP object" of the north star): problem data in CSR
// form, the projected embedding point, the prepared D Pi, work units and the
// LSMR workspace.  All device-resident; immutable after qg_create_batch
// except for the per-call workspace.
#pragma once

#include <memory>
#include <mutex>
#include <vector>

#include "comm.h"
#include "cone_table.h"
#include "qg_common.cuh"

namespace qg {

// Per-problem embedding constants (embedding.py:337-344, 399-417).
struct Embed {
  double tau;   // (Pi z)_N = max(z_N, 0)
  double zN;    // z_N (= 1 from embed)
  double last;  // D Pi on the last coordinate: 1 if z_N > 0 else 0
  double xPx;   // xbar' P xbar
};

// Per-problem LSMR state (lsmr.py:57-184), resident in HBM.
struct Lsmr {
  double alpha, beta, s_u, s_v, normb;
  double zetabar, alphabar, rho, rhobar, cbar, sbar;
  double betadd, betad, rhodold, tautildeold, thetatilde, zeta, d, normA2;
  double normr, normar, normA, normx;
  double c_hbar, c_x, c_h;
  double s_in, c_out;     // coefficients of the next half step
  double atol, btol;
  long long itn, max_iter;
  int active, converged, skip_v, status;
};

// Transposed / reinterpreted sparse structure on the device.
struct DevCsr {
  int32_t *rp = nullptr;   // row pointer (global rows)
  int32_t *col = nullptr;  // global column index
  double *val = nullptr;
  int32_t *perm = nullptr; // CSR position -> global CSC entry (transposes)
  int64_t nrows = 0, nnz = 0;
  void release();
};

struct SellMat {
  int64_t *off = nullptr;
  int32_t *w = nullptr;
  int32_t *col = nullptr;
  double *val = nullptr;
  int64_t entries = 0;
  SellView view() const { return SellView{off, w, col, val}; }
  void release();
};

struct DfCtl;  // operator.h

struct Workspace {
  double *u = nullptr, *v = nullptr, *h = nullptr, *hb = nullptr, *x = nullptr;  // EVec
  double *dpu = nullptr, *dpv = nullptr, *tY = nullptr, *tY2 = nullptr;          // Y
  double *part = nullptr;    // per work-unit partial sums (X units then Y units)
  double *rk1 = nullptr;     // EVec: refine rank-one vector (allocated on first use)
  Lsmr *st = nullptr;
  int *d_nactive = nullptr;
  int *d_claim = nullptr;    // problem claim counter of the resident engine
  double *part2 = nullptr;   // v-step partial sums of deferred-finalize loops (u-steps use part)
  DfCtl *df = nullptr;       // deferred-finalize control block (operator.h)
  long long *d_loop = nullptr;  // device-terminated graph loop: [iterations run, cap]
  int *h_nactive = nullptr;  // pinned
  void release();
};

struct Handle {
  int B = 0;
  std::vector<int64_t> n, m, xoff, yoff, nnzP, nnzA, noffP, noffA;
  int64_t NX = 0, NY = 0, NE = 0;  // NE = NX + NY + B
  DevCsr P;    // CSR of P (exact transpose of the CSC input)
  DevCsr Pc;   // CSC structure of P read as rows = columns (for dP emission)
  DevCsr A;    // CSR of A
  DevCsr AT;   // CSC of A read as CSR of A' (rows = columns of A, cols = global Y)
  ConeTable cones;
  SellMat sP, sAT, sA;          // SELL copies of P, A' (X rows) and A (Y rows)
  int32_t *x_rowof = nullptr;   // [32 * x slices] row of each slice lane (-1 = padding)
  int32_t *y_rowof = nullptr;
  int64_t nslice_x = 0, nslice_y = 0;
  bool has_wide = false;        // some unit runs CTA-per-row (MODE_WIDE)
  bool engine = false;          // LSMR solves run problem-resident (engine.cu)
  // engine layout: 16-bit problem-local columns parallel to the SELL entries
  // of P, A', A and 16-bit local rows of the slice lanes (0xffff = padding)
  uint16_t *c16P = nullptr, *c16AT = nullptr, *c16A = nullptr;
  unsigned char *eng_blob = nullptr;  // per-problem meta blobs (slice table, units, blocks, resident plan)
  int eng_res_cap = 0;                // resident matrix entries per CTA
  unsigned long long *eng_prof = nullptr;  // QG_ENG_PROF per-phase cycle counters
  std::vector<Unit> xunits;
  std::vector<int64_t> xunit_ptr;
  Unit *d_xunits = nullptr;
  int64_t *d_xoff = nullptr, *d_yoff = nullptr;
  int64_t *d_xunit_ptr = nullptr, *d_yunit_ptr = nullptr;
  int32_t *d_ft_order = nullptr;  // F' CTA -> unit order, PSD units first (null: natural order)
  int n_psd_units = 0;            // leading PSD units of d_ft_order (their own F' kernel, k_step_psd)
  bool defer_fin = false;       // single-problem graph loop with the deferred finalize (kFeatDF)
  bool df_mixed = false;        // (PSD blocks: only the F step defers)
  int max_unit_rows = 0;         // rows of the longest work unit (kFeatDF staging)
  bool psd_split = true;         // QG_PSD_SPLIT at creation (0: PSD units stay in k_step, A/B)
  double *q = nullptr, *b = nullptr, *xbar = nullptr, *ybar = nullptr, *sbar = nullptr;
  double *Pxbar = nullptr;
  Embed *emb = nullptr;
  Workspace ws;
  std::mutex mu;  // one jvp/vjp at a time per handle (workspace reuse)

  // row-partitioned mode (comm.h): this handle holds one rank's Y rows
  Comm *comm = nullptr;           // not owned; null = whole problems
  double *xred = nullptr;         // [NX] A_r' partial products, summed over ranks
  double *psum = nullptr;         // [2][B][kSlots] per-problem X / Y partial sums
  int64_t *d_iota = nullptr;      // [B+1] 0..B (one reduced "unit" per problem)
  bool x_owner() const { return comm == nullptr || comm->rank == 0; }

  // the point z the handle is prepared at (qg_set_point moves it)
  bool normalized = true;   // z_N == 1 for every problem (jvp / vjp formulas)
  bool deriv_ready = true;  // D Pi prepared at the current point
  bool use_rk1 = false;     // LSMR on J = F - rk1 e_N' (qg_lsmr_jacobian)

  // device time of the last jvp / vjp LSMR loop (qg_loop_time)
  cudaEvent_t ev_loop[2] = {nullptr, nullptr};
  double loop_ms[2] = {0.0, 0.0};
  int loop_pending = 0;  // 1: jvp, 2: vjp events recorded, not yet read
  bool while_pending = false;  // a device-terminated loop ran: count its launches at finish
  void loop_events();

  int nxu() const { return (int)xunits.size(); }
  int nyu() const { return (int)cones.units.size(); }
  ~Handle();
};

// CSC (int64, concatenated per problem) -> device CSR (int32) by a stable
// radix sort on global row keys.  Also returns the CSC structure itself in
// CSR-of-transpose form when `csc_as_rows` is non-null.
struct CscBatch {
  const int64_t *colptr, *rowidx;
  const double *vals;
  std::vector<int64_t> ncols, nrows, nnz;  // per problem
};
void csc_to_csr(const CscBatch &in, DevCsr &out, DevCsr *csc_as_rows, bool keep_perm, cudaStream_t st);

// SELL copies of P, A' (X units) and A (Y units); sets unit modes / slices
// (sell.cu).  rp* are host copies of the CSR row pointers.
// force: SELL on both sides (the resident engine walks SELL slices only).
void build_sell(Handle &H, const int32_t *rpP, const int32_t *rpAT, const int32_t *rpA, bool force, cudaStream_t st);

// Problem-resident LSMR engine (engine.cu): whether a batch qualifies
// (before the SELL build), whether every unit ended up SELL (after), and the
// launch that runs the whole loop of a solve after its init phases.
bool engine_candidate(const Handle &H);
bool engine_units_ok(const Handle &H);
void build_engine_layout(Handle &H, cudaStream_t st);

}  // namespace qg
