/* qcpgrad -- B200-native derivative/adjoint of the QCP solution map.
 *
 * C ABI of libqcpgrad.so (paper_2508_17522_b200/_lib/libqcpgrad.so).  Plain
 * pointers and sizes only.  Unless stated otherwise every array argument is a
 * DEVICE pointer (cudaMalloc / torch CUDA storage) owned by the caller; cone
 * block tables and size arrays are HOST pointers.  `stream` is a cudaStream_t
 * (NULL = legacy default stream).  Every call returns a qg_status; the
 * message of the last failure on the calling thread is qg_last_error().
 *
 * Reference interfaces replaced (paths relative to the reference's
 * pkg/src/conegrad/):
 *   qg_create / qg_create_batch  <- ProblemData + embed + _embedding_project +
 *                                   make_F preparation (embedding.py:59-115,
 *                                   337-427; solution_map.py:170-179)
 *   qg_jvp                       <- solution_map.jvp   (solution_map.py:325-355)
 *   qg_vjp                       <- solution_map.vjp   (solution_map.py:358-385)
 *   qg_apply_F                   <- make_F(...).matvec / .rmatvec
 *                                   (embedding.py:420-425)
 *   qg_check                     <- check_solution     (solution_map.py:263-288)
 *   qg_cones_*                   <- cones.project / project_dual /
 *                                   dprojection(_dual).matvec (cones.py:926-963)
 *   qg_spmv_csc                  <- _kernels.spmv / spmv_adjoint backend slot
 *                                   (_kernels/__init__.py:23-50, _csc.pyx:17-50)
 *   qg_set_point / qg_residual / <- testkit.refine internals: make_F at any z,
 *   qg_lsmr_jacobian                normalized_residual, the Gauss-Newton model
 *                                   solve (embedding.py:374-427; testkit.py:410-470)
 *   qg_comm_* / qg_create_batch_dist  no counterpart (row-partitioned multi-GPU,
 *                                   SURVEY.md §8(e))
 */
#ifndef QCPGRAD_H
#define QCPGRAD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes mirror the reference exception taxonomy (errors.py:13-38). */
typedef enum {
  QG_OK = 0,
  QG_ERR_VALIDATION = 1,        /* ValidationError                          */
  QG_ERR_DOMAIN = 2,            /* DomainError (tau <= 0, z_N <= 0)          */
  QG_ERR_NUMERICAL = 3,         /* NumericalError (root finding, non-finite) */
  QG_ERR_NOT_DIFFERENTIABLE = 4,/* NotDifferentiableError (pow apex)        */
  QG_ERR_CUDA = 5,              /* CUDA runtime failure                     */
  QG_ERR_UNSUPPORTED = 6        /* outside this build's limits              */
} qg_status;

/* Cone kinds in the reference's canonical order (cones.py:36-46). */
typedef enum {
  QG_CONE_ZERO = 0, QG_CONE_NONNEG = 1, QG_CONE_SOC = 2, QG_CONE_PSD = 3,
  QG_CONE_EXP = 4, QG_CONE_DEXP = 5, QG_CONE_POW = 6, QG_CONE_DPOW = 7
} qg_cone_kind;

typedef struct {
  int32_t kind;   /* qg_cone_kind                                  */
  int32_t dim;    /* vectorised length (psd: order*(order+1)/2)    */
  int32_t order;  /* psd matrix order, else 0                      */
  double alpha;   /* pow/dpow exponent in (0,1), else 0            */
} qg_cone_block;

/* A batch of independent problems, concatenated in problem order.  Sparse
 * matrices are CSC with int64 indices exactly as the reference stores them
 * (sparse.py:19-73), each problem's col_ptr starting at 0.  P carries both
 * triangles and is validated symmetric by the caller (sparse.py:173-194). */
typedef struct {
  int64_t nprob;
  const int64_t *n, *m;           /* host [nprob]                         */
  const int64_t *P_nnz, *A_nnz;   /* host [nprob]                         */
  const int64_t *nblocks;         /* host [nprob]                         */
  const qg_cone_block *blocks;    /* host, concatenated                    */
  const int64_t *P_colptr, *P_rowidx; const double *P_vals; /* device      */
  const int64_t *A_colptr, *A_rowidx; const double *A_vals; /* device      */
  const double *q, *b;            /* device, sum(n) / sum(m)              */
  const double *x, *y, *s;        /* device, sum(n) / sum(m) / sum(m)     */
} qg_batch_desc;

/* Perturbation (dP, dA, dq, db) for qg_jvp: CSC per problem, concatenated.
 * same_pattern != 0 promises dP/dA share P's/A's exact patterns (the common
 * case), which lets the kernels reuse the prepared transposes. */
typedef struct {
  const int64_t *dP_nnz, *dA_nnz;                            /* host [nprob] */
  const int64_t *dP_colptr, *dP_rowidx; const double *dP_vals; /* device     */
  const int64_t *dA_colptr, *dA_rowidx; const double *dA_vals; /* device     */
  const double *dq, *db;                                       /* device     */
  int32_t same_pattern;
} qg_perturbation;

typedef struct {
  double atol, btol;   /* lsmr.py:57 defaults 1e-10                      */
  int64_t max_iter;    /* 0 -> 10*(in_dim+out_dim) (lsmr.py:69-70);
                          < 0 -> no iterations (explicit cap of zero)     */
} qg_lsmr_opts;

/* Per-problem diagnostics (solution_map.py:139-167, 313-322). */
typedef struct {
  int64_t iterations;
  int32_t converged;
  int32_t derivative_unreliable;
  double residual_norm;   /* LSMR recurrence estimate normr (lsmr.py:161) */
  double atr_norm;
  double rhs_norm;
} qg_diag;

typedef struct qg_handle qg_handle;
typedef struct qg_cones qg_cones;

const char *qg_last_error(void);
const char *qg_version(void);

/* Prepare a batch: CSC->CSR transposes, z = (x, y-s, 1), Pi_K*(z) and the
 * prepared projection derivative, P xbar and xbar'P xbar. */
int qg_create_batch(qg_handle **out, const qg_batch_desc *desc, void *stream);
int qg_destroy(qg_handle *h);
int qg_handle_sizes(const qg_handle *h, int64_t *nprob, int64_t *total_n, int64_t *total_m);
/* SpMV layout chosen at create (diagnostic; no reference counterpart): number
 * of SELL-32 slices on the X side (rows of P and A') and on the Y side (rows
 * of A); 0 = that side runs the CSR group-per-row path. */
int qg_handle_layout(const qg_handle *h, int64_t *sell_slices_x, int64_t *sell_slices_y);
/* LSMR loop mode chosen at create (diagnostic): *resident = 1 when every
 * solve runs problem-resident (one persistent kernel, a CTA per problem,
 * vectors in shared memory: small problems / large batches), 0 = the
 * 4-launches-per-iteration CUDA-graph loop. */
int qg_handle_engine(const qg_handle *h, int32_t *resident);
/* Device time of the LSMR loop (after the init phases) of the last jvp and
 * the last vjp on this handle, CUDA events on the call's stream (0 = none). */
int qg_loop_time(const qg_handle *h, double *jvp_ms, double *vjp_ms);

/* jvp: outputs dx (sum n), dy, ds (sum m), diag[nprob] (host). */
int qg_jvp(qg_handle *h, const qg_perturbation *dtheta, const qg_lsmr_opts *opts,
           double *dx, double *dy, double *ds, qg_diag *diag, void *stream);
/* vjp: inputs dx, dy, ds; outputs dP values (sum P_nnz, CSC order of P),
 * dA values (CSC order of A), dq, db; diag[nprob] (host). */
int qg_vjp(qg_handle *h, const double *dx, const double *dy, const double *ds,
           const qg_lsmr_opts *opts, double *dP_vals, double *dA_vals, double *dq,
           double *db, qg_diag *diag, void *stream);

/* One operator application F w (transpose=0) or F' w (transpose=1) on the
 * batch embedding vector laid out as [X (sum n) | Y (sum m) | T (nprob)]. */
int qg_apply_F(qg_handle *h, int transpose, const double *w, double *out, void *stream);
/* The projected embedding point Pi z in the same layout. */
int qg_embedding_point(qg_handle *h, double *pz, void *stream);

/* KKT residuals of (x, y, s) per problem: report[5*p + {primal,
 * stationarity, gap, primal_cone_distance, dual_cone_distance}] (host). */
int qg_check(qg_handle *h, const double *x, const double *y, const double *s, double *report, void *stream);

/* Standalone cone calculus over a block table (host). */
int qg_cones_create(qg_cones **out, const qg_cone_block *blocks, int64_t nblocks, void *stream);
int qg_cones_destroy(qg_cones *c);
int qg_cones_project(qg_cones *c, int dual, const double *z, double *out, void *stream);
/* Prepare D Pi at z (dual or primal); subsequent applies reuse it. */
int qg_cones_prepare(qg_cones *c, int dual, const double *z, void *stream);
int qg_cones_apply(qg_cones *c, const double *dz, double *out, void *stream);

/* Plain CSC products with int64 indices (the reference's SpMV backend slot). */
int qg_spmv_csc(int64_t nrows, int64_t ncols, const int64_t *col_ptr, const int64_t *row_idx,
                const double *values, int64_t nnz, int adjoint, const double *x, double *out,
                void *stream);

/* Benchmark hook: launch one hot-path kernel of the prepared batch -- which =
 * 0: fused F step (SpMV + epilogue), 1: fused F' step (SpMV + D Pi epilogues),
 * 2: LSMR vector update, 3: the F' step's PSD units alone (k_step_psd; batches
 * with PSD blocks) -- `reps` times on `stream` between CUDA events;
 * *avg_ms receives the mean device time per launch. */
int qg_time_kernel(qg_handle *h, int which, int reps, double *avg_ms, void *stream);

/* Number of kernels this library launched since load (telemetry). */
int64_t qg_kernel_launches(void);

/* ---- re-solving oracle (testkit.refine / fd_jvp, testkit.py:410-497) ----
 * Move the handle to an arbitrary embedding point z = [X | Y | T] (device,
 * NE = sum n + sum m + nprob doubles, every z_N > 0 else QG_ERR_DOMAIN):
 * Pi z, P xbar, and with want_deriv the projection derivative at z.  jvp /
 * vjp need z_N = 1 (QG_ERR_DOMAIN otherwise, solution_map.py:197-203). */
int qg_set_point(qg_handle *h, const double *z, int want_deriv, void *stream);
/* normalized residual N(z) = (Q(Pi z) - Pi z + z)/|z_N| at the handle's point
 * (embedding.normalized_residual, embedding.py:374-396); out: NE doubles */
int qg_residual(qg_handle *h, double *out, void *stream);
/* LSMR on J = F - rank1 e_N' (rank1: NE doubles, or NULL for F itself) at the
 * handle's point from rhs (NE), solution to sol (NE); the Gauss-Newton model
 * of testkit.refine (testkit.py:439-454).  diag[nprob] (host). */
int qg_lsmr_jacobian(qg_handle *h, const double *rhs, const double *rank1, const qg_lsmr_opts *opts,
                     double *sol, qg_diag *diag, void *stream);

/* ---- row-partitioned mode (no reference counterpart:
 * the reference is single-process).  The Y rows of A -- with b, y, s and
 * whole cone blocks (zero / nonneg blocks may be cut anywhere) -- are split
 * over ranks; every rank holds the full X side (P, q, x) and the T entry.
 * Each rank creates a handle from ITS shard (qg_batch_desc with the local m,
 * local A rows as CSC over all n columns, local b, y, s, blocks) plus a
 * communicator; jvp / vjp then run the same LSMR on every rank with one
 * sum-allreduce of the A' partials per operator step and one of the
 * per-problem partial sums per finalize.  Outputs: dx, dq, dP replicated;
 * dy, ds, db and dA (local rows, CSC order of the local A) per rank.
 * qg_check is not available on a partitioned handle. */
typedef struct qg_comm qg_comm;
/* rank 0 creates the NCCL unique id and ships it to the others (any channel) */
int qg_comm_nccl_id(unsigned char id[128]);
/* one rank per GPU / process; NCCL resolved at run time from libnccl.so.2 */
int qg_comm_create_nccl(qg_comm **out, const unsigned char id[128], int world, int rank);
/* `world` (1..8) shards on the current device, one host thread per shard:
 * out[r] is shard r's communicator.  Not graph-capturable (host barrier). */
int qg_comm_create_local(qg_comm **out, int world);
int qg_comm_destroy(qg_comm *c);
int qg_comm_rank(const qg_comm *c, int *rank, int *world);
/* in-place sum over ranks of n doubles (device buffer), synchronous */
int qg_comm_allreduce(qg_comm *c, double *buf, int64_t n, void *stream);
/* create a handle over this rank's shard; `comm` must outlive the handle */
int qg_create_batch_dist(qg_handle **out, const qg_batch_desc *desc, qg_comm *comm, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* QCPGRAD_H */
