/*
 * qpk.h -- C ABI of libqpk.so, the B200 (sm_100a) Jacobi-PCG direction
 * solver for the Forsgren-Gill doubly augmented KKT system
 *
 *     K = [[Q + 2 B' D^-1 B, B'], [B, D]],   Q = H + diag(q_extra),
 *     B = (C; A_l; -A_u),  D = diag(d_diag)
 *
 * It is the native side of the reference's direction-solver hook
 *     DirectionSolver = Callable[[KktOperator, ndarray, PcgConfig], PcgResult]
 *     (/root/reference/pkg/src/qpipm/ipm.py:176, called at ipm.py:206)
 * and replaces, function by function:
 *     qpk_problem_begin, _add_rows, qpk_set_hessian_<kind>, _finalize
 *                           -> the per-problem data of KktOperator
 *                              (kkt.py:146-160, 203-208; model.py:17-162);
 *                              B is uploaded once per problem instead of the
 *                              row_submatrix copies made each IPM iteration
 *     qpk_set_diagonals     -> build_operator's d_diag / q_diag_extra
 *                              (kkt.py:190-202), once per IPM iteration
 *     qpk_jacobi            -> jacobi_diagonal (kkt.py:224-239) and the
 *                              inv_diag of _pcg_direction (ipm.py:180)
 *     qpk_apply             -> apply_doubly_augmented (kkt.py:211-221)
 *     qpk_pcg               -> pcg(apply_op, apply_prec, rhs, cfg)
 *                              (linalg.py:66-133) with x0 = 0, as
 *                              _pcg_direction calls it (ipm.py:181-182)
 *
 * Conventions: every function returns QPK_OK (0) or a negative QPK_E* code;
 * qpk_last_error() returns a thread-local message for the last failure.
 * Pointers are HOST pointers unless the function name ends in _dev, in which
 * case they are device pointers on the context's device.  All sizes are
 * element counts.  Not reentrant per context (one caller thread, as the
 * reference).  A breakdown (p'Kp <= 0, linalg.py:102-103) is not
 * an error: qpk_pcg returns QPK_OK with info.status == QPK_PCG_BREAKDOWN and
 * the best iterate in x (the reference raises PcgBreakdownError carrying the
 * same result).
 */
#ifndef QPK_H
#define QPK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QPK_ABI_VERSION 1

enum {
  QPK_OK = 0,
  QPK_E_ARG = -1,      /* invalid argument / dimension (reference DimensionError) */
  QPK_E_STATE = -2,    /* call out of order (e.g. qpk_pcg before qpk_set_diagonals) */
  QPK_E_CUDA = -3,     /* CUDA runtime failure */
  QPK_E_NOMEM = -4,    /* device or host allocation failed */
  QPK_E_UNSUPPORTED = -5
};

enum { QPK_HESS_DIAG = 0, QPK_HESS_CSR = 1, QPK_HESS_DENSE = 2, QPK_HESS_LOWRANK = 3 };

enum { QPK_PCG_OK = 0, QPK_PCG_BREAKDOWN = 1 };

/* scatter strategy for the B' z product of the operator apply */
enum {
  QPK_SCATTER_AUTO = 0,    /* chosen per matrix at finalize */
  QPK_SCATTER_ATOMIC = 1,  /* one pass over B, fp64 atomics (order not reproducible) */
  QPK_SCATTER_CSC = 2,     /* second, gather-only pass over a resident CSC copy:
                              bitwise reproducible run to run */
  QPK_SCATTER_DICT = 3,    /* one pass; rows grouped into blocks with a shared-memory
                              column dictionary, per-block partials combined in a
                              fixed order: no atomics, bitwise reproducible */
  QPK_SCATTER_PANEL = 4    /* one pass; columns present in most rows stored as a dense
                              row-major panel (B'z partials in registers, combined
                              per CTA in a fixed order), the rest of each row as a
                              narrow ELL strip: bitwise reproducible */
};

typedef struct qpk_ctx qpk_ctx;

/* result record of qpk_pcg: PcgResult (linalg.py:42-47) plus diagnostics */
typedef struct {
  int32_t iterations;          /* PcgResult.iterations */
  int32_t converged;           /* PcgResult.converged */
  int32_t status;              /* QPK_PCG_OK or QPK_PCG_BREAKDOWN */
  int32_t restarts;            /* true-residual restarts (linalg.py:117-125) */
  int32_t applies;             /* operator applications performed */
  int32_t reserved;
  double final_residual_norm;  /* PcgResult.final_residual_norm (true residual,
                                  or best recurrence residual on breakdown) */
  double threshold;            /* tol * ||rhs|| (relative) or tol */
  double rhs_norm;             /* ||rhs|| */
  double kernel_ms;            /* device time of the solve (CUDA events) */
  double phase_ms[4];          /* time inside the solve kernel spent in the
                                  direction/top phase, the rows (B, B') phase,
                                  the residual-update phase, and the rest
                                  (init, true residuals), from %globaltimer */
} qpk_pcg_info;

int qpk_abi_version(void);
const char* qpk_last_error(void);

/* one context per device (one process per GPU) */
int qpk_create(int device, qpk_ctx** out);
int qpk_destroy(qpk_ctx* ctx);
/* use an external cudaStream_t (e.g. torch's current stream); NULL = own stream */
int qpk_set_stream(qpk_ctx* ctx, void* stream);
int qpk_synchronize(qpk_ctx* ctx);

/* ---- multi-GPU: row sharding of B over ranks (one process per GPU) ------
 * Rank r holds rows [lo_r, hi_r) of B and the matching slice of every bottom
 * vector; the top block (n) is replicated, every rank owning a slice of its
 * terms.  Per PCG iteration the ranks all-reduce [y_top partial | slot scalars]
 * with NCCL; the tile format folds [r'r, r'z] into that one
 * all-reduce, the other formats reduce them in a second, 2-value all-reduce.
 * Rank 0 obtains the id, the launcher broadcasts it (e.g. through
 * torch.distributed), every rank calls qpk_shard_init before
 * qpk_problem_begin with its local sizes. */
int qpk_nccl_get_unique_id(unsigned char id[128]);
int qpk_shard_init(qpk_ctx* ctx, int world, int rank, const unsigned char id[128]);
/* test hook: rank `rank` of `world` without a communicator -- qpk_apply and
 * qpk_jacobi return this rank's un-reduced share (before qpk_problem_begin) */
int qpk_shard_emulate(qpk_ctx* ctx, int world, int rank);

/* ---- multi-GPU from ONE process (the reference's solve() is a single
 * process, ipm.py:185-206) ----------------------------------------------------
 * qpk_multi owns one context per listed device, shards B by rows over them
 * (contiguous, nnz-balanced blocks, as the one-process-per-GPU layout) and
 * runs every call on one host thread per device; the per-iteration
 * all-reduces go through one NCCL communicator per device.  All vectors are
 * GLOBAL host vectors (d: m_B, q: n, v / rhs / x: n + m_B).  The arrays given
 * to qpk_multi_problem_add_rows / qpk_multi_set_hessian_* are read at
 * qpk_multi_problem_finalize and must stay valid until it returns. */
typedef struct qpk_multi qpk_multi;
int qpk_multi_create(int n_devices, const int* device_ids, qpk_multi** out);
int qpk_multi_destroy(qpk_multi* mm);
/* test hook: n_ranks contexts on ONE device with host-mediated all-reduces --
 * the whole N > 1 sharded engine on a single GPU, no kernel waiting on a peer */
int qpk_multi_create_emulated(int n_ranks, int device, qpk_multi** out);
int qpk_multi_devices(qpk_multi* mm);
qpk_ctx* qpk_multi_context(qpk_multi* mm, int rank);
int qpk_multi_problem_begin(qpk_multi* mm, int64_t n, int64_t m_e, int64_t m_l, int64_t m_u);
int qpk_multi_problem_add_rows(qpk_multi* mm, int64_t n_rows, const int64_t* row_offsets,
                               const int64_t* col_indices, const double* values,
                               const int64_t* rows, int64_t n_sel, double sign);
int qpk_multi_set_hessian_diag(qpk_multi* mm, const double* d);
int qpk_multi_set_hessian_csr(qpk_multi* mm, const int64_t* row_offsets, const int64_t* col_indices,
                              const double* values);
int qpk_multi_set_hessian_dense(qpk_multi* mm, const double* m_rowmajor);
int qpk_multi_set_hessian_lowrank(qpk_multi* mm, const double* h0, int64_t k, const double* u_rowmajor,
                                  const double* w);
int qpk_multi_problem_finalize(qpk_multi* mm, int scatter);
int qpk_multi_set_diagonals(qpk_multi* mm, const double* d_diag, const double* q_diag_extra);
int qpk_multi_jacobi(qpk_multi* mm, double* diag_out);
int qpk_multi_apply(qpk_multi* mm, const double* v, double* y);
int qpk_multi_pcg(qpk_multi* mm, const double* rhs, double tol, int tol_is_relative, int64_t max_iters,
                  double* x_out, qpk_pcg_info* info, double* resid_hist);
int64_t qpk_multi_query(qpk_multi* mm, int rank, const char* key);

/* ---- problem upload (once per QpProblem) ------------------------------ */
/* n variables; m_e equality rows (C), m_l rows of A with a finite lower bound,
 * m_u rows of A with a finite upper bound; m_B = m_e + m_l + m_u. */
int qpk_problem_begin(qpk_ctx* ctx, int64_t n, int64_t m_e, int64_t m_l, int64_t m_u);
/* Append rows to B in reference order (C, then A_l, then A_u with sign = -1).
 * row_offsets/col_indices/values: a CSR matrix (int64 offsets and columns as
 * SparseMatrix stores them, model.py:30-33); rows: the row indices of that
 * matrix to append, in order (NULL = all n_rows rows). */
int qpk_problem_add_rows(qpk_ctx* ctx, int64_t n_rows, const int64_t* row_offsets,
                         const int64_t* col_indices, const double* values,
                         const int64_t* rows, int64_t n_sel, double sign);
int qpk_set_hessian_diag(qpk_ctx* ctx, const double* d);
int qpk_set_hessian_csr(qpk_ctx* ctx, const int64_t* row_offsets, const int64_t* col_indices,
                        const double* values);
int qpk_set_hessian_dense(qpk_ctx* ctx, const double* m_rowmajor);
int qpk_set_hessian_lowrank(qpk_ctx* ctx, const double* h0, int64_t k, const double* u_rowmajor,
                            const double* w);
/* dense H from a DEVICE matrix (n x n row-major, copied at finalize): the SVM
 * dual's Gram-based Hessian never leaves the GPU */
int qpk_set_hessian_dense_dev(qpk_ctx* ctx, const double* m_rowmajor_dev);

/* ---- SVM dual frontend ----------------------------
 * H[i][j] = y_i y_j exp(-max(|x_i|^2 + |x_j|^2 - 2 x_i.x_j, 0) / (2 sigma)),
 * exactly symmetric: the Hessian build_svm_dual makes from _gram_matrix
 * (qpipm/svm.py:166-176, 185).  X (n x d row-major), y (n), H (n x n
 * row-major): device pointers; runs on the context's stream.  Usable before
 * or without a problem. */
int qpk_rbf_hessian_dev(qpk_ctx* ctx, const double* X, int64_t n, int64_t d, const double* y, double sigma,
                        double* H);
/* out = H v with the finalized problem's Hessian (hessian_apply, model.py:165-176,
 * without q_extra); dense and diagonal H.  Device pointers. */
int qpk_hessian_apply_dev(qpk_ctx* ctx, const double* v, double* out);
/* out = M v for a dense n x n row-major DEVICE matrix (the SVM decision values
 * g = y o (H alpha), svm.py:194-196, with the Hessian already on the device) */
int qpk_dense_gemv_dev(qpk_ctx* ctx, const double* m_rowmajor_dev, int64_t n, const double* v, double* out);

/* builds the device layout; scatter = QPK_SCATTER_* */
int qpk_problem_finalize(qpk_ctx* ctx, int scatter);

/* ---- per IPM iteration --------------------------------------------------- */
int qpk_set_diagonals(qpk_ctx* ctx, const double* d_diag, const double* q_extra);
int qpk_set_diagonals_dev(qpk_ctx* ctx, const double* d_diag, const double* q_extra);
/* builds the Jacobi diagonal on the device; diag_out (length n+m_B, nullable) receives it */
int qpk_jacobi(qpk_ctx* ctx, double* diag_out);

/* y = K v (length n + m_B) */
int qpk_apply(qpk_ctx* ctx, const double* v, double* y);
int qpk_apply_dev(qpk_ctx* ctx, const double* v, double* y);

/* PCG from x0 = 0.  resid_hist (nullable, length max_iters + 1) receives the
 * recurrence residual norm after each iteration k (index k; index 0 = ||rhs||);
 * entries past info.iterations are untouched. */
int qpk_pcg(qpk_ctx* ctx, const double* rhs, double tol, int tol_is_relative, int64_t max_iters,
            double* x, qpk_pcg_info* info, double* resid_hist);
int qpk_pcg_dev(qpk_ctx* ctx, const double* rhs, double tol, int tol_is_relative, int64_t max_iters,
                double* x, qpk_pcg_info* info, double* resid_hist_dev);

/* ---- device-resident interior-point loop -------
 * qpk_ipm_solve runs qpipm.ipm.solve (ipm.py:185-240) with the iterate,
 * residuals, right-hand side, direction recovery, ratio test and step on the
 * device; only the per-iteration scalars cross to the host.  Single GPU. */
typedef struct {
  double gamma, mu_init, mu_tol, mu_shrink;   /* IpmConfig (ipm.py:31-46) */
  int64_t max_iters;
  double pcg_tol;                             /* PcgConfig (linalg.py:29-39) */
  int64_t pcg_max_iters;
  int32_t pcg_tol_is_relative;
  int32_t verbose;
} qpk_ipm_config;

typedef struct {                              /* TraceRecord (ipm.py:49-59) */
  int32_t iter, cg_iters;
  double mu, primal_inf, dual_inf, compl_inf, cg_resid, alpha_x, alpha_lam;
} qpk_ipm_trace;

typedef struct {
  int32_t status;                             /* 0 converged, 1 iteration_limit, 2 linear_solver_failure */
  int32_t iterations;
  int64_t cg_total;
  double objective;                           /* 1/2 x'Hx + p'x (model.py:257-258) */
  double wall_ms;
} qpk_ipm_result;

/* p (n); bnd (m_B, B-row order: b of the C rows | lower bounds of the A_l rows
 * | upper bounds of the A_u rows); variable bounds as index lists + values. */
int qpk_ipm_set_bounds(qpk_ctx* ctx, const double* p, const double* bnd, int64_t n_lower, const int64_t* var_lower,
                       const double* lower, int64_t n_upper, const int64_t* var_upper, const double* upper);
/* x_out (n, nullable); trace (capacity cfg->max_iters records, nullable) */
int qpk_ipm_solve(qpk_ctx* ctx, const qpk_ipm_config* cfg, double* x_out, qpk_ipm_trace* trace,
                  qpk_ipm_result* result);

/* ---- introspection ------------------------------------------------------ */
/* keys: "n", "m", "nnz", "nnz_padded", "lanes", "scatter", "grid", "block",
 * "sms", "hess_kind", "device_bytes", "kernel_launches" */
int64_t qpk_query(qpk_ctx* ctx, const char* key);

#ifdef __cplusplus
}
#endif
#endif /* QPK_H */
