/*
 * lyap_ir.h -- C ABI of the B200-native mixed-precision iterative-refinement
 * solver for low-rank Lyapunov equations  A X + X A^T + W = 0,  W = L L^T or
 * W = L S L^T  (PAPER.md Eq. eq:lyap l.40-42, Eq. eq:lyap-W-fac l.44-47;
 * Benner & Liu, arXiv 2510.02126).
 *
 * Every entry point below runs entirely in hand-written sm_100a CUDA kernels
 * of liblyapir.so.  There is no CPU fallback: without a CUDA device every
 * call returns LYAP_ERR_CUDA.
 *
 * Conventions
 *  - Precision codes (Table 1, l.73-95): LYAP_FP64=0, LYAP_FP32=1,
 *    LYAP_FP16=2, LYAP_BF16=3.
 *  - A is an n x n matrix stored ROW-MAJOR (C order, element (i,j) at
 *    A[i*n+j]).  Tall factors L (n x m), Z (n x c) are stored COLUMN-MAJOR
 *    (column j contiguous at L + j*n) so that appending the columns
 *    A_k^{-1} Z_k of the factored Newton iteration is a contiguous write.
 *    Small square matrices S, Y are column-major.
 *  - "device" pointers are CUDA global-memory pointers on the current device;
 *    "host" pointers are ordinary CPU memory.  The library never frees
 *    caller memory; it owns only the workspace behind a handle.
 *  - stream: a cudaStream_t passed as void*; NULL = legacy default stream.
 *    All calls are stream-ordered and synchronise the stream before
 *    returning (the IR loop makes host decisions from device scalars).
 *  - Return value: LYAP_OK (0) or a negative error code.
 */
#ifndef LYAP_IR_H
#define LYAP_IR_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define LYAP_FP64 0
#define LYAP_FP32 1
#define LYAP_FP16 2
#define LYAP_BF16 3

#define LYAP_OK              0
#define LYAP_ERR_ARG        -1   /* invalid argument (size, precision, pointer) */
#define LYAP_ERR_CUDA       -2   /* CUDA runtime error or no device */
#define LYAP_ERR_SINGULAR   -3   /* exactly zero pivot column in an inversion */
#define LYAP_ERR_OVERFLOW   -4   /* inf/nan produced in the solver precision */
#define LYAP_ERR_CAPACITY   -5   /* factor width exceeds the handle's max_cols */

/* IR status (PAPER.md Algorithms 1-2 l.284-307 / l.835-858; stagnation rule
 * l.1413-1417). */
#define LYAP_STATUS_CONVERGED 0
#define LYAP_STATUS_STAGNATED 1
#define LYAP_STATUS_MAXSTEPS  2
#define LYAP_STATUS_SOLVER_FAILED 3
#define LYAP_STATUS_CAPACITY  4   /* refinement stopped: the next factor would exceed max_cols */

/* Algorithmic parameters (Section 4.1 l.1419-1428 for defaults). */
typedef struct {
    int    kmax;        /* max Newton steps per solve (l.1422: 50) */
    int    scaling;     /* mu_k (l.1139): 0 none, 1 Frobenius-norm scaling (the
                           paper's choice, l.1406; default), 2 determinantal
                           scaling |det A_k|^{-1/n} from the inversion's pivots */
    int    extra;       /* Newton iterations after Eq. newton-stop-tau holds
                           (reading R-EXTRA: 1, matches Table 3, l.1449) */
    double rho;         /* rank truncation threshold rho (l.1424: 0.1) */
    double eta_r;       /* residual truncation, relative (l.1428: 1e-4) */
    double eta_s;       /* solution truncation, relative (l.1427: 10u) */
    int    cache;       /* reuse the A_k^{-1} sequence across refinement steps
                           (Section 3.4, l.1358-1375): 1 */
    int    newton_cols; /* capacity of the Newton factor Z_k (columns before a
                           truncation); 0 = 2 max(2 max_cols + 64, ceil(rho n)) + 16 */
    int    work_cols;   /* capacity of the fp64 residual / update factors
                           ([Z, AZ, L] and [Z, Z_+, Z_-]); 0 = newton_cols + 2 max_cols + 64 */
} lyap_ir_options;

/* Per-solve report. */
#define LYAP_MAX_REPORT 128
typedef struct {
    int    status;                  /* LYAP_STATUS_* */
    int    steps;                   /* refinement corrections applied */
    int    newton_steps;            /* Newton steps per solver call (alpha) */
    int    newton_calls;            /* solver calls */
    int    inversions;              /* n x n inversions performed */
    int    rank;                    /* columns of the returned Z */
    int    nres;                    /* residual evaluations */
    double res[LYAP_MAX_REPORT];    /* relative residual (Eq. res-fac-sol) of Z_1, Z_2, ... */
    int    ranks[LYAP_MAX_REPORT];
    double final_res;
    double newton_ms, residual_ms, update_ms, total_ms;   /* device time split */
    double newton_flops;            /* algorithmic flops of the inversions (2 n^3 each) */
} lyap_ir_report;

typedef struct lyap_ir_ctx *lyap_ir_handle;

/* Fill *opt with the paper's defaults. */
void lyap_ir_default_options(lyap_ir_options *opt);

/* Create a solver handle for order n, factor widths up to max_cols
 * (max_cols >= 2*ceil(rho*n) recommended) and solver precision us.
 * Allocates all device workspace (A_k in us, the cached inverse sequence,
 * fp64 residual buffers).  opt may be NULL (defaults).  Errors: ARG, CUDA. */
int lyap_ir_create(lyap_ir_handle *h, int n, int max_cols, int us,
                   const lyap_ir_options *opt, void *stream);
int lyap_ir_destroy(lyap_ir_handle h);

/* Solve A X + X A^T + L S L^T = 0 by Algorithm 2 (S != NULL, LDL^T type:
 * X = Z Y Z^T) or Algorithm 1 (S == NULL, Cholesky type: X = Z Z^T), with
 * the sign-function Newton solver (Algorithms 3/4) at precision us and the
 * residual factorization / solution update at ur (LYAP_FP64).
 *   A  device, row-major n x n fp64          (read only)
 *   L  device, column-major n x m fp64       (read only)
 *   S  device, column-major m x m fp64 or NULL
 *   us solver precision u_s (LYAP_FP64/FP32/FP16/BF16, Table 3 l.1078), or -1 for
 *      the handle's current one; a different u_s re-allocates the u_s-typed
 *      workspace and drops the cached A_k^{-1} sequence
 *   ur residual precision u_r: LYAP_FP64 (the only supported value)
 *   tol  relative-residual tolerance (Eq. res-fac-sol), maxit = i_max
 *   Z  device, column-major n x max_cols fp64 (output, first *rank columns)
 *   Y  device, column-major max_cols x max_cols fp64 (output; LDL^T only,
 *      leading *rank x *rank block, diagonal) or NULL
 *   rep  host pointer or NULL.
 * Errors: ARG, CUDA, CAPACITY (only if the initial solve does not fit); solver
 * breakdowns are reported in rep->status = LYAP_STATUS_SOLVER_FAILED, and a factor
 * outgrowing max_cols later in rep->status = LYAP_STATUS_CAPACITY, both with the last
 * iterate returned. */
int lyap_ir_solve(lyap_ir_handle h, const double *A, const double *L, int m,
                  const double *S, int us, int ur, double tol, int maxit,
                  double *Z, double *Y, int *rank, lyap_ir_report *rep);

/* Same, with HOST buffers: copies A, L, S host->device and Z, Y back inside
 * the call (the end-to-end path). */
int lyap_ir_solve_host(lyap_ir_handle h, const double *A, const double *L, int m,
                       const double *S, int us, int ur, double tol, int maxit,
                       double *Z, double *Y, int *rank, lyap_ir_report *rep);

/* ---------------- individual steps of the hot path (for parity tests) ------ */

/* In-place blocked inversion of an n x n row-major matrix in precision prec
 * (Gauss-Jordan sweep = LU with partial pivoting fused with the triangular
 * inversions; Eq. newton-lyapu1 l.1125 needs A_{k-1}^{-1}).
 *   A     device, row-major, element type of prec (double/float/__half/
 *         __nv_bfloat16), overwritten by A^{-1}
 *   ipiv  device int[n] or NULL: LAPACK-style pivots (row j swapped with row
 *         ipiv[j] at step j, 0-based) -- identical to LU with partial pivoting.
 * Errors: ARG, CUDA, SINGULAR, OVERFLOW. */
int lyap_invert(int n, int prec, void *A, int *ipiv, void *stream);

/* A-side of the sign-function Newton iteration (Algorithms 3/4 line 3,
 * Eq. newton-stop-tau l.1309, scaling rules l.1406-1411) on the handle's
 * matrix: A (device fp64 row-major n x n) is rounded to the handle's us and
 * iterated; the inverse sequence is cached in the handle.  Outputs (host):
 * *steps, mu[k], delta[k], infnorm[k] (arrays of length >= opt.kmax, may be
 * NULL).  Returns ARG/CUDA/SINGULAR/OVERFLOW. */
int lyap_newton_aseq(lyap_ir_handle h, const double *A, int *steps,
                     double *mu, double *delta, double *infnorm);

/* Copy cached inverse j (in the handle's us, row-major) to device memory. */
int lyap_newton_get_inverse(lyap_ir_handle h, int j, void *out);

/* Z-side of Algorithm 4 (ldlt=1, S required) or Algorithm 3 (ldlt=0) on the
 * cached A-sequence: L device col-major n x m fp64, S device col-major m x m;
 * Z out device col-major n x max_cols fp64, Y out device max_cols^2 fp64
 * (col-major, leading c x c).  *c receives the column count. */
int lyap_newton_z(lyap_ir_handle h, int ldlt, const double *L, int m,
                  const double *S, double *Z, double *Y, int *c);

/* Thin Householder QR of a column-major m x n fp64 matrix (device):
 * Q m x k, R k x n (k = min(m,n)), diag(R) >= 0 (Fragments 1-4 "thin QR"). */
int lyap_qr(int m, int n, const double *A, double *Q, double *R, void *stream);

/* Symmetric eigendecomposition of a column-major n x n fp64 matrix (device):
 * w descending, V columns (largest-|component| positive). */
int lyap_syev(int n, const double *A, double *w, double *V, void *stream);

/* RankTruncChol (Algorithm 3 sub-function, l.1256-1266) of Z (device
 * col-major n x c fp64) with relative tolerance tol; Zout device n x c,
 * *k receives the kept rank.  Internals fp64, output rounded to prec. */
int lyap_rank_trunc_chol(int n, int c, const double *Z, double tol, int prec,
                         double *Zout, int *k, void *stream);

/* RankTruncLdlt (Algorithm 4 sub-function, l.1295-1304). */
int lyap_rank_trunc_ldlt(int n, int c, const double *Z, const double *Y, int prec,
                         double *Zout, double *Yout, int *k, void *stream);

/* Fragment 3 (l.771-798) / Fragment 1 (l.151-173) at fp64.  Outputs are
 * device buffers sized n x (2c+m) for Ld/Lp/Lm and (2c+m)^2 for Sd; the
 * kept ranks and ||R||_F are returned through host pointers. */
int lyap_res_fac_ldlt(lyap_ir_handle h, const double *A, const double *L, int m,
                      const double *S, int c, const double *Z, const double *Y,
                      double eta_r, double *Ld, double *Sd, int *r, double *resF);
int lyap_res_fac_chol(lyap_ir_handle h, const double *A, const double *L, int m,
                      int c, const double *Z, double eta_r, double *Lp, int *rp,
                      double *Lm, int *rm, double *resF);

/* Fragment 4 (l.809-830) / Fragment 2 (l.226-245) at fp64. */
int lyap_sol_upt_ldlt(lyap_ir_handle h, int c, const double *Z, const double *Y,
                      int cd, const double *Zd, const double *Yd, double eta_s,
                      double *Zn, double *Yn, int *r);
int lyap_sol_upt_chol(lyap_ir_handle h, int c, const double *Z, int cp,
                      const double *Zp, int cm, const double *Zm, double eta_s,
                      double *Zn, int *r);

/* Tensor-core (tcgen05, TMEM accumulator, TMA-fed) product of the 16-bit solver
 * precisions used by the inversion update and the A_k^{-1} Z_k products
 * (Eq. newton-lyapu1 l.1125, Alg. 3/4 line 4):
 *   C = alpha * A * B^T + beta * C
 *   A  device, M x K row-major (ld lda), B device, N x K row-major (ld ldb),
 *   C  device, M x N row-major (ld ldc); all of type prec (LYAP_BF16/LYAP_FP16),
 *   fp32 accumulation.  lda, ldb multiples of 8; A, B 16-byte aligned.
 * Errors: ARG (precision / alignment), CUDA. */
int lyap_tc_gemm(int prec, int M, int N, int K, float alpha, const void *A, long lda,
                 const void *B, long ldb, float beta, void *C, long ldc, void *stream);

/* Number of this library's kernel launches since load (a counter the bench
 * reports as gpu_launches). */
int64_t lyap_launch_count(void);

/* Kernel-class timing for the roofline report: after lyap_kernel_timing(cls)
 * every launch of class cls (0 Gauss-Jordan rank-b update GEMM, 1 pivoted
 * panel, 2 A_k^{-1} Z products, 3 Jacobi eigensolver, 4 Householder QR,
 * 5 fp64 A Z, 6 Newton update, 7 fp64 DMMA GEMM, 8 tcgen05 GEMM, 9 Householder
 * panel, 10 tridiagonalisation, 11 compact-WY application, 12 column-pivoted QR;
 * -1 disables) is bracketed by CUDA events on its
 * launch stream.  lyap_kernel_stats synchronises and returns the summed
 * device milliseconds and the number of timed launches since the last
 * lyap_kernel_timing call. */
int lyap_kernel_timing(int cls);
int lyap_kernel_stats(double *ms, int64_t *launches);
/* Algorithmic flops and bytes of the launches timed since lyap_kernel_timing
 * (classes 7 fp64 DMMA GEMM, 8 tcgen05 GEMM, 9 Householder panel, 10
 * tridiagonalisation, 11 compact-WY application report them). */
int lyap_kernel_work(double *flops, double *bytes);

#ifdef __cplusplus
}
#endif
#endif
