/*
 * oracle.h -- CPU oracle for the mixed-precision IR / sign-function Newton
 * method of PAPER.md (arXiv 2510.02126, Benner & Liu).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA product path
 * (paper_2510_02126_b200/).
 *
 * Conventions: every matrix is a column-major array of doubles with leading
 * dimension == number of rows.  "Computation at precision p" follows the
 * paper's emulation model (bf16 "simulated by using the
 * chop function"): every elementary operation is evaluated in binary64 and
 * immediately rounded to p (round-to-nearest-even, subnormals kept,
 * overflow -> inf).  p is one of ORC_FP64, ORC_FP32, ORC_FP16, ORC_BF16
 * (Table 1, l.73-95).
 */
#ifndef LYAP_ORACLE_H
#define LYAP_ORACLE_H
#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_FP64 = 0, ORC_FP32 = 1, ORC_FP16 = 2, ORC_BF16 = 3 };

/* Table 1 */
double orc_unit_roundoff(int prec);
double orc_xmin(int prec);
double orc_xmax(int prec);
double orc_round(double x, int prec);      /* fast exact path */
double orc_round_ref(double x, int prec);  /* the definition */
void   orc_round_array(double *x, long len, int prec);

/* precision model of u_s matrix operations: 0 = chop (per operation),
 * 1 = tensor-core (u_s storage, fp32 accumulation); see oracle.c */
void orc_set_model(int model);
int  orc_get_model(void);

/* C(m x n) = op(A) op(B), every product and partial sum rounded to prec,
 * inner products accumulated in index order. */
void orc_gemm(int prec, int ta, int tb, int m, int n, int k,
              const double *A, int lda, const double *B, int ldb,
              double *C, int ldc);

/* LU with partial pivoting (largest |a|, lowest index on ties), in place.
 * piv[j] = row swapped with row j at step j (0-based).
 * returns 0 ok, j+1 on an exactly zero pivot column, -1 on inf/nan. */
int orc_getrf(int prec, int n, double *A, int lda, int *piv);

/* Ainv = A^{-1} via LU + solve against the identity, all at prec.
 * piv (may be NULL) receives the pivot sequence. Same return codes. */
int orc_inverse(int prec, int n, const double *A, double *Ainv, int *piv);
/* same, with log|det A| = sum log|u_ii| of the LU (NULL: not wanted) */
int orc_inverse_ld(int prec, int n, const double *A, double *Ainv, int *piv, double *logabsdet);

/* Thin Householder QR, k = min(m,n): Q (m x k), R (k x n) upper
 * trapezoidal with non-negative diagonal. */
void orc_qr(int prec, int m, int n, const double *A, double *Q, double *R);

/* Symmetric eigendecomposition by cyclic Jacobi at prec.  w descending,
 * V columns matching (largest-|component| made positive).  Returns sweeps. */
int orc_syev(int prec, int n, const double *A, double *w, double *V);

/* RankTruncChol (Algorithm 3 sub-function).
 * Z n x c.  Returns k (columns written into Zout, n x k, capacity n*c). */
int orc_rank_trunc_chol(int prec, int n, int c, const double *Z, double tol_rel,
                        double *Zout);

/* RankTruncLdlt (Algorithm 4 sub-function).
 * Z n x c, Y c x c.  Returns k; Zout n x k, Yout k x k (diagonal). */
int orc_rank_trunc_ldlt(int prec, int n, int c, const double *Z, const double *Y,
                        double *Zout, double *Yout);

/* ---- sign-function Newton iteration (Section 3) ---- */
typedef struct {
    int kmax;          /* maximal Newton steps (50) */
    int scaling;       /* mu_k (l.1139): 0 none, 1 Frobenius norm (l.1406), 2 |det A_k|^{-1/n} */
    int extra;         /* iterations after tolerance (l.1312: 2) */
    double rho;        /* rank truncation threshold (l.1424: 0.1) */
} orc_newton_params;

typedef struct orc_aseq orc_aseq;   /* cached A-side sequence (Section 3.4) */

/* A-side of Algorithms 3/4: A_k = (mu A_{k-1} + mu^{-1} A_{k-1}^{-1})/2. */
orc_aseq *orc_aseq_compute(int prec, int n, const double *A,
                           const orc_newton_params *P, int *info);
int    orc_aseq_steps(const orc_aseq *q);
int    orc_aseq_converged(const orc_aseq *q);
double orc_aseq_mu(const orc_aseq *q, int j);
double orc_aseq_delta(const orc_aseq *q, int j);
double orc_aseq_inf(const orc_aseq *q, int j);   /* ||A_{j+1} + I||_inf */
const double *orc_aseq_inverse(const orc_aseq *q, int j);
const int *orc_aseq_pivots(const orc_aseq *q, int j);
void   orc_aseq_free(orc_aseq *q);

/* Z-side of Algorithm 4 (LDL^T).  Returns the number of columns c of Z;
 * *Zout (n x c) and *Yout (c x c) are malloc'ed (free with orc_free). */
int orc_newton_ldlt_z(int prec, const orc_aseq *q, int n, int m,
                      const double *L, const double *S, double rho,
                      double **Zout, double **Yout, int *ntrunc);
/* Z-side of Algorithm 3 (Cholesky).  Returns c; *Zout n x c malloc'ed. */
int orc_newton_chol_z(int prec, const orc_aseq *q, int n, int m,
                      const double *L, double rho, double **Zout, int *ntrunc);

/* ---- fragments (Section 2) ---- all return the kept rank ---- */
int orc_res_fac_ldlt(int prec, int n, int m, const double *A, const double *L,
                     const double *S, int c, const double *Z, const double *Y,
                     double eta_r, double **Ld, double **Sd, double *resF);
int orc_sol_upt_ldlt(int prec, int n, int c, const double *Z, const double *Y,
                     int cd, const double *Zd, const double *Yd, double eta_s,
                     double **Zn, double **Yn);
int orc_res_fac_chol(int prec, int n, int m, const double *A, const double *L,
                     int c, const double *Z, double eta_r,
                     double **Lp, int *kp, double **Lm, int *km, double *resF);
int orc_sol_upt_chol(int prec, int n, int c, const double *Z, int cp,
                     const double *Zp, int cm, const double *Zm, double eta_s,
                     double **Zn);

/* ---- IR frameworks (Algorithms 1 and 2) ---- */
typedef struct {
    int us, ur, uc;    /* solver / residual / update precisions (u = fp64) */
    double tol;        /* relative-residual tolerance (Eq. res-fac-sol) */
    int imax;          /* maximal refinement steps */
    double eta_r, eta_s;
    orc_newton_params newton;
    int cache;         /* Section 3.4 inverse-sequence cache (results identical) */
} orc_ir_params;

#define ORC_MAX_REPORT 128
typedef struct {
    int steps;                         /* refinement corrections applied */
    int status;                        /* 0 converged, 1 stagnated, 2 max_steps, 3 solver failure */
    int newton_calls, newton_total, newton_max, inversions;
    int nres;                          /* number of residual evaluations */
    double res[ORC_MAX_REPORT];        /* relative residual of Z_1, Z_2, ... */
    int rank[ORC_MAX_REPORT];
    double final_res;
} orc_ir_report;

int orc_ir_ldlt(const orc_ir_params *P, int n, int m, const double *A,
                const double *L, const double *S, double **Z, double **Y,
                orc_ir_report *rep);
int orc_ir_chol(const orc_ir_params *P, int n, int m, const double *A,
                const double *L, double **Z, orc_ir_report *rep);

/* ---- residual and brute force (Eq. lyap-ls, Eq. res-fac-sol) ---- */
/* X (n x n) from (Z, Y) or Z Z^T (Y == NULL). */
void orc_form_x(int n, int c, const double *Z, const double *Y, double *X);
/* relative residual ||AX+XA^T+W||_F / (||W||_F + 2||X||_F ||A||_F), explicit fp64 */
double orc_rel_residual_explicit(int n, const double *A, const double *X, const double *W);
/* Kronecker brute force (I (x) A + A (x) I) vec X = -vec W, fp64, n <= 40 */
int orc_kron_solve(int n, const double *A, const double *W, double *X);

void orc_free(void *p);

#ifdef __cplusplus
}
#endif
#endif
