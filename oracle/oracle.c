/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for PAPER.md
 * (Benner & Liu, "Mixed-precision iterative refinement for low-rank Lyapunov
 * equations", arXiv 2510.02126).
 *
 * TEST INFRASTRUCTURE ONLY -- see oracle.h.  Compile with -ffp-contract=off
 * so that every a*b and a+b is a separately rounded binary64 operation which
 * is then rounded again to the emulated precision.
 *
 * Each function names the passage it follows.  "l.N" = PAPER.md line N.
 */
#include "oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>
#include <stdint.h>

#define IDX(i, j, ld) ((long)(i) + (long)(j) * (long)(ld))

/* ------------------------------------------------------------------ */
/* Table 1 (l.73-95): t = significand bits incl. implicit bit, emin.    */
/* ------------------------------------------------------------------ */
static int fmt_t(int p)    { return p == ORC_FP64 ? 53 : p == ORC_FP32 ? 24 : p == ORC_FP16 ? 11 : 8; }
static int fmt_emin(int p) { return p == ORC_FP64 ? -1022 : p == ORC_FP32 ? -126 : p == ORC_FP16 ? -14 : -126; }
static int fmt_emax(int p) { return p == ORC_FP64 ? 1023 : p == ORC_FP32 ? 127 : p == ORC_FP16 ? 15 : 127; }

double orc_unit_roundoff(int p) { return ldexp(1.0, -fmt_t(p)); }
double orc_xmin(int p) { return ldexp(1.0, fmt_emin(p)); }
double orc_xmax(int p) { return ldexp(2.0 - ldexp(1.0, 1 - fmt_t(p)), fmt_emax(p)); }

/* Reference rounding (the definition): round a binary64 value to the nearest
 * value of format p, ties to even.  x = f * 2^e (frexp, f in [0.5,1)) lies in
 * binade [2^E, 2^{E+1}), E = e-1; the spacing there is
 * q = 2^{max(E,emin) - (t-1)}; x/q is exact and nearbyint rounds it to the
 * nearest integer (ties to even, default rounding mode). */
double orc_round_ref(double x, int p)
{
    if (p == ORC_FP64 || x == 0.0 || isnan(x) || isinf(x)) return x;
    int e;
    frexp(x, &e);
    int E = e - 1;
    if (E < fmt_emin(p)) E = fmt_emin(p);
    double q = ldexp(1.0, E - (fmt_t(p) - 1));
    double r = nearbyint(x / q) * q;
    if (fabs(r) > orc_xmax(p)) return copysign(INFINITY, x);
    return r;
}

/* Same function, fast path for results in the normal range of p: add half an
 * ulp (minus one unless the kept lsb is odd: ties to even) to the binary64
 * bit pattern and clear the dropped significand bits; a carry moves into the
 * exponent exactly as rounding up to the next binade does.  Everything else
 * (zero, subnormal range of p, overflow, inf/nan) takes the reference path.
 * tests/test_oracle_pins.py checks fast == reference on random and boundary
 * values for every format. */
static inline double rnd(double x, int p)
{
    if (p == ORC_FP64) return x;
    if (p == ORC_FP32) return (double)(float)x;
    uint64_t b;
    memcpy(&b, &x, 8);
    int ex = (int)((b >> 52) & 0x7ff) - 1023;
    int t = (p == ORC_FP16) ? 11 : 8;
    int emin = (p == ORC_FP16) ? -14 : -126;
    int emax = (p == ORC_FP16) ? 15 : 127;
    if (ex < emin || ex > emax) return orc_round_ref(x, p);
    int sh = 52 - (t - 1);
    uint64_t lsb = (b >> sh) & 1u;
    b += ((uint64_t)1 << (sh - 1)) - 1u + lsb;
    b &= ~(((uint64_t)1 << sh) - 1u);
    double r;
    memcpy(&r, &b, 8);
    double xm = (p == ORC_FP16) ? 65504.0 : 0x1.fep127;
    if (fabs(r) > xm) return copysign(INFINITY, x);
    return r;
}

double orc_round(double x, int p) { return rnd(x, p); }

void orc_round_array(double *x, long len, int p)
{
    if (p == ORC_FP64) return;
    for (long i = 0; i < len; i++) x[i] = rnd(x[i], p);
}

#define FL(x) rnd((x), p)

void orc_free(void *ptr) { free(ptr); }

static double *dalloc(long n) { double *a = (double *)calloc(n > 0 ? n : 1, sizeof(double)); return a; }
static double *dcopy(const double *a, long n) { double *b = dalloc(n); if (n > 0) memcpy(b, a, n * sizeof(double)); return b; }

/* ------------------------------------------------------------------ */
/* Diagnostics in binary64 (norms are diagnostics, l.1396 "residuals    */
/* are computed in fp64 throughout").                                   */
/* ------------------------------------------------------------------ */
static double nrm_fro(long len, const double *a)
{
    double s = 0.0;
    for (long i = 0; i < len; i++) s += a[i] * a[i];
    return sqrt(s);
}

static int exponent_of_max(long len, const double *a)
{
    double mx = 0.0;
    for (long i = 0; i < len; i++) if (fabs(a[i]) > mx) mx = fabs(a[i]);
    if (mx == 0.0 || !isfinite(mx)) return 0;
    int e;
    frexp(mx, &e);           /* mx in [2^{e-1}, 2^e) */
    return e;                /* 2^{-e} * max in [0.5, 1) */
}

/* ------------------------------------------------------------------ */
/* Matrix product at precision p (used for every "A_{k-1}^{-1} Z_{k-1}", */
/* "A Z_i", "T_i N_i T_i^T", ... of the paper).                          */
/* ------------------------------------------------------------------ */
/* Precision model of "computation at precision u_s" for the u_s matrix
 * operations (products, inversions):
 *   ORC_MODEL_CHOP (0): every scalar operation rounded to u_s -- the paper's
 *       chop-based simulation (l.1400-1401);
 *   ORC_MODEL_TC (1): operands and results stored in u_s, inner products and
 *       eliminations carried in fp32 -- the tensor-core arithmetic the paper
 *       targets (fp16 tensor cores with fp32 accumulation, l.67-70).
 * For u_s in {fp32, fp64} both models coincide.  Reading R-TC. */
static int g_model = 0;
void orc_set_model(int model) { g_model = model; }
int orc_get_model(void) { return g_model; }
static int acc_prec(int p) { return (g_model == 1 && (p == ORC_FP16 || p == ORC_BF16)) ? ORC_FP32 : p; }

void orc_gemm(int p, int ta, int tb, int m, int n, int k,
              const double *A, int lda, const double *B, int ldb,
              double *C, int ldc)
{
    const int q = acc_prec(p);     /* accumulation precision */
    for (int j = 0; j < n; j++)
        for (int i = 0; i < m; i++) {
            double s = 0.0;
            for (int l = 0; l < k; l++) {
                double a = ta ? A[IDX(l, i, lda)] : A[IDX(i, l, lda)];
                double b = tb ? B[IDX(j, l, ldb)] : B[IDX(l, j, ldb)];
                double pr = rnd(a * b, q);
                s = (l == 0) ? pr : rnd(s + pr, q);
            }
            C[IDX(i, j, ldc)] = rnd(s, p);
        }
}

/* ------------------------------------------------------------------ */
/* LU with partial pivoting and the inverse (the Newton step's          */
/* A_{k-1}^{-1}, Eq. newton-lyapu1, l.1125).  The paper does not fix the  */
/* inversion method; LU with partial pivoting + solve against I is the   */
/* textbook choice (SPEC kernels.invert).                                */
/* ------------------------------------------------------------------ */
int orc_getrf(int p, int n, double *A, int lda, int *piv)
{
    for (int j = 0; j < n; j++) {
        int ip = j;
        double amax = fabs(A[IDX(j, j, lda)]);
        for (int i = j + 1; i < n; i++) {
            double v = fabs(A[IDX(i, j, lda)]);
            if (v > amax) { amax = v; ip = i; }
        }
        piv[j] = ip;
        if (isnan(amax) || isinf(amax)) return -1;
        if (amax == 0.0) return j + 1;
        if (ip != j)
            for (int k = 0; k < n; k++) {
                double t = A[IDX(j, k, lda)];
                A[IDX(j, k, lda)] = A[IDX(ip, k, lda)];
                A[IDX(ip, k, lda)] = t;
            }
        double d = A[IDX(j, j, lda)];
        for (int i = j + 1; i < n; i++) A[IDX(i, j, lda)] = FL(A[IDX(i, j, lda)] / d);
        for (int k = j + 1; k < n; k++) {
            double u = A[IDX(j, k, lda)];
            if (u == 0.0) continue;            /* a - fl(l*0) == a exactly */
            for (int i = j + 1; i < n; i++)
                A[IDX(i, k, lda)] = FL(A[IDX(i, k, lda)] - FL(A[IDX(i, j, lda)] * u));
        }
    }
    for (long t = 0; t < (long)n * n; t++) if (!isfinite(A[t])) return -1;
    return 0;
}

/* Inverse and, if logabsdet != NULL, log|det A| = sum_i log|u_ii| from the same LU
 * (for the determinantal scaling mu_k = |det A_k|^{-1/n}, l.1139). */
int orc_inverse_ld(int pout, int n, const double *A, double *Ainv, int *piv_out, double *logabsdet)
{
    const int p = acc_prec(pout);   /* TC model: eliminations in fp32, result stored in u_s */
    double *LU = dcopy(A, (long)n * n);
    int *piv = (int *)malloc(sizeof(int) * (n > 0 ? n : 1));
    int info = orc_getrf(p, n, LU, n, piv);
    if (info != 0) { free(LU); free(piv); return info; }
    if (logabsdet) {
        double ld = 0.0;
        for (int i = 0; i < n; i++) ld += log(fabs(LU[IDX(i, i, n)]));
        *logabsdet = ld;
    }
    /* Solve A X = I column by column: X(:,j) = U^{-1} L^{-1} P e_j. */
    double *y = dalloc(n);
    for (int j = 0; j < n; j++) {
        for (int i = 0; i < n; i++) y[i] = (i == j) ? 1.0 : 0.0;
        for (int i = 0; i < n; i++) if (piv[i] != i) { double t = y[i]; y[i] = y[piv[i]]; y[piv[i]] = t; }
        /* forward, unit lower: y_i -= L_il y_l, l increasing */
        for (int l = 0; l < n; l++) {
            double yl = y[l];
            if (yl == 0.0) continue;           /* exact no-op */
            for (int i = l + 1; i < n; i++) y[i] = FL(y[i] - FL(LU[IDX(i, l, n)] * yl));
        }
        /* backward: x_i = (y_i - sum_{l>i} U_il x_l) / U_ii, l decreasing */
        for (int l = n - 1; l >= 0; l--) {
            y[l] = FL(y[l] / LU[IDX(l, l, n)]);
            double xl = y[l];
            if (xl == 0.0) continue;
            for (int i = 0; i < l; i++) y[i] = FL(y[i] - FL(LU[IDX(i, l, n)] * xl));
        }
        for (int i = 0; i < n; i++) Ainv[IDX(i, j, n)] = rnd(y[i], pout);
    }
    if (piv_out) memcpy(piv_out, piv, sizeof(int) * n);
    free(y); free(LU); free(piv);
    for (long t = 0; t < (long)n * n; t++) if (!isfinite(Ainv[t])) return -1;
    return 0;
}

int orc_inverse(int pout, int n, const double *A, double *Ainv, int *piv_out)
{
    return orc_inverse_ld(pout, n, A, Ainv, piv_out, NULL);
}

/* ------------------------------------------------------------------ */
/* Thin Householder QR (Fragments 1-4 "Compute a thin QR decomposition", */
/* l.164, l.239, l.789, l.823; error model l.357 cites Householder QR).  */
/* H_j = I - (2/v^T v) v v^T with v = x - alpha e_1, alpha = -sign(x_1)||x||. */
/* ------------------------------------------------------------------ */
void orc_qr(int p, int m, int n, const double *A, double *Q, double *R)
{
    int k = m < n ? m : n;
    double *W = dcopy(A, (long)m * n);
    double *V = dalloc((long)m * (k > 0 ? k : 1));
    double *vtv = dalloc(k);
    for (int j = 0; j < k; j++) {
        double s = 0.0;
        for (int i = j; i < m; i++) { double t = FL(W[IDX(i, j, m)] * W[IDX(i, j, m)]); s = (i == j) ? t : FL(s + t); }
        double nrm = FL(sqrt(s));
        if (nrm == 0.0) { vtv[j] = 0.0; continue; }
        double x0 = W[IDX(j, j, m)];
        double alpha = (x0 >= 0.0) ? -nrm : nrm;
        double *v = V + (long)j * m;
        v[j] = FL(x0 - alpha);
        for (int i = j + 1; i < m; i++) v[i] = W[IDX(i, j, m)];
        double t2 = 0.0;
        for (int i = j; i < m; i++) { double t = FL(v[i] * v[i]); t2 = (i == j) ? t : FL(t2 + t); }
        vtv[j] = t2;
        W[IDX(j, j, m)] = alpha;
        for (int i = j + 1; i < m; i++) W[IDX(i, j, m)] = 0.0;
        for (int c = j + 1; c < n; c++) {
            double d = 0.0;
            for (int i = j; i < m; i++) { double t = FL(v[i] * W[IDX(i, c, m)]); d = (i == j) ? t : FL(d + t); }
            double f = FL(FL(2.0 * d) / t2);
            for (int i = j; i < m; i++) W[IDX(i, c, m)] = FL(W[IDX(i, c, m)] - FL(f * v[i]));
        }
    }
    /* R = upper k x n part */
    for (int c = 0; c < n; c++)
        for (int i = 0; i < k; i++) R[IDX(i, c, k)] = (i <= c) ? W[IDX(i, c, m)] : 0.0;
    /* Q = H_0 ... H_{k-1} [I_k; 0] */
    for (int c = 0; c < k; c++)
        for (int i = 0; i < m; i++) Q[IDX(i, c, m)] = (i == c) ? 1.0 : 0.0;
    for (int j = k - 1; j >= 0; j--) {
        if (vtv[j] == 0.0) continue;
        double *v = V + (long)j * m;
        for (int c = j; c < k; c++) {
            double d = 0.0;
            for (int i = j; i < m; i++) { double t = FL(v[i] * Q[IDX(i, c, m)]); d = (i == j) ? t : FL(d + t); }
            double f = FL(FL(2.0 * d) / vtv[j]);
            for (int i = j; i < m; i++) Q[IDX(i, c, m)] = FL(Q[IDX(i, c, m)] - FL(f * v[i]));
        }
    }
    /* sign convention: non-negative diag(R) (exact negations) */
    for (int j = 0; j < k; j++)
        if (R[IDX(j, j, k)] < 0.0) {
            for (int c = 0; c < n; c++) R[IDX(j, c, k)] = -R[IDX(j, c, k)];
            for (int i = 0; i < m; i++) Q[IDX(i, j, m)] = -Q[IDX(i, j, m)];
        }
    free(W); free(V); free(vtv);
}

/* ------------------------------------------------------------------ */
/* Symmetric eigendecomposition (Fragment 1 line 3, l.165: "compute a    */
/* spectral decomposition H_i = Q_i Lambda_i Q_i^T").  Cyclic Jacobi,     */
/* Golub & Van Loan sym.schur2 rotations, off-diagonal zeroed exactly.    */
/* ------------------------------------------------------------------ */
int orc_syev(int p, int n, const double *A, double *w, double *V)
{
    double *a = dalloc((long)n * n);
    for (int j = 0; j < n; j++)
        for (int i = 0; i < n; i++)
            a[IDX(i, j, n)] = FL(FL(A[IDX(i, j, n)] + A[IDX(j, i, n)]) * 0.5);
    for (int j = 0; j < n; j++)
        for (int i = 0; i < n; i++) V[IDX(i, j, n)] = (i == j) ? 1.0 : 0.0;
    double fro = nrm_fro((long)n * n, a);
    double u = orc_unit_roundoff(p);
    int sweep;
    for (sweep = 0; sweep < 60; sweep++) {
        double off = 0.0;
        for (int j = 0; j < n; j++) for (int i = 0; i < n; i++) if (i != j) off += a[IDX(i, j, n)] * a[IDX(i, j, n)];
        off = sqrt(off);
        if (off <= u * fro || off == 0.0) break;
        int rotated = 0;
        for (int pp = 0; pp < n - 1; pp++)
            for (int q = pp + 1; q < n; q++) {
                double apq = a[IDX(pp, q, n)];
                /* skip entries already negligible relative to their diagonal pair
                 * (Demmel-Veselic criterion); exact zero always skipped */
                if (apq == 0.0 || fabs(apq) <= u * sqrt(fabs(a[IDX(pp, pp, n)] * a[IDX(q, q, n)]))) continue;
                rotated = 1;
                double app = a[IDX(pp, pp, n)], aqq = a[IDX(q, q, n)];
                double tau = FL(FL(aqq - app) / FL(2.0 * apq));
                double t;
                if (isinf(tau)) t = 0.0;
                else t = (tau >= 0.0 ? 1.0 : -1.0) / FL(fabs(tau) + FL(sqrt(FL(1.0 + FL(tau * tau)))));
                t = FL(t);
                double c = FL(1.0 / FL(sqrt(FL(1.0 + FL(t * t)))));
                double s = FL(t * c);
                for (int kk = 0; kk < n; kk++) {           /* A <- A J */
                    double akp = a[IDX(kk, pp, n)], akq = a[IDX(kk, q, n)];
                    a[IDX(kk, pp, n)] = FL(FL(c * akp) - FL(s * akq));
                    a[IDX(kk, q, n)]  = FL(FL(s * akp) + FL(c * akq));
                }
                for (int kk = 0; kk < n; kk++) {           /* A <- J^T A */
                    double apk = a[IDX(pp, kk, n)], aqk = a[IDX(q, kk, n)];
                    a[IDX(pp, kk, n)] = FL(FL(c * apk) - FL(s * aqk));
                    a[IDX(q, kk, n)]  = FL(FL(s * apk) + FL(c * aqk));
                }
                a[IDX(pp, q, n)] = 0.0;
                a[IDX(q, pp, n)] = 0.0;
                for (int kk = 0; kk < n; kk++) {           /* V <- V J */
                    double vkp = V[IDX(kk, pp, n)], vkq = V[IDX(kk, q, n)];
                    V[IDX(kk, pp, n)] = FL(FL(c * vkp) - FL(s * vkq));
                    V[IDX(kk, q, n)]  = FL(FL(s * vkp) + FL(c * vkq));
                }
            }
        if (!rotated) break;
    }
    /* sort descending (stable selection), normalise eigenvector signs */
    int *ord = (int *)malloc(sizeof(int) * (n > 0 ? n : 1));
    for (int i = 0; i < n; i++) ord[i] = i;
    for (int i = 0; i < n; i++) {
        int b = i;
        for (int j = i + 1; j < n; j++) if (a[IDX(ord[j], ord[j], n)] > a[IDX(ord[b], ord[b], n)]) b = j;
        int t = ord[i]; ord[i] = ord[b]; ord[b] = t;
    }
    double *Vs = dalloc((long)n * n);
    for (int j = 0; j < n; j++) {
        w[j] = a[IDX(ord[j], ord[j], n)];
        int im = 0;
        for (int i = 0; i < n; i++) if (fabs(V[IDX(i, ord[j], n)]) > fabs(V[IDX(im, ord[j], n)])) im = i;
        double sg = V[IDX(im, ord[j], n)] < 0.0 ? -1.0 : 1.0;
        for (int i = 0; i < n; i++) Vs[IDX(i, j, n)] = sg * V[IDX(i, ord[j], n)];
    }
    memcpy(V, Vs, sizeof(double) * (long)n * n);
    free(Vs); free(ord); free(a);
    return sweep;
}

/* ------------------------------------------------------------------ */
/* Reading R-TRUNC-PREC: the rank truncations are O(n c^2)   */
/* side computations; as in the paper's chop-based simulation (only the   */
/* n x n work emulated, l.1400-1401) they run in binary64 and their       */
/* outputs are rounded to the solver precision.  Evidence: with this      */
/* reading the LDL^T bf16 column of Table 3 (n=100, l.1449-1506) is reproduced         */
/* (12(2) at cond 1.3 vs the paper's 12(2)); with emulated internals it   */
/* is 42(2).                                                              */
/* RankTruncChol (l.1256-1266): rank-revealing QR Z^T Pi = Q [T C; 0 S]  */
/* with ||S||_2 <= sqrt(u) ||Z||_2, return Pi [T C]^T.                    */
/* Reading R-RRQR: Householder QR with column pivoting (max   */
/* remaining column norm, lowest index on ties); stop at the first k with */
/* ||S_k||_F <= tol * |r_11|.  Since ||S||_2 <= ||S||_F and |r_11| <=     */
/* ||Z||_2 this implies the paper's condition.                             */
/* ------------------------------------------------------------------ */
int orc_rank_trunc_chol(int pout, int n, int c, const double *Z, double tol_rel, double *Zout)
{
    const int p = ORC_FP64;    /* reading R-TRUNC-PREC: internals in binary64, output at pout */
    /* M = Z^T, c x n column-major */
    double *M = dalloc((long)c * n);
    for (int i = 0; i < c; i++)
        for (int j = 0; j < n; j++) M[IDX(i, j, c)] = Z[IDX(j, i, n)];
    int *perm = (int *)malloc(sizeof(int) * (n > 0 ? n : 1));
    for (int j = 0; j < n; j++) perm[j] = j;
    int kmax = c < n ? c : n;
    int rank = kmax;
    double r11 = 0.0;
    double *v = dalloc(c);
    for (int j = 0; j < kmax; j++) {
        double tr = 0.0;                         /* ||S_j||_F, recomputed */
        for (int col = j; col < n; col++) for (int i = j; i < c; i++) tr += M[IDX(i, col, c)] * M[IDX(i, col, c)];
        tr = sqrt(tr);
        if (j > 0 && tr <= tol_rel * r11) { rank = j; break; }
        if (tr == 0.0) { rank = j; break; }
        int pc = j; double best = -1.0;
        for (int col = j; col < n; col++) {
            double s = 0.0;
            for (int i = j; i < c; i++) s += M[IDX(i, col, c)] * M[IDX(i, col, c)];
            if (s > best) { best = s; pc = col; }
        }
        if (pc != j) {
            for (int i = 0; i < c; i++) { double t = M[IDX(i, j, c)]; M[IDX(i, j, c)] = M[IDX(i, pc, c)]; M[IDX(i, pc, c)] = t; }
            int t = perm[j]; perm[j] = perm[pc]; perm[pc] = t;
        }
        /* Householder on M[j:c, j] */
        double s = 0.0;
        for (int i = j; i < c; i++) { double t = FL(M[IDX(i, j, c)] * M[IDX(i, j, c)]); s = (i == j) ? t : FL(s + t); }
        double nrm = FL(sqrt(s));
        double x0 = M[IDX(j, j, c)];
        double alpha = (x0 >= 0.0) ? -nrm : nrm;
        v[j] = FL(x0 - alpha);
        for (int i = j + 1; i < c; i++) v[i] = M[IDX(i, j, c)];
        double vv = 0.0;
        for (int i = j; i < c; i++) { double t = FL(v[i] * v[i]); vv = (i == j) ? t : FL(vv + t); }
        M[IDX(j, j, c)] = alpha;
        for (int i = j + 1; i < c; i++) M[IDX(i, j, c)] = 0.0;
        if (vv != 0.0)
            for (int col = j + 1; col < n; col++) {
                double d = 0.0;
                for (int i = j; i < c; i++) { double t = FL(v[i] * M[IDX(i, col, c)]); d = (i == j) ? t : FL(d + t); }
                double f = FL(FL(2.0 * d) / vv);
                for (int i = j; i < c; i++) M[IDX(i, col, c)] = FL(M[IDX(i, col, c)] - FL(f * v[i]));
            }
        if (j == 0) r11 = fabs(alpha);
    }
    if (rank == 0) {                             /* all-zero Z: one zero column */
        for (int i = 0; i < n; i++) Zout[i] = 0.0;
        free(M); free(perm); free(v);
        return 1;
    }
    /* Zout(perm[jj], r) = R(r, jj), R = first `rank` rows of M (upper trapezoidal) */
    for (int r = 0; r < rank; r++)
        for (int jj = 0; jj < n; jj++)
            Zout[IDX(perm[jj], r, n)] = (r <= jj) ? rnd(M[IDX(r, jj, c)], pout) : 0.0;
    free(M); free(perm); free(v);
    return rank;
}

/* ------------------------------------------------------------------ */
/* RankTruncLdlt (l.1295-1304): thin QR Z = QR, spectral decomposition   */
/* R Y R^T = V~ Lambda~ V~^T, keep lambda_i > u ||Lambda~||_inf.           */
/* Reading R-LDLT-ABS: kept set is |lambda_i| > u ||Lambda~||  */
/* so that indefinite inner factors (Fragment 3's S_i^Delta) survive.     */
/* ------------------------------------------------------------------ */
int orc_rank_trunc_ldlt(int pout, int n, int c, const double *Z, const double *Y,
                        double *Zout, double *Yout)
{
    const int p = ORC_FP64;    /* reading R-TRUNC-PREC: internals in binary64, output at pout */
    int k = n < c ? n : c;
    double *Q = dalloc((long)n * k), *R = dalloc((long)k * c);
    orc_qr(p, n, c, Z, Q, R);
    double *RY = dalloc((long)k * c), *M = dalloc((long)k * k);
    orc_gemm(p, 0, 0, k, c, c, R, k, Y, c, RY, k);
    orc_gemm(p, 0, 1, k, k, c, RY, k, R, k, M, k);
    double *w = dalloc(k), *V = dalloc((long)k * k);
    orc_syev(p, k, M, w, V);
    double lmax = 0.0;
    for (int i = 0; i < k; i++) if (fabs(w[i]) > lmax) lmax = fabs(w[i]);
    double thr = orc_unit_roundoff(pout) * lmax;
    int r = 0;
    double *Vk = dalloc((long)k * k);
    for (int i = 0; i < k; i++)
        if (fabs(w[i]) > thr) {
            memcpy(Vk + (long)r * k, V + (long)i * k, sizeof(double) * k);
            w[r] = w[i];
            r++;
        }
    orc_gemm(p, 0, 0, n, r, k, Q, n, Vk, k, Zout, n);
    orc_round_array(Zout, (long)n * r, pout);
    for (int j = 0; j < r; j++) for (int i = 0; i < r; i++) Yout[IDX(i, j, r)] = (i == j) ? rnd(w[i], pout) : 0.0;
    free(Q); free(R); free(RY); free(M); free(w); free(V); free(Vk);
    return r;
}

/* ------------------------------------------------------------------ */
/* Sign-function Newton iteration, A-side (Eq. newton-lyapu1 l.1125,      */
/* Algorithms 3/4 line 3, stopping rule Eq. newton-stop-tau l.1309-1315,   */
/* Frobenius scaling l.1139 + l.1406, scaling freeze at delta_k < 1e-2    */
/* and roundoff indicator delta_k > delta_{k-1}/2, l.1406-1411).           */
/* The A-sequence does not depend on Z, so it is computed once and cached  */
/* (Section 3.4, l.1358-1375); every solver call replays it.               */
/* ------------------------------------------------------------------ */
struct orc_aseq {
    int n, prec, k, converged;
    double *inv;      /* k * n * n */
    double mu[256], delta[256], infn[256];
    int *piv;         /* k * n */
};

int orc_aseq_steps(const orc_aseq *q) { return q->k; }
int orc_aseq_converged(const orc_aseq *q) { return q->converged; }
double orc_aseq_mu(const orc_aseq *q, int j) { return q->mu[j]; }
double orc_aseq_delta(const orc_aseq *q, int j) { return q->delta[j]; }
double orc_aseq_inf(const orc_aseq *q, int j) { return q->infn[j]; }
const double *orc_aseq_inverse(const orc_aseq *q, int j) { return q->inv + (long)j * q->n * q->n; }
const int *orc_aseq_pivots(const orc_aseq *q, int j) { return q->piv + (long)j * q->n; }
void orc_aseq_free(orc_aseq *q) { if (q) { free(q->inv); free(q->piv); free(q); } }

orc_aseq *orc_aseq_compute(int p, int n, const double *A, const orc_newton_params *P, int *info)
{
    long nn = (long)n * n;
    int kmax = P->kmax > 255 ? 255 : P->kmax;
    orc_aseq *q = (orc_aseq *)calloc(1, sizeof(orc_aseq));
    q->n = n; q->prec = p;
    q->inv = dalloc(nn * kmax);
    q->piv = (int *)calloc((size_t)n * kmax + 1, sizeof(int));
    double *Ak = dcopy(A, nn);
    orc_round_array(Ak, nn, p);
    double *As = dalloc(nn), *Ai = dalloc(nn), *An = dalloc(nn);
    double tauN = 10.0 * sqrt((double)n * orc_unit_roundoff(p));
    int scaling_on = P->scaling, countdown = -1, in_region = 0;
    double dprev = INFINITY;
    *info = 0;
    for (int it = 1; it <= kmax; it++) {
        /* range scaling by an exact power of two (reading R-RANGE): the
         * inverse of 2^-e A_k is 2^e A_k^{-1}; exact unless under/overflow */
        int e = exponent_of_max(nn, Ak);
        for (long t = 0; t < nn; t++) As[t] = ldexp(Ak[t], -e);
        double ldw = 0.0;
        int r = orc_inverse_ld(p, n, As, Ai, q->piv + (long)(it - 1) * n, &ldw);
        if (r != 0) { *info = r; break; }
        for (long t = 0; t < nn; t++) Ai[t] = FL(ldexp(Ai[t], -e));
        double mu = 1.0;
        int region_step = in_region;   /* convergence region reached at an earlier step */
        if (scaling_on && P->scaling == 2) {
            /* determinantal scaling mu = |det A_k|^{-1/n} (l.1139); det(2^-e A_k) = 2^{-en} det A_k */
            double ld = ldw + (double)n * e * log(2.0);
            if (isfinite(ld)) mu = exp(-ld / (double)n);
            if (!(mu > 0.0) || !isfinite(mu)) mu = 1.0;
        } else if (scaling_on) {
            double na = nrm_fro(nn, Ak), ni = nrm_fro(nn, Ai);
            if (na > 0.0 && ni > 0.0 && isfinite(na) && isfinite(ni)) mu = sqrt(ni / na);
        }
        memcpy(q->inv + (long)(it - 1) * nn, Ai, sizeof(double) * nn);
        q->mu[it - 1] = mu;
        double a = mu, b = 1.0 / mu;
        for (long t = 0; t < nn; t++) An[t] = FL(FL(FL(a * Ak[t]) + FL(b * Ai[t])) * 0.5);
        double dn = 0.0, nn2 = 0.0;
        for (long t = 0; t < nn; t++) { double d = An[t] - Ak[t]; dn += d * d; nn2 += An[t] * An[t]; }
        double delta = sqrt(dn) / sqrt(nn2);
        double inf = 0.0;
        for (int i = 0; i < n; i++) {
            double s = 0.0;
            for (int j = 0; j < n; j++) s += fabs(An[IDX(i, j, n)] + (i == j ? 1.0 : 0.0));
            if (s > inf) inf = s;
        }
        memcpy(Ak, An, sizeof(double) * nn);
        q->delta[it - 1] = delta;
        q->infn[it - 1] = inf;
        q->k = it;
        for (long t = 0; t < nn; t++) if (!isfinite(Ak[t])) { *info = -1; break; }
        if (*info) break;
        /* Higham [FM, sect. 5.8] as adopted at l.1410-1411: once delta_k < 1e-2 the
         * convergence region is reached; scaling stops from the next step on and the
         * roundoff indicator delta_k > delta_{k-1}/2 becomes active (reading R-DELTA). */
        if (delta < 1e-2) { scaling_on = 0; in_region = 1; }
        if (countdown < 0) {
            int trig = (inf <= tauN);
            if (region_step && delta > dprev / 2.0) trig = 1;
            if (trig) {
                q->converged = 1;
                countdown = P->extra;
                if (countdown == 0) break;
            }
        } else {
            countdown--;
            if (countdown == 0) break;
        }
        dprev = delta;
    }
    if (countdown < 0) q->converged = 0;
    free(Ak); free(As); free(Ai); free(An);
    return q;
}

/* Z-side of Algorithm 4 (l.1270-1292, Eq. newton-lyapu-factored-ldlt):
 * Z_k = [Z_{k-1}, A_{k-1}^{-1} Z_{k-1}], Y_k = blkdiag(mu Y, mu^{-1} Y)/2,
 * RankTruncLdlt when size(Z_k,2) > rho n; Y = Y_k / 2. */
int orc_newton_ldlt_z(int p, const orc_aseq *q, int n, int m,
                      const double *L, const double *S, double rho,
                      double **Zout, double **Yout, int *ntrunc)
{
    int eL = exponent_of_max((long)n * m, L), eS = exponent_of_max((long)m * m, S);
    int c = m;
    double *Z = dalloc((long)n * c), *Y = dalloc((long)c * c);
    for (long t = 0; t < (long)n * m; t++) Z[t] = FL(ldexp(L[t], -eL));
    for (long t = 0; t < (long)m * m; t++) Y[t] = FL(ldexp(S[t], -eS));
    int nt = 0;
    for (int j = 0; j < q->k; j++) {
        const double *Ai = q->inv + (long)j * n * n;
        double mu = q->mu[j];
        double *Zn = dalloc((long)n * 2 * c), *Yn = dalloc((long)4 * c * c);
        memcpy(Zn, Z, sizeof(double) * (long)n * c);
        orc_gemm(p, 0, 0, n, c, n, Ai, n, Z, n, Zn + (long)n * c, n);
        double a = mu / 2.0, b = 1.0 / (2.0 * mu);
        for (int jj = 0; jj < c; jj++)
            for (int ii = 0; ii < c; ii++) {
                Yn[IDX(ii, jj, 2 * c)] = FL(a * Y[IDX(ii, jj, c)]);
                Yn[IDX(ii + c, jj + c, 2 * c)] = FL(b * Y[IDX(ii, jj, c)]);
            }
        free(Z); free(Y);
        Z = Zn; Y = Yn; c = 2 * c;
        if ((double)c > rho * n) {
            double *Zt = dalloc((long)n * c), *Yt = dalloc((long)c * c);
            int r = orc_rank_trunc_ldlt(p, n, c, Z, Y, Zt, Yt);
            free(Z); free(Y);
            Z = Zt; Y = Yt; c = r; nt++;
        }
    }
    for (long t = 0; t < (long)n * c; t++) Z[t] = ldexp(Z[t], eL);
    for (long t = 0; t < (long)c * c; t++) Y[t] = ldexp(Y[t], eS - 1);   /* Y = Y_k / 2 */
    *Zout = Z; *Yout = Y;
    if (ntrunc) *ntrunc = nt;
    return c;
}

/* Z-side of Algorithm 3 (l.1231-1252, Eq. newton-lyapu-factored-chol):
 * Z_k = [mu^{1/2} Z_{k-1}, mu^{-1/2} A_{k-1}^{-1} Z_{k-1}] / sqrt(2),
 * RankTruncChol with tolerance sqrt(u) when size(Z_k,2) > rho n; Z = Z_k/sqrt2. */
int orc_newton_chol_z(int p, const orc_aseq *q, int n, int m,
                      const double *L, double rho, double **Zout, int *ntrunc)
{
    int eL = exponent_of_max((long)n * m, L);
    int c = m;
    double *Z = dalloc((long)n * c);
    for (long t = 0; t < (long)n * m; t++) Z[t] = FL(ldexp(L[t], -eL));
    int nt = 0;
    double tol = sqrt(orc_unit_roundoff(p));
    for (int j = 0; j < q->k; j++) {
        const double *Ai = q->inv + (long)j * n * n;
        double mu = q->mu[j];
        double a = sqrt(mu / 2.0), b = 1.0 / sqrt(2.0 * mu);
        double *Zn = dalloc((long)n * 2 * c);
        orc_gemm(p, 0, 0, n, c, n, Ai, n, Z, n, Zn + (long)n * c, n);
        for (long t = 0; t < (long)n * c; t++) {
            Zn[t] = FL(a * Z[t]);
            Zn[(long)n * c + t] = FL(b * Zn[(long)n * c + t]);
        }
        free(Z); Z = Zn; c = 2 * c;
        if ((double)c > rho * n) {
            double *Zt = dalloc((long)n * c);
            int r = orc_rank_trunc_chol(p, n, c, Z, tol, Zt);
            free(Z); Z = Zt; c = r; nt++;
        }
    }
    double is2 = 1.0 / sqrt(2.0);
    for (long t = 0; t < (long)n * c; t++) Z[t] = ldexp(FL(Z[t] * is2), eL);
    *Zout = Z;
    if (ntrunc) *ntrunc = nt;
    return c;
}

/* ------------------------------------------------------------------ */
/* Fragment 3 ResFacLdlt (l.771-798).  Reading R-TRUNC-REL: the kept set */
/* is |lambda_j| >= eta_r max|lambda| (analysis l.520 uses relative       */
/* truncation ||Lambda_{i,0}|| <= eta_r ||Lambda_i||).                    */
/* resF = sqrt(sum lambda_j^2) = ||R||_F (l.311, "readily available").    */
/* ------------------------------------------------------------------ */
static int build_F(int p, int n, int m, const double *A, const double *L, int c, const double *Z, double **Fout)
{
    int pc = 2 * c + m;
    double *F = dalloc((long)n * pc);
    memcpy(F, Z, sizeof(double) * (long)n * c);
    orc_gemm(p, 0, 0, n, c, n, A, n, Z, n, F + (long)n * c, n);
    memcpy(F + (long)n * 2 * c, L, sizeof(double) * (long)n * m);
    *Fout = F;
    return pc;
}

static int select_abs(int k, const double *w, double thr, int *idx, int sign)
{
    int r = 0;
    for (int i = 0; i < k; i++) {
        if (sign == 0 && fabs(w[i]) >= thr) idx[r++] = i;
        if (sign > 0 && w[i] >= thr) idx[r++] = i;
        if (sign < 0 && w[i] <= -thr) idx[r++] = i;
    }
    return r;
}

int orc_res_fac_ldlt(int p, int n, int m, const double *A, const double *L,
                     const double *S, int c, const double *Z, const double *Y,
                     double eta_r, double **Ld, double **Sd, double *resF)
{
    double *F;
    int pc = build_F(p, n, m, A, L, c, Z, &F);
    double *N = dalloc((long)pc * pc);
    for (int j = 0; j < c; j++)
        for (int i = 0; i < c; i++) {
            N[IDX(i, c + j, pc)] = Y[IDX(i, j, c)];
            N[IDX(c + i, j, pc)] = Y[IDX(i, j, c)];
        }
    for (int j = 0; j < m; j++)
        for (int i = 0; i < m; i++) N[IDX(2 * c + i, 2 * c + j, pc)] = S[IDX(i, j, m)];
    int k = n < pc ? n : pc;
    double *U = dalloc((long)n * k), *T = dalloc((long)k * pc);
    orc_qr(p, n, pc, F, U, T);
    double *TN = dalloc((long)k * pc), *H = dalloc((long)k * k);
    orc_gemm(p, 0, 0, k, pc, pc, T, k, N, pc, TN, k);
    orc_gemm(p, 0, 1, k, k, pc, TN, k, T, k, H, k);
    double *w = dalloc(k), *Qh = dalloc((long)k * k);
    orc_syev(p, k, H, w, Qh);
    double s2 = 0.0, lmax = 0.0;
    for (int i = 0; i < k; i++) { s2 += w[i] * w[i]; if (fabs(w[i]) > lmax) lmax = fabs(w[i]); }
    *resF = sqrt(s2);
    int *idx = (int *)malloc(sizeof(int) * (k > 0 ? k : 1));
    int r = select_abs(k, w, eta_r * lmax, idx, 0);
    double *Qt = dalloc((long)k * r);
    for (int j = 0; j < r; j++) memcpy(Qt + (long)j * k, Qh + (long)idx[j] * k, sizeof(double) * k);
    double *Lo = dalloc((long)n * r), *So = dalloc((long)r * r);
    orc_gemm(p, 0, 0, n, r, k, U, n, Qt, k, Lo, n);
    for (int j = 0; j < r; j++) So[IDX(j, j, r)] = w[idx[j]];
    *Ld = Lo; *Sd = So;
    free(F); free(N); free(U); free(T); free(TN); free(H); free(w); free(Qh); free(idx); free(Qt);
    return r;
}

/* Fragment 4 SolUptLdlt (l.809-830): G = [Z, Z^D], Upsilon = blkdiag(Y, Y^D),
 * G = V Gamma, K = Gamma Upsilon Gamma^T = Theta Sigma Theta^T, keep
 * sigma_j >= eta_s max|sigma| (reading R-TRUNC-REL), Y = diag, Z = V Theta_t. */
int orc_sol_upt_ldlt(int p, int n, int c, const double *Z, const double *Y,
                     int cd, const double *Zd, const double *Yd, double eta_s,
                     double **Zn, double **Yn)
{
    int pc = c + cd;
    double *G = dalloc((long)n * pc), *Ups = dalloc((long)pc * pc);
    memcpy(G, Z, sizeof(double) * (long)n * c);
    memcpy(G + (long)n * c, Zd, sizeof(double) * (long)n * cd);
    for (int j = 0; j < c; j++) for (int i = 0; i < c; i++) Ups[IDX(i, j, pc)] = Y[IDX(i, j, c)];
    for (int j = 0; j < cd; j++) for (int i = 0; i < cd; i++) Ups[IDX(c + i, c + j, pc)] = Yd[IDX(i, j, cd)];
    int k = n < pc ? n : pc;
    double *V = dalloc((long)n * k), *Gm = dalloc((long)k * pc);
    orc_qr(p, n, pc, G, V, Gm);
    double *GU = dalloc((long)k * pc), *K = dalloc((long)k * k);
    orc_gemm(p, 0, 0, k, pc, pc, Gm, k, Ups, pc, GU, k);
    orc_gemm(p, 0, 1, k, k, pc, GU, k, Gm, k, K, k);
    double *w = dalloc(k), *Th = dalloc((long)k * k);
    orc_syev(p, k, K, w, Th);
    double smax = 0.0;
    for (int i = 0; i < k; i++) if (fabs(w[i]) > smax) smax = fabs(w[i]);
    int *idx = (int *)malloc(sizeof(int) * (k > 0 ? k : 1));
    int r = select_abs(k, w, eta_s * smax, idx, +1);
    double *Tt = dalloc((long)k * r);
    for (int j = 0; j < r; j++) memcpy(Tt + (long)j * k, Th + (long)idx[j] * k, sizeof(double) * k);
    double *Zo = dalloc((long)n * r), *Yo = dalloc((long)r * r);
    orc_gemm(p, 0, 0, n, r, k, V, n, Tt, k, Zo, n);
    for (int j = 0; j < r; j++) Yo[IDX(j, j, r)] = w[idx[j]];
    *Zn = Zo; *Yn = Yo;
    free(G); free(Ups); free(V); free(Gm); free(GU); free(K); free(w); free(Th); free(idx); free(Tt);
    return r;
}

/* Fragment 1 ResFacChol (l.151-173): P_i = [0 I 0; I 0 0; 0 0 I] (l.208),
 * L+ = U Q+ (Lambda+)^{1/2}, L- = U Q- (-Lambda-)^{1/2}. */
int orc_res_fac_chol(int p, int n, int m, const double *A, const double *L,
                     int c, const double *Z, double eta_r,
                     double **Lp, int *kp, double **Lm, int *km, double *resF)
{
    double *F;
    int pc = build_F(p, n, m, A, L, c, Z, &F);
    int k = n < pc ? n : pc;
    double *U = dalloc((long)n * k), *T = dalloc((long)k * pc);
    orc_qr(p, n, pc, F, U, T);
    /* T P: swap column blocks 1 and 2 (exact permutation, l.404) */
    double *TP = dalloc((long)k * pc);
    for (int j = 0; j < pc; j++) {
        int src = j < c ? c + j : (j < 2 * c ? j - c : j);
        memcpy(TP + (long)j * k, T + (long)src * k, sizeof(double) * k);
    }
    double *H = dalloc((long)k * k);
    orc_gemm(p, 0, 1, k, k, pc, TP, k, T, k, H, k);
    double *w = dalloc(k), *Qh = dalloc((long)k * k);
    orc_syev(p, k, H, w, Qh);
    double s2 = 0.0, lmax = 0.0;
    for (int i = 0; i < k; i++) { s2 += w[i] * w[i]; if (fabs(w[i]) > lmax) lmax = fabs(w[i]); }
    *resF = sqrt(s2);
    int *ip = (int *)malloc(sizeof(int) * (k + 1)), *im = (int *)malloc(sizeof(int) * (k + 1));
    int rp = select_abs(k, w, eta_r * lmax, ip, +1);
    int rm = select_abs(k, w, eta_r * lmax, im, -1);
    double *Qp = dalloc((long)k * rp), *Qm = dalloc((long)k * rm);
    for (int j = 0; j < rp; j++) {
        double sq = FL(sqrt(w[ip[j]]));
        for (int i = 0; i < k; i++) Qp[IDX(i, j, k)] = FL(Qh[IDX(i, ip[j], k)] * sq);
    }
    for (int j = 0; j < rm; j++) {
        double sq = FL(sqrt(-w[im[j]]));
        for (int i = 0; i < k; i++) Qm[IDX(i, j, k)] = FL(Qh[IDX(i, im[j], k)] * sq);
    }
    double *Lpo = dalloc((long)n * rp), *Lmo = dalloc((long)n * rm);
    orc_gemm(p, 0, 0, n, rp, k, U, n, Qp, k, Lpo, n);
    orc_gemm(p, 0, 0, n, rm, k, U, n, Qm, k, Lmo, n);
    *Lp = Lpo; *kp = rp; *Lm = Lmo; *km = rm;
    free(F); free(U); free(T); free(TP); free(H); free(w); free(Qh); free(ip); free(im); free(Qp); free(Qm);
    return rp + rm;
}

/* Fragment 2 SolUptChol (l.226-245): G = [Z, Z+, Z-], J = blkdiag(I, I, -I),
 * K = Gamma J Gamma^T, keep sigma_j >= eta_s max|sigma|, Z = V Theta+ Sigma+^{1/2}. */
int orc_sol_upt_chol(int p, int n, int c, const double *Z, int cp,
                     const double *Zp, int cm, const double *Zm, double eta_s,
                     double **Zn)
{
    int pc = c + cp + cm;
    double *G = dalloc((long)n * pc);
    memcpy(G, Z, sizeof(double) * (long)n * c);
    memcpy(G + (long)n * c, Zp, sizeof(double) * (long)n * cp);
    memcpy(G + (long)n * (c + cp), Zm, sizeof(double) * (long)n * cm);
    int k = n < pc ? n : pc;
    double *V = dalloc((long)n * k), *Gm = dalloc((long)k * pc);
    orc_qr(p, n, pc, G, V, Gm);
    double *GJ = dalloc((long)k * pc);
    for (long t = 0; t < (long)k * pc; t++) GJ[t] = (t / k >= c + cp) ? -Gm[t] : Gm[t];
    double *K = dalloc((long)k * k);
    orc_gemm(p, 0, 1, k, k, pc, GJ, k, Gm, k, K, k);
    double *w = dalloc(k), *Th = dalloc((long)k * k);
    orc_syev(p, k, K, w, Th);
    double smax = 0.0;
    for (int i = 0; i < k; i++) if (fabs(w[i]) > smax) smax = fabs(w[i]);
    int *idx = (int *)malloc(sizeof(int) * (k + 1));
    int r = select_abs(k, w, eta_s * smax, idx, +1);
    double *Tt = dalloc((long)k * r);
    for (int j = 0; j < r; j++) {
        double sq = FL(sqrt(w[idx[j]]));
        for (int i = 0; i < k; i++) Tt[IDX(i, j, k)] = FL(Th[IDX(i, idx[j], k)] * sq);
    }
    double *Zo = dalloc((long)n * r);
    orc_gemm(p, 0, 0, n, r, k, V, n, Tt, k, Zo, n);
    *Zn = Zo;
    free(G); free(V); free(Gm); free(GJ); free(K); free(w); free(Th); free(idx); free(Tt);
    return r;
}

/* ------------------------------------------------------------------ */
/* Norms for Eq. res-fac-sol (l.1384-1394), evaluated in fp64 without    */
/* forming n x n products: ||Z Y Z^T||_F = ||R Y R^T||_F for Z = QR.      */
/* ------------------------------------------------------------------ */
static double fro_ZYZt(int n, int c, const double *Z, const double *Y)
{
    if (c == 0) return 0.0;
    int k = n < c ? n : c;
    double *Q = dalloc((long)n * k), *R = dalloc((long)k * c);
    orc_qr(ORC_FP64, n, c, Z, Q, R);
    double *RY = dalloc((long)k * c), *M = dalloc((long)k * k);
    if (Y) {
        orc_gemm(ORC_FP64, 0, 0, k, c, c, R, k, Y, c, RY, k);
        orc_gemm(ORC_FP64, 0, 1, k, k, c, RY, k, R, k, M, k);
    } else {
        orc_gemm(ORC_FP64, 0, 1, k, k, c, R, k, R, k, M, k);
    }
    double f = nrm_fro((long)k * k, M);
    free(Q); free(R); free(RY); free(M);
    return f;
}

/* ------------------------------------------------------------------ */
/* Algorithm 2: mixed-precision LDL^T-type IR (l.835-858), stagnation    */
/* rule theta_i > 0.9 twice in a row (l.1413-1417).  Reading R-TOL: the  */
/* convergence test is on the relative residual of Eq. res-fac-sol.      */
/* ------------------------------------------------------------------ */
int orc_ir_ldlt(const orc_ir_params *P, int n, int m, const double *A,
                const double *L, const double *S, double **Zo, double **Yo,
                orc_ir_report *rep)
{
    memset(rep, 0, sizeof(*rep));
    int info = 0;
    orc_aseq *q = orc_aseq_compute(P->us, n, A, &P->newton, &info);
    rep->inversions += q->k;
    if (info != 0) { orc_aseq_free(q); rep->status = 3; *Zo = dalloc(1); *Yo = dalloc(1); return 0; }
    double *Z, *Y;
    int c = orc_newton_ldlt_z(P->us, q, n, m, L, S, P->newton.rho, &Z, &Y, NULL);
    rep->newton_calls = 1; rep->newton_total = q->k; rep->newton_max = q->k;
    double nA = nrm_fro((long)n * n, A);
    double nW = fro_ZYZt(n, m, L, S);
    int stagn = 0;
    rep->status = 2;
    for (int i = 1; ; i++) {
        double *Ld, *Sd, resF;
        int r = orc_res_fac_ldlt(P->ur, n, m, A, L, S, c, Z, Y, P->eta_r, &Ld, &Sd, &resF);
        double rel = resF / (nW + 2.0 * fro_ZYZt(n, c, Z, Y) * nA);
        if (rep->nres < ORC_MAX_REPORT) { rep->res[rep->nres] = rel; rep->rank[rep->nres] = c; }
        rep->nres++;
        rep->final_res = rel;
        int stop = 0;
        if (rel <= P->tol) { rep->status = 0; stop = 1; }
        else if (i >= 2) {
            double theta = rel / rep->res[rep->nres - 2];
            stagn = (theta > 0.9) ? stagn + 1 : 0;
            if (stagn >= 2) { rep->status = 1; stop = 1; }
        }
        if (!stop && i > P->imax) { rep->status = 2; stop = 1; }
        if (stop) { free(Ld); free(Sd); break; }
        /* round L^D, S^D to u_s happens inside the solver (first FL) */
        if (!P->cache) {
            orc_aseq_free(q);
            q = orc_aseq_compute(P->us, n, A, &P->newton, &info);
            rep->inversions += q->k;
        }
        double *Zd, *Yd;
        int cd = orc_newton_ldlt_z(P->us, q, n, r, Ld, Sd, P->newton.rho, &Zd, &Yd, NULL);
        rep->newton_calls++; rep->newton_total += q->k;
        double *Zn, *Yn;
        int cn = orc_sol_upt_ldlt(P->uc, n, c, Z, Y, cd, Zd, Yd, P->eta_s, &Zn, &Yn);
        free(Z); free(Y); free(Zd); free(Yd); free(Ld); free(Sd);
        Z = Zn; Y = Yn; c = cn;
        rep->steps = i;
    }
    orc_aseq_free(q);
    *Zo = Z; *Yo = Y;
    return c;
}

/* Algorithm 1: mixed-precision Cholesky-type IR (l.284-307).  The two
 * correction equations share the A-sequence (l.1333-1336). */
int orc_ir_chol(const orc_ir_params *P, int n, int m, const double *A,
                const double *L, double **Zo, orc_ir_report *rep)
{
    memset(rep, 0, sizeof(*rep));
    int info = 0;
    orc_aseq *q = orc_aseq_compute(P->us, n, A, &P->newton, &info);
    rep->inversions += q->k;
    if (info != 0) { orc_aseq_free(q); rep->status = 3; *Zo = dalloc(1); return 0; }
    double *Z;
    int c = orc_newton_chol_z(P->us, q, n, m, L, P->newton.rho, &Z, NULL);
    rep->newton_calls = 1; rep->newton_total = q->k; rep->newton_max = q->k;
    double nA = nrm_fro((long)n * n, A);
    double nW = fro_ZYZt(n, m, L, NULL);
    int stagn = 0;
    for (int i = 1; ; i++) {
        double *Lp, *Lm, resF;
        int kp, km;
        orc_res_fac_chol(P->ur, n, m, A, L, c, Z, P->eta_r, &Lp, &kp, &Lm, &km, &resF);
        double rel = resF / (nW + 2.0 * fro_ZYZt(n, c, Z, NULL) * nA);
        if (rep->nres < ORC_MAX_REPORT) { rep->res[rep->nres] = rel; rep->rank[rep->nres] = c; }
        rep->nres++;
        rep->final_res = rel;
        int stop = 0;
        if (rel <= P->tol) { rep->status = 0; stop = 1; }
        else if (i >= 2) {
            double theta = rel / rep->res[rep->nres - 2];
            stagn = (theta > 0.9) ? stagn + 1 : 0;
            if (stagn >= 2) { rep->status = 1; stop = 1; }
        }
        if (!stop && i > P->imax) { rep->status = 2; stop = 1; }
        if (stop) { free(Lp); free(Lm); break; }
        if (!P->cache) {
            orc_aseq_free(q);
            q = orc_aseq_compute(P->us, n, A, &P->newton, &info);
            rep->inversions += q->k;
        }
        double *Zp = NULL, *Zm = NULL;
        int cp = 0, cm = 0;
        if (kp > 0) cp = orc_newton_chol_z(P->us, q, n, kp, Lp, P->newton.rho, &Zp, NULL);
        else Zp = dalloc(1);
        if (km > 0) cm = orc_newton_chol_z(P->us, q, n, km, Lm, P->newton.rho, &Zm, NULL);
        else Zm = dalloc(1);
        rep->newton_calls++; rep->newton_total += q->k;
        double *Zn;
        int cn = orc_sol_upt_chol(P->uc, n, c, Z, cp, Zp, cm, Zm, P->eta_s, &Zn);
        free(Z); free(Zp); free(Zm); free(Lp); free(Lm);
        Z = Zn; c = cn;
        rep->steps = i;
    }
    orc_aseq_free(q);
    *Zo = Z;
    return c;
}

/* ------------------------------------------------------------------ */
/* Brute force and explicit residual (Eq. lyap-ls l.122-128;             */
/* Eq. res-fac-sol l.1384-1394).                                         */
/* ------------------------------------------------------------------ */
void orc_form_x(int n, int c, const double *Z, const double *Y, double *X)
{
    double *ZY = dalloc((long)n * (c > 0 ? c : 1));
    if (Y) orc_gemm(ORC_FP64, 0, 0, n, c, c, Z, n, Y, c, ZY, n);
    else memcpy(ZY, Z, sizeof(double) * (long)n * c);
    orc_gemm(ORC_FP64, 0, 1, n, n, c, ZY, n, Z, n, X, n);
    free(ZY);
}

double orc_rel_residual_explicit(int n, const double *A, const double *X, const double *W)
{
    double *AX = dalloc((long)n * n), *XAt = dalloc((long)n * n);
    orc_gemm(ORC_FP64, 0, 0, n, n, n, A, n, X, n, AX, n);
    orc_gemm(ORC_FP64, 0, 1, n, n, n, X, n, A, n, XAt, n);
    double num = 0.0;
    for (long t = 0; t < (long)n * n; t++) { double r = AX[t] + XAt[t] + W[t]; num += r * r; }
    double den = nrm_fro((long)n * n, W) + 2.0 * nrm_fro((long)n * n, X) * nrm_fro((long)n * n, A);
    free(AX); free(XAt);
    return sqrt(num) / den;
}

int orc_kron_solve(int n, const double *A, const double *W, double *X)
{
    if (n > 40) return -2;
    int N = n * n;
    double *M = dalloc((long)N * N), *b = dalloc(N);
    /* M = I (x) A + A (x) I ; (I (x) A)_{(i,j),(k,l)} = d_jl a_ik, (A (x) I) = a_jl d_ik,
     * with vec index (i,j) -> i + j n (column stacking). */
    for (int j = 0; j < n; j++)
        for (int i = 0; i < n; i++)
            for (int l = 0; l < n; l++)
                for (int k = 0; k < n; k++) {
                    double v = 0.0;
                    if (j == l) v += A[IDX(i, k, n)];
                    if (i == k) v += A[IDX(j, l, n)];
                    M[IDX(i + j * n, k + l * n, N)] = v;
                }
    for (int t = 0; t < N; t++) b[t] = -W[t];
    int *piv = (int *)malloc(sizeof(int) * N);
    int info = orc_getrf(ORC_FP64, N, M, N, piv);
    if (info == 0) {
        for (int i = 0; i < N; i++) if (piv[i] != i) { double t = b[i]; b[i] = b[piv[i]]; b[piv[i]] = t; }
        for (int l = 0; l < N; l++) for (int i = l + 1; i < N; i++) b[i] -= M[IDX(i, l, N)] * b[l];
        for (int l = N - 1; l >= 0; l--) { b[l] /= M[IDX(l, l, N)]; for (int i = 0; i < l; i++) b[i] -= M[IDX(i, l, N)] * b[l]; }
        for (int j = 0; j < n; j++)
            for (int i = 0; i < n; i++) X[IDX(i, j, n)] = 0.5 * (b[i + j * n] + b[j + i * n]);
    }
    free(M); free(b); free(piv);
    return info;
}
