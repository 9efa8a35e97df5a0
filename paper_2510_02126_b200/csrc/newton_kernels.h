// newton_kernels.h -- launchers of newton.cu and the device-scalar layout.
#pragma once
#include <cuda_runtime.h>

namespace lyap {

// device scalar slots (double array `scal`)
enum {
    SC_RED = 0,      // 4 reduction outputs: sum part0, sum part1, max part2, max part3
    SC_MAXA = 4,     // max|A_k|  (range scaling of the inversion)
    SC_NA2 = 5,      // ||A_k||_F^2
    SC_EXP = 6,      // exponent e of the current inversion scaling
    SC_MU = 7,       // Frobenius scaling mu_k
    SC_EL = 8,       // exponent of the right-hand-side factor (Z side, slot 0)
    SC_ES = 9,       // exponent of the inner factor S (Z side)
    SC_EL2 = 10,     // second right-hand side (Cholesky minus equation)
    SC_TR = 11,      // trace results (norms of implied products)
    SC_TR2 = 12,
    SC_MAXB = 13,    // scratch: bit pattern of a grid-wide max|x| (atomicMax on non-negative doubles)
    SC_ORTH = 14,    // ||Z^T Q2||_F^2 of the block Gram-Schmidt fast path
    SC_COUNT = 16
};

int nk_cast(cudaStream_t s, int prec, int n, const double *A, void *Ak, double *part, double *out);
int nk_scale(cudaStream_t s, int prec, long nn, const void *Ak, void *W, double *scal);
int nk_mu(cudaStream_t s, int prec, int n, const void *G, double *part, double *scal, int scaling);
int nk_mu_det(cudaStream_t s, int n, const double *ldet, double *scal, int scaling);
int nk_row_gather(cudaStream_t s, int prec, int n, int c, const void *Z, const int *rowperm, void *out);
int nk_ldexp(cudaStream_t s, int prec, long len, void *x, int e);
int nk_update(cudaStream_t s, int prec, int n, const void *Ak, const void *G, const int *invperm, void *Anext,
              void *Ainv, double *scal, double *part);
int nk_roll(cudaStream_t s, double *scal);
int nk_load_factor(cudaStream_t s, int prec, long len, const double *L, void *Zt, double *scal, int slot);
int nk_load_inner(cudaStream_t s, int prec, int m, const double *S, double *Y, int ldy, double *scal, int slot);
int nk_y_blkdiag(cudaStream_t s, int c, const double *Y, int ldy, double *Yn, int ldn, double a, double b, int prec);
int nk_chol_scale(cudaStream_t s, int prec, long nc, void *Z, double a, double b);
int nk_to_f64(cudaStream_t s, int prec, long len, const void *x, double *y, double f);
int nk_from_f64(cudaStream_t s, int prec, long len, const double *x, void *y);
int nk_finish_factor(cudaStream_t s, int prec, long len, const void *x, double *y, double s1, const double *scal, int slot);
int nk_select(cudaStream_t s, int k, const double *w, double rel, int mode, int *idx, int *cnt);
int nk_gather_cols(cudaStream_t s, int rows, int cnt, const double *V, int ldv, const int *idx, const double *w,
                   int fmode, double *out, int ldo);
int nk_diag_from_sel(cudaStream_t s, int cnt, const double *w, const int *idx, int prec, double *Y, int ldy);
int nk_round(cudaStream_t s, long len, double *x, int prec);
int nk_copy_block(cudaStream_t s, int rows, int cols, const double *a, int lda, double *b, int ldb, double f);
int nk_zero(cudaStream_t s, long len, double *x);
int nk_build_N(cudaStream_t s, int c, int m, const double *Y, int ldy, const double *S, double *N);
int nk_sym_add(cudaStream_t s, int k, double *H, int ldh);
int nk_scale_cols(cudaStream_t s, int k, int c, const double *T, int ldt, const double *D, int ldd, double *out, int ldo);
int nk_build_blkdiag(cudaStream_t s, int c, int cd, const double *Y, int ldy, const double *Yd, int ldyd, int cp,
                     double *U);
int nk_trace_prod(cudaStream_t s, int k, const double *P, double *out);
int nk_sumsq(cudaStream_t s, long len, const double *x, double *out);
int nk_diag_range(cudaStream_t s, int k, const double *R, int ldr, double *out);
int nk_axpy(cudaStream_t s, long len, double a, const double *x, double *y);
int nk_assemble_T(cudaStream_t s, int c, int q, int k2, const double *Rz, const double *R2, double *T);

}  // namespace lyap
