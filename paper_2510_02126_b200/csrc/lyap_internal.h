// lyap_internal.h -- internal interfaces between the library's translation units.
#pragma once
#include <cuda_runtime.h>
#include <cstddef>

namespace lyap {

// Workspace of the blocked Gauss-Jordan inversion (gje.cu).
// outer block of the two-level Gauss-Jordan scheme (16-bit types and fp32).  Measured with the
// implicit-pivoting sweep (ms per fp16 inversion at n = 4096 / 8192 / 16384): 128 columns 6.37 /
// 17.6 / 47.5, 192: 6.34 / 17.3 / 44.0, 256: 6.21 / 17.0 / 42.3, 384: 6.20 / 17.4 / 43.4, 512: 6.29 /
// 17.7 / 43.9, 1024: 6.58 / 19.1 / 49.2 -- narrower blocks halve the rank-32 updates' traffic, and
// the look-ahead hides the extra rank-NB updates
constexpr int GJE_NB = 256;
constexpr int GJE_NB_MAX = 1024;   // capacity of the outer-block workspace (tuning of gje_ip.cu's block)
struct GjeWork {
    int n = 0, prec = 0;
    void *X = nullptr, *B = nullptr, *tmp = nullptr, *Pglob = nullptr, *Tg = nullptr, *Bo = nullptr, *tmp2 = nullptr;
    int *oints = nullptr, *omoved = nullptr, *onmoved = nullptr, *slot_of = nullptr, *invprev = nullptr;
    cudaStream_t side = nullptr;          // look-ahead stream of the two-level scheme
    cudaEvent_t ev_a = nullptr, ev_b = nullptr;
    int *ints = nullptr;
    int *ipiv = nullptr, *rowperm = nullptr, *invperm = nullptr, *moved = nullptr;
    int *nmoved = nullptr, *info = nullptr, *tmp_perm = nullptr;
    double *ldet = nullptr;               // log|pivot| sums per panel start (log|det| of the matrix)
    int alloc(int n, int prec);
    void release();
};

int gje_invert(cudaStream_t s, int n, int prec, void *A, GjeWork &w);
// implicit-pivoting sweep (gje_ip.cu): A is destroyed, the result (gje_invert's layout) goes to G != A
bool gje_ip_eligible(int n, int prec, const GjeWork &w);
int gje_ip_invert(cudaStream_t s, int n, int prec, void *A, void *G, GjeWork &w);
// LYAP_GEMM=simt routes the 16-bit products through the SIMT kernel (cross-checking)
inline bool use_simt_gemm() {
    static int v = -1;
    if (v < 0) { const char *e = getenv("LYAP_GEMM"); v = (e && e[0] == 's') ? 1 : 0; }
    return v == 1;
}
// tcgen05 GEMM (tc_gemm.cu): C = alpha A B^T + beta C, 16-bit A (M x K), B (N x K) row-major
// max_ctas > 0 caps the persistent kernel's grid (SMs left free for concurrent work), < 0: one CTA per
// tile; pdl: programmatic dependent launch (the kernel's setup overlaps the previous kernel's tail)
int tc_gemm(cudaStream_t s, int prec, int M, int N, int K, float alpha, const void *A, long lda, const void *B,
            long ldb, float beta, void *C, long ldc, int colmajor, int max_ctas = 0, bool pdl = false);
// rank-32 update C (M x N, ld ldc) += X (M x 32) Bt^T (Bt: N x 32), 16-bit storage (rank_update.cu)
bool rank32_update_ok(int prec, int N, const void *X, const void *Bt, const void *C, long ldc);
int rank32_update(cudaStream_t s, int prec, int M, int N, const void *X, const void *Bt, void *C, long ldc,
                  bool pdl = false);
// the same with the X tile formed in the kernel from the panel's export (see rank_update.cu)
int rank32_fused_update(cudaStream_t s, int prec, int M, int N, int k, int K0, const float *P, const float *TL,
                        const int *pos, const void *Bt, void *C, long ldc, bool pdl = false);
int col_gather(cudaStream_t s, int n, int prec, const void *G, const int *invperm, void *out);
template <typename T> int gemm_update(cudaStream_t s, int n, int b, const T *X, const T *B, T *A);

// fp64 dense kernels (qr.cu, eig.cu, rrqr.cu)
struct QrWork {
    int mmax = 0, nmax = 0;
    double *V = nullptr, *T = nullptr, *W = nullptr, *tau = nullptr, *Wk = nullptr;
    double *gin = nullptr;     // global inbox of the grid-cooperative panel
    double *Tbig = nullptr, *G = nullptr, *W1 = nullptr, *W2 = nullptr;   // two-level blocking
    int gin_ctas = 0;
    int alloc(int mmax, int nmax);
    void release();
};
// Q (m x k) and R (k x n), k = min(m, n), column-major, diag(R) >= 0.
int qr_f64(cudaStream_t s, int m, int n, const double *A, double *Q, double *R, QrWork &w);

// Tridiagonalisation + divide-and-conquer eigensolver (syevd.cu)
struct SyevdWork {
    int pmax = 0;
    double *A = nullptr, *Q = nullptr, *Qg = nullptr, *Qk = nullptr, *U = nullptr, *Qn = nullptr, *R = nullptr;
    double *vec = nullptr, *rot = nullptr;
    double *gvec = nullptr;      // tridiagonalisation vectors in global memory (p > 6400)
    int gvec_ctas = 0;
    int *ivec = nullptr;
    int alloc(int pmax);
    void release();
};
int syevd_f64(cudaStream_t s, int p, const double *A, double *w, double *V, SyevdWork &W);

struct EigWork {
    int nmax = 0;
    double *A = nullptr, *V = nullptr, *scal = nullptr;
    int *ints = nullptr;
    SyevdWork sd;
    int alloc(int nmax);
    void release();
};
// sizes above this use syevd_f64, below the one-CTA Jacobi
constexpr int kJacobiMax = 32;
// w descending, V columns (largest-|component| positive); A is not modified.
int syev_f64(cudaStream_t s, int n, const double *A, double *w, double *V, EigWork &e);

struct RrqrWork {
    int nmax = 0, cmax = 0;
    double *M = nullptr, *nrm = nullptr, *scal = nullptr;
    int *ints = nullptr;
    // blocked QRCP: reflectors (cmax x 32), F (nmax x 32), partials, state
    double *V3 = nullptr, *F3 = nullptr, *p3 = nullptr, *st3 = nullptr, *ug3 = nullptr, *pw3 = nullptr;
    int *act3 = nullptr, *ist3 = nullptr;
    int p3_ctas = 0;
    int alloc(int nmax, int cmax);
    void release();
};
// RankTruncChol: returns the kept rank in *k (host), Zout n x k.
int rank_trunc_chol_f64(cudaStream_t s, int n, int c, const double *Z, double tol, int prec_out,
                        double *Zout, int *k, RrqrWork &w);

}  // namespace lyap
