// qr.cu -- thin Householder QR of tall-skinny fp64 matrices (Fragments 1-4:
// "Compute a thin QR decomposition F_i = U_i T_i", PAPER.md l.164, l.239,
// l.789, l.823; the error analysis l.357 assumes Householder QR).
//
// Blocked right-looking Householder with compact-WY panels of width 16:
//   panel kernel (one CTA): reflectors H_j = I - tau_j v_j v_j^T,
//     v_j = x - alpha e_1, alpha = -sign(x_1)||x||, tau_j = 2 / v_j^T v_j,
//     plus the panel's triangular factor T (H_0..H_{b-1} = I - V T V^T);
//   trailing update W <- W - V (T^T (V^T W)) with the strided GEMM;
//   Q = H_0 ... H_{k-1} [I_k; 0] accumulated backwards the same way.
// The sign convention diag(R) >= 0 makes the factorization unique for full
// column rank, so it matches any other Householder QR up to rounding.
#include "common.cuh"
#include "gemm_simt.cuh"
#include "lyap_internal.h"

namespace lyap {

static constexpr int QB = 16;

// Factor panel columns [j0, j0+jb) of W (m x n, ld m), rows j0..m-1.
// Writes V (m x k, ld m; zero above the diagonal), tau, and T_panel (QB x QB).
__global__ void __launch_bounds__(512)
qr_panel_kernel(int m, int j0, int jb, double *__restrict__ W, double *__restrict__ V,
                double *__restrict__ tau, double *__restrict__ Tp)
{
    __shared__ double red[32];
    __shared__ double sh_alpha, sh_tau;
    __shared__ double G[QB][QB];
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int jj = 0; jj < jb; jj++) {
        const int j = j0 + jj;
        double *x = W + (long)j * m;
        double s = 0.0;
        for (int i = j + tid; i < m; i += nt) s = fma(x[i], x[i], s);
        s = block_sum(s, red);
        const double nrm = sqrt(s);
        double *v = V + (long)j * m;
        if (tid == 0) {
            if (nrm == 0.0) { sh_tau = 0.0; sh_alpha = 0.0; }
            else {
                double x0 = x[j];
                double alpha = (x0 >= 0.0) ? -nrm : nrm;
                sh_alpha = alpha;
                // v^T v = (x0-alpha)^2 + (s - x0^2) = 2 nrm (nrm + |x0|)
                double v0 = x0 - alpha;
                sh_tau = 2.0 / (v0 * v0 + (s - x0 * x0));
                v[j] = v0;
            }
        }
        __syncthreads();
        const double tj = sh_tau;
        for (int i = tid; i < m; i += nt) {
            if (i < j) v[i] = 0.0;
            else if (i > j) v[i] = (tj == 0.0) ? 0.0 : x[i];
        }
        if (tid == 0 && tj == 0.0) v[j] = 0.0;
        __syncthreads();
        // apply H_j to the remaining panel columns
        for (int cc = jj + 1; cc < jb; cc++) {
            double *y = W + (long)(j0 + cc) * m;
            double d = 0.0;
            if (tj != 0.0)
                for (int i = j + tid; i < m; i += nt) d = fma(v[i], y[i], d);
            d = block_sum(d, red);
            const double f = tj * d;
            if (tj != 0.0)
                for (int i = j + tid; i < m; i += nt) y[i] = fma(-f, v[i], y[i]);
            __syncthreads();
        }
        if (tid == 0) { tau[j] = tj; }
        // column j of W becomes alpha e_j
        for (int i = j + tid; i < m; i += nt) x[i] = (i == j) ? ((tj == 0.0) ? x[j] : sh_alpha) : 0.0;
        __syncthreads();
    }
    // Gram G = V_p^T V_p (warp per entry), then T (forward, columnwise)
    const int lane = tid & 31, w = tid >> 5, nw = nt >> 5;
    for (int e = w; e < jb * jb; e += nw) {
        int a = e / jb, c = e % jb;
        double d = 0.0;
        if (a <= c) {
            const double *va = V + (long)(j0 + a) * m, *vc = V + (long)(j0 + c) * m;
            for (int i = j0 + lane; i < m; i += 32) d = fma(va[i], vc[i], d);
            d = warp_sum(d);
        }
        if (lane == 0) G[a][c] = d;
    }
    __syncthreads();
    if (tid == 0) {
        double T[QB][QB];
        for (int a = 0; a < QB; a++) for (int c = 0; c < QB; c++) T[a][c] = 0.0;
        for (int c = 0; c < jb; c++) {
            double tc = tau[j0 + c];
            T[c][c] = tc;
            // T[0:c, c] = -tau_c T[0:c, 0:c] (V[:,0:c]^T v_c)
            for (int a = 0; a < c; a++) {
                double sacc = 0.0;
                for (int l = a; l < c; l++) sacc += T[a][l] * G[l][c];
                T[a][c] = -tc * sacc;
            }
        }
        for (int a = 0; a < QB; a++) for (int c = 0; c < QB; c++) Tp[a + c * QB] = T[a][c];
    }
}

__global__ void set_identity_kernel(int m, int k, double *Q) {
    long tot = (long)m * k;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < tot; idx += (long)gridDim.x * blockDim.x) {
        long i = idx % m, c = idx / m;
        Q[idx] = (i == c) ? 1.0 : 0.0;
    }
}

// R = upper k x n part of W, then the sign fix on R rows and Q columns.
__global__ void qr_finish_kernel(int m, int n, int k, const double *__restrict__ W, double *__restrict__ Q,
                                 double *__restrict__ R)
{
    long tot = (long)k * n;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < tot; idx += (long)gridDim.x * blockDim.x) {
        int i = (int)(idx % k), c = (int)(idx / k);
        double sg = (W[(long)i * m + i] < 0.0) ? -1.0 : 1.0;
        R[idx] = (i <= c) ? sg * W[(long)c * m + i] : 0.0;
    }
    long totq = (long)m * k;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < totq; idx += (long)gridDim.x * blockDim.x) {
        int c = (int)(idx / m);
        if (W[(long)c * m + c] < 0.0) Q[idx] = -Q[idx];
    }
}

int QrWork::alloc(int mmax_, int nmax_) {
    mmax = mmax_; nmax = nmax_;
    int kmax = mmax < nmax ? mmax : nmax;
    LYAP_CUDA_TRY(cudaMalloc(&V, sizeof(double) * (size_t)mmax * kmax));
    LYAP_CUDA_TRY(cudaMalloc(&T, sizeof(double) * (size_t)QB * QB * (kmax / QB + 1)));
    LYAP_CUDA_TRY(cudaMalloc(&W, sizeof(double) * (size_t)2 * QB * (nmax > mmax ? nmax : mmax)));
    LYAP_CUDA_TRY(cudaMalloc(&tau, sizeof(double) * (size_t)kmax));
    LYAP_CUDA_TRY(cudaMalloc(&Wk, sizeof(double) * (size_t)mmax * nmax));
    return LYAP_OK;
}
void QrWork::release() { cudaFree(V); cudaFree(T); cudaFree(W); cudaFree(tau); cudaFree(Wk); V = T = W = tau = Wk = nullptr; }

int qr_f64(cudaStream_t s, int m, int n, const double *A, double *Q, double *R, QrWork &w)
{
    if (m <= 0 || n <= 0) return LYAP_OK;
    if (m > w.mmax || n > w.nmax) return LYAP_ERR_CAPACITY;
    const int k = m < n ? m : n;
    double *Wm = w.Wk;
    LYAP_CUDA_TRY(cudaMemcpyAsync(Wm, A, sizeof(double) * (size_t)m * n, cudaMemcpyDeviceToDevice, s));
    for (int j0 = 0; j0 < k; j0 += QB) {
        int jb = (k - j0 < QB) ? k - j0 : QB;
        double *Tp = w.T + (size_t)(j0 / QB) * QB * QB;
        qr_panel_kernel<<<1, 512, 0, s>>>(m, j0, jb, Wm, w.V, w.tau, Tp);
        LYAP_TRY(launched());
        int nt = n - (j0 + jb);
        if (nt > 0) {
            const double *Vp = w.V + (size_t)j0 * m;
            double *Wt = Wm + (size_t)(j0 + jb) * m;
            // Y = V_p^T Wt (jb x nt)      (rows j0..m-1 suffice: V zero above)
            LYAP_TRY(dgemm_cm(s, true, false, jb, nt, m - j0, 1.0, Vp + j0, m, Wt + j0, m, 0.0, w.W, QB));
            // Y = T^T Y  (in place via a second buffer region: use Q as scratch? no - small copy)
            LYAP_TRY(gemm_strided<double, double, double, double>(s, jb, nt, jb, 1.0, Tp, QB, 1, w.W, 1, QB,
                                                                  0.0, w.W + (size_t)QB * nt, 1, QB));
            // Wt -= V_p Y
            LYAP_TRY(dgemm_cm(s, false, false, m - j0, nt, jb, -1.0, Vp + j0, m, w.W + (size_t)QB * nt, QB, 1.0,
                              Wt + j0, m));
        }
    }
    // Q = H_0 ... H_{k-1} [I; 0]
    set_identity_kernel<<<ceil_div((long)m * k, 256) < 1024 ? ceil_div((long)m * k, 256) : 1024, 256, 0, s>>>(m, k, Q);
    LYAP_TRY(launched());
    for (int j0 = ((k - 1) / QB) * QB; j0 >= 0; j0 -= QB) {
        int jb = (k - j0 < QB) ? k - j0 : QB;
        const double *Tp = w.T + (size_t)(j0 / QB) * QB * QB;
        const double *Vp = w.V + (size_t)j0 * m;
        int nc = k - j0;               // columns j0..k-1 of Q are affected
        double *Qc = Q + (size_t)j0 * m;
        LYAP_TRY(dgemm_cm(s, true, false, jb, nc, m - j0, 1.0, Vp + j0, m, Qc + j0, m, 0.0, w.W, QB));
        LYAP_TRY(gemm_strided<double, double, double, double>(s, jb, nc, jb, 1.0, Tp, 1, QB, w.W, 1, QB,
                                                              0.0, w.W + (size_t)QB * nc, 1, QB));
        LYAP_TRY(dgemm_cm(s, false, false, m - j0, nc, jb, -1.0, Vp + j0, m, w.W + (size_t)QB * nc, QB, 1.0,
                          Qc + j0, m));
    }
    int tot = (int)(((long)k * n + (long)m * k + 255) / 256);
    qr_finish_kernel<<<tot < 1024 ? tot : 1024, 256, 0, s>>>(m, n, k, Wm, Q, R);
    return launched();
}

}  // namespace lyap

extern "C" int lyap_qr(int m, int n, const double *A, double *Q, double *R, void *stream)
{
    using namespace lyap;
    if (m <= 0 || n <= 0 || !A || !Q || !R) return LYAP_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    QrWork w;
    int rc = w.alloc(m, n);
    if (rc == LYAP_OK) rc = qr_f64(s, m, n, A, Q, R, w);
    if (cudaStreamSynchronize(s) != cudaSuccess) rc = LYAP_ERR_CUDA;
    w.release();
    return rc;
}
