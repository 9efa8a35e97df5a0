// eig.cu -- symmetric eigendecomposition of the small kernel matrices
// H_i = T_i N_i T_i^T, K_i = Gamma_i Upsilon_i Gamma_i^T and R Y R^T
// (PAPER.md Fragment 1 l.165, Fragment 2 l.240, Fragments 3/4 l.790/l.824,
// RankTruncLdlt l.1298).
//
// Parallel cyclic Jacobi in round-robin ("tournament") order: each round
// rotates n/2 disjoint pairs at once.  A <- J^T A J is applied as independent
// 2x2 block updates (one thread per block), V <- V J as column-pair updates.
// Rotation formulas (Golub & Van Loan sym.schur2) and the stopping rule
// (off(A) <= u ||A||_F, or a sweep without rotations; entries below
// u sqrt(|a_pp a_qq|) are skipped) are those of the oracle's cyclic Jacobi;
// only the rotation order differs, so eigenvalues agree to rounding and
// eigenvectors up to the sign normalisation applied at the end.
#include "common.cuh"
#include "lyap_internal.h"
#include "ktimer.h"

namespace lyap {

// LYAP_EIG=jacobi forces the one-CTA Jacobi at every size (cross-checking).
static bool force_jacobi() {
    static int v = -1;
    if (v < 0) { const char *e = getenv("LYAP_EIG"); v = (e && e[0] == 'j') ? 1 : 0; }
    return v == 1;
}

__device__ __forceinline__ void rr_pair(int r, int i, int N, int &a, int &b) {
    if (i == 0) { a = r; b = N - 1; }
    else { a = (r + i) % (N - 1); b = (r - i + (N - 1)) % (N - 1); }
    if (a > b) { int t = a; a = b; b = t; }
}

// One CTA; A (n x n, ld n) and V in global workspace.  scal[0] = sweeps.
__global__ void __launch_bounds__(1024)
jacobi_kernel(int n, double *__restrict__ A, double *__restrict__ V, double *__restrict__ cs,
              int *__restrict__ partner, double *__restrict__ scal)
{
    __shared__ double red[32];
    __shared__ int any_rot;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int N = n + (n & 1);
    const double u = 0x1p-53;
    // symmetrize, V = I
    for (long idx = tid; idx < (long)n * n; idx += nt) {
        int i = (int)(idx % n), j = (int)(idx / n);
        if (i < j) {
            double v = 0.5 * (A[idx] + A[(long)i * n + j]);
            A[idx] = v; A[(long)i * n + j] = v;
        }
        V[idx] = (i == j) ? 1.0 : 0.0;
    }
    __syncthreads();
    double fro2 = 0.0;
    for (long idx = tid; idx < (long)n * n; idx += nt) fro2 = fma(A[idx], A[idx], fro2);
    const double fro = sqrt(block_sum(fro2, red));
    int sweep = 0;
    for (sweep = 0; sweep < 60; sweep++) {
        double off2 = 0.0;
        for (long idx = tid; idx < (long)n * n; idx += nt) {
            int i = (int)(idx % n), j = (int)(idx / n);
            if (i != j) off2 = fma(A[idx], A[idx], off2);
        }
        const double off = sqrt(block_sum(off2, red));
        if (off <= u * fro || off == 0.0) break;
        if (tid == 0) any_rot = 0;
        __syncthreads();
        for (int r = 0; r < N - 1; r++) {
            // phase 1: rotations of this round
            for (int i = tid; i < N / 2; i += nt) {
                int a, b;
                rr_pair(r, i, N, a, b);
                double c = 1.0, s = 0.0;
                if (b < n) {
                    double apq = A[(long)b * n + a];
                    double app = A[(long)a * n + a], aqq = A[(long)b * n + b];
                    if (apq != 0.0 && fabs(apq) > u * sqrt(fabs(app * aqq))) {
                        double tau = (aqq - app) / (2.0 * apq);
                        double t = isinf(tau) ? 0.0 : ((tau >= 0.0) ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                        c = 1.0 / sqrt(1.0 + t * t);
                        s = t * c;
                        any_rot = 1;
                    }
                    partner[a] = b; partner[b] = a;
                    cs[2 * a] = c; cs[2 * a + 1] = s; cs[2 * b] = c; cs[2 * b + 1] = s;
                } else {
                    partner[a] = -1;
                    cs[2 * a] = 1.0; cs[2 * a + 1] = 0.0;
                }
            }
            __syncthreads();
            // phase 2: A <- J^T A J by 2x2 blocks (pair P rows, pair Q cols)
            const int np = N / 2;
            for (int e = tid; e < np * np; e += nt) {
                int P = e % np, Q = e / np;
                int a, b, a2, b2;
                rr_pair(r, P, N, a, b);
                rr_pair(r, Q, N, a2, b2);
                const bool bv = b < n, b2v = b2 < n;
                double c1 = cs[2 * a], s1 = cs[2 * a + 1], c2 = cs[2 * a2], s2 = cs[2 * a2 + 1];
                double m00 = A[(long)a2 * n + a];
                double m01 = b2v ? A[(long)b2 * n + a] : 0.0;
                double m10 = bv ? A[(long)a2 * n + b] : 0.0;
                double m11 = (bv && b2v) ? A[(long)b2 * n + b] : 0.0;
                // right: columns a2 <- c2*a2 - s2*b2 ; b2 <- s2*a2 + c2*b2
                double n00 = c2 * m00 - s2 * m01, n01 = s2 * m00 + c2 * m01;
                double n10 = c2 * m10 - s2 * m11, n11 = s2 * m10 + c2 * m11;
                // left: rows a <- c1*a - s1*b ; b <- s1*a + c1*b
                double o00 = c1 * n00 - s1 * n10, o01 = c1 * n01 - s1 * n11;
                double o10 = s1 * n00 + c1 * n10, o11 = s1 * n01 + c1 * n11;
                if (P == Q && bv && s1 != 0.0) { o01 = 0.0; o10 = 0.0; }
                A[(long)a2 * n + a] = o00;
                if (b2v) A[(long)b2 * n + a] = o01;
                if (bv) A[(long)a2 * n + b] = o10;
                if (bv && b2v) A[(long)b2 * n + b] = o11;
            }
            // V <- V J (column pairs)
            for (int e = tid; e < n * np; e += nt) {
                int k = e % n, P = e / n;
                int a, b;
                rr_pair(r, P, N, a, b);
                if (b >= n) continue;
                double c = cs[2 * a], s = cs[2 * a + 1];
                if (s == 0.0) continue;
                double va = V[(long)a * n + k], vb = V[(long)b * n + k];
                V[(long)a * n + k] = c * va - s * vb;
                V[(long)b * n + k] = s * va + c * vb;
            }
            __syncthreads();
        }
        if (!any_rot) { sweep++; break; }
    }
    if (tid == 0) scal[0] = sweep;
}

// Sort eigenvalues descending (rank by comparison, ties by index) and write
// w / V with the sign normalisation (largest |component| positive, lowest index).
__global__ void eig_sort_kernel(int n, const double *__restrict__ A, const double *__restrict__ V,
                                double *__restrict__ w, double *__restrict__ Vout)
{
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int i = gw; i < n; i += nw) {
        double di = A[(long)i * n + i];
        int rank = 0;
        for (int j = lane; j < n; j += 32) {
            double dj = A[(long)j * n + j];
            if (dj > di || (dj == di && j < i)) rank++;
        }
        rank = warp_sum(rank);
        // argmax |V[:, i]|, lowest index on ties
        double bv = -1.0; int bi = n;
        for (int k = lane; k < n; k += 32) {
            double v = fabs(V[(long)i * n + k]);
            if (v > bv || (v == bv && k < bi)) { bv = v; bi = k; }
        }
        for (int o = 16; o > 0; o >>= 1) {
            double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
            int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
            if (v2 > bv || (v2 == bv && i2 < bi)) { bv = v2; bi = i2; }
        }
        double sg = (V[(long)i * n + bi] < 0.0) ? -1.0 : 1.0;
        if (lane == 0) w[rank] = di;
        for (int k = lane; k < n; k += 32) Vout[(long)rank * n + k] = sg * V[(long)i * n + k];
    }
}

int EigWork::alloc(int nmax_) {
    nmax = nmax_;
    LYAP_CUDA_TRY(cudaMalloc(&A, sizeof(double) * (size_t)nmax * nmax));
    LYAP_CUDA_TRY(cudaMalloc(&V, sizeof(double) * (size_t)nmax * nmax));
    LYAP_CUDA_TRY(cudaMalloc(&scal, sizeof(double) * (size_t)(2 * nmax + 16)));
    LYAP_CUDA_TRY(cudaMalloc(&ints, sizeof(int) * (size_t)(nmax + 8)));
    if (nmax > kJacobiMax) LYAP_TRY(sd.alloc(nmax));
    return LYAP_OK;
}
void EigWork::release() {
    cudaFree(A); cudaFree(V); cudaFree(scal); cudaFree(ints);
    A = V = scal = nullptr; ints = nullptr;
    if (sd.pmax) sd.release();
}

int syev_f64(cudaStream_t s, int n, const double *Ain, double *w, double *Vout, EigWork &e)
{
    if (n <= 0) return LYAP_OK;
    if (n > e.nmax) return LYAP_ERR_CAPACITY;
    if (n > kJacobiMax && !force_jacobi()) {
        KTimer kt(KC_JACOBI, s);
        return syevd_f64(s, n, Ain, w, Vout, e.sd);
    }
    LYAP_CUDA_TRY(cudaMemcpyAsync(e.A, Ain, sizeof(double) * (size_t)n * n, cudaMemcpyDeviceToDevice, s));
    // cs uses scal[8 ...], partner uses ints
    {
        KTimer kt(KC_JACOBI, s);
        jacobi_kernel<<<1, 1024, 0, s>>>(n, e.A, e.V, e.scal + 8, e.ints, e.scal);
    }
    LYAP_TRY(launched());
    int blocks = ceil_div((long)n * 32, 256);
    eig_sort_kernel<<<blocks < 512 ? blocks : 512, 256, 0, s>>>(n, e.A, e.V, w, Vout);
    return launched();
}

}  // namespace lyap

extern "C" int lyap_syev(int n, const double *A, double *w, double *V, void *stream)
{
    using namespace lyap;
    if (n <= 0 || !A || !w || !V) return LYAP_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    EigWork e;
    int rc = e.alloc(n);
    if (rc == LYAP_OK) rc = syev_f64(s, n, A, w, V, e);
    if (cudaStreamSynchronize(s) != cudaSuccess) rc = LYAP_ERR_CUDA;
    e.release();
    return rc;
}
