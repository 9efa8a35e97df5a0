// gemm_simt.cuh -- strided SIMT GEMM  C = alpha * A * B + beta * C.
//
// Used for the fp64 (residual path, small kernels) and fp32 products, and as
// the reference path for the 16-bit products.  Operands are addressed through
// explicit (row, col) strides so one template serves row-major, column-major
// and transposed views:
//   A(i,l) = A[i*sam + l*sak],  B(l,j) = B[l*sbk + j*sbn],  C(i,j) = C[i*scm + j*scn].
// Skinny products (few output tiles, long K) are split along K into a
// workspace and reduced in a fixed order (deterministic).
#pragma once
#include "common.cuh"

namespace lyap {

template <typename TA, typename TB, typename TC, typename Acc, int BM, int BN, int BK, int TM, int TN>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
gemm_strided_kernel(int M, int N, int K, int kchunk, Acc alpha,
                    const TA *__restrict__ A, long sam, long sak,
                    const TB *__restrict__ B, long sbk, long sbn,
                    Acc beta, TC *__restrict__ C, long scm, long scn, Acc *__restrict__ work)
{
    constexpr int NT = (BM / TM) * (BN / TN);
    __shared__ Acc As[BK][BM + 1];
    __shared__ Acc Bs[BK][BN + 1];
    const int tid = threadIdx.x;
    const int tx = tid % (BN / TN), ty = tid / (BN / TN);
    const long m0 = (long)blockIdx.y * BM, n0 = (long)blockIdx.x * BN;
    const int kb = blockIdx.z * kchunk, ke = min(K, kb + kchunk);
    Acc acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; i++)
#pragma unroll
        for (int j = 0; j < TN; j++) acc[i][j] = Acc(0);
    const bool a_kfast = (sak == 1), b_kfast = (sbk == 1);
    for (int k0 = kb; k0 < ke; k0 += BK) {
        for (int idx = tid; idx < BM * BK; idx += NT) {
            int mm, kk;
            if (a_kfast) { kk = idx % BK; mm = idx / BK; } else { mm = idx % BM; kk = idx / BM; }
            long gm = m0 + mm, gk = k0 + kk;
            Acc v = Acc(0);
            if (gm < M && gk < ke) v = (Acc)to_d<TA>(A[gm * sam + gk * sak]);
            As[kk][mm] = v;
        }
        for (int idx = tid; idx < BN * BK; idx += NT) {
            int nn, kk;
            if (b_kfast) { kk = idx % BK; nn = idx / BK; } else { nn = idx % BN; kk = idx / BN; }
            long gn = n0 + nn, gk = k0 + kk;
            Acc v = Acc(0);
            if (gn < N && gk < ke) v = (Acc)to_d<TB>(B[gk * sbk + gn * sbn]);
            Bs[kk][nn] = v;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; kk++) {
            Acc a[TM], b[TN];
#pragma unroll
            for (int i = 0; i < TM; i++) a[i] = As[kk][ty + i * (BM / TM)];
#pragma unroll
            for (int j = 0; j < TN; j++) b[j] = Bs[kk][tx + j * (BN / TN)];
#pragma unroll
            for (int i = 0; i < TM; i++)
#pragma unroll
                for (int j = 0; j < TN; j++) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < TM; i++) {
        long gm = m0 + ty + i * (BM / TM);
        if (gm >= M) continue;
#pragma unroll
        for (int j = 0; j < TN; j++) {
            long gn = n0 + tx + j * (BN / TN);
            if (gn >= N) continue;
            if (work) {
                work[(long)blockIdx.z * M * N + gm + gn * (long)M] = alpha * acc[i][j];
            } else {
                TC *cp = C + gm * scm + gn * scn;
                Acc v = alpha * acc[i][j];
                if (beta != Acc(0)) v = fma(beta, (Acc)to_d<TC>(*cp), v);
                *cp = from_d<TC>((double)v);
            }
        }
    }
}

template <typename TC, typename Acc>
__global__ void splitk_reduce_kernel(int M, int N, int splits, const Acc *__restrict__ work, Acc beta,
                                     TC *__restrict__ C, long scm, long scn)
{
    long tot = (long)M * N;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < tot; e += (long)gridDim.x * blockDim.x) {
        Acc s = Acc(0);
        for (int z = 0; z < splits; z++) s += work[(long)z * tot + e];
        long gm = e % M, gn = e / M;
        TC *cp = C + gm * scm + gn * scn;
        if (beta != Acc(0)) s = fma(beta, (Acc)to_d<TC>(*cp), s);
        *cp = from_d<TC>((double)s);
    }
}

// grow-only device workspace for split-K partials
inline void *splitk_workspace(size_t bytes) {
    static void *ptr = nullptr;
    static size_t cap = 0;
    if (bytes > cap) {
        if (ptr) { cudaDeviceSynchronize(); cudaFree(ptr); }
        cap = bytes + bytes / 2;
        if (cudaMalloc(&ptr, cap) != cudaSuccess) { ptr = nullptr; cap = 0; }
    }
    return ptr;
}

template <typename TA, typename TB, typename TC, typename Acc>
int gemm_strided(cudaStream_t s, int M, int N, int K, Acc alpha,
                 const TA *A, long sam, long sak, const TB *B, long sbk, long sbn,
                 Acc beta, TC *C, long scm, long scn)
{
    if (M <= 0 || N <= 0) return LYAP_OK;
    constexpr int BM = 64, BN = 64, BK = 16, TM = 4, TN = 4;
    const int tiles = ceil_div(N, BN) * ceil_div(M, BM);
    int splits = 1;
    if (tiles < 148 && K >= 512) {
        splits = std::min(ceil_div(K, 256), std::max(1, 296 / tiles));
        splits = std::min(splits, 64);
    }
    if (K <= 0) splits = 1;
    Acc *work = nullptr;
    if (splits > 1) {
        work = (Acc *)splitk_workspace(sizeof(Acc) * (size_t)splits * M * N);
        if (!work) splits = 1;
    }
    const int kchunk = (splits > 1) ? ceil_div(ceil_div(K, splits), BK) * BK : std::max(K, 1);
    if (splits > 1) splits = ceil_div(K, kchunk);
    dim3 grid(ceil_div(N, BN), ceil_div(M, BM), splits);
    gemm_strided_kernel<TA, TB, TC, Acc, BM, BN, BK, TM, TN><<<grid, (BM / TM) * (BN / TN), 0, s>>>(
        M, N, K, kchunk, alpha, A, sam, sak, B, sbk, sbn, beta, C, scm, scn, splits > 1 ? work : nullptr);
    LYAP_TRY(launched());
    if (splits > 1) {
        int g = std::min(ceil_div((long)M * N, 256), 2048);
        splitk_reduce_kernel<TC, Acc><<<g, 256, 0, s>>>(M, N, splits, work, beta, C, scm, scn);
        LYAP_TRY(launched());
    }
    return LYAP_OK;
}

// Column-major convenience wrappers (fp64): C(m x n) = alpha op(A) op(B) + beta C.
inline int dgemm_cm(cudaStream_t s, bool ta, bool tb, int m, int n, int k, double alpha,
                    const double *A, int lda, const double *B, int ldb, double beta,
                    double *C, int ldc)
{
    long sam = ta ? lda : 1, sak = ta ? 1 : lda;
    long sbk = tb ? ldb : 1, sbn = tb ? 1 : ldb;
    return gemm_strided<double, double, double, double>(s, m, n, k, alpha, A, sam, sak, B, sbk, sbn,
                                                        beta, C, 1, ldc);
}

}  // namespace lyap
