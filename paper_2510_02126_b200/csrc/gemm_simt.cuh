// gemm_simt.cuh -- strided SIMT GEMM  C = alpha * A * B + beta * C.
//
// Used for the fp64 (residual path, small kernels) and fp32 products, and as
// the reference path for the 16-bit products until the tcgen05 kernel takes
// over.  Operands are addressed through explicit (row, col) strides so one
// template serves row-major, column-major and transposed views:
//   A(i,l) = A[i*sam + l*sak],  B(l,j) = B[l*sbk + j*sbn],  C(i,j) = C[i*scm + j*scn].
#pragma once
#include "common.cuh"

namespace lyap {

template <typename TA, typename TB, typename TC, typename Acc, int BM, int BN, int BK, int TM, int TN>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
gemm_strided_kernel(int M, int N, int K, Acc alpha,
                    const TA *__restrict__ A, long sam, long sak,
                    const TB *__restrict__ B, long sbk, long sbn,
                    Acc beta, TC *__restrict__ C, long scm, long scn)
{
    constexpr int NT = (BM / TM) * (BN / TN);
    __shared__ Acc As[BK][BM + 1];
    __shared__ Acc Bs[BK][BN + 1];
    const int tid = threadIdx.x;
    const int tx = tid % (BN / TN), ty = tid / (BN / TN);
    const long m0 = (long)blockIdx.y * BM, n0 = (long)blockIdx.x * BN;
    Acc acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; i++)
#pragma unroll
        for (int j = 0; j < TN; j++) acc[i][j] = Acc(0);
    const bool a_kfast = (sak == 1), b_kfast = (sbk == 1);
    for (int k0 = 0; k0 < K; k0 += BK) {
        for (int idx = tid; idx < BM * BK; idx += NT) {
            int mm, kk;
            if (a_kfast) { kk = idx % BK; mm = idx / BK; } else { mm = idx % BM; kk = idx / BM; }
            long gm = m0 + mm, gk = k0 + kk;
            Acc v = Acc(0);
            if (gm < M && gk < K) v = (Acc)to_d<TA>(A[gm * sam + gk * sak]);
            As[kk][mm] = v;
        }
        for (int idx = tid; idx < BN * BK; idx += NT) {
            int nn, kk;
            if (b_kfast) { kk = idx % BK; nn = idx / BK; } else { nn = idx % BN; kk = idx / BN; }
            long gn = n0 + nn, gk = k0 + kk;
            Acc v = Acc(0);
            if (gn < N && gk < K) v = (Acc)to_d<TB>(B[gk * sbk + gn * sbn]);
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
            TC *cp = C + gm * scm + gn * scn;
            Acc v = alpha * acc[i][j];
            if (beta != Acc(0)) v = fma(beta, (Acc)to_d<TC>(*cp), v);
            *cp = from_d<TC>((double)v);
        }
    }
}

template <typename TA, typename TB, typename TC, typename Acc>
int gemm_strided(cudaStream_t s, int M, int N, int K, Acc alpha,
                 const TA *A, long sam, long sak, const TB *B, long sbk, long sbn,
                 Acc beta, TC *C, long scm, long scn)
{
    if (M <= 0 || N <= 0) return LYAP_OK;
    constexpr int BM = 64, BN = 64, BK = 16, TM = 4, TN = 4;
    dim3 grid(ceil_div(N, BN), ceil_div(M, BM));
    gemm_strided_kernel<TA, TB, TC, Acc, BM, BN, BK, TM, TN><<<grid, (BM / TM) * (BN / TN), 0, s>>>(
        M, N, K, alpha, A, sam, sak, B, sbk, sbn, beta, C, scm, scn);
    return launched();
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
