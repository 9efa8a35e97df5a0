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
#include <mutex>
#include <unordered_map>
#include <type_traits>
#include "common.cuh"
#include "ktimer.h"

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

// grow-only device workspace for split-K partials, one per stream (concurrent solver
// handles on different streams must not share it; growth synchronises only that stream)
inline void *splitk_workspace(size_t bytes, cudaStream_t s) {
    struct Buf { void *ptr = nullptr; size_t cap = 0; };
    static std::mutex mu;
    static std::unordered_map<cudaStream_t, Buf> bufs;
    std::lock_guard<std::mutex> lock(mu);
    Buf &b = bufs[s];
    if (bytes > b.cap) {
        if (b.ptr) { cudaStreamSynchronize(s); cudaFree(b.ptr); }
        b.cap = bytes + bytes / 2;
        if (cudaMalloc(&b.ptr, b.cap) != cudaSuccess) { b.ptr = nullptr; b.cap = 0; }
    }
    return b.ptr;
}

// ---------------------------------------------------------------- fp64 on the DMMA pipe
// C tile 64 x 64 per CTA, 4 warps (2 x 2) of 32 x 32, k-tiles of 16 staged in shared
// memory (double-buffered through registers); mma.sync.m8n8k4.f64 (the fp64 tensor
// path of sm_100a -- tcgen05 has no f64 kind).  Fragment layouts (PTX ISA m8n8k4 .f64):
// A: row = lane/4, k = lane%4; B: k = lane%4, col = lane/4; C: row = lane/4,
// cols 2*(lane%4) + {0,1}.
__device__ __forceinline__ void dmma8x8x4(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// one 64 x 64 tile of C = alpha A B (+ beta C), k range [kb, ke); 128 threads.  work != 0:
// write the split-K partial to work + wz instead (M x N, column-major)
__device__ __forceinline__ void dmma_tile(int M, int N, int kb, int ke, long m0, long n0, double alpha,
                                          const double *__restrict__ A, long sam, long sak,
                                          const double *__restrict__ B, long sbk, long sbn,
                                          double beta, double *__restrict__ C, long scm, long scn,
                                          double *__restrict__ work, long wz)
{
    constexpr int BM = 64, BN = 64, BK = 16, PAD = 4;
    __shared__ double As[2][BK][BM + PAD];
    __shared__ double Bs[2][BK][BN + PAD];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
    const bool a_kfast = (sak == 1), b_kfast = (sbk == 1);
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j][0] = acc[i][j][1] = 0.0;
    double ra[8], rb[8];
    auto gload = [&](int k0) {
#pragma unroll
        for (int e = 0; e < 8; e++) {
            int idx = tid + e * 128, mm, kk;
            if (a_kfast) { kk = idx % BK; mm = idx / BK; } else { mm = idx % BM; kk = idx / BM; }
            long gm = m0 + mm, gk = k0 + kk;
            ra[e] = (gm < M && gk < ke) ? A[gm * sam + gk * sak] : 0.0;
            int nn;
            if (b_kfast) { kk = idx % BK; nn = idx / BK; } else { nn = idx % BN; kk = idx / BN; }
            long gn = n0 + nn;
            gk = k0 + kk;
            rb[e] = (gn < N && gk < ke) ? B[gk * sbk + gn * sbn] : 0.0;
        }
    };
    auto sstore = [&](int buf) {
#pragma unroll
        for (int e = 0; e < 8; e++) {
            int idx = tid + e * 128, mm, kk;
            if (a_kfast) { kk = idx % BK; mm = idx / BK; } else { mm = idx % BM; kk = idx / BM; }
            As[buf][kk][mm] = ra[e];
            int nn;
            if (b_kfast) { kk = idx % BK; nn = idx / BK; } else { nn = idx % BN; kk = idx / BN; }
            Bs[buf][kk][nn] = rb[e];
        }
    };
    const int ntiles = (ke > kb) ? (ke - kb + BK - 1) / BK : 0;
    if (ntiles > 0) { gload(kb); sstore(0); }
    __syncthreads();
    const int lr = lane >> 2, lk = lane & 3;
    for (int t = 0; t < ntiles; t++) {
        const int buf = t & 1;
        if (t + 1 < ntiles) gload(kb + (t + 1) * BK);
#pragma unroll
        for (int k4 = 0; k4 < BK; k4 += 4) {
            double a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; i++) a[i] = As[buf][k4 + lk][wm + i * 8 + lr];
#pragma unroll
            for (int j = 0; j < 4; j++) b[j] = Bs[buf][k4 + lk][wn + j * 8 + lr];
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
                for (int j = 0; j < 4; j++) dmma8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
        }
        if (t + 1 < ntiles) sstore(buf ^ 1);
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const long gm = m0 + wm + i * 8 + lr;
        if (gm >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; j++)
#pragma unroll
            for (int v = 0; v < 2; v++) {
                const long gn = n0 + wn + j * 8 + 2 * lk + v;
                if (gn >= N) continue;
                const double r = alpha * acc[i][j][v];
                if (work) work[wz + gm + gn * (long)M] = r;
                else {
                    double *cp = C + gm * scm + gn * scn;
                    *cp = (beta != 0.0) ? fma(beta, *cp, r) : r;
                }
            }
    }
}

static __global__ void __launch_bounds__(128)
dgemm_dmma_kernel(int M, int N, int K, int kchunk, double alpha,
                  const double *__restrict__ A, long sam, long sak,
                  const double *__restrict__ B, long sbk, long sbn,
                  double beta, double *__restrict__ C, long scm, long scn, double *__restrict__ work)
{
    const int kb = blockIdx.z * kchunk, ke = min(K, kb + kchunk);
    dmma_tile(M, N, kb, ke, (long)blockIdx.y * 64, (long)blockIdx.x * 64, alpha, A, sam, sak, B, sbk, sbn, beta, C,
              scm, scn, work, (long)blockIdx.z * M * N);
}


// ---------------------------------------------------------------- fp32 SIMT, 128 x 128 tiles
// C = alpha A B^T + beta C for fp32 with both operands K-contiguous (A(i,l) = A[i sam + l],
// B(l,j) = B[l + j sbn]) -- the shapes of the fp32 solver's Gauss-Jordan update and of its
// A_k^{-1} Z products.  256 threads, 8 x 8 outputs per thread, BK = 16 k-slices staged
// transposed in shared memory (double-buffered through registers, 16-byte loads when the
// rows are 16-byte aligned); split-K partials go to `work` like gemm_strided_kernel.
constexpr int SG_BM = 128, SG_BN = 128, SG_BK = 16;
static __global__ void __launch_bounds__(256)
sgemm_nt_kernel(int M, int N, int K, int kchunk, float alpha, const float *__restrict__ A, long sam,
                const float *__restrict__ B, long sbn, float beta, float *__restrict__ C, long scm, long scn,
                float *__restrict__ work, int vec)
{
    __shared__ __align__(16) float As[2][SG_BK][SG_BM + 4];
    __shared__ __align__(16) float Bs[2][SG_BK][SG_BN + 4];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const long m0 = (long)blockIdx.y * SG_BM, n0 = (long)blockIdx.x * SG_BN;
    const int kb = blockIdx.z * kchunk, ke = min(K, kb + kchunk);
    // loader: thread -> (row r = tid / 4 + 64 h, k quad q = tid % 4), h = 0, 1
    const int lr = tid >> 2, lq = (tid & 3) * 4;
    float ra[2][4], rb[2][4];
    auto gload = [&](int k0) {
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const long gm = m0 + lr + 64 * h, gn = n0 + lr + 64 * h;
            const int gk = k0 + lq;
            if (vec && gk + 4 <= ke) {
                float4 a4 = (gm < M) ? *reinterpret_cast<const float4 *>(A + gm * sam + gk) : make_float4(0.f, 0.f, 0.f, 0.f);
                float4 b4 = (gn < N) ? *reinterpret_cast<const float4 *>(B + gn * sbn + gk) : make_float4(0.f, 0.f, 0.f, 0.f);
                ra[h][0] = a4.x; ra[h][1] = a4.y; ra[h][2] = a4.z; ra[h][3] = a4.w;
                rb[h][0] = b4.x; rb[h][1] = b4.y; rb[h][2] = b4.z; rb[h][3] = b4.w;
            } else {
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    ra[h][e] = (gm < M && gk + e < ke) ? A[gm * sam + gk + e] : 0.f;
                    rb[h][e] = (gn < N && gk + e < ke) ? B[gn * sbn + gk + e] : 0.f;
                }
            }
        }
    };
    auto sstore = [&](int buf) {
#pragma unroll
        for (int h = 0; h < 2; h++)
#pragma unroll
            for (int e = 0; e < 4; e++) {
                As[buf][lq + e][lr + 64 * h] = ra[h][e];
                Bs[buf][lq + e][lr + 64 * h] = rb[h][e];
            }
    };
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = 0; j < 8; j++) acc[i][j] = 0.f;
    const int ntiles = (ke > kb) ? (ke - kb + SG_BK - 1) / SG_BK : 0;
    if (ntiles > 0) { gload(kb); sstore(0); }
    __syncthreads();
    for (int t = 0; t < ntiles; t++) {
        const int buf = t & 1;
        if (t + 1 < ntiles) gload(kb + (t + 1) * SG_BK);
#pragma unroll
        for (int kk = 0; kk < SG_BK; kk++) {
            // rows ty*4 + {0..3} and 64 + ty*4 + {0..3}; columns likewise (conflict-free float4)
            const float4 a0 = *reinterpret_cast<const float4 *>(&As[buf][kk][ty * 4]);
            const float4 a1 = *reinterpret_cast<const float4 *>(&As[buf][kk][64 + ty * 4]);
            const float4 b0 = *reinterpret_cast<const float4 *>(&Bs[buf][kk][tx * 4]);
            const float4 b1 = *reinterpret_cast<const float4 *>(&Bs[buf][kk][64 + tx * 4]);
            const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int i = 0; i < 8; i++)
#pragma unroll
                for (int j = 0; j < 8; j++) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        if (t + 1 < ntiles) sstore(buf ^ 1);
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 8; i++) {
        const long gm = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
        if (gm >= M) continue;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const long gn = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
            if (gn >= N) continue;
            const float r = alpha * acc[i][j];
            if (work) {
                work[(long)blockIdx.z * M * N + gm + gn * (long)M] = r;
            } else {
                float *cp = C + gm * scm + gn * scn;
                *cp = (beta != 0.f) ? fmaf(beta, *cp, r) : r;
            }
        }
    }
}

template <typename TA, typename TB, typename TC, typename Acc>
int gemm_strided(cudaStream_t s, int M, int N, int K, Acc alpha,
                 const TA *A, long sam, long sak, const TB *B, long sbk, long sbn,
                 Acc beta, TC *C, long scm, long scn)
{
    if (M <= 0 || N <= 0) return LYAP_OK;
    constexpr bool all_f64 = std::is_same<TA, double>::value && std::is_same<TB, double>::value &&
                             std::is_same<TC, double>::value && std::is_same<Acc, double>::value;
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
        work = (Acc *)splitk_workspace(sizeof(Acc) * (size_t)splits * M * N, s);
        if (!work) splits = 1;
    }
    const int kchunk = (splits > 1) ? ceil_div(ceil_div(K, splits), BK) * BK : std::max(K, 1);
    if (splits > 1) splits = ceil_div(K, kchunk);
    dim3 grid(ceil_div(N, BN), ceil_div(M, BM), splits);
    constexpr bool all_f32 = std::is_same<TA, float>::value && std::is_same<TB, float>::value &&
                             std::is_same<TC, float>::value && std::is_same<Acc, float>::value;
    if constexpr (all_f32) {
        // 128 x 128 tiles for K-contiguous operands (both fp32 solver shapes) with enough tiles
        const long tiles128 = (long)ceil_div(N, SG_BN) * ceil_div(M, SG_BM);
        if (sak == 1 && sbk == 1 && tiles128 >= 64 && !env_flag("LYAP_SGEMM_OLD")) {
            int sp = 1;
            if (tiles128 < 148 && K >= 512) sp = std::min(std::min(ceil_div(K, 256), std::max(1, (int)(296 / tiles128))), 64);
            float *wk = nullptr;
            if (sp > 1) { wk = (float *)splitk_workspace(sizeof(float) * (size_t)sp * M * N, s); if (!wk) sp = 1; }
            const int kc = (sp > 1) ? ceil_div(ceil_div(K, sp), SG_BK) * SG_BK : std::max(K, 1);
            if (sp > 1) sp = ceil_div(K, kc);
            const int vec = (sam % 4 == 0 && sbn % 4 == 0 && ((uintptr_t)A % 16) == 0 && ((uintptr_t)B % 16) == 0) ? 1 : 0;
            dim3 g2(ceil_div(N, SG_BN), ceil_div(M, SG_BM), sp);
            sgemm_nt_kernel<<<g2, 256, 0, s>>>(M, N, K, kc, alpha, A, sam, B, sbn, beta, C, scm, scn,
                                               sp > 1 ? wk : nullptr, vec);
            LYAP_TRY(launched());
            if (sp > 1) {
                int gr = std::min(ceil_div((long)M * N, 256), 2048);
                splitk_reduce_kernel<TC, Acc><<<gr, 256, 0, s>>>(M, N, sp, wk, beta, C, scm, scn);
                LYAP_TRY(launched());
            }
            return LYAP_OK;
        }
    }
    if constexpr (all_f64) {
        KTimer kt(KC_DGEMM, s, 2.0 * M * N * K, 8.0 * ((double)M * K + (double)K * N + 2.0 * M * N));
        dgemm_dmma_kernel<<<grid, 128, 0, s>>>(M, N, K, kchunk, alpha, A, sam, sak, B, sbk, sbn, beta, C, scm,
                                               scn, splits > 1 ? work : nullptr);
    } else {
        gemm_strided_kernel<TA, TB, TC, Acc, BM, BN, BK, TM, TN><<<grid, (BM / TM) * (BN / TN), 0, s>>>(
            M, N, K, kchunk, alpha, A, sam, sak, B, sbk, sbn, beta, C, scm, scn, splits > 1 ? work : nullptr);
    }
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
