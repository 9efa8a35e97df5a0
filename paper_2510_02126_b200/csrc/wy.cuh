// wy.cuh -- fused application of a compact-WY block reflector to a tall matrix,
//     C <- (I - V T V^T) C      (trans = 0: Q = H_0 ... H_{b-1} applied from the left)
//     C <- (I - V T^T V^T) C    (trans = 1: Q^T applied from the left)
// V is m x jb (column-major, ld ldv, zero above its unit diagonal), T is jb x jb
// (column-major, ld 32), C is m x ncols (column-major, ld ldc).  One CTA owns 16
// columns of C for all m rows, so Y = V^T C, Y <- T Y and C -= V Y need no cross-CTA
// reduction: one launch replaces three GEMM launches (+ split-K reductions) per
// Householder panel in the QR factorisation, the Q formation and the eigenvector
// back-transformation.
#pragma once
#include "common.cuh"
#include "ktimer.h"

namespace lyap {

constexpr int WY_NB = 8, WY_CH = 128, WY_THREADS = 256;
constexpr int WY_VS = WY_CH * 33, WY_CS = WY_CH * WY_NB;
constexpr size_t WY_SMEM = sizeof(double) * (2 * WY_VS + 2 * WY_CS + 32 * WY_NB);
// NB = columns of C per CTA (8, or 4 when fewer than ~one CTA per SM would result)

__device__ __forceinline__ void wy_cp8(double *sdst, const double *gsrc, bool pred)
{
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gsrc), "r"(pred ? 8 : 0));
}
__device__ __forceinline__ void wy_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void wy_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// 256 threads; CTA = 8 columns of C; row chunks of 128 staged by cp.async into a
// double buffer so the next chunk's loads overlap this chunk's FMAs.
// Phase 1 (Y = V^T C): warp w accumulates rows w*16..w*16+15 of each chunk, lane =
// reflector index a, 8 column accumulators in registers.  Phase 3 (C -= V Y2):
// thread = (row, half of the 8 columns), Y2 read as broadcasts.
template <int NB>
static __global__ void __launch_bounds__(WY_THREADS)
wy_apply_kernel(int m, int ncols, int jb, int row0, const double *__restrict__ V, int ldv,
                const double *__restrict__ T, int trans, double *__restrict__ C, int ldc)
{
    extern __shared__ __align__(16) double wy_sm[];
    double *Vs = wy_sm;                         // [2][WY_CH][33]
    double *Cs = wy_sm + 2 * WY_VS;             // [2][WY_CH * NB]; later the 8 warp partials of Y
    double *Y2 = Cs + 2 * WY_CS;                // [32][NB]
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int c0 = blockIdx.x * NB;
    const int ncb = min(NB, ncols - c0);
    const int nch = (m - row0 + WY_CH - 1) / WY_CH;
    auto load_v = [&](int k) {
        const int r0 = row0 + k * WY_CH, rows = min(WY_CH, m - r0);
        double *vb = Vs + (k & 1) * WY_VS;
        for (int e = tid; e < WY_CH * 32; e += WY_THREADS) {
            const int i = e & (WY_CH - 1), a = e / WY_CH;
            const bool ok = i < rows && a < jb;
            wy_cp8(vb + i * 33 + a, ok ? V + (long)a * ldv + r0 + i : V, ok);
        }
    };
    auto load_c = [&](int k) {
        const int r0 = row0 + k * WY_CH, rows = min(WY_CH, m - r0);
        double *cb = Cs + (k & 1) * WY_CS;
        for (int e = tid; e < WY_CH * NB; e += WY_THREADS) {
            const int i = e & (WY_CH - 1), c = e / WY_CH;
            const bool ok = i < rows && c < ncb;
            wy_cp8(cb + i * NB + c, ok ? C + (long)(c0 + c) * ldc + r0 + i : C, ok);
        }
    };
    double acc[NB];
#pragma unroll
    for (int c = 0; c < NB; c++) acc[c] = 0.0;
    // ---- phase 1: Y = V^T C
    load_v(0);
    load_c(0);
    wy_commit();
    for (int k = 0; k < nch; k++) {
        if (k + 1 < nch) {
            load_v(k + 1);
            load_c(k + 1);
            wy_commit();
            wy_wait<1>();
        } else {
            wy_wait<0>();
        }
        __syncthreads();
        const double *vb = Vs + (k & 1) * WY_VS;
        const double *cb = Cs + (k & 1) * WY_CS;
#pragma unroll 4
        for (int ii = 0; ii < WY_CH / 8; ii++) {
            const int i = wid * (WY_CH / 8) + ii;
            const double v = vb[i * 33 + lane];
            const double2 *cr = reinterpret_cast<const double2 *>(cb + i * NB);
#pragma unroll
            for (int q = 0; q < NB / 2; q++) {
                const double2 cc = cr[q];
                acc[2 * q] = fma(v, cc.x, acc[2 * q]);
                acc[2 * q + 1] = fma(v, cc.y, acc[2 * q + 1]);
            }
        }
        __syncthreads();
    }
    // phase-3 chunk 0 in flight while Y is reduced
    load_v(0);
    wy_commit();
    // ---- reduce the eight warp partials, then Y2 = op(T) Y
#pragma unroll
    for (int c = 0; c < NB; c++) Cs[(wid * 32 + lane) * NB + c] = acc[c];
    __syncthreads();
    {
        double ys = 0.0;
#pragma unroll
        if (tid < 32 * NB)
            for (int w = 0; w < 8; w++) ys += Cs[w * 32 * NB + tid];
        __syncthreads();
        if (tid < 32 * NB) Cs[tid] = ys;
        __syncthreads();
        if (tid < 32 * NB) {
            const int a = tid / NB, c = tid % NB;
            double sacc = 0.0;
            if (a < jb)
                for (int l = 0; l < jb; l++) sacc = fma(trans ? T[l + a * 32] : T[a + l * 32], Cs[l * NB + c], sacc);
            Y2[tid] = sacc;
        }
    }
    // ---- phase 3: C -= V Y2
    constexpr int HC = NB / 2;                  // columns per thread in phase 3
    const int ri = tid & (WY_CH - 1), ch = (tid >> 7) * HC;
    for (int k = 0; k < nch; k++) {
        if (k + 1 < nch) {
            load_v(k + 1);
            wy_commit();
            wy_wait<1>();
        } else {
            wy_wait<0>();
        }
        __syncthreads();
        const int r0 = row0 + k * WY_CH, rows = min(WY_CH, m - r0);
        double cv[HC];
#pragma unroll
        for (int c = 0; c < HC; c++)
            cv[c] = (ri < rows && ch + c < ncb) ? C[(long)(c0 + ch + c) * ldc + r0 + ri] : 0.0;
        const double *vb = Vs + (k & 1) * WY_VS;
        double sacc[HC];
#pragma unroll
        for (int c = 0; c < HC; c++) sacc[c] = 0.0;
#pragma unroll 8
        for (int a = 0; a < 32; a++) {
            const double v = vb[ri * 33 + a];
            const double2 *yr = reinterpret_cast<const double2 *>(Y2 + a * NB + ch);
#pragma unroll
            for (int q = 0; q < HC / 2; q++) {
                const double2 y = yr[q];
                sacc[2 * q] = fma(v, y.x, sacc[2 * q]);
                sacc[2 * q + 1] = fma(v, y.y, sacc[2 * q + 1]);
            }
        }
        if (ri < rows) {
#pragma unroll
            for (int c = 0; c < HC; c++)
                if (ch + c < ncb) C[(long)(c0 + ch + c) * ldc + r0 + ri] = cv[c] - sacc[c];
        }
        __syncthreads();
    }
}

// launcher: rows [row0, m) of V and C take part (V is zero above row0 for this panel)
static inline int wy_apply(cudaStream_t s, int m, int ncols, int jb, int row0, const double *V, int ldv, const double *T,
                    int trans, double *C, int ldc)
{
    if (ncols <= 0 || jb <= 0) return LYAP_OK;
    const double mr = m - row0;
    KTimer kt(KC_WY, s, 4.0 * mr * jb * ncols, 8.0 * (2.0 * mr * ncols + mr * jb));
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(wy_apply_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)WY_SMEM);
        cudaFuncSetAttribute(wy_apply_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)WY_SMEM);
        attr = true;
    }
    if (ceil_div(ncols, 8) < 160)
        wy_apply_kernel<4><<<ceil_div(ncols, 4), WY_THREADS, WY_SMEM, s>>>(m, ncols, jb, row0, V, ldv, T, trans, C, ldc);
    else
        wy_apply_kernel<8><<<ceil_div(ncols, 8), WY_THREADS, WY_SMEM, s>>>(m, ncols, jb, row0, V, ldv, T, trans, C, ldc);
    return launched();
}

}  // namespace lyap
