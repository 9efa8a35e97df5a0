// qr.cu -- thin Householder QR of tall-skinny fp64 matrices (Fragments 1-4:
// "Compute a thin QR decomposition F_i = U_i T_i", PAPER.md l.164, l.239,
// l.789, l.823; the error analysis l.357 assumes Householder QR).
//
// Blocked right-looking Householder with compact-WY panels of width 32:
//   panel kernel (one CTA, panel staged in shared memory when it fits):
//     reflectors H_j = I - tau_j v_j v_j^T, v_j = x - alpha e_1,
//     alpha = -sign(x_1)||x||, tau_j = 2 / v_j^T v_j; the reflector is applied
//     to the remaining panel columns one warp per column; then the panel's
//     triangular factor T (H_0..H_{b-1} = I - V T V^T);
//   trailing update W <- W - V (T^T (V^T W)) with the strided GEMM;
//   Q = H_0 ... H_{k-1} [I_k; 0] accumulated backwards the same way.
// The sign convention diag(R) >= 0 makes the factorization unique for full
// column rank, so it matches any other Householder QR up to rounding.
#include <vector>
#include <cooperative_groups.h>
#include "common.cuh"
#include "gemm_simt.cuh"
#include "wy.cuh"
#include "lyap_internal.h"
#include "ktimer.h"

namespace lyap {

static constexpr int QB = 32;

// Warp reduce-scatter: lane l ends with sum over the warp of d[l].  31 shuffles.
__device__ __forceinline__ double reduce_scatter32(double (&d)[QB], int lane)
{
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const bool upper = (lane & off) != 0;
#pragma unroll
        for (int k = 0; k < off; k++) {
            const double send = upper ? d[k] : d[k + off];
            const double keep = upper ? d[k + off] : d[k];
            d[k] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
    }
    return d[0];
}

__device__ __forceinline__ double sel_col32(const double (&r)[QB], int j) {
    double v = r[0];
#pragma unroll
    for (int c = 1; c < QB; c++) v = (c == j) ? r[c] : v;
    return v;
}
__device__ __forceinline__ void set_col32(double (&r)[QB], int j, double x) {
#pragma unroll
    for (int c = 0; c < QB; c++) r[c] = (c == j) ? x : r[c];
}

// Factor panel columns [j0, j0+jb) of W (m x n, ld m), rows j0..m-1.
// Writes V (m x k, ld m; zero above the diagonal), tau, and T_panel (QB x QB).
// Row-distributed: per reflector, every thread forms the dot products of v with all
// panel columns for its rows (32 register accumulators), one warp reduce-scatter +
// one shared-memory pass give the totals; the products with earlier columns are the
// Gram entries V^T v needed for T, so T costs no extra pass.  Two block barriers per
// column (the dots; the look-ahead norm of the next column).
template <bool SM>
__global__ void __launch_bounds__(512)
qr_panel_kernel(int m, int j0, int jb, double *__restrict__ W, double *__restrict__ V,
                double *__restrict__ tau, double *__restrict__ Tp)
{
    extern __shared__ double smp[];
    __shared__ double red[16][QB + 1];
    __shared__ double rnorm[16];
    __shared__ double G[QB][QB + 1];
    const int tid = threadIdx.x, nt = blockDim.x;
    const int lane = tid & 31, wid = tid >> 5;
    const int R = m - j0;                          // panel rows j0..m-1
    double *P = SM ? smp : W + (long)j0 * m + j0;
    const int ldp = SM ? R : m;
    if (SM) {
        for (int c = 0; c < jb; c++)
            for (int i = tid; i < R; i += nt) P[c * R + i] = W[(long)(j0 + c) * m + j0 + i];
    }
    __syncthreads();
    {
        double s0 = 0.0;
        for (int i = 1 + tid; i < R; i += nt) s0 = fma(P[i], P[i], s0);
        s0 = warp_sum(s0);
        if (lane == 0) rnorm[wid] = s0;
        __syncthreads();
    }
    for (int jj = 0; jj < jb; jj++) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < 16; w++) s += rnorm[w];
        const double x0 = P[jj * ldp + jj];
        double tj = 0.0, v0 = 0.0;
        const double nrm2 = s + x0 * x0;
        if (nrm2 != 0.0) {
            const double alpha = (x0 >= 0.0) ? -sqrt(nrm2) : sqrt(nrm2);
            v0 = x0 - alpha;
            tj = 2.0 / (v0 * v0 + s);
        }
        // d[c] = v^T P[:, c] over rows jj..R-1 (c < jj: Gram entries v_c^T v)
        double d[QB];
#pragma unroll
        for (int c = 0; c < QB; c++) d[c] = 0.0;
        if (tj != 0.0) {
            for (int i = jj + tid; i < R; i += nt) {
                const double vi = (i == jj) ? v0 : P[jj * ldp + i];
#pragma unroll
                for (int c = 0; c < QB; c++)
                    if (c < jb) d[c] = fma(vi, P[c * ldp + i], d[c]);
            }
        }
        red[wid][lane] = reduce_scatter32(d, lane);
        __syncthreads();
        double dl = 0.0;
#pragma unroll
        for (int w = 0; w < 16; w++) dl += red[w][lane];
        if (wid == 0 && lane < jj) G[lane][jj] = dl;
#pragma unroll
        for (int c = 0; c < QB; c++) d[c] = __shfl_sync(0xffffffffu, dl, c);
        // apply H_jj to columns jj+1.. and the look-ahead norm of column jj+1
        double s2 = 0.0;
        for (int i = jj + tid; i < R; i += nt) {
            const double vi = (i == jj) ? v0 : P[jj * ldp + i];
            const double f = tj * vi;
#pragma unroll
            for (int c = 0; c < QB; c++) {
                if (c > jj && c < jb) {
                    const double y = fma(-f, d[c], P[c * ldp + i]);
                    P[c * ldp + i] = y;
                    if (c == jj + 1 && i > jj + 1) s2 = fma(y, y, s2);
                }
            }
            if (i == jj && tj != 0.0) P[jj * ldp + jj] = v0;   // column jj now holds v
        }
        if (tid == 0) tau[j0 + jj] = tj;
        s2 = warp_sum(s2);
        if (lane == 0) rnorm[wid] = s2;
        __syncthreads();
    }
    // write V (full columns of length m); x[jj] holds v0
    for (int c = 0; c < jb; c++) {
        const int j = j0 + c;
        const bool nz = tau[j] != 0.0;
        for (int i = tid; i < m; i += nt) V[(long)j * m + i] = (nz && i >= j) ? P[c * ldp + (i - j0)] : 0.0;
    }
    __syncthreads();                // P may alias W (no shared-memory staging)
    if (tid < 32) {                 // row a of T in registers (see wy_T_kernel)
        const int a = tid;
        double Ta[QB];
#pragma unroll
        for (int c = 0; c < QB; c++) Ta[c] = 0.0;
#pragma unroll
        for (int c = 0; c < QB; c++) {
            if (c < jb) {
                double sacc = 0.0;
#pragma unroll
                for (int l = 0; l < c; l++)
                    if (l >= a) sacc = fma(Ta[l], G[l][c], sacc);
                const double tc = tau[j0 + c];
                Ta[c] = (a < c) ? -tc * sacc : ((a == c) ? tc : 0.0);
            }
        }
#pragma unroll
        for (int c = 0; c < QB; c++) Tp[a + c * QB] = Ta[c];
    }
    // R part of the panel columns: above the diagonal from P, below zero (the
    // diagonal is written by qr_finish from alpha)
    for (int c = 0; c < jb; c++)
        for (int i = tid; i < R; i += nt)
            if (i != c) W[(long)(j0 + c) * m + j0 + i] = (i < c) ? P[c * ldp + i] : 0.0;
}

// ---------------------------------------------------------------------------------
// Cluster panel: the same reflectors as qr_panel_kernel, with the panel's rows split
// over a cluster of QC CTAs (one SM each).  Every CTA keeps its RB-row slice of the
// 32-column panel in shared memory; per reflector the partial dot products (E1) and
// the look-ahead norm plus the next pivot entry (E2) are exchanged through
// distributed shared memory with one cluster barrier each.
constexpr int QC = 8, QCT = 256;

__device__ __forceinline__ double reduce_scatter16(double (&d)[16], int lane)
{
#pragma unroll
    for (int off = 8; off >= 1; off >>= 1) {
        const bool upper = (lane & off) != 0;
#pragma unroll
        for (int k = 0; k < off; k++) {
            const double send = upper ? d[k] : d[k + off];
            const double keep = upper ? d[k + off] : d[k];
            d[k] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
    }
    return d[0] + __shfl_xor_sync(0xffffffffu, d[0], 16);   // lane l: column (l & 15)
}

__global__ void __cluster_dims__(QC, 1, 1) __launch_bounds__(QCT)
qr_panel_cluster_kernel(int m, int j0, int jb, int RB, double *__restrict__ W, double *__restrict__ V,
                        double *__restrict__ tau, double *__restrict__ diag, double *__restrict__ Tp)
{
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ double Pl[];                 // RB x QB, column-major (ld RB)
    __shared__ double xch0[QB];                    // E1: this CTA's partial dots
    __shared__ double xch1[16];                    // E2: per warp (norm partial, next pivot entry)
    __shared__ double part[8][16];
    __shared__ double G[QB][QB + 1];
    __shared__ double tl[QB];                      // tau of this panel (every CTA has it)
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int q = (int)cl.block_rank();
    const int R = m - j0;
    const int g0 = q * RB;                         // first panel row of this CTA
    const int nloc = max(0, min(RB, R - g0));
    const int h = tid >> 7, lr0 = tid & 127;       // column half, first local row
    for (int c = 0; c < jb; c++)
        for (int i = tid; i < nloc; i += QCT) Pl[c * RB + i] = W[(long)(j0 + c) * m + j0 + g0 + i];
    __syncthreads();
    // E2 for column 0: norm of rows 1.. and the pivot entry
    {
        double s0 = 0.0, x0p = 0.0;
        if (h == 0)
            for (int i = lr0; i < nloc; i += 128) {
                const double x = Pl[i];
                if (g0 + i >= 1) s0 = fma(x, x, s0);
                else x0p = x;
            }
        s0 = warp_sum(s0);
        x0p = warp_sum(x0p);
        if (lane == 0) { xch1[2 * wid] = s0; xch1[2 * wid + 1] = x0p; }
    }
    auto gather_e2 = [&](double &s, double &x0) {
        const double *rem = cl.map_shared_rank(xch1, lane >> 2);
        double a = 0.0, b = 0.0;
#pragma unroll
        for (int t = 0; t < 2; t++) {
            a += rem[(lane & 3) * 4 + 2 * t];
            b += rem[(lane & 3) * 4 + 2 * t + 1];
        }
        s = warp_sum(a);
        x0 = warp_sum(b);
    };
    cl.sync();
    double s, x0;
    gather_e2(s, x0);
    for (int jj = 0; jj < jb; jj++) {
        double tj = 0.0, v0 = 0.0, alpha = 0.0;
        const double nrm2 = s + x0 * x0;
        if (nrm2 != 0.0) {
            alpha = (x0 >= 0.0) ? -sqrt(nrm2) : sqrt(nrm2);
            v0 = x0 - alpha;
            tj = 2.0 / (v0 * v0 + s);
        }
        // E1: d[c] = v^T P[:, c] (c < jj: Gram entries v_c^T v)
        double d[16];
#pragma unroll
        for (int c = 0; c < 16; c++) d[c] = 0.0;
        if (tj != 0.0) {
            for (int i = lr0; i < nloc; i += 128) {
                const int gi = g0 + i;
                if (gi < jj) continue;
                const double vi = (gi == jj) ? v0 : Pl[jj * RB + i];
#pragma unroll
                for (int c = 0; c < 16; c++)
                    if (h * 16 + c < jb) d[c] = fma(vi, Pl[(h * 16 + c) * RB + i], d[c]);
            }
        }
        const double wv = reduce_scatter16(d, lane);
        if (lane < 16) part[wid][lane] = wv;
        __syncthreads();
        if (tid < QB) {
            const int hb = (tid >> 4) * 4;
            xch0[tid] = part[hb][tid & 15] + part[hb + 1][tid & 15] + part[hb + 2][tid & 15] + part[hb + 3][tid & 15];
        }
        cl.sync();
        double dt = 0.0;
        {
            const int col = h * 16 + (lane & 15);
#pragma unroll
            for (int r = 0; r < QC / 2; r++) dt += cl.map_shared_rank(xch0, 2 * r + (lane >> 4))[col];
            dt += __shfl_xor_sync(0xffffffffu, dt, 16);
            if (q == 0 && lane < 16 && col < jj) G[col][jj] = dt;
        }
#pragma unroll
        for (int c = 0; c < 16; c++) d[c] = __shfl_sync(0xffffffffu, dt, c);
        // apply H_jj to columns jj+1.., look-ahead norm and pivot entry of column jj+1
        double s2 = 0.0, xn = 0.0;
        for (int i = lr0; i < nloc; i += 128) {
            const int gi = g0 + i;
            if (gi < jj) continue;
            const double vi = (gi == jj) ? v0 : Pl[jj * RB + i];
            const double f = tj * vi;
#pragma unroll
            for (int c = 0; c < 16; c++) {
                const int cc = h * 16 + c;
                if (cc > jj && cc < jb) {
                    const double y = fma(-f, d[c], Pl[cc * RB + i]);
                    Pl[cc * RB + i] = y;
                    if (cc == jj + 1) {
                        if (gi > jj + 1) s2 = fma(y, y, s2);
                        else if (gi == jj + 1) xn = y;
                    }
                }
            }
            if (gi == jj && h == 0 && tj != 0.0) Pl[jj * RB + i] = v0;   // column jj now holds v
        }
        if (tid == 0) {
            tl[jj] = tj;
            if (q == 0) { tau[j0 + jj] = tj; diag[j0 + jj] = (tj == 0.0) ? 0.0 : alpha; }
        }
        s2 = warp_sum(s2);
        xn = warp_sum(xn);
        if (lane == 0) { xch1[2 * wid] = s2; xch1[2 * wid + 1] = xn; }
        cl.sync();
        gather_e2(s, x0);
    }
    // V (full columns of length m), the R part above the diagonal, T from the Gram entries
    for (int c = 0; c < jb; c++) {
        const int j = j0 + c;
        const bool nz = tl[c] != 0.0;
        for (int i = tid; i < nloc; i += QCT) {
            const int gi = g0 + i;
            const double pv = Pl[c * RB + i];
            V[(long)j * m + j0 + gi] = (nz && gi >= c) ? pv : 0.0;
            if (gi != c) W[(long)j * m + j0 + gi] = (gi < c) ? pv : 0.0;
        }
        if (q == 0)
            for (int i = tid; i < j0; i += QCT) V[(long)j * m + i] = 0.0;
    }
    if (q == 0) {
        __syncthreads();
        if (tid < 32) {
            const int a = tid;
            double Ta[QB];
#pragma unroll
            for (int c = 0; c < QB; c++) Ta[c] = 0.0;
#pragma unroll
            for (int c = 0; c < QB; c++) {
                if (c < jb) {
                    double sacc = 0.0;
#pragma unroll
                    for (int l = 0; l < c; l++)
                        if (l >= a) sacc = fma(Ta[l], G[l][c], sacc);
                    const double tc = tl[c];
                    Ta[c] = (a < c) ? -tc * sacc : ((a == c) ? tc : 0.0);
                }
            }
#pragma unroll
            for (int c = 0; c < QB; c++) Tp[a + c * QB] = Ta[c];
        }
    }
    cl.sync();                                     // no CTA leaves while its shared memory may be read
}

// ---------------------------------------------------------------------------------
// Register panel: the same reflectors with every panel row held in registers by one
// thread (256 threads per CTA, cluster of NC = ceil(R/256) CTAs, R <= 4096).  One
// cluster exchange per reflector in the common case: the partial dot products of v
// with all 32 panel columns are pushed into every CTA's inbox together with the
// pre-update sums that give the next column's trailing norm by downdating,
//     s' = S_xx - 2 f S_vx + f^2 S_vv   (f = tau d_{j+1}),
// which is used only when s' >= S_xx / 2 (no cancellation: error a few ulp);
// otherwise a second exchange computes s' directly.
constexpr int QRT = 256, QNV = QB + 5;
#ifdef LYAP_PANEL_PROF
__device__ unsigned long long g_qr_fallbacks = 0, g_qr_reflectors = 0;
#endif     // 32 dots + S_xx, S_vx, S_vv, x_{j+1}, v_{j+1}

template <int NV>
__device__ __forceinline__ void qr_cta_reduce_push(double (&vals)[NV], int lane, int wid, int q, int NC,
                                                   double (*part)[NV + 1], double (*inbox)[NV + 1],
                                                   cooperative_groups::cluster_group &cl)
{
    // lanes: reduce-scatter of the first 32 values, plain sums of the rest (lane 0)
    double d[QB];
#pragma unroll
    for (int c = 0; c < QB; c++) d[c] = vals[c];
    const double col = reduce_scatter32(d, lane);
    if constexpr (NV > QB) {
#pragma unroll
        for (int e = QB; e < NV; e++) vals[e] = warp_sum(vals[e]);
    }
    part[wid][lane] = col;
    if constexpr (NV > QB) {
        if (lane == 0)
#pragma unroll
            for (int e = QB; e < NV; e++) part[wid][e] = vals[e];
    }
    __syncthreads();
    const int t = threadIdx.x;
    if (t < NV) {
        double acc = 0.0;
        for (int w = 0; w < QRT / 32; w++) acc += part[w][t];
        for (int r = 0; r < NC; r++) cl.map_shared_rank(&inbox[0][0], r)[q * (NV + 1) + t] = acc;
    }
    cl.sync();
}

__global__ void __launch_bounds__(QRT)
qr_panel_reg_kernel(int m, int j0, int jb, double *__restrict__ W, double *__restrict__ V,
                    double *__restrict__ tau, double *__restrict__ diag, double *__restrict__ Tp)
{
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int q = (int)cl.block_rank(), NC = (int)cl.num_blocks();
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int R = m - j0;
    const int gi = q * QRT + tid;                          // this thread's panel row
    const bool has = gi < R;
    __shared__ double part[QRT / 32][QNV + 1];
    __shared__ double inbox[2][16][QNV + 1];
    __shared__ double tot[QNV];
    __shared__ double G[QB][QB + 1];
    __shared__ double tl[QB];
    double row[QB];
#pragma unroll
    for (int c = 0; c < QB; c++) row[c] = (has && c < jb) ? W[(long)(j0 + c) * m + j0 + gi] : 0.0;
    // column 0: trailing norm and pivot entry (second-exchange path)
    double s, x0;
    {
        double vals[2] = {(has && gi >= 1) ? row[0] * row[0] : 0.0, (has && gi == 0) ? row[0] : 0.0};
#pragma unroll
        for (int e = 0; e < 2; e++) vals[e] = warp_sum(vals[e]);
        if (lane == 0) { part[wid][0] = vals[0]; part[wid][1] = vals[1]; }
        __syncthreads();
        if (tid < 2) {
            double acc = 0.0;
            for (int w = 0; w < QRT / 32; w++) acc += part[w][tid];
            for (int r = 0; r < NC; r++) cl.map_shared_rank(&inbox[1][0][0], r)[q * (QNV + 1) + tid] = acc;
        }
        cl.sync();
        s = 0.0; x0 = 0.0;
        for (int r = 0; r < NC; r++) { s += inbox[1][r][0]; x0 += inbox[1][r][1]; }
        __syncthreads();
    }
    for (int jj = 0; jj < jb; jj++) {
        const int buf = jj & 1;
#ifdef LYAP_PANEL_PROF
        if (q == 0 && tid == 0) atomicAdd(&g_qr_reflectors, 1ull);
#endif
        double tj = 0.0, v0 = 0.0, alpha = 0.0;
        const double nrm2 = s + x0 * x0;
        if (nrm2 != 0.0) {
            alpha = (x0 >= 0.0) ? -sqrt(nrm2) : sqrt(nrm2);
            v0 = x0 - alpha;
            tj = 2.0 / (v0 * v0 + s);
        }
        const double vi = (!has || gi < jj || tj == 0.0) ? 0.0 : (gi == jj ? v0 : sel_col32(row, jj));
        const double xn = sel_col32(row, jj + 1 < QB ? jj + 1 : QB - 1);
        const bool below = has && gi > jj + 1 && jj + 1 < jb;
        double vals[QNV];
#pragma unroll
        for (int c = 0; c < QB; c++) vals[c] = vi * row[c];
        vals[QB + 0] = below ? xn * xn : 0.0;
        vals[QB + 1] = below ? vi * xn : 0.0;
        vals[QB + 2] = below ? vi * vi : 0.0;
        vals[QB + 3] = (has && gi == jj + 1) ? xn : 0.0;
        vals[QB + 4] = (has && gi == jj + 1) ? vi : 0.0;
        qr_cta_reduce_push<QNV>(vals, lane, wid, q, NC, part, inbox[buf], cl);
        if (tid < QNV) {
            double acc = 0.0;
            for (int r = 0; r < NC; r++) acc += inbox[buf][r][tid];
            tot[tid] = acc;
        }
        __syncthreads();
        if (q == 0 && tid < jj) G[tid][jj] = tot[tid];
        if (tid == 0) {
            tl[jj] = tj;
            if (q == 0) { tau[j0 + jj] = tj; diag[j0 + jj] = (tj == 0.0) ? 0.0 : alpha; }
        }
        // apply H_jj to columns jj+1..; column jj keeps v (v0 on the diagonal row)
        if (has && gi >= jj) {
            const double f = tj * vi;
#pragma unroll
            for (int c = 0; c < QB; c++) {
                const double y = fma(-f, tot[c], row[c]);
                row[c] = (c > jj && c < jb) ? y : row[c];
            }
            if (gi == jj && tj != 0.0) set_col32(row, jj, v0);
        }
        if (jj + 1 < jb) {
            // next column: downdated trailing norm, or a second exchange on cancellation
            const double f = tj * tot[jj + 1];
            const double sxx = tot[QB], svx = tot[QB + 1], svv = tot[QB + 2];
            const double sd = sxx - 2.0 * f * svx + f * f * svv;
            x0 = tot[QB + 3] - f * tot[QB + 4];
            if (sd >= 0.5 * sxx) {
                s = sd;
            } else {
#ifdef LYAP_PANEL_PROF
                if (q == 0 && tid == 0) atomicAdd(&g_qr_fallbacks, 1ull);
#endif
                const double xv = sel_col32(row, jj + 1);
                double v2[2] = {below ? xv * xv : 0.0, 0.0};
                v2[0] = warp_sum(v2[0]);
                __syncthreads();                                // tot / part reads above are done
                if (lane == 0) part[wid][0] = v2[0];
                __syncthreads();
                if (tid == 0) {
                    double acc = 0.0;
                    for (int w = 0; w < QRT / 32; w++) acc += part[w][0];
                    for (int r = 0; r < NC; r++) cl.map_shared_rank(&inbox[buf ^ 1][0][0], r)[q * (QNV + 1) + QNV] = acc;
                }
                cl.sync();
                s = 0.0;
                for (int r = 0; r < NC; r++) s += inbox[buf ^ 1][r][QNV];
            }
        }
        __syncthreads();
    }
    // V (this CTA's rows), the R part above the diagonal, T on CTA 0
    if (has) {
#pragma unroll
        for (int c = 0; c < QB; c++) {
            if (c < jb) {
                const int j = j0 + c;
                V[(long)j * m + j0 + gi] = (tl[c] != 0.0 && gi >= c) ? row[c] : 0.0;
                if (gi != c) W[(long)j * m + j0 + gi] = (gi < c) ? row[c] : 0.0;
            }
        }
    }
    if (q == 0)
        for (int c = 0; c < jb; c++)
            for (int i = tid; i < j0; i += QRT) V[(long)(j0 + c) * m + i] = 0.0;
    if (q == 0 && tid < 32) {
        const int a = tid;
        double Ta[QB];
#pragma unroll
        for (int c = 0; c < QB; c++) Ta[c] = 0.0;
#pragma unroll
        for (int c = 0; c < QB; c++) {
            if (c < jb) {
                double sacc = 0.0;
#pragma unroll
                for (int l = 0; l < c; l++)
                    if (l >= a) sacc = fma(Ta[l], G[l][c], sacc);
                const double tc = tl[c];
                Ta[c] = (a < c) ? -tc * sacc : ((a == c) ? tc : 0.0);
            }
        }
#pragma unroll
        for (int c = 0; c < QB; c++) Tp[a + c * QB] = Ta[c];
    }
    cl.sync();
}

__global__ void set_identity_kernel(int m, int k, double *Q) {
    long tot = (long)m * k;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < tot; idx += (long)gridDim.x * blockDim.x) {
        long i = idx % m, c = idx / m;
        Q[idx] = (i == c) ? 1.0 : 0.0;
    }
}

// R = upper k x n part of W, then the sign fix on R rows and Q columns.
__global__ void qr_finish_kernel(int m, int n, int k, const double *__restrict__ W, const double *__restrict__ diag,
                                 double *__restrict__ Q, double *__restrict__ R)
{
    long tot = (long)k * n;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < tot; idx += (long)gridDim.x * blockDim.x) {
        int i = (int)(idx % k), c = (int)(idx / k);
        double sg = (diag[i] < 0.0) ? -1.0 : 1.0;
        double v = (i < c) ? W[(long)c * m + i] : (i == c ? diag[i] : 0.0);
        R[idx] = sg * v;
    }
    long totq = (long)m * k;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < totq; idx += (long)gridDim.x * blockDim.x) {
        int c = (int)(idx / m);
        if (diag[c] < 0.0) Q[idx] = -Q[idx];
    }
}

// diag_j = alpha_j (or the untouched x0 when tau_j = 0) from V's leading entry:
// alpha = x0 - v0 where x0 = v0 + alpha ... we recompute alpha from ||x||: the panel
// stores ||x|| implicitly in tau: tau = 2/(v0^2 + s), v0 = x0 - alpha, alpha^2 = x0^2 + s.
// Simplest exact route: alpha_j = -(sign v0) * ... -> keep an explicit array instead.

int QrWork::alloc(int mmax_, int nmax_) {
    mmax = mmax_; nmax = nmax_;
    int kmax = mmax < nmax ? mmax : nmax;
    LYAP_CUDA_TRY(cudaMalloc(&V, sizeof(double) * (size_t)mmax * kmax));
    LYAP_CUDA_TRY(cudaMalloc(&T, sizeof(double) * (size_t)QB * QB * (kmax / 8 + 2)));
    LYAP_CUDA_TRY(cudaMalloc(&W, sizeof(double) * (size_t)2 * QB * (nmax > mmax ? nmax : mmax)));
    LYAP_CUDA_TRY(cudaMalloc(&tau, sizeof(double) * (size_t)2 * kmax));
    LYAP_CUDA_TRY(cudaMalloc(&Wk, sizeof(double) * (size_t)mmax * nmax));
    return LYAP_OK;
}
void QrWork::release() { cudaFree(V); cudaFree(T); cudaFree(W); cudaFree(tau); cudaFree(Wk); V = T = W = tau = Wk = nullptr; }

// alpha_j from the reflector: v = x - alpha e1 and tau = 2/(v^T v), ||v||^2 = 2 ||x||(||x|| + |x0|)
// -> with v0 = x0 - alpha, alpha = -sign(x0) ||x||:  v0 = x0 + sign(x0)||x||, so
// alpha = -sign(v0) * (|v0| - |x0|) = x0 - v0.  x0 is not kept, but v^T v = 2/tau and
// v0^2 - (v0^T v - v0^2)... -> we simply compute alpha = x0 - v0 inside the panel kernel.
__global__ void qr_alpha_kernel(int m, int j0, int jb, const double *__restrict__ V, const double *__restrict__ tau,
                                double *__restrict__ diag)
{
    // ||x||^2 = v0^2 + s where s = sum_{i>j} v_i^2 and v^T v = v0^2 + s = 2/tau -> the
    // norm of x is sqrt(x0^2 + s); with x0 = v0 + alpha and alpha^2 = x0^2 + s:
    //   alpha = -(v0^2 + s) / (2 v0) = -(1/tau)/v0
    const int c = threadIdx.x;
    if (c < jb) {
        const int j = j0 + c;
        const double t = tau[j];
        diag[j] = (t == 0.0) ? 0.0 : -(1.0 / t) / V[(long)j * m + j];
    }
}

int qr_f64(cudaStream_t s, int m, int n, const double *A, double *Q, double *R, QrWork &w)
{
    if (m <= 0 || n <= 0) return LYAP_OK;
    if (m > w.mmax || n > w.nmax) return LYAP_ERR_CAPACITY;
    KTimer kt(KC_QR, s);
    const int k = m < n ? m : n;
    double *Wm = w.Wk;
    double *diag = w.tau + k;
    // one-time setup (function-local static: thread-safe initialisation)
    static const bool attr = [] {
        cudaFuncSetAttribute(qr_panel_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(qr_panel_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        return true;
    }();
    (void)attr;
    LYAP_CUDA_TRY(cudaMemcpyAsync(Wm, A, sizeof(double) * (size_t)m * n, cudaMemcpyDeviceToDevice, s));
    // cluster panels (32 wide) while a CTA's row slice fits in shared memory; otherwise
    // the one-CTA panel with widths 32, or 16/8 while the panel would not fit
    const bool use_cluster = ceil_div(m, QC) * QB * sizeof(double) <= 200 * 1024 && !env_flag("LYAP_QR_1CTA");
    std::vector<int> starts;
    for (int j0 = 0, jb; j0 < k; j0 += jb) {
        jb = QB;
        while (!use_cluster && jb > 8 && sizeof(double) * (size_t)(m - j0) * jb > 200 * 1024) jb /= 2;
        jb = std::min(jb, k - j0);
        starts.push_back(j0);
    }
    starts.push_back(k);
    for (size_t pi = 0; pi + 1 < starts.size(); pi++) {
        const int j0 = starts[pi], jb = starts[pi + 1] - j0;
        double *Tp = w.T + pi * QB * QB;
        if (m - j0 <= 16 * QRT && !env_flag("LYAP_QR_SMEM")) {
            const int nc = ceil_div(m - j0, QRT);
            KTimer kp(KC_QR_PANEL, s, 4.0 * (m - j0) * jb * jb, 16.0 * (m - j0) * jb);
            // one-time setup (function-local static: thread-safe initialisation)
            static const bool attr_r = [] {
                cudaFuncSetAttribute(qr_panel_reg_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
                return true;
            }();
            (void)attr_r;
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(nc, 1, 1);
            cfg.blockDim = dim3(QRT, 1, 1);
            cfg.stream = s;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = nc;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            LYAP_CUDA_TRY(cudaLaunchKernelEx(&cfg, qr_panel_reg_kernel, m, j0, jb, Wm, w.V, w.tau, diag, Tp));
            LYAP_TRY(launched());
        } else if (use_cluster) {
            const int RB = ceil_div(m - j0, QC);
            KTimer kp(KC_QR_PANEL, s, 4.0 * (m - j0) * jb * jb, 16.0 * (m - j0) * jb);
            qr_panel_cluster_kernel<<<QC, QCT, sizeof(double) * RB * QB, s>>>(m, j0, jb, RB, Wm, w.V, w.tau, diag,
                                                                           Tp);
            LYAP_TRY(launched());
        } else {
            const size_t smem = sizeof(double) * (size_t)(m - j0) * jb;
            const bool use_smem = smem <= 200 * 1024;
            {
                KTimer kp(KC_QR_PANEL, s, 4.0 * (m - j0) * jb * jb, 16.0 * (m - j0) * jb);
                if (use_smem) qr_panel_kernel<true><<<1, 512, smem, s>>>(m, j0, jb, Wm, w.V, w.tau, Tp);
                else qr_panel_kernel<false><<<1, 512, 0, s>>>(m, j0, jb, Wm, w.V, w.tau, Tp);
            }
            LYAP_TRY(launched());
            qr_alpha_kernel<<<1, 32, 0, s>>>(m, j0, jb, w.V, w.tau, diag);
            LYAP_TRY(launched());
        }
        int nt = n - (j0 + jb);
        if (nt > 0) {
            const double *Vp = w.V + (size_t)j0 * m;
            double *Wt = Wm + (size_t)(j0 + jb) * m;
            // Wt <- (I - V T^T V^T) Wt, rows j0..m-1 (V is zero above)
            LYAP_TRY(wy_apply(s, m, nt, jb, j0, Vp, m, Tp, 1, Wt, m));
        }
    }
    // Q = H_0 ... H_{k-1} [I; 0]
    set_identity_kernel<<<ceil_div((long)m * k, 256) < 1024 ? ceil_div((long)m * k, 256) : 1024, 256, 0, s>>>(m, k, Q);
    LYAP_TRY(launched());
    for (int pi = (int)starts.size() - 2; pi >= 0; pi--) {
        const int j0 = starts[pi], jb = starts[pi + 1] - j0;
        const double *Tp = w.T + (size_t)pi * QB * QB;
        const double *Vp = w.V + (size_t)j0 * m;
        int nc = k - j0;               // columns j0..k-1 of Q are affected
        double *Qc = Q + (size_t)j0 * m;
        LYAP_TRY(wy_apply(s, m, nc, jb, j0, Vp, m, Tp, 0, Qc, m));
    }
    int tot = (int)(((long)k * n + (long)m * k + 255) / 256);
    qr_finish_kernel<<<tot < 1024 ? tot : 1024, 256, 0, s>>>(m, n, k, Wm, diag, Q, R);
    return launched();
}

}  // namespace lyap

#ifdef LYAP_PANEL_PROF
extern "C" void lyap_debug_qr_counters(unsigned long long *fb, unsigned long long *refl)
{
    cudaMemcpyFromSymbol(fb, lyap::g_qr_fallbacks, sizeof(*fb));
    cudaMemcpyFromSymbol(refl, lyap::g_qr_reflectors, sizeof(*refl));
}
#endif
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
