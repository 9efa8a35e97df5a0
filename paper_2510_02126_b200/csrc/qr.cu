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
#include <type_traits>
#include <cooperative_groups.h>
#include "common.cuh"
#include "gemm_simt.cuh"
#include "wy.cuh"
#include "lyap_internal.h"
#include "ktimer.h"

namespace lyap {

static constexpr int QB = 32;
constexpr int QB2 = 256;      // outer block of the two-level blocking

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

// Exchange of the per-CTA partial sums of one reflector step between the CTAs that
// hold the panel rows.  Cluster flavour (R <= 16 x 256 rows): every CTA pushes its
// partials into every CTA's shared-memory inbox (DSMEM) and one cluster barrier
// publishes them.  Grid flavour (taller panels, a cooperative launch of ceil(R/256)
// CTAs): every CTA stores its partials once in a global inbox and one grid barrier
// publishes them.  Both inboxes are double-buffered by step parity (a fast CTA writes
// step j+1's partials while a slow one may still read step j's); every CTA then sums
// the NC partials of a slot in the same fixed order (deterministic).
struct QrXCluster {
    cooperative_groups::cluster_group cl;
    double (*inbox)[16][QNV + 1];                  // shared [2][16][QNV + 1]
    int q, NC;
    __device__ QrXCluster(double (*ib)[16][QNV + 1], double *)
        : cl(cooperative_groups::this_cluster()), inbox(ib), q((int)cl.block_rank()), NC((int)cl.num_blocks()) {}
    __device__ void put(int buf, int slot, double v) {
        for (int r = 0; r < NC; r++) cl.map_shared_rank(&inbox[buf][0][0], r)[q * (QNV + 1) + slot] = v;
    }
    __device__ double get(int buf, int r, int slot) const { return inbox[buf][r][slot]; }
    __device__ void sync() { cl.sync(); }
};
struct QrXGrid {
    cooperative_groups::grid_group g;
    double *gin;                                   // global [2][NC][QNV + 1]
    int q, NC;
    __device__ QrXGrid(double (*)[16][QNV + 1], double *g_in)
        : g(cooperative_groups::this_grid()), gin(g_in), q((int)blockIdx.x), NC((int)gridDim.x) {}
    __device__ void put(int buf, int slot, double v) { gin[((long)buf * NC + q) * (QNV + 1) + slot] = v; }
    __device__ double get(int buf, int r, int slot) const { return __ldcg(gin + ((long)buf * NC + r) * (QNV + 1) + slot); }
    __device__ void sync() { g.sync(); }
};

template <int NV, class X>
__device__ __forceinline__ void qr_cta_reduce_push(double (&vals)[NV], int lane, int wid, int buf,
                                                   double (*part)[NV + 1], X &x)
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
        x.put(buf, t, acc);
    }
    x.sync();
}

// Sum over the NC CTAs of inbox slot `slot` (fixed order r = 0..NC-1).
template <class X>
__device__ __forceinline__ double qr_gather(const X &x, int buf, int slot)
{
    double acc = 0.0;
    for (int r = 0; r < x.NC; r++) acc += x.get(buf, r, slot);
    return acc;
}

template <bool GRID>
__global__ void __launch_bounds__(QRT)
qr_panel_reg_kernel(int m, int j0, int jb, double *__restrict__ W, double *__restrict__ V,
                    double *__restrict__ tau, double *__restrict__ diag, double *__restrict__ Tp,
                    double *__restrict__ gin)
{
    namespace cg = cooperative_groups;
    using X = std::conditional_t<GRID, QrXGrid, QrXCluster>;
    __shared__ double inbox_sh[GRID ? 1 : 2][16][QNV + 1];
    X x(inbox_sh, gin);
    const int q = x.q;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int R = m - j0;
    const int gi = q * QRT + tid;                          // this thread's panel row
    const bool has = gi < R;
    __shared__ double part[QRT / 32][QNV + 1];
    __shared__ double tot[QNV + 1];
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
            x.put(1, tid, acc);
        }
        x.sync();
        if (tid < 2) tot[tid] = qr_gather(x, 1, tid);
        __syncthreads();
        s = tot[0]; x0 = tot[1];
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
        qr_cta_reduce_push<QNV>(vals, lane, wid, buf, part, x);
        if (tid < QNV) tot[tid] = qr_gather(x, buf, tid);
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
                    x.put(buf ^ 1, QNV, acc);
                }
                x.sync();
                if (tid == 0) tot[QNV] = qr_gather(x, buf ^ 1, QNV);
                __syncthreads();
                s = tot[QNV];
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
    if constexpr (!GRID) x.sync();                 // no CTA leaves while its shared memory may be read
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
    gin_ctas = ceil_div(mmax, QRT);
    LYAP_CUDA_TRY(cudaMalloc(&gin, sizeof(double) * (size_t)2 * gin_ctas * (QNV + 1)));
    if (kmax > QB2) {
        LYAP_CUDA_TRY(cudaMalloc(&Tbig, sizeof(double) * (size_t)QB2 * QB2 * (kmax / QB2 + 1)));
        LYAP_CUDA_TRY(cudaMalloc(&G, sizeof(double) * (size_t)QB2 * QB2));
        LYAP_CUDA_TRY(cudaMalloc(&W1, sizeof(double) * (size_t)QB2 * nmax));
        LYAP_CUDA_TRY(cudaMalloc(&W2, sizeof(double) * (size_t)QB2 * nmax));
    }
    return LYAP_OK;
}
void QrWork::release() {
    for (double *p : {V, T, W, tau, Wk, gin, Tbig, G, W1, W2}) if (p) cudaFree(p);
    V = T = W = tau = Wk = gin = Tbig = G = W1 = W2 = nullptr;
}

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

// Compact-WY factor of an outer block of up to QB2 = 256 reflectors (8 panels of 32):
// T = [[T_11, T_12], [0, T_22]] with the panel factors T_bb (from the panel kernels) on
// the diagonal and, block column by block column,
//     T(0:32b, b) = -T(0:32b, 0:32b) (G(0:32b, b) T_bb),   G = V^T V,
// the LAPACK xLARFT recurrence taken 32 columns at a time.  One CTA; T (ld QB2) is
// upper triangular with zeros below the diagonal.
__global__ void __launch_bounds__(1024)
qr_bigT_kernel(int Jb, const double *__restrict__ G, const double *__restrict__ Tsmall, double *__restrict__ Tb)
{
    extern __shared__ double m1_sm[];
    double (*M1)[QB + 1] = reinterpret_cast<double (*)[QB + 1]>(m1_sm);   // [QB2 - QB][QB + 1]
    const int tid = threadIdx.x, nt = blockDim.x;
    const int nb = (Jb + QB - 1) / QB;
    for (int e = tid; e < QB2 * QB2; e += nt) {
        const int i = e % QB2, c = e / QB2;
        const int bi = i / QB, bc = c / QB;
        Tb[e] = (bi == bc && i < Jb && c < Jb) ? Tsmall[(long)bc * QB * QB + (i % QB) + (c % QB) * QB] : 0.0;
    }
    __syncthreads();
    for (int b = 1; b < nb; b++) {
        const int r = QB * b, cb = min(QB, Jb - r);
        const double *Tbb = Tsmall + (long)b * QB * QB;
        for (int e = tid; e < r * QB; e += nt) {
            const int i = e % r, c = e / r;
            double acc = 0.0;
            if (c < cb)
                for (int l = 0; l <= c; l++) acc = fma(G[i + (long)(r + l) * Jb], Tbb[l + c * QB], acc);
            M1[i][c] = acc;
        }
        __syncthreads();
        for (int e = tid; e < r * QB; e += nt) {
            const int i = e % r, c = e / r;
            if (c < cb) {
                double acc = 0.0;
                for (int l = i; l < r; l++) acc = fma(Tb[i + (long)l * QB2], M1[l][c], acc);
                Tb[i + (long)(r + c) * QB2] = -acc;
            }
        }
        __syncthreads();
    }
}

// C (rows row0..m-1, ncols columns, ld ldc) <- (I - V op(T) V^T) C with the outer-block
// reflectors V (rows row0.., Jb columns, ld ldv) and T (ld QB2): three DMMA GEMMs,
// op(T) = T^T for Q^T (trans = 1) and T for Q (trans = 0).
static int qr_block_apply(cudaStream_t s, int m, int row0, int ncols, int Jb, const double *V, int ldv,
                          const double *Tb, int trans, double *C, int ldc, double *W1, double *W2)
{
    if (ncols <= 0) return LYAP_OK;
    const int mr = m - row0;
    const double *Vs = V + row0;
    double *Cs = C + row0;
    LYAP_TRY(dgemm_cm(s, true, false, Jb, ncols, mr, 1.0, Vs, ldv, Cs, ldc, 0.0, W1, Jb));
    LYAP_TRY(dgemm_cm(s, trans != 0, false, Jb, ncols, Jb, 1.0, Tb, QB2, W1, Jb, 0.0, W2, Jb));
    return dgemm_cm(s, false, false, mr, ncols, Jb, -1.0, Vs, ldv, W2, Jb, 1.0, Cs, ldc);
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
    // register panels (32 wide, one row per thread): a cluster of up to 16 CTAs for R <=
    // 4096 panel rows, a cooperative grid of ceil(R / 256) co-resident CTAs above; the
    // shared-memory cluster panel and the one-CTA panel (widths 32, or 16/8 while the panel
    // would not fit) remain for panels taller than one co-resident grid
    static const int grid_max = [] {
        int dev = 0, nsm = 0, per = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(qr_panel_reg_kernel<false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, qr_panel_reg_kernel<true>, QRT, 0);
        return nsm * std::max(per, 0);
    }();
    const bool use_grid = ceil_div(m, QRT) <= std::min(grid_max, w.gin_ctas) && !env_flag("LYAP_QR_NOGRID");
    const bool use_cluster = ceil_div(m, QC) * QB * sizeof(double) <= 200 * 1024 && !env_flag("LYAP_QR_1CTA");
    std::vector<int> starts;
    for (int j0 = 0, jb; j0 < k; j0 += jb) {
        jb = QB;
        while (!use_cluster && !use_grid && jb > 8 && sizeof(double) * (size_t)(m - j0) * jb > 200 * 1024) jb /= 2;
        jb = std::min(jb, k - j0);
        starts.push_back(j0);
    }
    starts.push_back(k);
    // two-level blocking for tall, wide factorizations (all panels 32 wide), one level
    // below (measured: the per-panel fused application wins while the matrix sits in L2)
    bool two_level = (use_grid || use_cluster) && (long)m * n >= (1L << 22) && k > QB2 && w.Tbig != nullptr;
    if (env_flag("LYAP_QR_1LEVEL")) two_level = false;
    if (env_flag("LYAP_QR_2LEVEL") && (use_grid || use_cluster) && w.Tbig) two_level = true;
    for (size_t pi = 0; pi + 1 < starts.size(); pi++) {
        const int j0 = starts[pi], jb = starts[pi + 1] - j0;
        double *Tp = w.T + pi * QB * QB;
        if (m - j0 <= 16 * QRT && !env_flag("LYAP_QR_SMEM")) {
            const int nc = ceil_div(m - j0, QRT);
            KTimer kp(KC_QR_PANEL, s, 4.0 * (m - j0) * jb * jb, 16.0 * (m - j0) * jb);
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
            LYAP_CUDA_TRY(cudaLaunchKernelEx(&cfg, qr_panel_reg_kernel<false>, m, j0, jb, Wm, w.V, w.tau, diag, Tp,
                                             (double *)nullptr));
            LYAP_TRY(launched());
        } else if (use_grid) {
            const int nc = ceil_div(m - j0, QRT);
            KTimer kp(KC_QR_PANEL, s, 4.0 * (m - j0) * jb * jb, 16.0 * (m - j0) * jb);
            int mm = m, jj0 = j0, jjb = jb;
            double *Wp = Wm, *Vp = w.V, *tp = w.tau, *dp = diag, *Tq = Tp, *gp = w.gin;
            void *args[] = {&mm, &jj0, &jjb, &Wp, &Vp, &tp, &dp, &Tq, &gp};
            LYAP_CUDA_TRY(cudaLaunchCooperativeKernel((void *)qr_panel_reg_kernel<true>, dim3(nc), dim3(QRT), args, 0, s));
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
        // two-level: the panel's reflectors update the rest of their outer block (wy_apply);
        // at the end of an outer block its 256 reflectors update the trailing columns at
        // once (G = V^T V, T_big, three DMMA GEMMs).  One level: every panel updates all
        // trailing columns.
        const int J0 = two_level ? (j0 / QB2) * QB2 : j0;
        const int Jend = two_level ? std::min(J0 + QB2, k) : n;
        int nt = std::min(n, Jend) - (j0 + jb);
        if (nt > 0) {
            const double *Vp = w.V + (size_t)j0 * m;
            double *Wt = Wm + (size_t)(j0 + jb) * m;
            // Wt <- (I - V T^T V^T) Wt, rows j0..m-1 (V is zero above)
            LYAP_TRY(wy_apply(s, m, nt, jb, j0, Vp, m, Tp, 1, Wt, m));
        }
        if (two_level && j0 + jb == Jend) {
            const int Jb = Jend - J0, ob = J0 / QB2;
            const double *Vb = w.V + (size_t)J0 * m;
            double *Tb = w.Tbig + (size_t)ob * QB2 * QB2;
            LYAP_TRY(dgemm_cm(s, true, false, Jb, Jb, m - J0, 1.0, Vb + J0, m, Vb + J0, m, 0.0, w.G, Jb));
            constexpr size_t bigT_smem = sizeof(double) * (QB2 - QB) * (QB + 1);
            static const bool bigT_attr = [] {
                cudaFuncSetAttribute(qr_bigT_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bigT_smem);
                return true;
            }();
            (void)bigT_attr;
            qr_bigT_kernel<<<1, 1024, bigT_smem, s>>>(Jb, w.G, w.T + (size_t)(J0 / QB) * QB * QB, Tb);
            LYAP_TRY(launched());
            LYAP_TRY(qr_block_apply(s, m, J0, n - Jend, Jb, Vb, m, Tb, 1, Wm + (size_t)Jend * m, m, w.W1, w.W2));
        }
    }
    // Q = H_0 ... H_{k-1} [I; 0]
    set_identity_kernel<<<ceil_div((long)m * k, 256) < 1024 ? ceil_div((long)m * k, 256) : 1024, 256, 0, s>>>(m, k, Q);
    LYAP_TRY(launched());
    if (two_level) {
        for (int ob = (k - 1) / QB2; ob >= 0; ob--) {
            const int J0 = ob * QB2, Jb = std::min(QB2, k - J0);
            LYAP_TRY(qr_block_apply(s, m, J0, k - J0, Jb, w.V + (size_t)J0 * m, m, w.Tbig + (size_t)ob * QB2 * QB2, 0,
                                    Q + (size_t)J0 * m, m, w.W1, w.W2));
        }
    } else {
        for (int pi = (int)starts.size() - 2; pi >= 0; pi--) {
            const int j0 = starts[pi], jb = starts[pi + 1] - j0;
            const double *Tp = w.T + (size_t)pi * QB * QB;
            const double *Vp = w.V + (size_t)j0 * m;
            int nc = k - j0;               // columns j0..k-1 of Q are affected
            double *Qc = Q + (size_t)j0 * m;
            LYAP_TRY(wy_apply(s, m, nc, jb, j0, Vp, m, Tp, 0, Qc, m));
        }
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
