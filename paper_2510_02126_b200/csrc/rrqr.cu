// rrqr.cu -- RankTruncChol (Algorithm 3 sub-function, l.1256-1266):
// rank-revealing QR  Z^T Pi = Q [T C; 0 S],  ||S|| <= sqrt(u) ||Z||,
// return Pi [T C]^T.
//
// Householder QR with column pivoting on M = Z^T (c x n), in binary64
// (reading R-TRUNC-PREC), as one cooperative kernel: per step j
//   A) warp-per-column norms of the trailing block M[j:c, j:n] + block argmax
//   B) every CTA reduces the per-CTA results identically (stop test
//      ||S_j||_F <= tol |r_11|, reading R-RRQR; pivot = max norm, lowest
//      index); CTA 0 swaps the pivot column in and forms the reflector
//   C) warp-per-column application of the reflector.
// Grid-wide barriers separate the phases.
#include <cooperative_groups.h>
#include "common.cuh"
#include "gemm_simt.cuh"
#include "lyap_internal.h"
#include "ktimer.h"

namespace cg = cooperative_groups;

namespace lyap {

struct RrqrArgs {
    int n, c, kmax;
    double tol;
    double *M;          // c x n col-major
    double *nrm;        // n
    double *bsum;       // gridDim
    double *bbest;      // gridDim
    int *bidx;          // gridDim
    int *perm;          // n
    double *v;          // c
    double *scal;       // [0] r11, [1] vtv, [2] alpha
    int *rank;          // 1
};

__global__ void __launch_bounds__(256)
rrqr_kernel(RrqrArgs a)
{
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nwb = blockDim.x >> 5;
    const int gw = blockIdx.x * nwb + wib, nwg = gridDim.x * nwb;
    const int n = a.n, c = a.c;
    __shared__ double s_sum[8], s_best[8];
    __shared__ int s_idx[8];
    __shared__ int s_stop, s_piv;
    int rank = a.kmax;
    for (int j = 0; j < a.kmax; j++) {
        // ---- A: column norms over rows j..c-1
        double bsum = 0.0, bbest = -1.0; int bidx = n;
        for (int col = j + gw; col < n; col += nwg) {
            const double *x = a.M + (long)col * c;
            double s = 0.0;
            for (int i = j + lane; i < c; i += 32) s = fma(x[i], x[i], s);
            s = warp_sum(s);
            bsum += s;
            if (s > bbest || (s == bbest && col < bidx)) { bbest = s; bidx = col; }
        }
        if (lane == 0) { s_sum[wib] = bsum; s_best[wib] = bbest; s_idx[wib] = bidx; }
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0, bv = -1.0; int bi = n;
            for (int w = 0; w < nwb; w++) {
                t += s_sum[w];
                if (s_best[w] > bv || (s_best[w] == bv && s_idx[w] < bi)) { bv = s_best[w]; bi = s_idx[w]; }
            }
            a.bsum[blockIdx.x] = t; a.bbest[blockIdx.x] = bv; a.bidx[blockIdx.x] = bi;
        }
        grid.sync();
        // ---- B: identical reduction in every CTA
        if (wib == 0) {
            double t = 0.0, bv = -1.0; int bi = n;
            for (int b = lane; b < (int)gridDim.x; b += 32) {
                t += a.bsum[b];
                double v = a.bbest[b]; int i2 = a.bidx[b];
                if (v > bv || (v == bv && i2 < bi)) { bv = v; bi = i2; }
            }
            t = warp_sum(t);
            for (int o = 16; o > 0; o >>= 1) {
                double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
                int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
                if (v2 > bv || (v2 == bv && i2 < bi)) { bv = v2; bi = i2; }
            }
            if (lane == 0) {
                double tr = sqrt(t);
                int stop = 0;
                if (j > 0 && tr <= a.tol * a.scal[0]) stop = 1;
                if (tr == 0.0) stop = 1;
                s_stop = stop; s_piv = bi;
            }
        }
        __syncthreads();
        if (s_stop) { rank = j; break; }
        if (blockIdx.x == 0) {
            const int pc = s_piv;
            double *xj = a.M + (long)j * c, *xp = a.M + (long)pc * c;
            if (pc != j) {
                for (int i = threadIdx.x; i < c; i += blockDim.x) { double t = xj[i]; xj[i] = xp[i]; xp[i] = t; }
                if (threadIdx.x == 0) { int t = a.perm[j]; a.perm[j] = a.perm[pc]; a.perm[pc] = t; }
            }
            __syncthreads();
            if (wib == 0) {
                double s = 0.0;
                for (int i = j + lane; i < c; i += 32) s = fma(xj[i], xj[i], s);
                s = warp_sum(s);
                double nrm = sqrt(s), x0 = xj[j];
                double alpha = (x0 >= 0.0) ? -nrm : nrm;
                double v0 = x0 - alpha;
                double vtv = v0 * v0 + (s - x0 * x0);
                for (int i = j + lane; i < c; i += 32) a.v[i] = (i == j) ? v0 : xj[i];
                __syncwarp();
                for (int i = j + lane; i < c; i += 32) xj[i] = (i == j) ? alpha : 0.0;
                if (lane == 0) {
                    a.scal[1] = vtv;
                    if (j == 0) a.scal[0] = fabs(alpha);
                }
            }
        }
        grid.sync();
        // ---- C: apply H_j to columns j+1..n-1
        const double vtv = a.scal[1];
        if (vtv != 0.0) {
            for (int col = j + 1 + gw; col < n; col += nwg) {
                double *y = a.M + (long)col * c;
                double d = 0.0;
                for (int i = j + lane; i < c; i += 32) d = fma(a.v[i], y[i], d);
                d = warp_sum(d);
                const double f = 2.0 * d / vtv;
                for (int i = j + lane; i < c; i += 32) y[i] = fma(-f, a.v[i], y[i]);
            }
        }
        grid.sync();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *a.rank = rank;
}

// Second version: one grid barrier per pivot step.  Physical columns never move (the
// pivot order is kept in perm, and the output needs none: Zout(col, r) = M[col][r]);
// every warp owns the same columns for the whole factorisation and keeps their
// trailing norms, downdated after each reflector (||x[j+1:]||^2 = ||x[j:]||^2 - x_j^2)
// and recomputed exactly when the downdate cancels (LAPACK xLAQP2 rule).  Per step:
//   grid barrier -> every CTA reduces the per-CTA (sum, argmax) partials identically,
//   forms the reflector of the pivot column in shared memory -> owners finalise the
//   previous pivot column, apply H_j to their active columns, downdate, and publish
//   the next partials.
struct Rrqr2Args {
    int n, c, kmax;
    double tol;
    double *M;          // c x n col-major
    double *nrm2;       // n: trailing norm^2 (rows >= current step)
    double *nrm0;       // n: norm^2 at the last exact recomputation
    double *bsum;       // 2 x gridDim (double-buffered by step parity)
    double *bbest;      // 2 x gridDim
    int *bidx;          // 2 x gridDim
    int *perm;          // n: pivot order
    int *active;        // n: 1 while not pivoted
    double *scal;       // [0] |r_11|
    int *rank;
};

template <int RPL>
__global__ void __launch_bounds__(256, RPL == 0 ? 4 : 2)
rrqr2_kernel(Rrqr2Args a)
{
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double vsh[];                  // reflector, c entries
    __shared__ double red[32];
    __shared__ double s_best[8], s_sum[8];
    __shared__ int s_idx[8];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nwb = blockDim.x >> 5;
    const int gw = blockIdx.x * nwb + wib, nwg = gridDim.x * nwb;
    const int n = a.n, c = a.c, G = gridDim.x;
    // Owned columns col = gw + t nwg (t < 32): lane t keeps that column's trailing norm^2,
    // its norm^2 at the last exact recomputation and its active flag in registers (no
    // global metadata loads in front of the column loads).
    double m_n2 = 0.0, m_n0 = 0.0;
    bool m_act = false;
    // initial norms (rows 0..c-1), partials of step 0
    {
        double bsum = 0.0, bbest = -1.0; int bidx = n;
        for (int col = gw, t = 0; col < n; col += nwg, t++) {
            const double *x = a.M + (long)col * c;
            double s = 0.0;
            for (int i = lane; i < c; i += 32) s = fma(x[i], x[i], s);
            s = warp_sum(s);
            if (lane == t) { m_n2 = s; m_n0 = s; m_act = true; }
            bsum += s;
            if (s > bbest || (s == bbest && col < bidx)) { bbest = s; bidx = col; }
        }
        if (lane == 0) { s_sum[wib] = bsum; s_best[wib] = bbest; s_idx[wib] = bidx; }
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0, bv = -1.0; int bi = n;
            for (int w = 0; w < nwb; w++) {
                t += s_sum[w];
                if (s_best[w] > bv || (s_best[w] == bv && s_idx[w] < bi)) { bv = s_best[w]; bi = s_idx[w]; }
            }
            a.bsum[blockIdx.x] = t; a.bbest[blockIdx.x] = bv; a.bidx[blockIdx.x] = bi;
        }
    }
    int rank = a.kmax, prev = -1;
    double r11 = 0.0, prev_alpha = 0.0;
#ifdef LYAP_PANEL_PROF
    long long pt[5] = {0, 0, 0, 0, 0}, tl = clock64();
#define RPROF(i) do { if (blockIdx.x == 0 && threadIdx.x == 0) { long long t_ = clock64(); pt[i] += t_ - tl; tl = t_; } } while (0)
#else
#define RPROF(i) do { } while (0)
#endif
    for (int j = 0; j < a.kmax; j++) {
        grid.sync();
        RPROF(0);
        const int buf = j & 1;
        const double *bs = a.bsum + buf * G, *bb = a.bbest + buf * G;
        const int *bx = a.bidx + buf * G;
        // ---- every CTA: identical reduction of the partials (warp 0 only: the G partials are
        // the same few L2 lines for every CTA), stop test, pivot
        __shared__ double s_t;
        __shared__ int s_bi;
        if (wib == 0) {
            double t = 0.0, bv = -1.0; int bi = n;
#pragma unroll 4
            for (int b = lane; b < G; b += 32) {
                t += bs[b];
                const double v = bb[b]; const int i2 = bx[b];
                if (v > bv || (v == bv && i2 < bi)) { bv = v; bi = i2; }
            }
            t = warp_sum(t);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
                const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
                if (v2 > bv || (v2 == bv && i2 < bi)) { bv = v2; bi = i2; }
            }
            if (lane == 0) { s_t = t; s_bi = bi; }
        }
        __syncthreads();
        const double t = s_t;
        const int bi = s_bi;
        const double tr = sqrt(t);
        const bool stop = (j > 0 && tr <= a.tol * r11) || tr == 0.0 || bi >= n;
        // owners finalise the previous pivot column (all CTAs have finished reading it)
        if (prev >= 0 && (prev % nwg) == gw) {
            double *xp = a.M + (long)prev * c;
            for (int i = j - 1 + lane; i < c; i += 32) xp[i] = (i == j - 1) ? prev_alpha : 0.0;
        }
        RPROF(1);
        if (stop) { rank = j; break; }
        const int pc = bi;
        // ---- reflector of column pc, rows j..c-1, in shared memory
        const double *xp = a.M + (long)pc * c;
        double part = 0.0;
        for (int i = j + threadIdx.x; i < c; i += blockDim.x) {
            const double x = xp[i];
            vsh[i] = x;
            if (i > j) part = fma(x, x, part);
        }
        part = block_sum(part, red);
        const double x0 = vsh[j];
        const double nrm = sqrt(part + x0 * x0);
        const double alpha = (x0 >= 0.0) ? -nrm : nrm;
        const double v0 = x0 - alpha;
        const double vtv = v0 * v0 + part;
        __syncthreads();
        if (threadIdx.x == 0) vsh[j] = v0;
        if (j == 0) r11 = fabs(alpha);
        if (blockIdx.x == 0 && threadIdx.x == 0) { a.perm[j] = pc; if (j == 0) a.scal[0] = fabs(alpha); }
        __syncthreads();
        RPROF(2);
        // ---- owners: apply H_j to active columns, downdate norms, next partials
        double bsum = 0.0, bbest = -1.0; int bidx = n;
        for (int col = gw, t = 0; col < n; col += nwg, t++) {
            if (col == pc) { if (lane == t) m_act = false; continue; }
            if (!__shfl_sync(0xffffffffu, (int)m_act, t)) continue;
            double *y = a.M + (long)col * c;
            double yj, s2 = __shfl_sync(0xffffffffu, m_n2, t);
            const double n0 = __shfl_sync(0xffffffffu, m_n0, t);
            if constexpr (RPL > 0) {
                // the column's active rows in registers: all loads in flight at once, one
                // load and one store per element
                double yr[RPL];
#pragma unroll
                for (int u = 0; u < RPL; u++) { const int i = j + lane + 32 * u; yr[u] = (i < c) ? y[i] : 0.0; }
                if (vtv != 0.0) {
                    double d = 0.0;
#pragma unroll
                    for (int u = 0; u < RPL; u++) { const int i = j + lane + 32 * u; if (i < c) d = fma(vsh[i], yr[u], d); }
                    d = warp_sum(d);
                    const double f = 2.0 * d / vtv;
#pragma unroll
                    for (int u = 0; u < RPL; u++) {
                        const int i = j + lane + 32 * u;
                        if (i < c) { yr[u] = fma(-f, vsh[i], yr[u]); y[i] = yr[u]; }
                    }
                }
                yj = __shfl_sync(0xffffffffu, yr[0], 0);
                const double r = (s2 > 0.0) ? 1.0 - (yj * yj) / s2 : 0.0;
                const double temp2 = fmax(r, 0.0) * (s2 / fmax(n0, 1e-300));
                if (temp2 <= 1.5e-8) {                 // sqrt(eps) rule: recompute exactly
                    double e = 0.0;
#pragma unroll
                    for (int u = 0; u < RPL; u++) { const int i = j + lane + 32 * u; if (i > j && i < c) e = fma(yr[u], yr[u], e); }
                    s2 = warp_sum(e);
                    if (lane == t) m_n0 = s2;
                } else {
                    s2 = s2 - yj * yj;
                }
            } else {
                double d = 0.0;
                if (vtv != 0.0) {
#pragma unroll 8
                    for (int i = j + lane; i < c; i += 32) d = fma(vsh[i], y[i], d);
                    d = warp_sum(d);
                    const double f = 2.0 * d / vtv;
#pragma unroll 8
                    for (int i = j + lane; i < c; i += 32) y[i] = fma(-f, vsh[i], y[i]);
                    __syncwarp();
                }
                yj = y[j];
                const double r = (s2 > 0.0) ? 1.0 - (yj * yj) / s2 : 0.0;
                const double temp = fmax(r, 0.0);
                const double temp2 = temp * (s2 / fmax(n0, 1e-300));
                if (temp2 <= 1.5e-8) {                 // sqrt(eps) rule: recompute exactly
                    double e = 0.0;
#pragma unroll 8
                    for (int i = j + 1 + lane; i < c; i += 32) e = fma(y[i], y[i], e);
                    s2 = warp_sum(e);
                    if (lane == t) m_n0 = s2;
                } else {
                    s2 = s2 - yj * yj;
                }
            }
            if (lane == t) m_n2 = s2;
            bsum += s2;
            if (s2 > bbest || (s2 == bbest && col < bidx)) { bbest = s2; bidx = col; }
        }
        RPROF(3);
        prev = pc; prev_alpha = alpha;
        if (lane == 0) { s_sum[wib] = bsum; s_best[wib] = bbest; s_idx[wib] = bidx; }
        __syncthreads();
        if (threadIdx.x == 0) {
            double tt = 0.0, bvv = -1.0; int bii = n;
            for (int w = 0; w < nwb; w++) {
                tt += s_sum[w];
                if (s_best[w] > bvv || (s_best[w] == bvv && s_idx[w] < bii)) { bvv = s_best[w]; bii = s_idx[w]; }
            }
            const int nb = buf ^ 1;
            a.bsum[nb * G + blockIdx.x] = tt; a.bbest[nb * G + blockIdx.x] = bvv; a.bidx[nb * G + blockIdx.x] = bii;
        }
    }
    if (rank == a.kmax && prev >= 0) {                 // finalise the last pivot column
        grid.sync();
        if ((prev % nwg) == gw) {
            double *xp = a.M + (long)prev * c;
            for (int i = a.kmax - 1 + lane; i < c; i += 32) xp[i] = (i == a.kmax - 1) ? prev_alpha : 0.0;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *a.rank = rank;
#ifdef LYAP_PANEL_PROF
    if (blockIdx.x == 0 && threadIdx.x == 0 && rank > 0)
        printf("rrqr2 n=%d c=%d grid=%d rank=%d cycles/step: gridsync %lld pivot %lld reflector %lld apply %lld\n", n, c,
               gridDim.x, rank, pt[0] / rank, pt[1] / rank, pt[2] / rank, pt[3] / rank);
#endif
}


// ---------------------------------------------------------------------------------
// Blocked QRCP (LAPACK xLAQPS scheme).  Same pivots and
// reflectors as rrqr2 (up to rounding), but within a block of RQ_NB steps the trailing
// matrix is not updated: step j (= j0 + jj) forms
//   u   = M[j0:, pc] - V[j0:, 0:jj] F[pc, 0:jj]^T         (the pivot column, updated)
//   v, tau from u[j:]                                        (reflector H_j)
//   F[col, jj] = tau (M[j:, col]^T v - F[col, 0:jj] (V[j:, 0:jj]^T v))   (read-only GEMV)
//   M[j, col] -= V[j, 0:jj+1] F[col, 0:jj+1]^T              (row j of R, final)
// and downdates the trailing norms with row j.  A block ends after RQ_NB steps, or early
// after a step whose downdate cancelled (the xLAQP2 sqrt(eps) rule); then one DMMA GEMM
// applies the block to the trailing rows, M[j0+nb:, :] -= V[j0+nb:, :] F^T, and the next
// launch recomputes every trailing norm exactly.  Per step the trailing matrix is read
// once and not written (rrqr2: read and written); one grid barrier per step.
constexpr int RQ_NB = 32;
struct Rrqr3Args {
    int n, c, kmax, j0;
    double tol;
    double *M;          // c x n col-major
    double *V;          // c x RQ_NB col-major (reflectors of this block, zero above their row)
    double *F;          // n x RQ_NB, row col at F + col * RQ_NB
    double *bsum, *bbest; int *bidx, *bflag;   // 2 x gridDim partials (step parity)
    int *perm;          // n: pivot order
    int *active;        // n: 1 while not pivoted
    double *state;      // [0] r11
    int *istate;        // [0] next j, [1] done (rank final), [2] rank
    double *ug;         // c: the updated pivot column u (row slices by CTA)
    double *pw;         // gridDim x (RQ_NB + 1): slice partials of V^T u and ||u||^2
};

// NT = 256 with two CTAs per SM while the pivot column (c doubles of shared memory per CTA)
// allows it; above ~13 K rows only one CTA fits, and 512 threads keep 16 warps of loads in
// flight per SM (the per-step GEMV is HBM bound: configs[3] with the fp32 solver, c ~ 12000).
template <int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB)
rrqr3_kernel(Rrqr3Args a)
{
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double rq_sm[];
    double *ush = rq_sm;                     // c: updated pivot column -> reflector v (rows j..)
    __shared__ double wv[RQ_NB];             // V[j:, 0:jj]^T v
    __shared__ double red[32];
    __shared__ double s_best[NT / 32], s_sum[NT / 32];
    __shared__ int s_idx[NT / 32], s_flag[NT / 32];
    __shared__ double s_t;
    __shared__ int s_bi, s_fl;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nwb = blockDim.x >> 5;
    const int gw = blockIdx.x * nwb + wib, nwg = gridDim.x * nwb;
    const int n = a.n, c = a.c, G = gridDim.x, j0 = a.j0;
    double r11 = (j0 > 0) ? a.state[0] : 0.0;
    // owned columns col = gw + t nwg: lane t keeps the trailing norm^2, its value at the
    // block start (exact), and the active flag
    double m_n2 = 0.0, m_n0 = 0.0;
    bool m_act = false;
    auto publish = [&](int buf, double bsum, double bbest, int bidx, int flag) {
        if (lane == 0) { s_sum[wib] = bsum; s_best[wib] = bbest; s_idx[wib] = bidx; s_flag[wib] = flag; }
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0, bv = -1.0; int bi = n, fl = 0;
            for (int w = 0; w < nwb; w++) {
                t += s_sum[w]; fl |= s_flag[w];
                if (s_best[w] > bv || (s_best[w] == bv && s_idx[w] < bi)) { bv = s_best[w]; bi = s_idx[w]; }
            }
            a.bsum[buf * G + blockIdx.x] = t; a.bbest[buf * G + blockIdx.x] = bv;
            a.bidx[buf * G + blockIdx.x] = bi; a.bflag[buf * G + blockIdx.x] = fl;
        }
    };
    {   // exact trailing norms (rows j0..c-1) of the active columns
        double bsum = 0.0, bbest = -1.0; int bidx = n;
        for (int col = gw, t = 0; col < n; col += nwg, t++) {
            const bool act = a.active[col] != 0;
            double sq = 0.0;
            if (act) {
                const double *x = a.M + (long)col * c;
#pragma unroll 8
                for (int i = j0 + lane; i < c; i += 32) sq = fma(x[i], x[i], sq);
                sq = warp_sum(sq);
                bsum += sq;
                if (sq > bbest || (sq == bbest && col < bidx)) { bbest = sq; bidx = col; }
            }
            if (lane == t) { m_n2 = sq; m_n0 = sq; m_act = act; }
        }
        publish(0, bsum, bbest, bidx, 0);
    }
    int prev = -1, jj = 0, stopped = 0;
    double prev_alpha = 0.0;
    for (; jj < RQ_NB && j0 + jj < a.kmax; jj++) {
        const int j = j0 + jj;
        grid.sync();
        const int buf = jj & 1;
        if (wib == 0) {
            double t = 0.0, bv = -1.0; int bi = n, fl = 0;
            for (int b = lane; b < G; b += 32) {
                t += a.bsum[buf * G + b]; fl |= a.bflag[buf * G + b];
                const double v = a.bbest[buf * G + b]; const int i2 = a.bidx[buf * G + b];
                if (v > bv || (v == bv && i2 < bi)) { bv = v; bi = i2; }
            }
            t = warp_sum(t);
            fl = __reduce_or_sync(0xffffffffu, fl);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
                const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
                if (v2 > bv || (v2 == bv && i2 < bi)) { bv = v2; bi = i2; }
            }
            if (lane == 0) { s_t = t; s_bi = bi; s_fl = fl; }
        }
        __syncthreads();
        const double tr = sqrt(s_t);
        const int bi = s_bi;
        // owners finalise the previous pivot column (every CTA has finished reading it)
        if (prev >= 0 && (prev % nwg) == gw) {
            double *xp = a.M + (long)prev * c;
            for (int i = j - 1 + lane; i < c; i += 32) xp[i] = (i == j - 1) ? prev_alpha : 0.0;
            if (lane < RQ_NB) a.F[(long)prev * RQ_NB + lane] = 0.0;
        }
        if (s_fl) break;                     // a downdate cancelled in the previous step: end the block
        if ((j > 0 && tr <= a.tol * r11) || tr == 0.0 || bi >= n) { stopped = 1; break; }
        const int pc = bi;
        // ---- u = M[j:, pc] - V[j:, 0:jj] F[pc, 0:jj]^T, split over the CTAs by row slices
        // (every CTA forming all of u would read V (c x jj) from L2 G times per step), with
        // each slice's partial ||u[j+1:]||^2 and V[j+1:, l]^T u[j+1:] (l < jj); one more
        // grid barrier publishes u and the partials
        const double *xp = a.M + (long)pc * c;
        const double *Fp = a.F + (long)pc * RQ_NB;
        if (wib == 0) {                              // one warp per CTA: <= ~50 rows per slice
            const int rows = c - j, per = (rows + G - 1) / G;
            const int r0 = j + blockIdx.x * per, r1 = min(c, r0 + per);
            double pn = 0.0;
            double pwl[RQ_NB];
#pragma unroll
            for (int l = 0; l < RQ_NB; l++) pwl[l] = 0.0;
            for (int i = r0 + lane; i < r1; i += 32) {
                double x = xp[i];
                for (int l = 0; l < jj; l++) x = fma(-a.V[(long)l * c + i], Fp[l], x);
                a.ug[i] = x;
                if (i > j) {
                    pn = fma(x, x, pn);
#pragma unroll
                    for (int l = 0; l < RQ_NB; l++)
                        if (l < jj) pwl[l] = fma(a.V[(long)l * c + i], x, pwl[l]);
                }
            }
            pn = warp_sum(pn);
            double *pq = a.pw + (long)blockIdx.x * (RQ_NB + 1);
            if (lane == 0) pq[RQ_NB] = pn;
#pragma unroll
            for (int l = 0; l < RQ_NB; l++) {
                if (l < jj) {                        // jj is uniform: no divergence
                    const double t2 = warp_sum(pwl[l]);
                    if (lane == 0) pq[l] = t2;
                }
            }
        }
        grid.sync();
        double part = 0.0;
        if (wib == 0) {
            for (int b = lane; b < G; b += 32) part += __ldcg(a.pw + (long)b * (RQ_NB + 1) + RQ_NB);
            part = warp_sum(part);
        }
        // warps 1..7 reduce w'_l for l = wib - 1, wib + 6, ... (fixed order over the CTAs)
        for (int l = wib - 1; l >= 0 && l < jj; l += nwb - 1) {
            double d = 0.0;
            for (int b = lane; b < G; b += 32) d += __ldcg(a.pw + (long)b * (RQ_NB + 1) + l);
            d = warp_sum(d);
            if (lane == 0) wv[l] = d;
        }
        if (wib == 0 && lane == 0) red[0] = part;
        for (int i = j + threadIdx.x; i < c; i += blockDim.x) ush[i] = __ldcg(a.ug + i);
        __syncthreads();
        part = red[0];
        const double x0 = ush[j];
        const double nrm = sqrt(part + x0 * x0);
        const double alpha = (x0 >= 0.0) ? -nrm : nrm;
        const double v0 = x0 - alpha;
        const double vtv = v0 * v0 + part;
        const double tau = (vtv != 0.0) ? 2.0 / vtv : 0.0;
        __syncthreads();
        if (threadIdx.x == 0) ush[j] = v0;
        if (j == 0) r11 = fabs(alpha);
        // w_l = V[j:, l]^T v = w'_l + V[j, l] v0
        if (threadIdx.x < jj) wv[threadIdx.x] += a.V[(long)threadIdx.x * c + j] * v0;
        __syncthreads();
        if (blockIdx.x == 0) {
            for (int i = threadIdx.x; i < c; i += blockDim.x) a.V[(long)jj * c + i] = (i >= j) ? ush[i] : 0.0;
            if (threadIdx.x == 0) {
                a.perm[j] = pc; a.active[pc] = 0;
                if (j == 0) a.state[0] = fabs(alpha);
            }
        }
        __syncthreads();
        // ---- owners: F[col, jj], row j of R, norm downdate, next partials
        double bsum = 0.0, bbest = -1.0; int bidx = n, flag = 0;
        const double vj = (lane <= jj) ? ((lane == jj) ? v0 : a.V[(long)lane * c + j]) : 0.0;   // V[j, lane]
        const double wl = (lane < jj) ? wv[lane] : 0.0;
        for (int col = gw, t = 0; col < n; col += nwg, t++) {
            if (col == pc) { if (lane == t) m_act = false; continue; }
            if (!__shfl_sync(0xffffffffu, (int)m_act, t)) continue;
            const double *y = a.M + (long)col * c;
            // four partial sums: the fp64 multiply-add chain of 16 in-flight loads would
            // otherwise serialise behind the loads of the next 16
            double d = 0.0;
            {
                double d1 = 0.0, d2 = 0.0, d3 = 0.0;
                int i = j + lane;
                for (; i + 96 < c; i += 128) {
                    d = fma(y[i], ush[i], d);
                    d1 = fma(y[i + 32], ush[i + 32], d1);
                    d2 = fma(y[i + 64], ush[i + 64], d2);
                    d3 = fma(y[i + 96], ush[i + 96], d3);
                }
                for (; i < c; i += 32) d = fma(y[i], ush[i], d);
                d = (d + d1) + (d2 + d3);
            }
            double *Fc = a.F + (long)col * RQ_NB;
            const double fl = (lane < jj) ? Fc[lane] : 0.0;
            const double corr = warp_sum(fl * wl);
            d = warp_sum(d);
            const double fnew = tau * (d - corr);
            const double fall = (lane == jj) ? fnew : fl;
            const double rj = y[j] - warp_sum(vj * fall);
            if (lane == 0) { Fc[jj] = fnew; a.M[(long)col * c + j] = rj; }
            double s2 = __shfl_sync(0xffffffffu, m_n2, t);
            const double n0 = __shfl_sync(0xffffffffu, m_n0, t);
            const double r = (s2 > 0.0) ? 1.0 - (rj * rj) / s2 : 0.0;
            const double temp2 = fmax(r, 0.0) * (s2 / fmax(n0, 1e-300));
            if (temp2 <= 1.5e-8) flag = 1;   // recomputed exactly at the next block start
            s2 = fmax(s2 - rj * rj, 0.0);
            if (lane == t) m_n2 = s2;
            bsum += s2;
            if (s2 > bbest || (s2 == bbest && col < bidx)) { bbest = s2; bidx = col; }
        }
        publish(buf ^ 1, bsum, bbest, bidx, flag);
        prev = pc; prev_alpha = alpha;
    }
    // block end: finalise the last pivot column once every CTA has read it
    grid.sync();
    if (prev >= 0 && (prev % nwg) == gw) {
        const int jl = j0 + jj;              // steps j0 .. jl-1 done; prev was pivot of step jl-1
        double *xp = a.M + (long)prev * c;
        for (int i = jl - 1 + lane; i < c; i += 32) xp[i] = (i == jl - 1) ? prev_alpha : 0.0;
        if (lane < RQ_NB) a.F[(long)prev * RQ_NB + lane] = 0.0;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const int jl = j0 + jj;
        a.istate[0] = jl;
        a.istate[1] = (stopped || jl >= a.kmax) ? 1 : 0;
        a.istate[2] = jl;
    }
}

// Zout(col, r) = M[col][r] for r < k, rounded to prec (physical columns = rows of Z)
__global__ void rrqr2_out_kernel(int n, int c, int k, const double *__restrict__ M, int prec, double *__restrict__ Zout)
{
    long tot = (long)n * k;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < tot; idx += (long)gridDim.x * blockDim.x) {
        const int col = (int)(idx % n), r = (int)(idx / n);
        Zout[(long)r * n + col] = round_to(M[(long)col * c + r], prec);
    }
}

__global__ void transpose_init_kernel(int n, int c, const double *__restrict__ Z, double *__restrict__ M, int *perm)
{
    long tot = (long)n * c;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < tot; idx += (long)gridDim.x * blockDim.x) {
        int i = (int)(idx % c), col = (int)(idx / c);     // M[i + col*c] = Z[col + i*n]
        M[idx] = Z[col + (long)i * n];
        if (i == 0) perm[col] = col;
    }
}

// Zout(perm[jj], r) = R(r, jj) for r < k (R upper trapezoidal), rounded to prec.
__global__ void rrqr_out_kernel(int n, int c, int k, const double *__restrict__ M, const int *__restrict__ perm,
                                int prec, double *__restrict__ Zout)
{
    long tot = (long)n * k;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < tot; idx += (long)gridDim.x * blockDim.x) {
        int jj = (int)(idx % n), r = (int)(idx / n);
        double v = (r <= jj) ? M[(long)jj * c + r] : 0.0;
        Zout[(long)r * n + perm[jj]] = round_to(v, prec);
    }
}

int RrqrWork::alloc(int nmax_, int cmax_) {
    nmax = nmax_; cmax = cmax_;
    LYAP_CUDA_TRY(cudaMalloc(&M, sizeof(double) * (size_t)nmax * cmax));
    LYAP_CUDA_TRY(cudaMalloc(&nrm, sizeof(double) * (size_t)(2 * nmax + 4 * 1024 + cmax + 8)));
    LYAP_CUDA_TRY(cudaMalloc(&ints, sizeof(int) * (size_t)(2 * nmax + 2048 + 16)));
    scal = nrm + nmax;
    p3_ctas = 512;
    LYAP_CUDA_TRY(cudaMalloc(&V3, sizeof(double) * (size_t)cmax * RQ_NB));
    LYAP_CUDA_TRY(cudaMalloc(&F3, sizeof(double) * (size_t)nmax * RQ_NB));
    LYAP_CUDA_TRY(cudaMalloc(&p3, sizeof(double) * (size_t)8 * p3_ctas));
    LYAP_CUDA_TRY(cudaMalloc(&st3, sizeof(double) * 4));
    LYAP_CUDA_TRY(cudaMalloc(&ug3, sizeof(double) * (size_t)cmax));
    LYAP_CUDA_TRY(cudaMalloc(&pw3, sizeof(double) * (size_t)p3_ctas * (RQ_NB + 1)));
    LYAP_CUDA_TRY(cudaMalloc(&act3, sizeof(int) * ((size_t)nmax + 8)));
    ist3 = act3 + nmax;
    return LYAP_OK;
}
void RrqrWork::release() {
    for (double *p : {M, nrm, V3, F3, p3, st3, ug3, pw3}) if (p) cudaFree(p);
    if (ints) cudaFree(ints);
    if (act3) cudaFree(act3);
    M = nrm = scal = V3 = F3 = p3 = st3 = ug3 = pw3 = nullptr;
    ints = act3 = ist3 = nullptr;
}

__global__ void fill_int_kernel(int len, int v, int *x)
{
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x) x[i] = v;
}

// Blocked driver: one cooperative launch per block of RQ_NB pivots, then the block's
// trailing update as one DMMA GEMM.  M = Z^T and perm are set up by the caller.
static int rank_trunc_chol_blocked(cudaStream_t s, int n, int c, double tol, int prec_out, double *Zout,
                                   int *k_out, RrqrWork &w)
{
    struct Cfg { int nsm, per; };
    static const Cfg cfg = [] {
        int dev = 0, nsm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(rrqr3_kernel<256, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(rrqr3_kernel<512, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        return Cfg{nsm, 0};
    }();
    const size_t smem = sizeof(double) * (size_t)c;
    if (smem > 200 * 1024) return LYAP_ERR_CAPACITY;
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, rrqr3_kernel<256, 2>, 256, smem);
    const bool wide = per < 2 && !env_flag("LYAP_RRQR_256");     // one CTA per SM: 512 threads
    const int nth = wide ? 512 : 256;
    const int grid = std::max(1, std::min(std::min(cfg.nsm * (wide ? 1 : std::min(per, 2)), w.p3_ctas), ceil_div(n, nth / 32)));
    if (n > 32 * (nth / 32) * grid) return LYAP_ERR_CAPACITY;
    fill_int_kernel<<<std::min(ceil_div(n, 256), 1024), 256, 0, s>>>(n, 1, w.act3);
    LYAP_TRY(launched());
    const int kmax = c < n ? c : n;
    int *ist = w.ist3;
    int j0 = 0, k = 0;
    int hs[3] = {0, 0, 0};
    KTimer kt(KC_RRQR, s);
    for (;;) {
        Rrqr3Args a{n, c, kmax, j0, tol, w.M, w.V3, w.F3, w.p3, w.p3 + 2 * w.p3_ctas,
                    (int *)(w.p3 + 4 * w.p3_ctas), (int *)(w.p3 + 4 * w.p3_ctas) + 2 * w.p3_ctas,
                    w.ints, w.act3, w.st3, ist, w.ug3, w.pw3};
        void *args[] = {&a};
        LYAP_CUDA_TRY(cudaLaunchCooperativeKernel(wide ? (void *)rrqr3_kernel<512, 1> : (void *)rrqr3_kernel<256, 2>, dim3(grid),
                                                  dim3(nth), args, smem, s));
        LYAP_TRY(launched());
        LYAP_CUDA_TRY(cudaMemcpyAsync(hs, ist, sizeof(int) * 3, cudaMemcpyDeviceToHost, s));
        LYAP_CUDA_TRY(cudaStreamSynchronize(s));
        if (hs[1]) { k = hs[2]; break; }
        const int j1 = hs[0], nbb = j1 - j0;
        if (nbb <= 0) return LYAP_ERR_CUDA;          // cannot happen: every launch makes a step or stops
        if (j1 < c)
            LYAP_TRY(dgemm_cm(s, false, false, c - j1, n, nbb, -1.0, w.V3 + j1, c, w.F3, RQ_NB, 1.0, w.M + j1, c));
        j0 = j1;
    }
    if (k == 0) {   // all-zero Z: a single zero column (as the oracle)
        LYAP_CUDA_TRY(cudaMemsetAsync(Zout, 0, sizeof(double) * (size_t)n, s));
        *k_out = 1;
        return LYAP_OK;
    }
    const long to = (long)n * k;
    rrqr2_out_kernel<<<ceil_div(to, 256) < 2048 ? ceil_div(to, 256) : 2048, 256, 0, s>>>(n, c, k, w.M, prec_out, Zout);
    LYAP_TRY(launched());
    *k_out = k;
    return LYAP_OK;
}

int rank_trunc_chol_f64(cudaStream_t s, int n, int c, const double *Z, double tol, int prec_out,
                        double *Zout, int *k_out, RrqrWork &w)
{
    if (n > w.nmax || c > w.cmax) return LYAP_ERR_CAPACITY;
    int *perm = w.ints, *bidx = w.ints + w.nmax, *rank = bidx + 2048;
    double *bsum = w.nrm + 2 * w.nmax, *bbest = bsum + 1024, *v = bbest + 1024, *scal = v + w.cmax;
    long tot = (long)n * c;
    transpose_init_kernel<<<ceil_div(tot, 256) < 2048 ? ceil_div(tot, 256) : 2048, 256, 0, s>>>(n, c, Z, w.M, perm);
    LYAP_TRY(launched());
    // blocked QRCP for factors that do not stay in L2 (the per-step GEMV reads the
    // trailing matrix once instead of reading and writing it); LYAP_RRQR_BLOCKED=0/1 forces
    const char *eb = getenv("LYAP_RRQR_BLOCKED");
    const bool blocked = eb ? (eb[0] == '1') : ((double)n * c * 8.0 > 96e6);
    if (blocked && w.V3) return rank_trunc_chol_blocked(s, n, c, tol, prec_out, Zout, k_out, w);
    const bool v2 = !env_flag("LYAP_RRQR_V1");
    // one-time setup (function-local static: thread-safe initialisation, published after
    // every attribute is set)
    struct Cfg { int max_blocks, nsm; };
    static const Cfg cfg = [] {
        int dev = 0, per = 0, nsm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, rrqr_kernel, 256, 0);
        int mb = nsm * (per < 2 ? per : 2);
        if (mb > 1024) mb = 1024;
        if (mb < 1) mb = 1;
        for (void *f : {(void *)rrqr2_kernel<0>, (void *)rrqr2_kernel<16>, (void *)rrqr2_kernel<32>,
                        (void *)rrqr2_kernel<48>})
            cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        return Cfg{mb, nsm};
    }();
    const int max_blocks = cfg.max_blocks, nsm = cfg.nsm;
    const int want = ceil_div(n, 8);
    const size_t smem2 = sizeof(double) * (size_t)c;
    // register-resident columns (one load and one store per element, all loads of a column in
    // flight at once) up to 16 rows per lane (two CTAs per SM); streamed columns above (64
    // registers, up to four CTAs per SM).  32 / 48 rows per lane spill: measured slower.
    void *fn = (c <= 512) ? (void *)rrqr2_kernel<16> : (void *)rrqr2_kernel<0>;
    if (env_flag("LYAP_RRQR_STREAM")) fn = (void *)rrqr2_kernel<0>;
    if (env_flag("LYAP_RRQR_REG"))
        fn = (c <= 1024) ? (void *)rrqr2_kernel<32> : (c <= 1536) ? (void *)rrqr2_kernel<48> : fn;
    int per2 = 0;
    if (v2 && smem2 <= 160 * 1024) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, fn, 256, smem2);
    const int cap = (fn == (void *)rrqr2_kernel<0> && !env_flag("LYAP_RRQR_2CTA")) ? 4 : 2;
    // at most 512 CTAs: the double-buffered partial arrays hold 2 x 512 entries
    const int max_blocks2 = std::min(512, nsm * std::min(per2, cap));
    if (v2 && max_blocks2 > 0 && n <= 32 * 8 * max_blocks2) {
        // the step time is set by the warps owning the most columns: take the fewest CTAs
        // that keep that maximum minimal (fewer partials, cheaper barrier; measured: n = 4096,
        // 256 CTAs x 2 columns/warp 17 us/step vs 296 CTAs x 1-2 columns/warp 23 us/step)
        const int cpw = ceil_div(n, 8 * max_blocks2);
        int grid = std::max(1, std::min(ceil_div(n, 8 * cpw), max_blocks2));
        if (const char *e = getenv("LYAP_RRQR_GRID")) grid = std::max(1, std::min(atoi(e), max_blocks2));
        Rrqr2Args a2{n, c, c < n ? c : n, tol, w.M, w.nrm, w.nrm + n, bsum, bbest, bidx, perm, w.ints + w.nmax + 2048 + 8,
                     scal, rank};
        void *args2[] = {&a2};
        KTimer kt(KC_RRQR, s);
        LYAP_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(256), args2, smem2, s));
    } else {
        const int grid = want < max_blocks ? want : max_blocks;
        RrqrArgs a{n, c, c < n ? c : n, tol, w.M, w.nrm, bsum, bbest, bidx, perm, v, scal, rank};
        void *args[] = {&a};
        KTimer kt(KC_RRQR, s);
        LYAP_CUDA_TRY(cudaLaunchCooperativeKernel((void *)rrqr_kernel, dim3(grid), dim3(256), args, 0, s));
    }
    LYAP_TRY(launched());
    int k = 0;
    LYAP_CUDA_TRY(cudaMemcpyAsync(&k, rank, sizeof(int), cudaMemcpyDeviceToHost, s));
    LYAP_CUDA_TRY(cudaStreamSynchronize(s));
    if (k == 0) {   // all-zero Z: a single zero column (as the oracle)
        LYAP_CUDA_TRY(cudaMemsetAsync(Zout, 0, sizeof(double) * (size_t)n, s));
        *k_out = 1;
        return LYAP_OK;
    }
    long to = (long)n * k;
    if (v2 && max_blocks2 > 0 && n <= 32 * 8 * max_blocks2)
        rrqr2_out_kernel<<<ceil_div(to, 256) < 2048 ? ceil_div(to, 256) : 2048, 256, 0, s>>>(n, c, k, w.M, prec_out, Zout);
    else
        rrqr_out_kernel<<<ceil_div(to, 256) < 2048 ? ceil_div(to, 256) : 2048, 256, 0, s>>>(n, c, k, w.M, perm, prec_out, Zout);
    LYAP_TRY(launched());
    *k_out = k;
    return LYAP_OK;
}

}  // namespace lyap

extern "C" int lyap_rank_trunc_chol(int n, int c, const double *Z, double tol, int prec,
                                    double *Zout, int *k, void *stream)
{
    using namespace lyap;
    if (n <= 0 || c <= 0 || !Z || !Zout || !k) return LYAP_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    RrqrWork w;
    int rc = w.alloc(n, c);
    if (rc == LYAP_OK) rc = rank_trunc_chol_f64(s, n, c, Z, tol, prec, Zout, k, w);
    if (cudaStreamSynchronize(s) != cudaSuccess) rc = LYAP_ERR_CUDA;
    w.release();
    return rc;
}
