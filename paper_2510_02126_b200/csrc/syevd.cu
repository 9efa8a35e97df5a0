// syevd.cu -- fp64 symmetric eigensolver for the kernel matrices of Fragments
// 1-4 and RankTruncLdlt when they are large (ranks of several hundred make
// H_i, K_i and R Y R^T ~1000 x 1000, PAPER.md l.165, l.240, l.790, l.824,
// l.1298).  Any backward-stable eigensolver computes "the spectral
// decomposition" the paper asks for; this one is built for the GPU:
//
//  1. Householder tridiagonalisation Q_H^T A Q_H = T in ONE cooperative
//     kernel: every CTA derives the reflector redundantly from column j, the
//     symmetric product p = tau A v is column-distributed, a grid barrier,
//     then the rank-2 update A -= v w^T + w v^T (2 grid barriers per column).
//  2. Cuppen divide and conquer on T with Gu-Eisenstat eigenvectors:
//     leaves (<= 32) by warp Jacobi; each merge D + rho z z^T is deflated
//     (LAPACK dlaed2 rules: rho|z_i| <= tol, close poles rotated together),
//     the secular roots are found by safeguarded bisection around the nearer
//     pole (tau stored relative to it), z is recomputed from the roots
//     (Loewner), and the eigenvector block is a GEMM Q U.
//  3. Back-transformation X = Q_H Q_T with compact-WY panels (GEMMs).
#include <cooperative_groups.h>
#include <algorithm>
#include <vector>
#include <cmath>
#include "common.cuh"
#include "gemm_simt.cuh"
#include "wy.cuh"
#include "lyap_internal.h"
#include "ktimer.h"

namespace cg = cooperative_groups;

namespace lyap {

// ---------------------------------------------------------------- 1. tridiagonalisation
struct TridArgs {
    int p;
    double *A;      // p x p col-major (symmetric), trailing block updated in place
    double *R;      // p x p col-major: reflector j in R[j+1:p, j] (R[j+1, j] = 1)
    double *d, *e, *tau;
    double *P;      // p
    double *gvec;   // tridiag_kernel: per-CTA v, vn, w, c (4 p doubles each) in global memory
                    // when 4 p doubles exceed shared memory (p > 6400); nullptr otherwise
};

// Reflector from x[0..L) (x[0] = alpha): v[0] = 1, v[i] = x[i]/(alpha - beta), tau, beta.
// Every CTA runs it on identical data with the same reduction tree -> identical results.
__device__ void make_reflector(const double *x, int L, double *v, double *red, double &tau, double &beta)
{
    double s = 0.0;
    for (int i = 1 + threadIdx.x; i < L; i += blockDim.x) s = fma(x[i], x[i], s);
    s = block_sum(s, red);
    const double alpha = x[0];
    if (s == 0.0) { tau = 0.0; beta = alpha; }
    else {
        beta = -copysign(sqrt(alpha * alpha + s), alpha);
        tau = (beta - alpha) / beta;
    }
    const double scale = (tau == 0.0) ? 0.0 : 1.0 / (alpha - beta);
    for (int i = threadIdx.x; i < L; i += blockDim.x) v[i] = (i == 0) ? 1.0 : x[i] * scale;
    __syncthreads();
}

#ifndef TRID_CHUNK
#define TRID_CHUNK 16
#endif
// One grid barrier per column: column g of the trailing matrix is owned by warp g mod
// (#warps) for the whole reduction, so the owner's update of step j and its product with
// v_{j+1} for step j+1 are fused (each column read and written once per step); only the
// vector P = tau A2 v crosses CTAs.  Column j+1 -- the source of the next reflector -- is
// not written in step j; every CTA applies step j's rank-2 update to it privately.
__global__ void __launch_bounds__(256)
tridiag_kernel(TridArgs a)
{
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double sm[];
    const int p = a.p;
    double *vb = a.gvec ? a.gvec + (long)blockIdx.x * 4 * p : sm;
    double *v = vb, *vn = vb + p, *w = vb + 2 * p, *c = vb + 3 * p;
    __shared__ double red[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwb = blockDim.x >> 5;
    const int gw = blockIdx.x * nwb + wid, nwg = gridDim.x * nwb;
    double *A = a.A;
    if (p <= 2) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            a.d[0] = A[0];
            if (p == 2) { a.e[0] = A[1]; a.d[1] = A[3]; a.tau[0] = 0.0; }
        }
        return;
    }
    // prologue: reflector 0 from column 0 (rows 1..p-1), products for step 0
    double tau, beta;
    make_reflector(A + 1, p - 1, v, red, tau, beta);
    for (int g = 1 + gw; g < p; g += nwg) {
        const double *col = A + (long)g * p + 1;
        double s = 0.0;
        for (int i = lane; i < p - 1; i += 32) s = fma(col[i], v[i], s);
        s = warp_sum(s);
        if (lane == 0) a.P[g] = tau * s;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) a.d[0] = A[0];
    grid.sync();
    for (int j = 0; j + 2 < p; j++) {
        const double *Pc = a.P + (long)(j & 1) * p;             // P double-buffered by step parity
        double *Pn = a.P + (long)((j + 1) & 1) * p;
        const int L = p - j - 1;                 // rows j+1 .. p-1
        const int r0 = j + 1;
        // (c) w = P - (tau/2)(P.v) v     (all CTAs, identical)
        double k = 0.0;
        for (int i = threadIdx.x; i < L; i += blockDim.x) { double t = Pc[r0 + i]; w[i] = t; k = fma(t, v[i], k); }
        k = 0.5 * tau * block_sum(k, red);
        for (int i = threadIdx.x; i < L; i += blockDim.x) w[i] = fma(-k, v[i], w[i]);
        __syncthreads();
        // (e) updated column j+1 (private copy), next reflector from rows j+2..
        const double *cj = A + (long)r0 * p + r0;
        for (int i = threadIdx.x; i < L; i += blockDim.x) c[i] = cj[i] - v[i] * w[0] - w[i] * v[0];
        __syncthreads();
        double taun = 0.0, betan = 0.0;
        const bool more = (j + 3 < p);
        if (more) make_reflector(c + 1, L - 1, vn, red, taun, betan);
        if (blockIdx.x == 0) {
            for (int i = threadIdx.x; i < L; i += blockDim.x) a.R[(long)j * p + r0 + i] = v[i];
            if (threadIdx.x == 0) {
                a.e[j] = beta; a.tau[j] = tau; a.d[j + 1] = c[0];
                if (!more) { a.e[j + 1] = c[1]; a.tau[j + 1] = 0.0; }
            }
        }
        // (d) owners: update columns g >= j+2 and, fused, P_{j+1}[g] = taun * col_g' . vn
        for (int g = r0 + 1 + gw; g < p; g += nwg) {
            double *col = A + (long)g * p + r0;
            const int ig = g - r0;
            const double vg = v[ig], wg = w[ig];
            double s = 0.0;
            // explicit chunks: all loads of a chunk in flight before its stores
            for (int i0 = 1 + lane; i0 < L; i0 += 32 * TRID_CHUNK) {
                double xr[TRID_CHUNK];
#pragma unroll
                for (int u = 0; u < TRID_CHUNK; u++) { const int i = i0 + 32 * u; if (i < L) xr[u] = col[i]; }
#pragma unroll
                for (int u = 0; u < TRID_CHUNK; u++) {
                    const int i = i0 + 32 * u;
                    if (i < L) {
                        const double x = xr[u] - v[i] * wg - w[i] * vg;
                        col[i] = x;
                        s = fma(x, vn[i - 1], s);
                    }
                }
            }
            if (more) {
                s = warp_sum(s);
                if (lane == 0) Pn[g] = taun * s;
            }
        }
        grid.sync();
        for (int i = threadIdx.x; i < L - 1; i += blockDim.x) v[i] = vn[i];
        tau = taun; beta = betan;
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) a.d[p - 1] = A[(long)(p - 1) * p + p - 1];
}

// Register-resident variant for p <= 1024: warp g owns column g for the whole
// reduction and keeps it in registers (lane holds rows lane + 32u), so the trailing
// matrix never leaves the register file; per step only P (p doubles) and the owner's
// copy of column j+2 (published for the next step's reflector) go through L2.
template <int CH>
__global__ void __launch_bounds__(256)
tridiag_reg_kernel(TridArgs a)
{
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double sm[];
    const int p = a.p;
    double *v = sm, *vn = sm + p, *w = sm + 2 * p, *c = sm + 3 * p;
    __shared__ double red[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwb = blockDim.x >> 5;
    const int g = blockIdx.x * nwb + wid;          // owned column (if < p)
    const bool owner = g < p;
    double *A = a.A;
    double col[CH];
#pragma unroll
    for (int u = 0; u < CH; u++) {
        int i = lane + 32 * u;
        col[u] = (owner && i < p) ? A[(long)g * p + i] : 0.0;
    }
    double tau, beta;
    make_reflector(A + 1, p - 1, v, red, tau, beta);
    if (owner && g >= 1) {
        double s = 0.0;
#pragma unroll
        for (int u = 0; u < CH; u++) { int i = lane + 32 * u; if (i >= 1 && i < p) s = fma(col[u], v[i - 1], s); }
        s = warp_sum(s);
        if (lane == 0) a.P[g] = tau * s;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) a.d[0] = A[0];
    grid.sync();
    for (int j = 0; j + 2 < p; j++) {
        const double *Pc = a.P + (long)(j & 1) * p;             // P double-buffered by step parity
        double *Pn = a.P + (long)((j + 1) & 1) * p;
        const int L = p - j - 1, r0 = j + 1;
        double k = 0.0;
        for (int i = threadIdx.x; i < L; i += blockDim.x) { double t = Pc[r0 + i]; w[i] = t; k = fma(t, v[i], k); }
        k = 0.5 * tau * block_sum(k, red);
        for (int i = threadIdx.x; i < L; i += blockDim.x) w[i] = fma(-k, v[i], w[i]);
        __syncthreads();
        // column j+1 as published by its owner (state after step j-1), updated privately
        const double *cj = A + (long)r0 * p + r0;
        for (int i = threadIdx.x; i < L; i += blockDim.x) c[i] = cj[i] - v[i] * w[0] - w[i] * v[0];
        __syncthreads();
        double taun = 0.0, betan = 0.0;
        const bool more = (j + 3 < p);
        if (more) make_reflector(c + 1, L - 1, vn, red, taun, betan);
        if (blockIdx.x == 0) {
            for (int i = threadIdx.x; i < L; i += blockDim.x) a.R[(long)j * p + r0 + i] = v[i];
            if (threadIdx.x == 0) {
                a.e[j] = beta; a.tau[j] = tau; a.d[j + 1] = c[0];
                if (!more) { a.e[j + 1] = c[1]; a.tau[j + 1] = 0.0; }
            }
        }
        if (owner && g >= r0 + 1) {
            const double vg = v[g - r0], wg = w[g - r0];
            double s = 0.0;
#pragma unroll
            for (int u = 0; u < CH; u++) {
                const int i = lane + 32 * u;
                if (i >= r0 + 1 && i < p) {
                    const double x = col[u] - v[i - r0] * wg - w[i - r0] * vg;
                    col[u] = x;
                    if (more) s = fma(x, vn[i - r0 - 1], s);
                }
            }
            if (more) {
                s = warp_sum(s);
                if (lane == 0) Pn[g] = taun * s;
            }
            if (g == r0 + 1) {                  // publish column j+2 for the next step
#pragma unroll
                for (int u = 0; u < CH; u++) {
                    const int i = lane + 32 * u;
                    if (i >= r0 + 1 && i < p) A[(long)g * p + i] = col[u];
                }
            }
            if (g == p - 1 && !more && lane == (p - 1) % 32) {
#pragma unroll
                for (int u = 0; u < CH; u++) if (lane + 32 * u == p - 1) a.d[p - 1] = col[u];
            }
        }
        grid.sync();
        for (int i = threadIdx.x; i < L - 1; i += blockDim.x) v[i] = vn[i];
        tau = taun; beta = betan;
        __syncthreads();
    }
}

// One grid barrier per column and one block barrier: warp 0 of every CTA forms, with
// warp-level reductions only, the quantities every CTA needs for step j (w = P - k v,
// column j+1 after step j, the next reflector vn) in shared memory; the owners then
// update their register-resident columns and publish P[g] = tau_{j+1} (col_g . vn).
// Same arithmetic as tridiag_reg_kernel up to the reduction trees.
template <int CH, int CPW>
__global__ void __launch_bounds__(256)
tridiag_w_kernel(TridArgs a)
{
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double sm[];
    const int p = a.p;
    double *vb[2] = {sm, sm + p};
    double *w = sm + 2 * p;
    __shared__ double s_tau[2], s_beta[2];
    __shared__ double red1[32], red2[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwb = blockDim.x >> 5;
    // warp gw owns columns gw + t * nwg (t < CPW): fewer CTAs -> a cheaper grid barrier
    const int gw = blockIdx.x * nwb + wid, nwg = gridDim.x * nwb;
    double *A = a.A;
    double col[CPW][CH];
#pragma unroll
    for (int t = 0; t < CPW; t++) {
        const int g = gw + t * nwg;
#pragma unroll
        for (int u = 0; u < CH; u++) {
            const int i = lane + 32 * u;
            col[t][u] = (g < p && i < p) ? A[(long)g * p + i] : 0.0;
        }
    }
    // reflector 0 from column 0, rows 1.. (warp 0 of every CTA)
    if (wid == 0) {
        double ss = 0.0;
        for (int i = 2 + lane; i < p; i += 32) { const double x = A[i]; ss = fma(x, x, ss); }
        ss = warp_sum(ss);
        const double alpha = A[1];
        double tau = 0.0, beta = alpha;
        if (ss != 0.0) { beta = -copysign(sqrt(alpha * alpha + ss), alpha); tau = (beta - alpha) / beta; }
        const double scale = (tau == 0.0) ? 0.0 : 1.0 / (alpha - beta);
        for (int i = lane; i < p; i += 32) vb[0][i] = (i < 1) ? 0.0 : (i == 1 ? 1.0 : A[i] * scale);
        if (lane == 0) { s_tau[0] = tau; s_beta[0] = beta; }
        if (blockIdx.x == 0 && lane == 0) a.d[0] = A[0];
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < CPW; t++) {
        const int g = gw + t * nwg;
        if (g < p && g >= 1) {
            const double *v = vb[0];
            double ss = 0.0;
#pragma unroll
            for (int u = 0; u < CH; u++) { const int i = lane + 32 * u; if (i >= 1 && i < p) ss = fma(col[t][u], v[i], ss); }
            ss = warp_sum(ss);
            if (lane == 0) a.P[g] = s_tau[0] * ss;
        }
    }
    grid.sync();
#ifdef LYAP_PANEL_PROF
    long long pt[6] = {0, 0, 0, 0, 0, 0}, tl = clock64();
#define TPROF(i) do { if (blockIdx.x == 0 && threadIdx.x == 0) { long long t_ = clock64(); pt[i] += t_ - tl; tl = t_; } } while (0)
#else
#define TPROF(i) do { } while (0)
#endif
    for (int j = 0; j + 2 < p; j++) {
        const int cur = j & 1, nxt = cur ^ 1;
        // P is double-buffered by step parity: a fast CTA's owners publish P for step j+1
        // while a slower CTA may still be reading step j's P
        const double *Pc = a.P + (long)cur * p;
        double *Pn = a.P + (long)nxt * p;
        const int r0 = j + 1;
        const double *v = vb[cur];
        double *vn = vb[nxt];
        const bool more = (j + 3 < p);
        // One block reduction per column: with y = x - P (x = column j+1 as published,
        // P = tau A v), the updated column is c = y + t v, t = 2k - P[r0], so
        //   k = (tau/2) P.v   and   ||c[r0+2:]||^2 = S_yy + 2 t S_yv + t^2 S_vv
        // come from four partial sums of one pass; on cancellation (result < 1/4 of the
        // terms) the norm is recomputed exactly with a second reduction.
        const double tau = s_tau[cur], beta = s_beta[cur];
        const double *cj = A + (long)r0 * p;
        double pv = 0.0, yy = 0.0, yv = 0.0, vv = 0.0;
        for (int i = r0 + threadIdx.x; i < p; i += blockDim.x) {
            const double Pi = Pc[i], vi = v[i], yi = cj[i] - Pi;
            w[i] = Pi;
            vn[i] = yi;
            pv = fma(Pi, vi, pv);
            if (i >= r0 + 2) { yy = fma(yi, yi, yy); yv = fma(yi, vi, yv); vv = fma(vi, vi, vv); }
        }
        pv = warp_sum(pv); yy = warp_sum(yy); yv = warp_sum(yv); vv = warp_sum(vv);
        if (lane == 0) { red1[wid] = pv; red1[8 + wid] = yy; red1[16 + wid] = yv; red2[wid] = vv; }
        const double P0 = Pc[r0], y0 = cj[r0] - P0;
        const double P1 = (r0 + 1 < p) ? Pc[r0 + 1] : 0.0, y1 = (r0 + 1 < p) ? cj[r0 + 1] - P1 : 0.0;
        TPROF(0);
        __syncthreads();
        TPROF(1);
        double spv = 0.0, syy = 0.0, syv = 0.0, svv = 0.0;
        for (int q = 0; q < nwb; q++) { spv += red1[q]; syy += red1[8 + q]; syv += red1[16 + q]; svv += red2[q]; }
        const double kk = 0.5 * tau * spv;
        const double t = 2.0 * kk - P0;
        double ss = syy + 2.0 * t * syv + t * t * svv;
        if (!(ss >= 0.25 * (syy + t * t * svv))) {                 // cancellation: exact norm
            __syncthreads();                                         // red1/red2 reads done
            double part = 0.0;
            for (int i = r0 + 2 + threadIdx.x; i < p; i += blockDim.x) {
                const double c = fma(t, v[i], vn[i]);
                part = fma(c, c, part);
            }
            part = warp_sum(part);
            if (lane == 0) red1[wid] = part;
            __syncthreads();
            ss = 0.0;
            for (int q = 0; q < nwb; q++) ss += red1[q];
        }
        TPROF(2);
        {
            const double alpha = fma(t, v[r0 + 1 < p ? r0 + 1 : r0], y1);
            const double dj1 = y0 + t;                               // v[r0] = 1
            double taun = 0.0, betan = alpha;
            if (more && ss != 0.0) { betan = -copysign(sqrt(alpha * alpha + ss), alpha); taun = (betan - alpha) / betan; }
            const double scale = (taun == 0.0) ? 0.0 : 1.0 / (alpha - betan);
            for (int i = r0 + threadIdx.x; i < p; i += blockDim.x) {
                const double vi = v[i];
                w[i] = fma(-kk, vi, w[i]);
                vn[i] = (i == r0) ? 0.0 : (i == r0 + 1 ? 1.0 : fma(t, vi, vn[i]) * scale);
            }
            if (threadIdx.x == 0) { s_tau[nxt] = taun; s_beta[nxt] = betan; }
            if (blockIdx.x == 0) {
                for (int i = r0 + threadIdx.x; i < p; i += blockDim.x) a.R[(long)j * p + i] = v[i];
                if (threadIdx.x == 0) {
                    a.e[j] = beta; a.tau[j] = tau; a.d[j + 1] = dj1;
                    if (!more) { a.e[j + 1] = alpha; a.tau[j + 1] = 0.0; }
                }
            }
        }
        __syncthreads();
        TPROF(3);
#pragma unroll
        for (int t = 0; t < CPW; t++) {
            const int g = gw + t * nwg;
            if (g < p && g >= r0 + 1) {
                const double vg = v[g], wg = w[g];
                double ss = 0.0;
#pragma unroll
                for (int u = 0; u < CH; u++) {
                    const int i = lane + 32 * u;
                    if (i >= r0 + 1 && i < p) {
                        const double x = col[t][u] - v[i] * wg - w[i] * vg;
                        col[t][u] = x;
                        if (more) ss = fma(x, vn[i], ss);
                    }
                }
                if (more) {
                    ss = warp_sum(ss);
                    if (lane == 0) Pn[g] = s_tau[nxt] * ss;
                }
                if (g == r0 + 1) {
#pragma unroll
                    for (int u = 0; u < CH; u++) {
                        const int i = lane + 32 * u;
                        if (i >= r0 + 1 && i < p) A[(long)g * p + i] = col[t][u];
                    }
                }
                if (g == p - 1 && !more) {
#pragma unroll
                    for (int u = 0; u < CH; u++) if (lane + 32 * u == p - 1) a.d[p - 1] = col[t][u];
                }
            }
        }
        TPROF(4);
        grid.sync();
        TPROF(5);
    }
#ifdef LYAP_PANEL_PROF
    if (blockIdx.x == 0 && threadIdx.x == 0)
        printf("tridiag p=%d grid=%d cycles/col: load+kk %lld bar1 %lld w,c,ss+bar2 %lld refl+bar3 %lld owner %lld gridsync %lld\n",
               p, gridDim.x, pt[0] / (p - 2), pt[1] / (p - 2), pt[2] / (p - 2), pt[3] / (p - 2), pt[4] / (p - 2), pt[5] / (p - 2));
#endif
}


// ---------------------------------------------------------------- 2. divide and conquer
// Leaf: dense eigendecomposition of the tridiagonal block [lo, hi) (size <= 32) by
// parallel (round-robin) Jacobi in one CTA; eigenvalues ascending into lam, vectors
// into the Q block.
__device__ __forceinline__ void leaf_pair(int r, int i, int N, int &a, int &b) {
    if (i == 0) { a = r; b = N - 1; }
    else { a = (r + i) % (N - 1); b = (r - i + (N - 1)) % (N - 1); }
    if (a > b) { int x = a; a = b; b = x; }
}

__global__ void __launch_bounds__(256)
dc_leaf_kernel(int p, const int *__restrict__ bounds, const double *__restrict__ d, const double *__restrict__ e,
               double *__restrict__ lam, double *__restrict__ Q)
{
    __shared__ double M[32][33], V[32][33], cs[32][2];
    __shared__ double red[32];
    __shared__ int any;
    const int lo = bounds[blockIdx.x], hi = bounds[blockIdx.x + 1], n = hi - lo;
    const int tid = threadIdx.x;
    const int N = n + (n & 1), np = N / 2;
    for (int idx = tid; idx < 32 * 32; idx += blockDim.x) {
        int r = idx / 32, t = idx % 32;
        double mv = 0.0;
        if (t < n && r < n) {
            if (r == t) mv = d[lo + r];
            else if (r == t + 1) mv = e[lo + t];
            else if (t == r + 1) mv = e[lo + r];
        }
        M[r][t] = mv;
        V[r][t] = (r == t) ? 1.0 : 0.0;
    }
    __syncthreads();
    double f2 = 0.0;
    for (int idx = tid; idx < n * n; idx += blockDim.x) f2 += M[idx / n][idx % n] * M[idx / n][idx % n];
    const double fro = sqrt(block_sum(f2, red));
    for (int sweep = 0; sweep < 40 && n > 1; sweep++) {
        double o2 = 0.0;
        for (int idx = tid; idx < n * n; idx += blockDim.x) { int r = idx / n, t = idx % n; if (r != t) o2 += M[r][t] * M[r][t]; }
        const double off = sqrt(block_sum(o2, red));
        if (off <= 0x1p-53 * fro || off == 0.0) break;
        if (tid == 0) any = 0;
        __syncthreads();
        for (int rr = 0; rr < N - 1; rr++) {
            if (tid < np) {
                int a, b;
                leaf_pair(rr, tid, N, a, b);
                double c = 1.0, s = 0.0;
                if (b < n) {
                    double apq = M[a][b];
                    if (apq != 0.0 && fabs(apq) > 0x1p-53 * sqrt(fabs(M[a][a] * M[b][b]))) {
                        double tt = (M[b][b] - M[a][a]) / (2.0 * apq);
                        double tn = isinf(tt) ? 0.0 : ((tt >= 0.0) ? 1.0 : -1.0) / (fabs(tt) + sqrt(1.0 + tt * tt));
                        c = 1.0 / sqrt(1.0 + tn * tn); s = tn * c;
                        any = 1;
                    }
                }
                cs[tid][0] = c; cs[tid][1] = s;
            }
            __syncthreads();
            for (int q = tid; q < np * np; q += blockDim.x) {       // A <- J^T A J, 2x2 blocks
                int P = q % np, R = q / np, a, b, a2, b2;
                leaf_pair(rr, P, N, a, b);
                leaf_pair(rr, R, N, a2, b2);
                const bool bv = b < n, b2v = b2 < n;
                double c1 = cs[P][0], s1 = cs[P][1], c2 = cs[R][0], s2 = cs[R][1];
                double m00 = M[a][a2], m01 = b2v ? M[a][b2] : 0.0;
                double m10 = bv ? M[b][a2] : 0.0, m11 = (bv && b2v) ? M[b][b2] : 0.0;
                double n00 = c2 * m00 - s2 * m01, n01 = s2 * m00 + c2 * m01;
                double n10 = c2 * m10 - s2 * m11, n11 = s2 * m10 + c2 * m11;
                double o00 = c1 * n00 - s1 * n10, o01 = c1 * n01 - s1 * n11;
                double o10 = s1 * n00 + c1 * n10, o11 = s1 * n01 + c1 * n11;
                if (P == R && bv && s1 != 0.0) { o01 = 0.0; o10 = 0.0; }
                M[a][a2] = o00;
                if (b2v) M[a][b2] = o01;
                if (bv) M[b][a2] = o10;
                if (bv && b2v) M[b][b2] = o11;
            }
            for (int q = tid; q < n * np; q += blockDim.x) {        // V <- V J
                int k = q % n, P = q / n, a, b;
                leaf_pair(rr, P, N, a, b);
                if (b >= n || cs[P][1] == 0.0) continue;
                double c = cs[P][0], s = cs[P][1];
                double va = V[k][a], vb = V[k][b];
                V[k][a] = c * va - s * vb;
                V[k][b] = s * va + c * vb;
            }
            __syncthreads();
        }
        if (!any) break;
    }
    // sort ascending (rank by comparison)
    const int t = tid;
    if (t < n) {
        double dt = M[t][t];
        int rank = 0;
        for (int r = 0; r < n; r++) { double dr = M[r][r]; if (dr < dt || (dr == dt && r < t)) rank++; }
        lam[lo + rank] = dt;
        for (int r = 0; r < n; r++) Q[(long)(lo + rank) * p + lo + r] = V[r][t];
    }
}

struct MergeInfo { int lo, mid, hi; };

__global__ void dc_tear_kernel(int nl, const int *__restrict__ bounds, const double *__restrict__ e,
                               double *__restrict__ d)
{
    const int i = 1 + blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nl) {
        const int m = bounds[i];
        const double r = fabs(e[m - 1]);
        d[m - 1] -= r;
        d[m] -= r;
    }
}

// M1: z, sort, deflation scan.  One CTA per merge.
//   out (per merge, indexed from lo): perm (sorted position -> local column),
//   Ds (sorted, deflation-modified), zK/DK (non-deflated compressed), K (positions),
//   defl positions; rot list; counts[2*m] = kk, counts[2*m+1] = nrot.
__global__ void __launch_bounds__(1024)
dc_merge_prep_kernel(int p, const MergeInfo *__restrict__ mi, const double *__restrict__ e,
                     const double *__restrict__ lam, const double *__restrict__ Q,
                     int *__restrict__ perm, double *__restrict__ Ds, double *__restrict__ zs,
                     double *__restrict__ DK, double *__restrict__ zK, int *__restrict__ Kpos,
                     int *__restrict__ Dpos, double *__restrict__ rot, int *__restrict__ counts,
                     double *__restrict__ rho_out, int use_smem)
{
    // the serial deflation scan runs on shared-memory copies when they fit (n <= nsmem):
    // its chain of dependent loads/stores then costs shared- instead of global-memory latency
    extern __shared__ double msm[];
    __shared__ double red[32];
    __shared__ int s_cnt[3];
    const MergeInfo m = mi[blockIdx.x];
    const int lo = m.lo, mid = m.mid, hi = m.hi, n = hi - lo, n1 = mid - lo;
    double *D = use_smem ? msm : Ds + lo;
    double *z = use_smem ? msm + n : zs + lo;
    double *R4 = use_smem ? msm + 2 * n : rot + 4 * lo;
    int *Dp = use_smem ? reinterpret_cast<int *>(msm + 6 * n) : Dpos + lo;
    int *Kp = use_smem ? Dp + n : Kpos + lo;
    const double rho_raw = e[mid - 1];
    const double sgn = (rho_raw < 0.0) ? -1.0 : 1.0;
    const double rho = 2.0 * fabs(rho_raw);
    const double isq2 = 0.70710678118654752440;
    // merge-sort positions: element i of child 1 (lam[lo+i]) and child 2 (lam[mid+i])
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double val = lam[lo + i];
        int pos;
        if (i < n1) {           // count elements of child 2 strictly smaller
            int a = 0, b = n - n1;
            while (a < b) { int c = (a + b) >> 1; if (lam[mid + c] < val) a = c + 1; else b = c; }
            pos = i + a;
        } else {                // count elements of child 1 <= val
            int a = 0, b = n1;
            while (a < b) { int c = (a + b) >> 1; if (lam[lo + c] <= val) a = c + 1; else b = c; }
            pos = (i - n1) + a;
        }
        perm[lo + pos] = i;
        D[pos] = val;
        double zz = (i < n1) ? Q[(long)(lo + i) * p + (mid - 1)] : sgn * Q[(long)(lo + i) * p + mid];
        z[pos] = zz * isq2;
    }
    __syncthreads();
    double mx = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) mx = fmax(mx, fmax(fabs(D[i]), fabs(z[i])));
    mx = block_max(mx, red);
    if (threadIdx.x == 0) {
        const double tol = 8.0 * 0x1p-52 * mx;
        int kk = 0, nd = 0, nr = 0, prev = -1;
        for (int k = 0; k < n; k++) {
            if (rho * fabs(z[k]) <= tol) { Dp[nd++] = k; continue; }
            if (prev < 0) { prev = k; continue; }
            double sn = z[prev], c = z[k];
            double tau = hypot(c, sn);
            double t = D[k] - D[prev];
            c /= tau; sn = -sn / tau;
            if (fabs(t * c * sn) <= tol) {
                z[k] = tau; z[prev] = 0.0;
                R4[4 * nr + 0] = prev; R4[4 * nr + 1] = k;
                R4[4 * nr + 2] = c; R4[4 * nr + 3] = sn;
                nr++;
                double tp = D[prev] * c * c + D[k] * sn * sn;
                D[k] = D[prev] * sn * sn + D[k] * c * c;
                D[prev] = tp;
                Dp[nd++] = prev;
                prev = k;
            } else {
                Kp[kk++] = prev;
                prev = k;
            }
        }
        if (prev >= 0) Kp[kk++] = prev;
        counts[2 * blockIdx.x] = kk;
        counts[2 * blockIdx.x + 1] = nr;
        rho_out[blockIdx.x] = rho;
        s_cnt[0] = kk; s_cnt[1] = nd; s_cnt[2] = nr;
    }
    __syncthreads();
    const int kk = s_cnt[0];
    if (use_smem) {
        const int nd = s_cnt[1], nr = s_cnt[2];
        for (int i = threadIdx.x; i < n; i += blockDim.x) { Ds[lo + i] = D[i]; zs[lo + i] = z[i]; }
        for (int i = threadIdx.x; i < nd; i += blockDim.x) Dpos[lo + i] = Dp[i];
        for (int i = threadIdx.x; i < kk; i += blockDim.x) Kpos[lo + i] = Kp[i];
        for (int i = threadIdx.x; i < 4 * nr; i += blockDim.x) rot[4 * lo + i] = R4[i];
    }
    for (int i = threadIdx.x; i < kk; i += blockDim.x) {
        DK[lo + i] = D[Kp[i]];
        zK[lo + i] = z[Kp[i]];
    }
}

// M2: gather Q block columns into sorted order (Qg[:, lo+k] = Q[:, lo+perm[k]], rows lo..hi),
// apply the deflation rotations in order (each thread one row), and compact the
// non-deflated columns into Qk[:, lo+k] = Qg[:, lo+Kpos[k]].  Gather and compaction run
// over (row, column) in parallel (grid.y strides columns, grid.z = subproblem); only the
// rotations, which must be applied in order, are one thread per row.
__global__ void dc_gather_kernel(int p, const MergeInfo *__restrict__ mi, const double *__restrict__ Q,
                                 const int *__restrict__ perm, double *__restrict__ Qg)
{
    const MergeInfo m = mi[blockIdx.z];
    const int lo = m.lo, n = m.hi - m.lo;
    for (int k = blockIdx.y; k < n; k += gridDim.y) {
        const double *src = Q + (long)(lo + perm[lo + k]) * p + lo;
        double *dst = Qg + (long)(lo + k) * p + lo;
        for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) dst[r] = src[r];
    }
}
__global__ void dc_rotate_kernel(int p, const MergeInfo *__restrict__ mi, const double *__restrict__ rot,
                                 const int *__restrict__ counts, double *__restrict__ Qg)
{
    const MergeInfo m = mi[blockIdx.y];
    const int lo = m.lo, n = m.hi - m.lo;
    const int nr = counts[2 * blockIdx.y + 1];
    if (nr == 0) return;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        for (int t = 0; t < nr; t++) {
            const double *R = rot + 4 * (lo + t);
            const int a = (int)R[0], b = (int)R[1];
            const double c = R[2], s = R[3];
            double *xa = Qg + (long)(lo + a) * p + lo + r, *xb = Qg + (long)(lo + b) * p + lo + r;
            const double x = *xa, y = *xb;
            *xa = c * x + s * y;
            *xb = c * y - s * x;
        }
    }
}
__global__ void dc_compact_kernel(int p, const MergeInfo *__restrict__ mi, const int *__restrict__ counts,
                                  const int *__restrict__ Kpos, const double *__restrict__ Qg, double *__restrict__ Qk)
{
    const MergeInfo m = mi[blockIdx.z];
    const int lo = m.lo, n = m.hi - m.lo;
    const int kk = counts[2 * blockIdx.z];
    for (int k = blockIdx.y; k < kk; k += gridDim.y) {
        const double *src = Qg + (long)(lo + Kpos[lo + k]) * p + lo;
        double *dst = Qk + (long)(lo + k) * p + lo;
        for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) dst[r] = src[r];
    }
}

// M3: secular roots by bisection around the nearer pole.  Thread per root.
__global__ void dc_secular_kernel(const MergeInfo *__restrict__ mi, const double *__restrict__ DK,
                                  const double *__restrict__ zK, const int *__restrict__ counts,
                                  const double *__restrict__ rho_in, double *__restrict__ taus,
                                  int *__restrict__ orig)
{
    const MergeInfo m = mi[blockIdx.y];
    const int lo = m.lo;
    const int kk = counts[2 * blockIdx.y];
    const double rho = rho_in[blockIdx.y];
    // one warp per root: the secular sum is split across the lanes
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const double *D = DK + lo, *z = zK + lo;
    double zz = 0.0;
    for (int i = lane; i < kk; i += 32) zz = fma(z[i], z[i], zz);
    zz = warp_sum(zz);
    for (int j = gw; j < kk; j += nw) {
        const double dl = D[j];
        const double du = (j + 1 < kk) ? D[j + 1] : D[j] + rho * zz;
        // choose the origin by the sign of f at the midpoint
        int o = j;
        if (j + 1 < kk) {
            const double mid = 0.5 * (du - dl);
            double f = 0.0;
            for (int i = lane; i < kk; i += 32) f += z[i] * z[i] / ((D[i] - dl) - mid);
            f = 1.0 + rho * warp_sum(f);
            if (f < 0.0) o = j + 1;          // root in (mid, du): measure from the upper pole
        }
        const double Do = D[o];
        double a, b;                          // tau interval
        if (o == j) { a = 0.0; b = (j + 1 < kk) ? 0.5 * (du - dl) : du - dl; }
        else { a = -(0.5 * (du - dl)); b = 0.0; }
        // Newton on h(tau) = (delta_o - tau) f(tau) = rho z_o^2 - tau (1 + rho S(tau)),
        // S = sum_{i != o} z_i^2 / (delta_i - tau): the pole at the origin is removed, so the
        // iteration converges fast for roots close to it (the usual case after deflation).
        // Started at tau = 0 (first step = the one-pole estimate rho z_o^2 / (1 + rho S(0))),
        // safeguarded by the bracket (a, b) of f's sign change and bisection.
        const double zo2 = rho * z[o] * z[o];
        double tau = 0.0;
        for (int it = 0; it < 200; it++) {
            double S = 0.0, dS = 0.0;
            for (int i = lane; i < kk; i += 32) {
                if (i == o) continue;
                const double t = z[i] / ((D[i] - Do) - tau);
                S = fma(t, z[i], S);
                dS = fma(t, t, dS);
            }
            S = rho * warp_sum(S);
            dS = rho * warp_sum(dS);
            const double h = zo2 - tau * (1.0 + S);
            const double dh = -(1.0 + S) - tau * dS;
            if (tau != 0.0) {
                if (h == 0.0) break;
                const double fs = (o == j) ? -h : h;             // sign of f (f increasing)
                if (fs > 0.0) b = tau; else a = tau;
            }
            double tn = (dh != 0.0) ? tau - h / dh : 0.5 * (a + b);
            if (!(tn > a && tn < b)) tn = 0.5 * (a + b);
            const bool done = (tn == a || tn == b || fabs(tn - tau) <= 4.4e-16 * fabs(tn));
            tau = tn;
            if (done) break;
        }
        if (lane == 0) { taus[lo + j] = tau; orig[lo + j] = o; }
    }
}

// M4: Loewner z-hat and the unnormalised eigenvector matrix U (kk x kk, at [lo,lo]).
__global__ void dc_vectors_kernel(int p, const MergeInfo *__restrict__ mi, const double *__restrict__ DK,
                                  const double *__restrict__ zK, const int *__restrict__ counts,
                                  const double *__restrict__ rho_in, const double *__restrict__ taus,
                                  const int *__restrict__ orig, double *__restrict__ zhat, double *__restrict__ U)
{
    const MergeInfo m = mi[blockIdx.y];
    const int lo = m.lo;
    const int kk = counts[2 * blockIdx.y];
    const double rho = rho_in[blockIdx.y];
    const double *D = DK + lo;
    // phase A: zhat (thread per i); phase B needs all zhat -> done in a second launch
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < kk; i += gridDim.x * blockDim.x) {
        // zhat_i^2 = (lambda_{kk-1} - d_i)/rho * prod_{j<i} (lambda_j - d_i)/(d_j - d_i)
        //            * prod_{i<=j<kk-1} (lambda_j - d_i)/(d_{j+1} - d_i)
        const double di = D[i];
        auto lmd = [&](int j) { return (D[orig[lo + j]] - di) + taus[lo + j]; };
        double prod = lmd(kk - 1) / rho;
        for (int j = 0; j < i; j++) prod *= lmd(j) / (D[j] - di);
        for (int j = i; j < kk - 1; j++) prod *= lmd(j) / (D[j + 1] - di);
        double zh = sqrt(fabs(prod));
        zhat[lo + i] = copysign(zh, zK[lo + i]);
    }
}

__global__ void dc_umatrix_kernel(int p, const MergeInfo *__restrict__ mi, const double *__restrict__ DK,
                                  const int *__restrict__ counts, const double *__restrict__ taus,
                                  const int *__restrict__ orig, const double *__restrict__ zhat,
                                  double *__restrict__ U)
{
    const MergeInfo m = mi[blockIdx.y];
    const int lo = m.lo;
    const int kk = counts[2 * blockIdx.y];
    const double *D = DK + lo;
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (int j = gw; j < kk; j += nw) {          // warp per eigenvector j
        const double Dj = D[orig[lo + j]], tj = taus[lo + j];
        double ss = 0.0;
        for (int i = lane; i < kk; i += 32) {
            double u = zhat[lo + i] / ((D[i] - Dj) - tj);
            U[(long)(lo + j) * p + lo + i] = u;
            ss = fma(u, u, ss);
        }
        ss = warp_sum(ss);
        const double inv = 1.0 / sqrt(ss);
        for (int i = lane; i < kk; i += 32) U[(long)(lo + j) * p + lo + i] *= inv;
    }
}

// M5: Qn = Qk U for every merge of the level in one launch (grid.z = merge), sizes read on
// the device (no host synchronisation): rows n_q = hi - lo, kk_q = counts[2q] non-deflated
// columns, fp64 DMMA tiles of 64 x 64.
static __global__ void __launch_bounds__(128)
dc_gemm_grouped_kernel(int p, const MergeInfo *__restrict__ mi, const int *__restrict__ counts,
                       const double *__restrict__ Qk, const double *__restrict__ U, double *__restrict__ Qn)
{
    const MergeInfo m = mi[blockIdx.z];
    const int n = m.hi - m.lo, kk = counts[2 * blockIdx.z];
    const long m0 = (long)blockIdx.y * 64, n0 = (long)blockIdx.x * 64;
    if (kk <= 0 || m0 >= n || n0 >= kk) return;
    const size_t off = (size_t)m.lo * p + m.lo;
    dmma_tile(n, kk, 0, kk, m0, n0, 1.0, Qk + off, 1, p, U + off, 1, p, 0.0, Qn + off, 1, p, nullptr, 0);
}

// M6: eigenvalues of the merged block and assembly of the (unsorted) columns:
// columns 0..kk-1: computed by GEMM into Qn; deflated columns copied; then sort.
__global__ void dc_finish_kernel(int p, const MergeInfo *__restrict__ mi, const double *__restrict__ Ds,
                                 const double *__restrict__ DK, const int *__restrict__ counts,
                                 const double *__restrict__ taus, const int *__restrict__ orig,
                                 const int *__restrict__ Dpos, const double *__restrict__ Qg,
                                 double *__restrict__ Qn, double *__restrict__ lamtmp)
{
    const MergeInfo m = mi[blockIdx.y];
    const int lo = m.lo, n = m.hi - m.lo;
    const int kk = counts[2 * blockIdx.y];
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        if (t < kk) {
            lamtmp[lo + t] = DK[lo + orig[lo + t]] + taus[lo + t];
        } else {
            int k = Dpos[lo + (t - kk)];
            lamtmp[lo + t] = Ds[lo + k];
            for (int r = 0; r < n; r++) Qn[(long)(lo + t) * p + lo + r] = Qg[(long)(lo + k) * p + lo + r];
        }
    }
}

// sort the n eigenvalues ascending (rank by comparison) and permute columns into Q
__global__ void dc_sort_kernel(int p, const MergeInfo *__restrict__ mi, const double *__restrict__ lamtmp,
                               const double *__restrict__ Qn, double *__restrict__ lam, double *__restrict__ Q)
{
    const MergeInfo m = mi[blockIdx.y];
    const int lo = m.lo, n = m.hi - m.lo;
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (int t = gw; t < n; t += nw) {
        double v = lamtmp[lo + t];
        int rank = 0;
        for (int s = lane; s < n; s += 32) { double u = lamtmp[lo + s]; if (u < v || (u == v && s < t)) rank++; }
        rank = warp_sum(rank);
        if (lane == 0) lam[lo + rank] = v;
        for (int r = lane; r < n; r += 32) Q[(long)(lo + rank) * p + lo + r] = Qn[(long)(lo + t) * p + lo + r];
    }
}

// ---------------------------------------------------------------- 3. back-transformation
// Compact-WY factor T (jb x jb, ld 32) of reflectors with Gram G = V^T V (ld 32):
// T[c][c] = tau_c, T[0:c, c] = -tau_c T[0:c, 0:c] G[0:c, c]  (forward, columnwise).
// One warp; column c is computed in parallel over its rows.
__global__ void wy_T_kernel(int jb, const double *__restrict__ G, const double *__restrict__ tau, double *__restrict__ Tp)
{
    // lane a keeps row a of T in registers (fully unrolled, static indexing); G is
    // read as warp-wide broadcasts from shared memory
    __shared__ double Gs[32][33];
    const int a = threadIdx.x;
    for (int c = 0; c < 32; c++) Gs[c][a] = (a < jb && c < jb) ? G[a + c * 32] : 0.0;   // Gs[l][c]... transposed load
    __syncwarp();
    double Ta[32];
#pragma unroll
    for (int c = 0; c < 32; c++) Ta[c] = 0.0;
#pragma unroll
    for (int c = 0; c < 32; c++) {
        if (c < jb) {
            double sacc = 0.0;
#pragma unroll
            for (int l = 0; l < c; l++)
                if (l >= a) sacc = fma(Ta[l], Gs[c][l], sacc);
            const double tc = tau[c];
            Ta[c] = (a < c) ? -tc * sacc : ((a == c) ? tc : 0.0);
        }
    }
#pragma unroll
    for (int c = 0; c < 32; c++) Tp[a + c * 32] = Ta[c];
}

// All compact-WY triangular factors of the back-transformation at once: CTA = panel of
// 32 reflectors; Gram G = V^T V over the panel's nonzero rows (staged 64 rows at a time),
// then T by the wy_T_kernel recurrence (lane a keeps row a of T).
__global__ void __launch_bounds__(256)
wy_gramT_batched_kernel(int p, int nref, const double *__restrict__ R, const double *__restrict__ tau,
                        double *__restrict__ Tall)
{
    const int panel = blockIdx.x, j0 = panel * 32, jb = min(32, nref - j0);
    const double *Vp = R + (long)j0 * p;
    __shared__ double Vs[64][33];
    __shared__ double Gs[32][33];
    const int tid = threadIdx.x;
    const int ga = tid >> 3, c0 = (tid & 7) * 4;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int r0 = j0 + 1; r0 < p; r0 += 64) {
        for (int e = tid; e < 64 * 32; e += 256) {
            const int i = e & 63, cc = e >> 6;
            Vs[i][cc] = (r0 + i < p && cc < jb) ? Vp[(long)cc * p + r0 + i] : 0.0;
        }
        __syncthreads();
#pragma unroll 8
        for (int i = 0; i < 64; i++) {
            const double va = Vs[i][ga];
#pragma unroll
            for (int t = 0; t < 4; t++) acc[t] = fma(va, Vs[i][c0 + t], acc[t]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int t = 0; t < 4; t++) Gs[c0 + t][ga] = acc[t];           // Gs[c][l] = G(l, c)
    __syncthreads();
    if (tid < 32) {
        const int a = tid;
        const double *tp = tau + j0;
        double Ta[32];
#pragma unroll
        for (int c = 0; c < 32; c++) Ta[c] = 0.0;
#pragma unroll
        for (int c = 0; c < 32; c++) {
            if (c < jb) {
                double sacc = 0.0;
#pragma unroll
                for (int l = 0; l < c; l++)
                    if (l >= a) sacc = fma(Ta[l], Gs[c][l], sacc);
                const double tc = tp[c];
                Ta[c] = (a < c) ? -tc * sacc : ((a == c) ? tc : 0.0);
            }
        }
        double *Tp = Tall + (long)panel * 1024;
#pragma unroll
        for (int c = 0; c < 32; c++) Tp[a + c * 32] = Ta[c];
    }
}

// eigenvalues descending + sign normalisation (largest |component| positive, lowest index)
__global__ void eigfinal_kernel(int p, const double *__restrict__ lam, const double *__restrict__ X,
                                double *__restrict__ w, double *__restrict__ V)
{
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (int j = gw; j < p; j += nw) {
        const int src = p - 1 - j;
        double bv = -1.0; int bi = p;
        for (int k = lane; k < p; k += 32) {
            double v = fabs(X[(long)src * p + k]);
            if (v > bv || (v == bv && k < bi)) { bv = v; bi = k; }
        }
        for (int o = 16; o > 0; o >>= 1) {
            double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
            int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
            if (v2 > bv || (v2 == bv && i2 < bi)) { bv = v2; bi = i2; }
        }
        const double sg = (X[(long)src * p + bi] < 0.0) ? -1.0 : 1.0;
        if (lane == 0) w[j] = lam[src];
        for (int k = lane; k < p; k += 32) V[(long)j * p + k] = sg * X[(long)src * p + k];
    }
}

__global__ void symmetrize_copy_kernel(int p, const double *__restrict__ Ain, double *__restrict__ A)
{
    long tot = (long)p * p;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < tot; idx += (long)gridDim.x * blockDim.x) {
        int i = (int)(idx % p), j = (int)(idx / p);
        A[idx] = 0.5 * (Ain[idx] + Ain[(long)i * p + j]);
    }
}

__global__ void zero_d_kernel(long len, double *x)
{
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < len; i += (long)gridDim.x * blockDim.x) x[i] = 0.0;
}

// ---------------------------------------------------------------- driver
int SyevdWork::alloc(int pmax_) {
    pmax = pmax_;
    size_t pp = (size_t)pmax * pmax;
    for (double **b : {&A, &Q, &Qg, &Qk, &U, &Qn, &R}) LYAP_CUDA_TRY(cudaMalloc(b, sizeof(double) * pp));
    LYAP_CUDA_TRY(cudaMalloc(&vec, sizeof(double) * (size_t)pmax * 16 + 32 * 33 * 64 * 8));
    LYAP_CUDA_TRY(cudaMalloc(&ivec, sizeof(int) * (size_t)pmax * 8 + 4096));
    LYAP_CUDA_TRY(cudaMalloc(&rot, sizeof(double) * (size_t)pmax * 4));
    if (sizeof(double) * 4 * (size_t)pmax > 200 * 1024) {
        gvec_ctas = 296;
        LYAP_CUDA_TRY(cudaMalloc(&gvec, sizeof(double) * (size_t)gvec_ctas * 4 * pmax));
    }
    return LYAP_OK;
}
void SyevdWork::release() {
    for (double *b : {A, Q, Qg, Qk, U, Qn, R, vec, rot, gvec}) if (b) cudaFree(b);
    gvec = nullptr;
    cudaFree(ivec);
    A = Q = Qg = Qk = U = Qn = R = vec = rot = nullptr;
    ivec = nullptr;
}

int syevd_f64(cudaStream_t s, int p, const double *Ain, double *w_out, double *V_out, SyevdWork &W)
{
    if (p > W.pmax) return LYAP_ERR_CAPACITY;
    const size_t pp = (size_t)p * p;
    double *d = W.vec, *e = d + p, *tau = e + p, *P = tau + p, *lam = P + p, *Ds = lam + p, *zs = Ds + p,
           *DK = zs + p, *zK = DK + p, *taus = zK + p, *zhat = taus + p, *lamtmp = zhat + p, *rho = lamtmp + p,
           *Tp = rho + p;
    int *perm = W.ivec, *Kpos = perm + p, *Dpos = Kpos + p, *orig = Dpos + p, *counts = orig + p,
        *bounds = counts + 2 * p;
    MergeInfo *mi = reinterpret_cast<MergeInfo *>(bounds + p + 2);
    const int gsz = std::min(ceil_div((long)pp, 256), 2048);
    static int prof = -1;
    static cudaEvent_t pev[4];
    if (prof < 0) {
        const char *ev = getenv("LYAP_PROFILE_EIG");
        prof = (ev && ev[0] == '1') ? 1 : 0;
        if (prof) for (auto &x : pev) cudaEventCreate(&x);
    }
    if (prof) cudaEventRecord(pev[0], s);
    // 1. tridiagonalisation (reflectors stay in W.A until the back-transformation)
    zero_d_kernel<<<gsz, 256, 0, s>>>((long)pp, W.R);
    LYAP_TRY(launched());
    symmetrize_copy_kernel<<<gsz, 256, 0, s>>>(p, Ain, W.A);
    LYAP_TRY(launched());
    {
        // shared memory for this p (the kernels address 4 p doubles), not the capacity;
        // above 200 KB the general kernel keeps the four vectors in a global slice per CTA
        const bool gvec = sizeof(double) * 4 * (size_t)p > 200 * 1024;
        const size_t smem = gvec ? 0 : sizeof(double) * 4 * (size_t)p;
        // one-time attribute setup (function-local static: thread-safe initialisation)
        static const int nsm_t = [] {
            int dev = 0, v = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
            cudaFuncSetAttribute(tridiag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            for (void *f : {(void *)tridiag_reg_kernel<8>, (void *)tridiag_reg_kernel<16>, (void *)tridiag_reg_kernel<32>,
                            (void *)tridiag_w_kernel<8, 1>, (void *)tridiag_w_kernel<16, 1>,
                            (void *)tridiag_w_kernel<32, 1>})
                cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            return v;
        }();
        const int max_blocks = nsm_t;                 // one CTA per SM for the register-resident kernels
        TridArgs ta{p, W.A, W.R, d, e, tau, P, gvec ? W.gvec : nullptr};
        void *args[] = {&ta};
        const int need = ceil_div(p, 8);             // one warp per column
        KTimer kt(KC_TRIDIAG, s, (4.0 / 3.0) * (double)p * p * p, 8.0 * (double)p * p);
        if (p >= 3 && p <= 1024 && need <= max_blocks && !gvec) {
            void *fn;
            int grid_t = need;
            if (env_flag("LYAP_TRIDIAG_REG")) {
                fn = (p <= 256) ? (void *)tridiag_reg_kernel<8>
                   : (p <= 512) ? (void *)tridiag_reg_kernel<16> : (void *)tridiag_reg_kernel<32>;
            } else {
                // one column per warp (two per warp measured slower: the owners' update is on
                // the critical path of every step, the grid barrier is not cheaper enough)
                fn = (p <= 256) ? (void *)tridiag_w_kernel<8, 1>
                   : (p <= 512) ? (void *)tridiag_w_kernel<16, 1> : (void *)tridiag_w_kernel<32, 1>;
            }
            LYAP_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(grid_t), dim3(256), args, smem, s));
        } else {
            // shared memory for this p (not the capacity): up to two CTAs per SM, one warp
            // per trailing column (the trailing block shrinks: the full grid is best)
            const size_t smem_p = smem;
            int dev, nsm, per = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, tridiag_kernel, 256, smem_p);
            int maxb = nsm * std::max(1, std::min(per, env_flag("LYAP_TRIDIAG_1CTA") ? 1 : 2));
            if (gvec) maxb = std::min(maxb, W.gvec_ctas);
            int grid = std::max(1, std::min(maxb, ceil_div(p - 1, 8)));
            if (const char *e = getenv("LYAP_TRIDIAG_GRID")) grid = std::max(1, std::min(maxb, atoi(e)));
            LYAP_CUDA_TRY(cudaLaunchCooperativeKernel((void *)tridiag_kernel, dim3(grid), dim3(256), args, smem_p, s));
        }
        LYAP_TRY(launched());
    }
    if (prof) cudaEventRecord(pev[1], s);
    // 2. divide and conquer on (d, e): leaves of size <= 32, power-of-two tree
    int nl = 1;
    static int leaf = 0;
    if (leaf == 0) { const char *e = getenv("LYAP_DC_LEAF"); leaf = e ? std::max(4, std::min(32, atoi(e))) : 16; }   // 16: measured best
    while ((p + nl - 1) / nl > leaf) nl *= 2;
    std::vector<int> hb(nl + 1);
    for (int i = 0; i <= nl; i++) hb[i] = (int)((long)i * p / nl);
    // Cuppen tears T = diag(T1', T2') + |e| v v^T at the leaf boundaries, on the device
    // (leaves are >= 16 long, so no two tears touch the same diagonal entry)
    LYAP_CUDA_TRY(cudaMemcpyAsync(bounds, hb.data(), sizeof(int) * (nl + 1), cudaMemcpyHostToDevice, s));
    if (nl > 1) {
        dc_tear_kernel<<<ceil_div(nl, 128), 128, 0, s>>>(nl, bounds, e, d);
        LYAP_TRY(launched());
    }
    zero_d_kernel<<<gsz, 256, 0, s>>>((long)pp, W.Q);
    LYAP_TRY(launched());
    dc_leaf_kernel<<<nl, 256, 0, s>>>(p, bounds, d, e, lam, W.Q);
    LYAP_TRY(launched());
    for (int width = 1; width < nl; width *= 2) {
        std::vector<MergeInfo> hm;
        for (int i = 0; i + width < nl; i += 2 * width)
            hm.push_back({hb[i], hb[i + width], hb[std::min(i + 2 * width, nl)]});
        const int nm = (int)hm.size();
        LYAP_CUDA_TRY(cudaMemcpyAsync(mi, hm.data(), sizeof(MergeInfo) * nm, cudaMemcpyHostToDevice, s));
        {
            int maxn0 = 0;
            for (auto &x : hm) maxn0 = std::max(maxn0, x.hi - x.lo);
            const size_t msm = 56 * (size_t)maxn0;           // D, z, rot (4n), Dpos, Kpos
            const int use = msm <= 200 * 1024 ? 1 : 0;
            // one-time setup (function-local static: thread-safe initialisation)
            static const bool attr_m = [] {
                cudaFuncSetAttribute(dc_merge_prep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
                return true;
            }();
            (void)attr_m;
            dc_merge_prep_kernel<<<nm, 1024, use ? msm : 0, s>>>(p, mi, e, lam, W.Q, perm, Ds, zs, DK, zK, Kpos, Dpos,
                                                                 W.rot, counts, rho, use);
        }
        LYAP_TRY(launched());
        int maxn = 0;
        for (auto &x : hm) maxn = std::max(maxn, x.hi - x.lo);
        dim3 g1(ceil_div(maxn, 128), nm);
        {
            const dim3 gc(ceil_div(maxn, 128), std::min(maxn, std::max(1, 2048 / nm)), nm);
            dc_gather_kernel<<<gc, 128, 0, s>>>(p, mi, W.Q, perm, W.Qg);
            LYAP_TRY(launched());
            dc_rotate_kernel<<<g1, 128, 0, s>>>(p, mi, W.rot, counts, W.Qg);
            LYAP_TRY(launched());
            dc_compact_kernel<<<gc, 128, 0, s>>>(p, mi, counts, Kpos, W.Qg, W.Qk);
            LYAP_TRY(launched());
        }
        dc_secular_kernel<<<dim3(ceil_div((long)maxn * 32, 256), nm), 256, 0, s>>>(mi, DK, zK, counts, rho, taus, orig);
        LYAP_TRY(launched());
        dc_vectors_kernel<<<g1, 128, 0, s>>>(p, mi, DK, zK, counts, rho, taus, orig, zhat, W.U);
        LYAP_TRY(launched());
        dim3 g2(ceil_div((long)maxn * 32, 256), nm);
        dc_umatrix_kernel<<<g2, 256, 0, s>>>(p, mi, DK, counts, taus, orig, zhat, W.U);
        LYAP_TRY(launched());
        {
            const dim3 gg(ceil_div(maxn, 64), ceil_div(maxn, 64), nm);
            KTimer kt(KC_DGEMM, s);
            dc_gemm_grouped_kernel<<<gg, 128, 0, s>>>(p, mi, counts, W.Qk, W.U, W.Qn);
            LYAP_TRY(launched());
        }
        dc_finish_kernel<<<g1, 128, 0, s>>>(p, mi, Ds, DK, counts, taus, orig, Dpos, W.Qg, W.Qn, lamtmp);
        LYAP_TRY(launched());
        dc_sort_kernel<<<g2, 256, 0, s>>>(p, mi, lamtmp, W.Qn, lam, W.Q);
        LYAP_TRY(launched());
    }
    if (prof) cudaEventRecord(pev[2], s);
    // 3. back-transformation X = Q_H Q_T: panels of 32 reflectors, last panel first
    const int nref = std::max(p - 2, 0);
    if (nref > 0) {
        wy_gramT_batched_kernel<<<ceil_div(nref, 32), 256, 0, s>>>(p, nref, W.R, tau, Tp);
        LYAP_TRY(launched());
    }
    for (int j0 = ((nref - 1) / 32) * 32; nref > 0 && j0 >= 0; j0 -= 32) {
        const int jb = std::min(32, nref - j0);
        // V = reflectors j0..j0+jb-1 as stored (zero above the unit entry), p x jb, ld p
        const double *Vp = W.R + (size_t)j0 * p;
        // X <- (I - V T V^T) X over rows j0+1..p-1 (reflector j0+a is zero above row j0+a+1)
        LYAP_TRY(wy_apply(s, p, p, jb, j0 + 1, Vp, p, Tp + (size_t)(j0 / 32) * 1024, 0, W.Q, p));
    }
    eigfinal_kernel<<<std::min(ceil_div((long)p * 32, 256), 1024), 256, 0, s>>>(p, lam, W.Q, w_out, V_out);
    LYAP_TRY(launched());
    if (prof) {
        cudaEventRecord(pev[3], s);
        cudaEventSynchronize(pev[3]);
        float a = 0, b = 0, c = 0;
        cudaEventElapsedTime(&a, pev[0], pev[1]);
        cudaEventElapsedTime(&b, pev[1], pev[2]);
        cudaEventElapsedTime(&c, pev[2], pev[3]);
        fprintf(stderr, "lyap: syevd p=%d tridiag %.3f ms  d&c %.3f ms  backtransform %.3f ms\n", p, a, b, c);
    }
    return LYAP_OK;
}

}  // namespace lyap
