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
#include "lyap_internal.h"

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
    LYAP_CUDA_TRY(cudaMalloc(&nrm, sizeof(double) * (size_t)(nmax + 3 * 1024 + cmax + 8)));
    LYAP_CUDA_TRY(cudaMalloc(&ints, sizeof(int) * (size_t)(nmax + 1024 + 8)));
    scal = nrm + nmax;
    return LYAP_OK;
}
void RrqrWork::release() { cudaFree(M); cudaFree(nrm); cudaFree(ints); M = nrm = scal = nullptr; ints = nullptr; }

int rank_trunc_chol_f64(cudaStream_t s, int n, int c, const double *Z, double tol, int prec_out,
                        double *Zout, int *k_out, RrqrWork &w)
{
    if (n > w.nmax || c > w.cmax) return LYAP_ERR_CAPACITY;
    int *perm = w.ints, *bidx = w.ints + w.nmax, *rank = bidx + 1024;
    double *bsum = w.nrm + w.nmax, *bbest = bsum + 1024, *v = bbest + 1024, *scal = v + w.cmax;
    long tot = (long)n * c;
    transpose_init_kernel<<<ceil_div(tot, 256) < 2048 ? ceil_div(tot, 256) : 2048, 256, 0, s>>>(n, c, Z, w.M, perm);
    LYAP_TRY(launched());
    static int max_blocks = 0;
    if (max_blocks == 0) {
        int dev, nsm, per;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, rrqr_kernel, 256, 0);
        max_blocks = nsm * (per < 2 ? per : 2);
        if (max_blocks > 1024) max_blocks = 1024;
        if (max_blocks < 1) max_blocks = 1;
    }
    int want = ceil_div(n, 8);
    int grid = want < max_blocks ? want : max_blocks;
    RrqrArgs a{n, c, c < n ? c : n, tol, w.M, w.nrm, bsum, bbest, bidx, perm, v, scal, rank};
    void *args[] = {&a};
    LYAP_CUDA_TRY(cudaLaunchCooperativeKernel((void *)rrqr_kernel, dim3(grid), dim3(256), args, 0, s));
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
