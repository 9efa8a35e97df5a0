// newton.cu -- element-wise / reduction kernels of the sign-function Newton
// iteration (Section 3, Eqs. newton-lyapu, newton-lyapu-factored-*)
// and of the fp64 fragments.
//
//  * cast kernel: A (fp64) -> A_0 in the solver precision u_s, with
//    max|a| and ||A_0||_F (the "norm-scaling and cast" step);
//  * scale kernel: W = 2^{-e} A_k (exact power-of-two range scaling so that
//    the inversion stays inside the fp16/bf16 range, reading R-RANGE);
//  * Newton update kernel (fused): A_{k+1} = (mu A_k + mu^{-1} A_k^{-1})/2
//    with the column un-permutation of the Gauss-Jordan result, the cached
//    copy of A_k^{-1}, and per-row partials of ||A_{k+1}-A_k||_F,
//    ||A_{k+1}||_F, ||A_{k+1}+I||_inf and max|A_{k+1}|;
//  * Z-side helpers (range scaling of L, blkdiag(mu Y, mu^{-1} Y)/2, the
//    Cholesky column scalings), selection / gather kernels for truncations.
#include "common.cuh"
#include "lyap_internal.h"
#include "newton_kernels.h"
#include "ktimer.h"
#include "ptx.cuh"

namespace lyap {

// ------------------------------------------------------------ row partials
// part[4*i + 0..3] = per-row partial sums, reduced by reduce_rows_kernel in a
// fixed order (deterministic).
template <typename T>
__global__ void __launch_bounds__(256)
cast_kernel(int n, const double *__restrict__ A, T *__restrict__ Ak, double *__restrict__ part)
{
    __shared__ double red[32];
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        double ss = 0.0, mx = 0.0;
        for (int j = threadIdx.x; j < n; j += blockDim.x) {
            T v = from_d<T>(A[(long)i * n + j]);
            Ak[(long)i * n + j] = v;
            double d = to_d<T>(v);
            ss = fma(d, d, ss);
            mx = fmax(mx, fabs(d));
        }
        ss = block_sum(ss, red);
        mx = block_max(mx, red);
        if (threadIdx.x == 0) { part[4 * i + 0] = 0.0; part[4 * i + 1] = ss; part[4 * i + 2] = 0.0; part[4 * i + 3] = mx; }
    }
}

// Same cast on row vectors: 16 bytes of A_k written per thread per pass, the fp64 source
// read as double2 (n a multiple of 16 / sizeof(T)).
template <typename T>
__global__ void __launch_bounds__(256)
cast_vec_kernel(int n, const double *__restrict__ A, T *__restrict__ Ak, double *__restrict__ part)
{
    __shared__ double red[32];
    constexpr int V = 16 / sizeof(T);
    const int nv = n / V;
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        const double2 *Ai = reinterpret_cast<const double2 *>(A + (long)i * n);
        uint4 *Oi = reinterpret_cast<uint4 *>(Ak + (long)i * n);
        double ss = 0.0, mx = 0.0;
        for (int j = threadIdx.x; j < nv; j += blockDim.x) {
            uint4 w;
            T *o = reinterpret_cast<T *>(&w);
#pragma unroll
            for (int t = 0; t < V / 2; t++) {
                const double2 a = __ldcs(Ai + (long)j * (V / 2) + t);
                o[2 * t] = from_d<T>(a.x);
                o[2 * t + 1] = from_d<T>(a.y);
            }
#pragma unroll
            for (int t = 0; t < V; t++) { const double d = to_d<T>(o[t]); ss = fma(d, d, ss); mx = fmax(mx, fabs(d)); }
            Oi[j] = w;
        }
        ss = block_sum(ss, red);
        mx = block_max(mx, red);
        if (threadIdx.x == 0) { part[4 * i + 0] = 0.0; part[4 * i + 1] = ss; part[4 * i + 2] = 0.0; part[4 * i + 3] = mx; }
    }
}

// out[0] = sum part[.,0], out[1] = sum part[.,1], out[2] = max part[.,2], out[3] = max part[.,3]
__global__ void __launch_bounds__(1024)
reduce_rows_kernel(int n, const double *__restrict__ part, double *__restrict__ out)
{
    __shared__ double red[32];
    double s0 = 0.0, s1 = 0.0, m2 = 0.0, m3 = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        s0 += part[4 * i]; s1 += part[4 * i + 1];
        m2 = fmax(m2, part[4 * i + 2]); m3 = fmax(m3, part[4 * i + 3]);
    }
    s0 = block_sum(s0, red); s1 = block_sum(s1, red);
    m2 = block_max(m2, red); m3 = block_max(m3, red);
    if (threadIdx.x == 0) { out[0] = s0; out[1] = s1; out[2] = m2; out[3] = m3; }
}

// W = 2^{-e} A_k with e = exponent of max|A_k| (scal[SC_MAXA]) so that max|W| in [0.5,1).
template <typename T>
__global__ void scale_kernel(long nn, const T *__restrict__ Ak, T *__restrict__ W, double *__restrict__ scal)
{
    int e;
    frexp(scal[SC_MAXA], &e);
    if (scal[SC_MAXA] == 0.0) e = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) scal[SC_EXP] = (double)e;
    const float f = ldexpf(1.0f, -e);
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < nn; idx += (long)gridDim.x * blockDim.x) {
        if constexpr (sizeof(T) == 8) W[idx] = ldexp(to_d<T>(Ak[idx]), -e);
        else W[idx] = from_f<T>(to_f<T>(Ak[idx]) * f);
    }
}

// Same scaling on 16-byte vectors (nn a multiple of 16 / sizeof(T)); exact, so bitwise
// equal to scale_kernel.
template <typename T>
__global__ void __launch_bounds__(256)
scale_vec_kernel(long nv, const uint4 *__restrict__ Ak, uint4 *__restrict__ W, double *__restrict__ scal)
{
    constexpr int V = 16 / sizeof(T);
    int e;
    frexp(scal[SC_MAXA], &e);
    if (scal[SC_MAXA] == 0.0) e = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) scal[SC_EXP] = (double)e;
    const float f = ldexpf(1.0f, -e);
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < nv; idx += (long)gridDim.x * blockDim.x) {
        uint4 v = __ldcs(Ak + idx), w;
        const T *a = reinterpret_cast<const T *>(&v);
        T *o = reinterpret_cast<T *>(&w);
#pragma unroll
        for (int t = 0; t < V; t++) {
            if constexpr (sizeof(T) == 8) o[t] = ldexp(to_d<T>(a[t]), -e);
            else o[t] = from_f<T>(to_f<T>(a[t]) * f);
        }
        W[idx] = w;
    }
}

template <typename T>
__global__ void __launch_bounds__(256)
sumsq_rows_kernel(int n, const T *__restrict__ G, double *__restrict__ part)
{
    __shared__ double red[32];
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        double ss = 0.0;
        for (int j = threadIdx.x; j < n; j += blockDim.x) { double d = to_d<T>(G[(long)i * n + j]); ss = fma(d, d, ss); }
        ss = block_sum(ss, red);
        if (threadIdx.x == 0) { part[4 * i] = ss; part[4 * i + 1] = 0.0; part[4 * i + 2] = 0.0; part[4 * i + 3] = 0.0; }
    }
}

// Same partials from 16-byte row vectors (n a multiple of 16 / sizeof(T)).
template <typename T>
__global__ void __launch_bounds__(256)
sumsq_rows_vec_kernel(int n, const T *__restrict__ G, double *__restrict__ part)
{
    __shared__ double red[32];
    constexpr int V = 16 / sizeof(T);
    const int nv = n / V;
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        const uint4 *Gi = reinterpret_cast<const uint4 *>(G + (long)i * n);
        double ss = 0.0;
        for (int j = threadIdx.x; j < nv; j += blockDim.x) {
            uint4 v = Gi[j];
            const T *g = reinterpret_cast<const T *>(&v);
#pragma unroll
            for (int t = 0; t < V; t++) { double d = to_d<T>(g[t]); ss = fma(d, d, ss); }
        }
        ss = block_sum(ss, red);
        if (threadIdx.x == 0) { part[4 * i] = ss; part[4 * i + 1] = 0.0; part[4 * i + 2] = 0.0; part[4 * i + 3] = 0.0; }
    }
}

// mu (Frobenius scaling, l.1139) from ||G||_F^2 (scal[SC_RED+0]), ||A_k||_F^2 (scal[SC_NA2]), e.
__global__ void mu_kernel(int scaling, double *scal)
{
    double e = scal[SC_EXP];
    double ng = sqrt(scal[SC_RED + 0]);
    double ninv = ldexp(ng, -(int)e);             // ||A_k^{-1}||_F = 2^{-e} ||G||_F
    double na = sqrt(scal[SC_NA2]);
    double mu = 1.0;
    if (scaling && na > 0.0 && ninv > 0.0 && isfinite(na) && isfinite(ninv)) mu = sqrt(ninv / na);
    scal[SC_MU] = mu;
}

// Determinantal scaling mu_k = |det A_k|^{-1/n}: the inversion leaves
// log|u_jj| summed per panel in ldet (zeros elsewhere); W = 2^{-e} A_k was inverted, so
// log|det A_k| = log|det W| + n e ln 2.  One CTA, fixed reduction order.
__global__ void __launch_bounds__(256) mu_det_kernel(int n, int scaling, const double *__restrict__ ldet, double *scal)
{
    __shared__ double red[32];
    double t = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) t += ldet[i];
    t = block_sum(t, red);
    if (threadIdx.x == 0) {
        const double e = scal[SC_EXP];
        const double ld = t + (double)n * e * 0.69314718055994530942;
        double mu = 1.0;
        if (scaling && isfinite(ld)) mu = exp(-ld / (double)n);
        if (!(mu > 0.0) || !isfinite(mu)) mu = 1.0;
        scal[SC_MU] = mu;
    }
}

// A_{k+1} = 0.5 (mu A_k + mu^{-1} A_k^{-1}),  A_k^{-1}[i][j] = 2^{-e} G[i][invperm[j]].
template <typename T>
__global__ void __launch_bounds__(256)
newton_update_kernel(int n, const T *__restrict__ Ak, const T *__restrict__ G, const int *__restrict__ invperm,
                     T *__restrict__ Anext, T *__restrict__ Ainv, const double *__restrict__ scal,
                     double *__restrict__ part)
{
    __shared__ double red[32];
    using Acc = typename Prec<T>::acc;
    const double mu = scal[SC_MU];
    const int e = (int)scal[SC_EXP];
    const Acc a = (Acc)mu, b = (Acc)(1.0 / mu);
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        double dd = 0.0, ss = 0.0, rs = 0.0, mx = 0.0;
        for (int j = threadIdx.x; j < n; j += blockDim.x) {
            T gi;
            if constexpr (sizeof(T) == 8) gi = ldexp(G[(long)i * n + invperm[j]], -e);
            else gi = from_f<T>(ldexpf(to_f<T>(G[(long)i * n + invperm[j]]), -e));
            if (Ainv) Ainv[(long)i * n + j] = gi;
            Acc x = to_acc<T>(Ak[(long)i * n + j]);
            Acc y = to_acc<T>(gi);
            T nv = from_acc<T>(Acc(0.5) * fma(a, x, b * y));
            Anext[(long)i * n + j] = nv;
            double nd = to_d<T>(nv), xd = (double)x;
            dd = fma(nd - xd, nd - xd, dd);
            ss = fma(nd, nd, ss);
            rs += fabs(nd + (i == j ? 1.0 : 0.0));
            mx = fmax(mx, fabs(nd));
            if (!isfinite(nd)) mx = INFINITY;
        }
        dd = block_sum(dd, red); ss = block_sum(ss, red);
        rs = block_sum(rs, red); mx = block_max(mx, red);
        if (threadIdx.x == 0) { part[4 * i] = dd; part[4 * i + 1] = ss; part[4 * i + 2] = rs; part[4 * i + 3] = mx; }
    }
}

// The same update, HBM-streaming form: row i of G (the column-permuted inverse) is staged
// in shared memory with 16-byte loads, so the invperm gather hits shared memory instead of
// scattered 32-byte sectors; A_k is read and A_{k+1}, A_k^{-1} are written as 16-byte
// vectors (V = 16 / sizeof(T) elements per thread per pass).  Per-element arithmetic is
// the kernel's above; only the order of the fp64 row partials differs.  Algorithmic
// traffic per row: read A_k, G (2 n sizeof(T)), write A_{k+1}, A_k^{-1} (2 n sizeof(T)).
// (Measured slower at n = 16384: a cp.async double-buffered G row, 2.5 vs 3.2 TB/s, the
// second buffer costing a resident CTA per SM; __launch_bounds__(256, 5), 810 vs 673 us,
// register spills; a 100 % shared-memory carveout, 2.75 TB/s: the invperm reads lose L1;
// invperm staged once per CTA as 16-bit indices in shared memory, 3.0 vs 3.2 TB/s: the
// extra 32 KB costs a resident CTA.)
template <typename T>
__global__ void __launch_bounds__(256)
newton_update_row_kernel(int n, const T *__restrict__ Ak, const T *__restrict__ G, const int *__restrict__ invperm,
                         T *__restrict__ Anext, T *__restrict__ Ainv, const double *__restrict__ scal,
                         double *__restrict__ part)
{
    extern __shared__ __align__(16) unsigned char nu_smem[];
    T *g = reinterpret_cast<T *>(nu_smem);
    __shared__ double red[32];
    constexpr int V = 16 / sizeof(T);
    using Acc = typename Prec<T>::acc;
    const double mu = scal[SC_MU];
    const int e = (int)scal[SC_EXP];
    const Acc a = (Acc)mu, b = (Acc)(1.0 / mu);
    const int nv = n / V;                       // caller guarantees n % V == 0
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        const uint4 *Gi = reinterpret_cast<const uint4 *>(G + (long)i * n);
        for (int j = threadIdx.x; j < nv; j += blockDim.x) reinterpret_cast<uint4 *>(g)[j] = __ldcs(Gi + j);
        __syncthreads();
        const uint4 *Ai = reinterpret_cast<const uint4 *>(Ak + (long)i * n);
        uint4 *Ni = reinterpret_cast<uint4 *>(Anext + (long)i * n);
        uint4 *Ii = Ainv ? reinterpret_cast<uint4 *>(Ainv + (long)i * n) : nullptr;
        double dd = 0.0, ss = 0.0, rs = 0.0, mx = 0.0;
        constexpr bool half_t = sizeof(T) == 2;
        const float scf = ldexpf(1.0f, -e);           // 2^-e: x * 2^-e rounds exactly as ldexp does
        const double scd = ldexp(1.0, -e);
        for (int jv = threadIdx.x; jv < nv; jv += blockDim.x) {
            uint4 av = __ldcs(Ai + jv), iv, nw;
            const T *ae = reinterpret_cast<const T *>(&av);
            T *ie = reinterpret_cast<T *>(&iv), *ne = reinterpret_cast<T *>(&nw);
            // 16-bit types: the row partials of the V = 8 elements of this vector in fp32
            // (squares of 11-bit significands and their differences are exact or rounded once),
            // then added to the fp64 accumulators -- fp64 work per vector, not per element
            float ddf = 0.f, ssf = 0.f, rsf = 0.f, mxf = 0.f;
#pragma unroll
            for (int t = 0; t < V; t++) {
                const int j = jv * V + t;
                T gi;
                if constexpr (sizeof(T) == 8) gi = g[invperm[j]] * scd;
                else gi = from_f<T>(to_f<T>(g[invperm[j]]) * scf);
                ie[t] = gi;
                Acc x = to_acc<T>(ae[t]);
                Acc y = to_acc<T>(gi);
                T nvt = from_acc<T>(Acc(0.5) * fma(a, x, b * y));
                ne[t] = nvt;
                if constexpr (half_t) {
                    const float nd = to_f<T>(nvt), df = nd - (float)x;
                    ddf = fmaf(df, df, ddf);
                    ssf = fmaf(nd, nd, ssf);
                    rsf += fabsf(nd + (i == j ? 1.0f : 0.0f));
                    mxf = fmaxf(mxf, fabsf(nd));
                    if (!isfinite(nd)) mxf = INFINITY;
                } else {
                    double nd = to_d<T>(nvt), xd = (double)x;
                    dd = fma(nd - xd, nd - xd, dd);
                    ss = fma(nd, nd, ss);
                    rs += fabs(nd + (i == j ? 1.0 : 0.0));
                    mx = fmax(mx, fabs(nd));
                    if (!isfinite(nd)) mx = INFINITY;
                }
            }
            if constexpr (half_t) {
                dd += (double)ddf; ss += (double)ssf; rs += (double)rsf;
                mx = fmax(mx, (double)mxf);
            }
            if (Ii) Ii[jv] = iv;
            Ni[jv] = nw;
        }
        dd = block_sum(dd, red); ss = block_sum(ss, red);     // block_sum's barriers also
        rs = block_sum(rs, red); mx = block_max(mx, red);     // free g for the next row
        if (threadIdx.x == 0) { part[4 * i] = dd; part[4 * i + 1] = ss; part[4 * i + 2] = rs; part[4 * i + 3] = mx; }
    }
}

// The update as a persistent streaming kernel (round 2): one CTA per SM pair slot, rows
// grid-strided.  invperm is staged ONCE per CTA as 16-bit indices; row i of G arrives by a
// 1-D bulk async copy (cp.async.bulk, mbarrier completion) into one of two shared
// buffers, the copy of row i + 2 grid being issued as soon as row i's buffer is free, so
// the G stream never waits on the SM; the A_k row is loaded with all of a thread's
// 16-byte vectors in flight before the wait.  Row partials: the sums ||A_{k+1} - A_k||_F^2
// and ||A_{k+1}||_F^2 stay in per-thread registers across rows; the row abs-sum (for
// ||A_{k+1} + I||_inf) is reduced per row through one parity-buffered warp slot and the
// one barrier per row that also frees the G buffer.  part[4 b + 0..3] holds CTA b's
// (sum dd, sum ss, max row sum, max |x|), reduced by reduce_rows_kernel over the grid.
// Per-element arithmetic is newton_update_kernel's.  Traffic: A_k, G in, A_{k+1} out.
template <typename T, int NT, int U>
__global__ void __launch_bounds__(NT, 2)
newton_update_stream_kernel(int n, const T *__restrict__ Ak, const T *__restrict__ G,
                            const int *__restrict__ invperm, T *__restrict__ Anext,
                            const double *__restrict__ scal, double *__restrict__ part)
{
    extern __shared__ __align__(128) unsigned char nus_smem[];
    constexpr int NW = NT / 32;
    constexpr int V = 16 / sizeof(T);
    using Acc = typename Prec<T>::acc;
    uint64_t *mbar = reinterpret_cast<uint64_t *>(nus_smem);
    T *const gbuf0 = reinterpret_cast<T *>(nus_smem + 128);
    uint16_t *ip = reinterpret_cast<uint16_t *>(gbuf0 + 2 * (long)n);
    __shared__ double wred[2][NW];
    __shared__ double red[32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int grid = gridDim.x, nv = n / V;
    const uint32_t rowbytes = (uint32_t)n * sizeof(T);
    const double mu = scal[SC_MU];
    const int e = (int)scal[SC_EXP];
    const Acc a = (Acc)mu, b = (Acc)(1.0 / mu);
    const float scf = ldexpf(1.0f, -e);
    const double scd = ldexp(1.0, -e);
    if (tid == 0) {
        ptx::mbar_init(&mbar[0], 1);
        ptx::mbar_init(&mbar[1], 1);
        ptx::fence_mbar_init();
        for (int t = 0; t < 2; t++) {
            const int i = blockIdx.x + t * grid;
            if (i < n) {
                ptx::mbar_arrive_expect_tx(&mbar[t], rowbytes);
                ptx::bulk_g2s(gbuf0 + (long)t * n, G + (long)i * n, rowbytes, &mbar[t]);
            }
        }
    }
    for (int j = tid; j < n; j += NT) ip[j] = (uint16_t)invperm[j];
    __syncthreads();
    double dd = 0.0, ss = 0.0, mx = 0.0, rsmax = 0.0;
    int t = 0;
    for (int i = blockIdx.x; i < n; i += grid, t++) {
        const int bsel = t & 1;
        const uint32_t parity = (uint32_t)(t >> 1) & 1u;
        const uint4 *Ai = reinterpret_cast<const uint4 *>(Ak + (long)i * n);
        uint4 *Ni = reinterpret_cast<uint4 *>(Anext + (long)i * n);
        const T *g = gbuf0 + (long)bsel * n;
        double rs = 0.0;
        for (int base = 0; base < nv; base += NT * U) {
            uint4 av[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int jv = base + u * NT + tid;
                if (jv < nv) av[u] = __ldcs(Ai + jv);
            }
            if (base == 0) ptx::mbar_wait(&mbar[bsel], parity);
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int jv = base + u * NT + tid;
                if (jv >= nv) continue;
                const T *ae = reinterpret_cast<const T *>(&av[u]);
                uint4 nw;
                T *ne = reinterpret_cast<T *>(&nw);
                uint16_t idx[V];
                if constexpr (V == 8) {
                    const uint4 iv = reinterpret_cast<const uint4 *>(ip)[jv];
                    const uint32_t w4[4] = {iv.x, iv.y, iv.z, iv.w};
#pragma unroll
                    for (int q = 0; q < 4; q++) { idx[2 * q] = (uint16_t)(w4[q] & 0xFFFFu); idx[2 * q + 1] = (uint16_t)(w4[q] >> 16); }
                } else if constexpr (V == 4) {
                    const uint2 iv = reinterpret_cast<const uint2 *>(ip)[jv];
                    idx[0] = (uint16_t)(iv.x & 0xFFFFu); idx[1] = (uint16_t)(iv.x >> 16);
                    idx[2] = (uint16_t)(iv.y & 0xFFFFu); idx[3] = (uint16_t)(iv.y >> 16);
                } else {
                    const uint32_t iv = reinterpret_cast<const uint32_t *>(ip)[jv];
                    idx[0] = (uint16_t)(iv & 0xFFFFu); idx[1] = (uint16_t)(iv >> 16);
                }
                float ddf = 0.f, ssf = 0.f, rsf = 0.f, mxf = 0.f;
#pragma unroll
                for (int q = 0; q < V; q++) {
                    const int j = jv * V + q;
                    T gi;
                    if constexpr (sizeof(T) == 8) gi = g[idx[q]] * scd;
                    else gi = from_f<T>(to_f<T>(g[idx[q]]) * scf);
                    const Acc x = to_acc<T>(ae[q]);
                    const Acc y = to_acc<T>(gi);
                    const T nvt = from_acc<T>(Acc(0.5) * fma(a, x, b * y));
                    ne[q] = nvt;
                    if constexpr (sizeof(T) == 2) {
                        const float nd = to_f<T>(nvt), df = nd - (float)x;
                        ddf = fmaf(df, df, ddf);
                        ssf = fmaf(nd, nd, ssf);
                        rsf += fabsf(nd + (i == j ? 1.0f : 0.0f));
                        mxf = fmaxf(mxf, fabsf(nd));
                        if (!isfinite(nd)) mxf = INFINITY;
                    } else {
                        const double nd = to_d<T>(nvt), xd = (double)x;
                        dd = fma(nd - xd, nd - xd, dd);
                        ss = fma(nd, nd, ss);
                        rs += fabs(nd + (i == j ? 1.0 : 0.0));
                        mx = fmax(mx, fabs(nd));
                        if (!isfinite(nd)) mx = INFINITY;
                    }
                }
                if constexpr (sizeof(T) == 2) {
                    dd += (double)ddf; ss += (double)ssf; rs += (double)rsf;
                    mx = fmax(mx, (double)mxf);
                }
                __stcs(Ni + jv, nw);
            }
        }
        rs = warp_sum(rs);
        if (lane == 0) wred[bsel][wid] = rs;
        __syncthreads();                       // G buffer bsel free, wred[bsel] complete
        if (tid == 0) {
            double r = 0.0;
#pragma unroll
            for (int w = 0; w < NW; w++) r += wred[bsel][w];
            rsmax = fmax(rsmax, r);
            const int inext = i + 2 * grid;
            if (inext < n) {
                ptx::mbar_arrive_expect_tx(&mbar[bsel], rowbytes);
                ptx::bulk_g2s(gbuf0 + (long)bsel * n, G + (long)inext * n, rowbytes, &mbar[bsel]);
            }
        }
    }
    dd = block_sum(dd, red);
    ss = block_sum(ss, red);
    mx = block_max(mx, red);
    if (tid == 0) {
        part[4 * blockIdx.x] = dd; part[4 * blockIdx.x + 1] = ss;
        part[4 * blockIdx.x + 2] = rsmax; part[4 * blockIdx.x + 3] = mx;
    }
}

// ------------------------------------------------------------ Z side
// Zt (n x m, T) = round(2^{-e} L) with e = exponent of max|L| (computed here, one CTA).
// grid-wide max|x| as the bit pattern of a non-negative double (integer order = value
// order), accumulated with atomicMax into a zeroed slot
__global__ void absmax_bits_kernel(long len, const double *__restrict__ x, unsigned long long *__restrict__ out)
{
    __shared__ double red[32];
    double mx = 0.0;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < len; i += (long)gridDim.x * blockDim.x)
        mx = fmax(mx, fabs(x[i]));
    mx = block_max(mx, red);
    if (threadIdx.x == 0) atomicMax(out, (unsigned long long)__double_as_longlong(mx));
}

__device__ __forceinline__ int exp_of_max(const double *scal) {
    const double mx = __longlong_as_double((long long)reinterpret_cast<const unsigned long long *>(scal)[SC_MAXB]);
    int e = 0;
    if (mx > 0.0 && isfinite(mx)) frexp(mx, &e);
    return e;
}

// Zt = 2^{-e} L rounded to T, e = exponent of max|L| (grid-wide, after absmax_bits_kernel)
template <typename T>
__global__ void load_factor_kernel(long len, const double *__restrict__ L, T *__restrict__ Zt, double *__restrict__ scal,
                                   int slot)
{
    const int e = exp_of_max(scal);
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < len; i += (long)gridDim.x * blockDim.x)
        Zt[i] = from_d<T>(ldexp(L[i], -e));
    if (blockIdx.x == 0 && threadIdx.x == 0) scal[slot] = (double)e;
}

// Y (m x m fp64) = round_us(2^{-e} S), e = exponent of max|S| (grid-wide)
__global__ void load_inner_kernel(int m, const double *__restrict__ S, double *__restrict__ Y, int ldy,
                                  int prec, double *__restrict__ scal, int slot)
{
    const int e = exp_of_max(scal);
    const long tot = (long)m * m;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < tot; idx += (long)gridDim.x * blockDim.x) {
        const int i = (int)(idx % m), j = (int)(idx / m);
        Y[i + (long)j * ldy] = round_to(ldexp(S[idx], -e), prec);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) scal[slot] = (double)e;
}

// Ynew (2c x 2c, ld ldn) = blkdiag(round(a Y), round(b Y)) with a = mu/2, b = 1/(2 mu).
__global__ void y_blkdiag_kernel(int c, const double *__restrict__ Y, int ldy, double *__restrict__ Yn, int ldn,
                                 double a, double b, int prec)
{
    long tot = (long)4 * c * c;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < tot; idx += (long)gridDim.x * blockDim.x) {
        int i = (int)(idx % (2 * c)), j = (int)(idx / (2 * c));
        double v = 0.0;
        if (i < c && j < c) v = round_to(a * Y[i + (long)j * ldy], prec);
        else if (i >= c && j >= c) v = round_to(b * Y[(i - c) + (long)(j - c) * ldy], prec);
        Yn[i + (long)j * ldn] = v;
    }
}

// Cholesky Z-side: Z[:, 0:c] *= a, Z[:, c:2c] *= b (rounded to T).
template <typename T>
__global__ void chol_scale_kernel(long nc, T *__restrict__ Z, float a, float b)
{
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < 2 * nc; idx += (long)gridDim.x * blockDim.x) {
        float f = (idx < nc) ? a : b;
        Z[idx] = from_f<T>(to_f<T>(Z[idx]) * f);
    }
}
template <>
__global__ void chol_scale_kernel<double>(long nc, double *__restrict__ Z, float a, float b) {}

__global__ void chol_scale_kernel_d(long nc, double *__restrict__ Z, double a, double b)
{
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < 2 * nc; idx += (long)gridDim.x * blockDim.x)
        Z[idx] *= (idx < nc) ? a : b;
}

template <typename T>
__global__ void to_f64_kernel(long len, const T *__restrict__ x, double *__restrict__ y, double f)
{
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < len; i += (long)gridDim.x * blockDim.x)
        y[i] = to_d<T>(x[i]) * f;
}
template <typename T>
__global__ void from_f64_kernel(long len, const double *__restrict__ x, T *__restrict__ y)
{
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < len; i += (long)gridDim.x * blockDim.x)
        y[i] = from_d<T>(x[i]);
}
// Z_final = round_T(Z * s1) * 2^{e}  (Cholesky: s1 = 1/sqrt(2); LDL^T: s1 = 1)
template <typename T>
__global__ void finish_factor_kernel(long len, const T *__restrict__ x, double *__restrict__ y, double s1,
                                     const double *__restrict__ scal, int slot)
{
    int e = (int)scal[slot];
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < len; i += (long)gridDim.x * blockDim.x) {
        double v = to_d<T>(x[i]);
        if (s1 != 1.0) v = to_d<T>(from_d<T>(v * s1));
        y[i] = ldexp(v, e);
    }
}

// ------------------------------------------------------------ selection
// mode 0: |w| >= thr ; 1: |w| > thr ; 2: w >= thr ; 3: w <= -thr.  thr = rel * max|w|.
// idx[0..cnt) in order; cnt written to *cnt (device).  One CTA.
__global__ void __launch_bounds__(1024)
select_kernel(int k, const double *__restrict__ w, double rel, int mode, int *__restrict__ idx, int *__restrict__ cnt)
{
    __shared__ double red[32];
    __shared__ int wc[32];
    double mx = 0.0;
    for (int i = threadIdx.x; i < k; i += blockDim.x) mx = fmax(mx, fabs(w[i]));
    mx = block_max(mx, red);
    const double thr = rel * mx;
    int base = 0;
    for (int i0 = 0; i0 < k; i0 += blockDim.x) {
        int i = i0 + threadIdx.x;
        bool keep = false;
        if (i < k) {
            double v = w[i];
            keep = (mode == 0) ? fabs(v) >= thr : (mode == 1) ? fabs(v) > thr : (mode == 2) ? v >= thr : v <= -thr;
            if (mx == 0.0) keep = false;
        }
        unsigned bal = __ballot_sync(0xffffffffu, keep);
        int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        if (lane == 0) wc[wid] = __popc(bal);
        __syncthreads();
        int off = base;
        for (int q = 0; q < wid; q++) off += wc[q];
        if (keep) idx[off + __popc(bal & ((1u << lane) - 1u))] = i;
        int tot = 0;
        for (int q = 0; q < (int)(blockDim.x >> 5); q++) tot += wc[q];
        base += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) *cnt = base;
}

// out[:, t] = V[:, idx[t]] * f(w[idx[t]]) ; fmode 0: 1, 1: sqrt(w), 2: sqrt(-w)
__global__ void gather_cols_kernel(int rows, int cnt, const double *__restrict__ V, int ldv, const int *__restrict__ idx,
                                   const double *__restrict__ w, int fmode, double *__restrict__ out, int ldo)
{
    long tot = (long)rows * cnt;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < tot; e += (long)gridDim.x * blockDim.x) {
        int i = (int)(e % rows), t = (int)(e / rows);
        int c = idx[t];
        double f = 1.0;
        if (fmode == 1) f = sqrt(w[c]);
        else if (fmode == 2) f = sqrt(-w[c]);
        out[i + (long)t * ldo] = V[i + (long)c * ldv] * f;
    }
}

// Y (cnt x cnt) = diag(round_prec(w[idx[t]])), zero elsewhere.
__global__ void diag_from_sel_kernel(int cnt, const double *__restrict__ w, const int *__restrict__ idx, int prec,
                                     double *__restrict__ Y, int ldy)
{
    long tot = (long)cnt * cnt;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < tot; e += (long)gridDim.x * blockDim.x) {
        int i = (int)(e % cnt), j = (int)(e / cnt);
        Y[i + (long)j * ldy] = (i == j) ? round_to(w[idx[i]], prec) : 0.0;
    }
}

__global__ void round_array_kernel(long len, double *__restrict__ x, int prec)
{
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < len; i += (long)gridDim.x * blockDim.x)
        x[i] = round_to(x[i], prec);
}

// copy a (rows x cols, ld lda) block into b (ld ldb), optional scale
__global__ void copy_block_kernel(int rows, int cols, const double *__restrict__ a, int lda, double *__restrict__ b,
                                  int ldb, double f)
{
    long tot = (long)rows * cols;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < tot; e += (long)gridDim.x * blockDim.x) {
        int i = (int)(e % rows), j = (int)(e / rows);
        b[i + (long)j * ldb] = f * a[i + (long)j * lda];
    }
}

__global__ void zero_kernel(long len, double *__restrict__ x)
{
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < len; i += (long)gridDim.x * blockDim.x) x[i] = 0.0;
}

// N = [0 Y 0; Y 0 0; 0 0 S] (p x p, p = 2c+m) or P (Y = I, S = I) when Y == nullptr.
__global__ void build_N_kernel(int c, int m, const double *__restrict__ Y, int ldy, const double *__restrict__ S,
                               double *__restrict__ N)
{
    const int p = 2 * c + m;
    long tot = (long)p * p;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < tot; e += (long)gridDim.x * blockDim.x) {
        int i = (int)(e % p), j = (int)(e / p);
        double v = 0.0;
        if (i < c && j >= c && j < 2 * c) v = Y ? Y[i + (long)(j - c) * ldy] : (i == j - c ? 1.0 : 0.0);
        else if (i >= c && i < 2 * c && j < c) v = Y ? Y[(i - c) + (long)j * ldy] : (i - c == j ? 1.0 : 0.0);
        else if (i >= 2 * c && j >= 2 * c) v = S ? S[(i - 2 * c) + (long)(j - 2 * c) * m] : (i == j ? 1.0 : 0.0);
        N[e] = v;
    }
}

// Ups = blkdiag(Y (c x c), Yd (cd x cd)) or signature J = blkdiag(I_c, I_cp, -I_cm) when Y == nullptr
__global__ void build_blkdiag_kernel(int c, int cd, const double *__restrict__ Y, int ldy, const double *__restrict__ Yd,
                                     int ldyd, int cp, double *__restrict__ U)
{
    const int p = c + cd;
    long tot = (long)p * p;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < tot; e += (long)gridDim.x * blockDim.x) {
        int i = (int)(e % p), j = (int)(e / p);
        double v = 0.0;
        if (Y) {
            if (i < c && j < c) v = Y[i + (long)j * ldy];
            else if (i >= c && j >= c) v = Yd[(i - c) + (long)(j - c) * ldyd];
        } else if (i == j) {
            v = (i < c + cp) ? 1.0 : -1.0;
        }
        U[e] = v;
    }
}

// trace(M) for the Frobenius norms of implied products, sum_i sum_j P_ij P_ji
__global__ void __launch_bounds__(1024)
trace_prod_kernel(int k, const double *__restrict__ P, double *__restrict__ out)
{
    __shared__ double red[32];
    double s = 0.0;
    for (long e = threadIdx.x; e < (long)k * k; e += blockDim.x) {
        int i = (int)(e % k), j = (int)(e / k);
        s = fma(P[e], P[j + (long)i * k], s);
    }
    s = block_sum(s, red);
    if (threadIdx.x == 0) *out = s;
}

// ------------------------------------------------------------ launchers
static inline int grid_for(long n, int bs = 256, int cap = 4096) { int g = ceil_div(n, bs); return g < 1 ? 1 : (g > cap ? cap : g); }

#define DISPATCH_T(prec, F, ...)                                        \
    switch (prec) {                                                     \
        case LYAP_FP64: F<double>(__VA_ARGS__); break;                  \
        case LYAP_FP32: F<float>(__VA_ARGS__); break;                   \
        case LYAP_FP16: F<__half>(__VA_ARGS__); break;                  \
        case LYAP_BF16: F<__nv_bfloat16>(__VA_ARGS__); break;           \
        default: return LYAP_ERR_ARG;                                   \
    }

template <typename T> static void k_cast(cudaStream_t s, int n, const double *A, void *Ak, double *part)
{
    // caller-owned A: the vector form needs 16-byte aligned rows
    if (n % (16 / (int)sizeof(T)) == 0 && reinterpret_cast<uintptr_t>(A) % 16 == 0) {
        cast_vec_kernel<T><<<n < 148 * 8 ? n : 148 * 8, 256, 0, s>>>(n, A, (T *)Ak, part);
        return;
    }
    cast_kernel<T><<<n < 4096 ? n : 4096, 256, 0, s>>>(n, A, (T *)Ak, part);
}
int nk_cast(cudaStream_t s, int prec, int n, const double *A, void *Ak, double *part, double *out)
{
    DISPATCH_T(prec, k_cast, s, n, A, Ak, part);
    LYAP_TRY(launched());
    reduce_rows_kernel<<<1, 1024, 0, s>>>(n, part, out);
    return launched();
}

template <typename T> static void k_scale(cudaStream_t s, long nn, const void *Ak, void *W, double *scal)
{
    constexpr int V = 16 / sizeof(T);
    if (nn % V == 0) {
        scale_vec_kernel<T><<<grid_for(nn / V, 256, 148 * 8), 256, 0, s>>>(nn / V, (const uint4 *)Ak, (uint4 *)W, scal);
        return;
    }
    scale_kernel<T><<<grid_for(nn), 256, 0, s>>>(nn, (const T *)Ak, (T *)W, scal);
}
int nk_scale(cudaStream_t s, int prec, long nn, const void *Ak, void *W, double *scal)
{
    DISPATCH_T(prec, k_scale, s, nn, Ak, W, scal);
    return launched();
}

template <typename T> static void k_sumsq(cudaStream_t s, int n, const void *G, double *part)
{
    if (n % (16 / (int)sizeof(T)) == 0) {
        sumsq_rows_vec_kernel<T><<<n < 148 * 8 ? n : 148 * 8, 256, 0, s>>>(n, (const T *)G, part);
        return;
    }
    sumsq_rows_kernel<T><<<n < 4096 ? n : 4096, 256, 0, s>>>(n, (const T *)G, part);
}
int nk_mu(cudaStream_t s, int prec, int n, const void *G, double *part, double *scal, int scaling)
{
    DISPATCH_T(prec, k_sumsq, s, n, G, part);
    LYAP_TRY(launched());
    reduce_rows_kernel<<<1, 1024, 0, s>>>(n, part, scal + SC_RED);
    LYAP_TRY(launched());
    mu_kernel<<<1, 1, 0, s>>>(scaling, scal);
    return launched();
}

// Z' (n x c, column-major) = rows of Z in the Gauss-Jordan pivot order: Z'[t] = Z[rowperm[t]],
// so that A_k^{-1} Z = 2^{-e} G Z' with the cached, column-permuted G (Section 3.4 cache).
template <typename T>
__global__ void row_gather_kernel(int n, long len, const T *__restrict__ Z, const int *__restrict__ rowperm,
                                  T *__restrict__ out)
{
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < len; idx += (long)gridDim.x * blockDim.x) {
        const long col = idx / n;
        const int t = (int)(idx - col * n);
        out[idx] = Z[col * n + rowperm[t]];
    }
}
template <typename T> static void k_row_gather(cudaStream_t s, int n, int c, const void *Z, const int *rp, void *out)
{
    const long len = (long)n * c;
    row_gather_kernel<T><<<grid_for(len), 256, 0, s>>>(n, len, (const T *)Z, rp, (T *)out);
}
int nk_row_gather(cudaStream_t s, int prec, int n, int c, const void *Z, const int *rowperm, void *out)
{
    if ((long)n * c <= 0) return LYAP_OK;
    DISPATCH_T(prec, k_row_gather, s, n, c, Z, rowperm, out);
    return launched();
}

// x <- 2^e x (exact power-of-two scaling in the element type)
template <typename T>
__global__ void ldexp_kernel(long len, T *__restrict__ x, int e)
{
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < len; i += (long)gridDim.x * blockDim.x) {
        if constexpr (sizeof(T) == 8) x[i] = ldexp(x[i], e);
        else x[i] = from_f<T>(ldexpf(to_f<T>(x[i]), e));
    }
}
template <typename T> static void k_ldexp(cudaStream_t s, long len, void *x, int e)
{
    ldexp_kernel<T><<<grid_for(len), 256, 0, s>>>(len, (T *)x, e);
}
int nk_ldexp(cudaStream_t s, int prec, long len, void *x, int e)
{
    DISPATCH_T(prec, k_ldexp, s, len, x, e);
    return launched();
}

int nk_mu_det(cudaStream_t s, int n, const double *ldet, double *scal, int scaling)
{
    mu_det_kernel<<<1, 256, 0, s>>>(n, scaling, ldet, scal);
    return launched();
}

// Launch forms of the update, by preference: the persistent streaming kernel (rows of
// 16-byte multiples, two G rows + 16-bit invperm in shared memory, n < 65536, no
// un-permuted copy requested); the row-staged kernel; the plain kernel.  Returns the
// number of partial rows written to part.
static constexpr int NU_SMEM_MAX = 96 * 1024;
static constexpr int NUS_NT = 512, NUS_U = 4;
static int sm_count() {
    static const int v = [] {
        int dev = 0, c = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev);
        return c;
    }();
    return v;
}
template <typename T> static int k_update(cudaStream_t s, int n, const void *Ak, const void *G, const int *ip,
                                          void *An, void *Ai, const double *scal, double *part)
{
    constexpr int V = 16 / (int)sizeof(T);
    const size_t smem_s = 128 + 2 * (size_t)n * sizeof(T) + 2 * (size_t)n;
    if (!Ai && n % V == 0 && n < 65536 && smem_s <= 200 * 1024 && !env_flag("LYAP_NU_ROW")) {
        static const bool attr = [] {
            cudaFuncSetAttribute(newton_update_stream_kernel<T, NUS_NT, NUS_U>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            return true;
        }();
        (void)attr;
        int per_sm = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, newton_update_stream_kernel<T, NUS_NT, NUS_U>, NUS_NT,
                                                      smem_s);
        per_sm = std::max(1, std::min(per_sm, 2));
        const int grid = std::min(n, sm_count() * per_sm);
        newton_update_stream_kernel<T, NUS_NT, NUS_U><<<grid, NUS_NT, smem_s, s>>>(
            n, (const T *)Ak, (const T *)G, ip, (T *)An, scal, part);
        return grid;
    }
    const size_t smem = (size_t)n * sizeof(T);
    if (n % V == 0 && smem <= (size_t)NU_SMEM_MAX) {
        static const bool attr = [] {
            cudaFuncSetAttribute(newton_update_row_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, NU_SMEM_MAX);
            return true;
        }();
        (void)attr;
        int per_sm = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, newton_update_row_kernel<T>, 256, smem);
        if (per_sm < 1) per_sm = 1;
        const int grid = n < sm_count() * per_sm ? n : sm_count() * per_sm;
        newton_update_row_kernel<T><<<grid, 256, smem, s>>>(n, (const T *)Ak, (const T *)G, ip, (T *)An, (T *)Ai,
                                                             scal, part);
        return n;
    }
    newton_update_kernel<T><<<n < 4096 ? n : 4096, 256, 0, s>>>(n, (const T *)Ak, (const T *)G, ip, (T *)An, (T *)Ai, scal, part);
    return n;
}
int nk_update(cudaStream_t s, int prec, int n, const void *Ak, const void *G, const int *invperm, void *Anext,
              void *Ainv, double *scal, double *part)
{
    int rows = n;
    {
        const double es = prec == LYAP_FP64 ? 8.0 : prec == LYAP_FP32 ? 4.0 : 2.0;
        // algorithmic bytes: A_k and G in, A_{k+1} out (+ the cached A_k^{-1} if requested)
        KTimer kt(KC_NEWTON_UPDATE, s, 0.0, (Ainv ? 4.0 : 3.0) * es * (double)n * n);
        switch (prec) {
            case LYAP_FP64: rows = k_update<double>(s, n, Ak, G, invperm, Anext, Ainv, scal, part); break;
            case LYAP_FP32: rows = k_update<float>(s, n, Ak, G, invperm, Anext, Ainv, scal, part); break;
            case LYAP_FP16: rows = k_update<__half>(s, n, Ak, G, invperm, Anext, Ainv, scal, part); break;
            case LYAP_BF16: rows = k_update<__nv_bfloat16>(s, n, Ak, G, invperm, Anext, Ainv, scal, part); break;
            default: return LYAP_ERR_ARG;
        }
    }
    LYAP_TRY(launched());
    reduce_rows_kernel<<<1, 1024, 0, s>>>(rows, part, scal + SC_RED);
    return launched();
}

template <typename T> static void k_loadf(cudaStream_t s, long len, const double *L, void *Zt, double *scal, int slot)
{ load_factor_kernel<T><<<grid_for(len), 256, 0, s>>>(len, L, (T *)Zt, scal, slot); }
static int absmax_bits(cudaStream_t s, long len, const double *x, double *scal)
{
    LYAP_CUDA_TRY(cudaMemsetAsync(scal + SC_MAXB, 0, sizeof(double), s));
    absmax_bits_kernel<<<grid_for(len), 256, 0, s>>>(len, x, reinterpret_cast<unsigned long long *>(scal) + SC_MAXB);
    return launched();
}
int nk_load_factor(cudaStream_t s, int prec, long len, const double *L, void *Zt, double *scal, int slot)
{
    LYAP_TRY(absmax_bits(s, len, L, scal));
    DISPATCH_T(prec, k_loadf, s, len, L, Zt, scal, slot);
    return launched();
}
int nk_load_inner(cudaStream_t s, int prec, int m, const double *S, double *Y, int ldy, double *scal, int slot)
{
    LYAP_TRY(absmax_bits(s, (long)m * m, S, scal));
    load_inner_kernel<<<grid_for((long)m * m), 256, 0, s>>>(m, S, Y, ldy, prec, scal, slot);
    return launched();
}
int nk_y_blkdiag(cudaStream_t s, int c, const double *Y, int ldy, double *Yn, int ldn, double a, double b, int prec)
{
    y_blkdiag_kernel<<<grid_for(4L * c * c), 256, 0, s>>>(c, Y, ldy, Yn, ldn, a, b, prec);
    return launched();
}
template <typename T> static void k_cs(cudaStream_t s, long nc, void *Z, double a, double b)
{
    if constexpr (sizeof(T) == 8) chol_scale_kernel_d<<<grid_for(2 * nc), 256, 0, s>>>(nc, (double *)Z, a, b);
    else chol_scale_kernel<T><<<grid_for(2 * nc), 256, 0, s>>>(nc, (T *)Z, (float)a, (float)b);
}
int nk_chol_scale(cudaStream_t s, int prec, long nc, void *Z, double a, double b)
{
    DISPATCH_T(prec, k_cs, s, nc, Z, a, b);
    return launched();
}
template <typename T> static void k_tof64(cudaStream_t s, long len, const void *x, double *y, double f)
{ to_f64_kernel<T><<<grid_for(len), 256, 0, s>>>(len, (const T *)x, y, f); }
int nk_to_f64(cudaStream_t s, int prec, long len, const void *x, double *y, double f)
{
    DISPATCH_T(prec, k_tof64, s, len, x, y, f);
    return launched();
}
template <typename T> static void k_fromf64(cudaStream_t s, long len, const double *x, void *y)
{ from_f64_kernel<T><<<grid_for(len), 256, 0, s>>>(len, x, (T *)y); }
int nk_from_f64(cudaStream_t s, int prec, long len, const double *x, void *y)
{
    DISPATCH_T(prec, k_fromf64, s, len, x, y);
    return launched();
}
template <typename T> static void k_finish(cudaStream_t s, long len, const void *x, double *y, double s1, const double *scal, int slot)
{ finish_factor_kernel<T><<<grid_for(len), 256, 0, s>>>(len, (const T *)x, y, s1, scal, slot); }
int nk_finish_factor(cudaStream_t s, int prec, long len, const void *x, double *y, double s1, const double *scal, int slot)
{
    DISPATCH_T(prec, k_finish, s, len, x, y, s1, scal, slot);
    return launched();
}
int nk_select(cudaStream_t s, int k, const double *w, double rel, int mode, int *idx, int *cnt)
{
    select_kernel<<<1, 1024, 0, s>>>(k, w, rel, mode, idx, cnt);
    return launched();
}
int nk_gather_cols(cudaStream_t s, int rows, int cnt, const double *V, int ldv, const int *idx, const double *w,
                   int fmode, double *out, int ldo)
{
    if (rows <= 0 || cnt <= 0) return LYAP_OK;
    gather_cols_kernel<<<grid_for((long)rows * cnt), 256, 0, s>>>(rows, cnt, V, ldv, idx, w, fmode, out, ldo);
    return launched();
}
int nk_diag_from_sel(cudaStream_t s, int cnt, const double *w, const int *idx, int prec, double *Y, int ldy)
{
    if (cnt <= 0) return LYAP_OK;
    diag_from_sel_kernel<<<grid_for((long)cnt * cnt), 256, 0, s>>>(cnt, w, idx, prec, Y, ldy);
    return launched();
}
int nk_round(cudaStream_t s, long len, double *x, int prec)
{
    if (prec == LYAP_FP64 || len <= 0) return LYAP_OK;
    round_array_kernel<<<grid_for(len), 256, 0, s>>>(len, x, prec);
    return launched();
}
int nk_copy_block(cudaStream_t s, int rows, int cols, const double *a, int lda, double *b, int ldb, double f)
{
    if (rows <= 0 || cols <= 0) return LYAP_OK;
    copy_block_kernel<<<grid_for((long)rows * cols), 256, 0, s>>>(rows, cols, a, lda, b, ldb, f);
    return launched();
}
int nk_zero(cudaStream_t s, long len, double *x)
{
    if (len <= 0) return LYAP_OK;
    zero_kernel<<<grid_for(len), 256, 0, s>>>(len, x);
    return launched();
}
// H <- H + H^T in place (k x k, ld ldh): each unordered pair {i, j} by the thread of (i <= j)
__global__ void sym_add_kernel(int k, double *__restrict__ H, int ldh)
{
    const long tot = (long)k * k;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < tot; e += (long)gridDim.x * blockDim.x) {
        const int i = (int)(e % k), j = (int)(e / k);
        if (i > j) continue;
        const double v = H[i + (long)j * ldh] + H[j + (long)i * ldh];
        H[i + (long)j * ldh] = v;
        H[j + (long)i * ldh] = v;
    }
}
// out[:, j] = T[:, j] * D[j][j]  (k x c; D with leading dimension ldd)
__global__ void scale_cols_kernel(int k, int c, const double *__restrict__ T, int ldt, const double *__restrict__ D,
                                  int ldd, double *__restrict__ out, int ldo)
{
    const long tot = (long)k * c;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < tot; e += (long)gridDim.x * blockDim.x) {
        const int i = (int)(e % k), j = (int)(e / k);
        out[i + (long)j * ldo] = T[i + (long)j * ldt] * D[j + (long)j * ldd];
    }
}
int nk_sym_add(cudaStream_t s, int k, double *H, int ldh)
{
    sym_add_kernel<<<grid_for((long)k * k), 256, 0, s>>>(k, H, ldh);
    return launched();
}
int nk_scale_cols(cudaStream_t s, int k, int c, const double *T, int ldt, const double *D, int ldd, double *out, int ldo)
{
    scale_cols_kernel<<<grid_for((long)k * c), 256, 0, s>>>(k, c, T, ldt, D, ldd, out, ldo);
    return launched();
}

int nk_build_N(cudaStream_t s, int c, int m, const double *Y, int ldy, const double *S, double *N)
{
    long p = 2L * c + m;
    build_N_kernel<<<grid_for(p * p), 256, 0, s>>>(c, m, Y, ldy, S, N);
    return launched();
}
int nk_build_blkdiag(cudaStream_t s, int c, int cd, const double *Y, int ldy, const double *Yd, int ldyd, int cp, double *U)
{
    long p = (long)c + cd;
    build_blkdiag_kernel<<<grid_for(p * p), 256, 0, s>>>(c, cd, Y, ldy, Yd, ldyd, cp, U);
    return launched();
}
__global__ void __launch_bounds__(1024)
sumsq_vec_kernel(long len, const double *__restrict__ x, double *__restrict__ out)
{
    __shared__ double red[32];
    double s = 0.0;
    for (long i = threadIdx.x; i < len; i += blockDim.x) s = fma(x[i], x[i], s);
    s = block_sum(s, red);
    if (threadIdx.x == 0) *out = s;
}
int nk_sumsq(cudaStream_t s, long len, const double *x, double *out)
{
    sumsq_vec_kernel<<<1, 1024, 0, s>>>(len, x, out);
    return launched();
}

__global__ void __launch_bounds__(1024)
diag_range_kernel(int k, const double *__restrict__ R, int ldr, double *__restrict__ out)
{
    __shared__ double red[32];
    double mx = 0.0, mn = INFINITY;
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
        double v = fabs(R[i + (long)i * ldr]);
        mx = fmax(mx, v);
        mn = fmin(mn, v);
    }
    mx = block_max(mx, red);
    mn = -block_max(-mn, red);
    if (threadIdx.x == 0) { out[0] = mn; out[1] = mx; }
}
int nk_diag_range(cudaStream_t s, int k, const double *R, int ldr, double *out)
{
    diag_range_kernel<<<1, 1024, 0, s>>>(k, R, ldr, out);
    return launched();
}

__global__ void axpy_kernel(long len, double a, const double *__restrict__ x, double *__restrict__ y)
{
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < len; i += (long)gridDim.x * blockDim.x)
        y[i] = fma(a, x[i], y[i]);
}
int nk_axpy(cudaStream_t s, long len, double a, const double *x, double *y)
{
    if (len <= 0) return LYAP_OK;
    axpy_kernel<<<grid_for(len), 256, 0, s>>>(len, a, x, y);
    return launched();
}

// T (k x p, ld k) = [[I_c, Rz (c x q)], [0, R2 (k2 x q)]], k = c + k2, p = c + q
__global__ void assemble_T_kernel(int c, int q, int k2, const double *__restrict__ Rz, const double *__restrict__ R2,
                                  double *__restrict__ T)
{
    const int k = c + k2, p = c + q;
    long tot = (long)k * p;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < tot; e += (long)gridDim.x * blockDim.x) {
        int i = (int)(e % k), j = (int)(e / k);
        double v = 0.0;
        if (j < c) v = (i == j) ? 1.0 : 0.0;
        else if (i < c) v = Rz[i + (long)(j - c) * c];
        else v = R2[(i - c) + (long)(j - c) * k2];
        T[e] = v;
    }
}
int nk_assemble_T(cudaStream_t s, int c, int q, int k2, const double *Rz, const double *R2, double *T)
{
    long tot = (long)(c + k2) * (c + q);
    assemble_T_kernel<<<grid_for(tot), 256, 0, s>>>(c, q, k2, Rz, R2, T);
    return launched();
}

__global__ void roll_kernel(double *scal) { scal[SC_NA2] = scal[SC_RED + 1]; scal[SC_MAXA] = scal[SC_RED + 3]; }
int nk_roll(cudaStream_t s, double *scal)
{
    roll_kernel<<<1, 1, 0, s>>>(scal);
    return launched();
}

int nk_trace_prod(cudaStream_t s, int k, const double *P, double *out)
{
    trace_prod_kernel<<<1, 1024, 0, s>>>(k, P, out);
    return launched();
}

}  // namespace lyap
