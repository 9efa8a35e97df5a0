// gje.cu -- blocked in-place inversion A <- A^{-1} for the Newton step
// A_k = (mu A_{k-1} + mu^{-1} A_{k-1}^{-1})/2 (PAPER.md Eq. newton-lyapu1 l.1125).
//
// Algorithm: blocked Gauss-Jordan elimination with partial pivoting.  Each
// block step k (panel width b) is
//   1. panel kernel (one CTA): LU with partial pivoting of the panel
//      A[k:n, k:k+b] (warp-shuffle argmax pivot search), inversion of the
//      b x b pivot block T = A11^{-1}, and the multiplier block
//      X = [-A[0:k,panel] T ; T ; -L21 L11^{-1}]            (n x b)
//   2. row-swap / prep kernels: apply the pivot rows to all n columns, copy
//      the pivot rows to B (b x n) with B[:, panel] = I, zero the pivot rows
//      and the panel columns of A,
//   3. rank-b update A += X B (n x n x b GEMM, fp32 accumulation for 16-bit
//      storage).
// After the last step A holds (PA)^{-1} = A^{-1} P^T, i.e. A^{-1}[:, rowperm[i]]
// = A[:, i]; the caller gathers columns with invperm.  The pivot sequence is
// exactly that of LU with partial pivoting (the rows below the block see the
// same Schur complement as right-looking LU).
#include <cooperative_groups.h>
#include "common.cuh"
#include "gemm_simt.cuh"
#include "lyap_internal.h"
#include "ktimer.h"

namespace lyap {

// -------------------------------------------------------------------- panel
template <typename Acc>
struct ArgMax { Acc v; int i; };

template <typename Acc>
__device__ __forceinline__ void argmax_merge(Acc &v, int &i, Acc v2, int i2) {
    if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
}

template <typename T>
__global__ void __launch_bounds__(1024)
gje_panel_kernel(int n, int k, int b, T *__restrict__ A, T *__restrict__ X,
                 int *__restrict__ ipiv, int *__restrict__ moved, int *__restrict__ nmoved,
                 int *__restrict__ info, typename Prec<T>::acc *__restrict__ Pglob, int use_smem,
                 double *__restrict__ ldet)
{
    using Acc = typename Prec<T>::acc;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int R = n - k;
    const int tid = threadIdx.x, nt = blockDim.x;
    Acc *Lw = reinterpret_cast<Acc *>(smem_raw);              // b*b : Linv
    Acc *Tw = Lw + 32 * 32;                                    // b*b : T = A11^{-1}
    Acc *redv = Tw + 32 * 32;                                  // 32
    int *redi = reinterpret_cast<int *>(redv + 32);            // 32
    int *pivl = redi + 32;                                     // 32 local pivots
    int *sflag = pivl + 32;                                    // 1
    Acc *P = use_smem ? reinterpret_cast<Acc *>(sflag + 4) : Pglob;   // R*b (row-major, ld b)

    for (int idx = tid; idx < R * b; idx += nt) {
        const int r = idx / b, c = idx - r * b;
        P[idx] = to_acc<T>(A[(long)(k + r) * n + k + c]);
    }
    if (tid == 0) *sflag = 0;
    __syncthreads();

    for (int j = 0; j < b; j++) {
        // ---- pivot search: max |P[r][j]|, r >= j, lowest index on ties
        Acc bv = Acc(-1); int bi = R;
        for (int r = j + tid; r < R; r += nt) {
            Acc v = fabs(P[(long)r * b + j]);
            argmax_merge(bv, bi, v, r);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            Acc v2 = __shfl_xor_sync(0xffffffffu, bv, o);
            int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
            argmax_merge(bv, bi, v2, i2);
        }
        if ((tid & 31) == 0) { redv[tid >> 5] = bv; redi[tid >> 5] = bi; }
        __syncthreads();
        if (tid < 32) {
            int nw = nt >> 5;
            bv = tid < nw ? redv[tid] : Acc(-1);
            bi = tid < nw ? redi[tid] : R;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                Acc v2 = __shfl_xor_sync(0xffffffffu, bv, o);
                int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
                argmax_merge(bv, bi, v2, i2);
            }
            int p = bi;
            if (tid == 0) {
                pivl[j] = p;
                if (!(bv > Acc(0))) {            // zero (or nan) pivot column
                    if (*sflag == 0) *sflag = k + j + 1;
                }
            }
            // swap rows j and p (one warp, b <= 32 columns)
            if (p != j && tid < b) {
                Acc t = P[(long)j * b + tid];
                P[(long)j * b + tid] = P[(long)p * b + tid];
                P[(long)p * b + tid] = t;
            }
        }
        __syncthreads();
        const Acc d = P[(long)j * b + j];
        if (d != Acc(0)) {
            const Acc inv = Acc(1) / d;
            for (int r = j + 1 + tid; r < R; r += nt) {
                Acc *row = P + (long)r * b;
                Acc l = row[j] * inv;
                row[j] = l;
                for (int c = j + 1; c < b; c++) row[c] = fma(-l, P[(long)j * b + c], row[c]);
            }
        }
        __syncthreads();
    }

    // ---- Linv = L11^{-1} (unit lower), Uinv = U11^{-1}; T = Uinv * Linv
    Acc *Uw = Tw;   // reuse T storage for Uinv first, then form T into Lw/Tw carefully
    if (tid < b) {
        int c = tid;
        // Linv column c
        for (int i = 0; i < b; i++) {
            Acc s = (i == c) ? Acc(1) : Acc(0);
            if (i > c)
                for (int t = c; t < i; t++) s = fma(-P[(long)i * b + t], Lw[t * 32 + c], s);
            Lw[i * 32 + c] = (i < c) ? Acc(0) : s;
        }
    } else if (tid >= 32 && tid < 32 + b) {
        int c = tid - 32;
        for (int i = b - 1; i >= 0; i--) {
            Acc s = (i == c) ? Acc(1) : Acc(0);
            if (i < c)
                for (int t = c; t >= i + 1; t--) s = fma(-P[(long)i * b + t], Uw[t * 32 + c], s);   // newest x last: short chain
            Uw[i * 32 + c] = (i > c) ? Acc(0) : s * (Acc(1) / P[(long)i * b + i]);   // reciprocal: off the chain
        }
    }
    __syncthreads();
    // T = Uinv * Linv, computed into registers then stored over Uw
    Acc tval = Acc(0);
    int ti = tid / 32, tc = tid % 32;
    if (ti < b && tc < b)
        for (int t = 0; t < b; t++) tval = fma(Uw[ti * 32 + t], Lw[t * 32 + tc], tval);
    __syncthreads();
    if (ti < b && tc < b) Tw[ti * 32 + tc] = tval;
    __syncthreads();

    // ---- X rows
    for (int idx = tid; idx < n * b; idx += nt) {
        const int i = idx / b, c = idx - i * b;
        Acc s = Acc(0);
        if (i >= k && i < k + b) {
            s = Tw[(i - k) * 32 + c];
        } else if (i >= k + b) {
            const Acc *row = P + (i - k) * b;
            for (int t = 0; t < b; t++) s = fma(-row[t], Lw[t * 32 + c], s);
        } else {
            const T *arow = A + (long)i * n + k;
            for (int t = 0; t < b; t++) s = fma(-to_acc<T>(arow[t]), Tw[t * 32 + c], s);
        }
        X[idx] = from_acc<T>(s);
    }
    // ---- pivots and the list of moved rows (dst local pos, src local row)
    if (tid == 0) {
        for (int j = 0; j < b; j++) ipiv[k + j] = k + pivl[j];
        // log|det| contribution of this panel: the Gauss-Jordan pivots are U's diagonal
        double sl = 0.0;
        for (int j = 0; j < b; j++) sl += log(fabs((double)P[(long)j * b + j]));
        ldet[k] = sl;
        if (*sflag && *info == 0) *info = *sflag;
        // replay the transpositions on a small position map of candidates
        int cand[64], src[64], nc = 0;
        for (int j = 0; j < b; j++) { cand[nc] = j; src[nc] = j; nc++; }
        for (int j = 0; j < b; j++) {
            int p = pivl[j];
            int ip = -1;
            for (int t = 0; t < nc; t++) if (cand[t] == p) { ip = t; break; }
            if (ip < 0) { cand[nc] = p; src[nc] = p; ip = nc; nc++; }
            int ij = j;   // position j is always cand[j]
            int tmp = src[ij]; src[ij] = src[ip]; src[ip] = tmp;
        }
        int m = 0;
        for (int t = 0; t < nc; t++)
            if (src[t] != cand[t]) { moved[2 * m] = cand[t]; moved[2 * m + 1] = src[t]; m++; }
        *nmoved = m;
    }
}

// -------------------------------------------------------------- cluster panel
// The same panel factorisation with the R = n-k panel rows split over a thread-block
// cluster of NC CTAs (one SM each, RB >= b rows per CTA).  Each thread keeps RPT panel
// rows in registers.  Per column one cluster exchange: every CTA publishes its local
// pivot candidate (|value|, row, the row itself) and, if it owns it, the current row
// j; after the cluster barrier every warp picks the same winner (largest |value|,
// lowest row on ties -- the single-CTA rule), the pivot row is broadcast by warp
// shuffles, and each thread swaps/eliminates its own rows.  Every matrix element
// sees exactly the arithmetic of the single-CTA kernel, so pivots and results are
// bitwise identical.
template <typename Acc, int BW>
__device__ __forceinline__ Acc sel_col(const Acc (&r)[BW], int j) {
    Acc v = r[0];
#pragma unroll
    for (int c = 1; c < BW; c++) v = (c == j) ? r[c] : v;
    return v;
}

// Warp argmax of (v >= 0 or -1 for "none", index), ties to the lower index, result in
// every lane.  Candidates must be ordered: lane order = index order among equal values
// (callers guarantee it).  fp32: one redux.sync max over the value bits + a ballot;
// fp64: butterfly of (value, index) pairs.
template <typename Acc>
__device__ __forceinline__ void warp_argmax(Acc &v, int &i, int lane) {
    if constexpr (sizeof(Acc) == 4) {
        // key 0 = no candidate / NaN (never selected, as in argmax_merge), else bits + 1
        const unsigned key = (v >= 0.f) ? __float_as_uint(v) + 1u : 0u;
        const unsigned mx = __reduce_max_sync(0xffffffffu, key);
        const unsigned who = __ballot_sync(0xffffffffu, key == mx);
        const int src = __ffs(who) - 1;
        v = __shfl_sync(0xffffffffu, v, src);
        i = __shfl_sync(0xffffffffu, i, src);
        if (mx == 0u) v = Acc(-1);
    } else {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            Acc v2 = __shfl_xor_sync(0xffffffffu, v, o);
            int i2 = __shfl_xor_sync(0xffffffffu, i, o);
            argmax_merge(v, i, v2, i2);
        }
    }
    (void)lane;
}

// a register row to / from 16-byte aligned shared memory, vectorised
template <typename Acc, int BW>
__device__ __forceinline__ void row_store(const Acc (&r)[BW], Acc *dst) {
    if constexpr (sizeof(Acc) == 4) {
#pragma unroll
        for (int c = 0; c < BW; c += 4) *reinterpret_cast<float4 *>(dst + c) = make_float4(r[c], r[c + 1], r[c + 2], r[c + 3]);
    } else {
#pragma unroll
        for (int c = 0; c < BW; c += 2) *reinterpret_cast<double2 *>(dst + c) = make_double2(r[c], r[c + 1]);
    }
}
template <typename Acc, int BW>
__device__ __forceinline__ void row_load(Acc (&r)[BW], const Acc *src) {
    if constexpr (sizeof(Acc) == 4) {
#pragma unroll
        for (int c = 0; c < BW; c += 4) {
            const float4 v = *reinterpret_cast<const float4 *>(src + c);
            r[c] = v.x; r[c + 1] = v.y; r[c + 2] = v.z; r[c + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int c = 0; c < BW; c += 2) {
            const double2 v = *reinterpret_cast<const double2 *>(src + c);
            r[c] = v.x; r[c + 1] = v.y;
        }
    }
}

// 16-byte vectors <-> elements (raw bits; the conversions are to_acc / from_acc's)
template <typename T> struct Vec16;
template <> struct Vec16<__nv_bfloat16> {
    static constexpr int E = 8;
    __device__ __forceinline__ static void unpack(const uint4 &v, float (&o)[E]) {
        const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; i++) {
            o[2 * i] = __bfloat162float(__ushort_as_bfloat16((unsigned short)(w[i] & 0xffffu)));
            o[2 * i + 1] = __bfloat162float(__ushort_as_bfloat16((unsigned short)(w[i] >> 16)));
        }
    }
    __device__ __forceinline__ static uint4 pack(const float (&x)[E]) {
        unsigned w[4];
#pragma unroll
        for (int i = 0; i < 4; i++)
            w[i] = (unsigned)__bfloat16_as_ushort(__float2bfloat16_rn(x[2 * i])) |
                   ((unsigned)__bfloat16_as_ushort(__float2bfloat16_rn(x[2 * i + 1])) << 16);
        return make_uint4(w[0], w[1], w[2], w[3]);
    }
};
template <> struct Vec16<__half> {
    static constexpr int E = 8;
    __device__ __forceinline__ static void unpack(const uint4 &v, float (&o)[E]) {
        const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; i++) {
            o[2 * i] = __half2float(__ushort_as_half((unsigned short)(w[i] & 0xffffu)));
            o[2 * i + 1] = __half2float(__ushort_as_half((unsigned short)(w[i] >> 16)));
        }
    }
    __device__ __forceinline__ static uint4 pack(const float (&x)[E]) {
        unsigned w[4];
#pragma unroll
        for (int i = 0; i < 4; i++)
            w[i] = (unsigned)__half_as_ushort(__float2half_rn(x[2 * i])) |
                   ((unsigned)__half_as_ushort(__float2half_rn(x[2 * i + 1])) << 16);
        return make_uint4(w[0], w[1], w[2], w[3]);
    }
};
template <> struct Vec16<float> {
    static constexpr int E = 4;
    __device__ __forceinline__ static void unpack(const uint4 &v, float (&o)[E]) {
        o[0] = __uint_as_float(v.x); o[1] = __uint_as_float(v.y); o[2] = __uint_as_float(v.z); o[3] = __uint_as_float(v.w);
    }
    __device__ __forceinline__ static uint4 pack(const float (&x)[E]) {
        return make_uint4(__float_as_uint(x[0]), __float_as_uint(x[1]), __float_as_uint(x[2]), __float_as_uint(x[3]));
    }
};
template <> struct Vec16<double> {
    static constexpr int E = 2;
    __device__ __forceinline__ static void unpack(const uint4 &v, double (&o)[E]) {
        o[0] = __hiloint2double((int)v.y, (int)v.x); o[1] = __hiloint2double((int)v.w, (int)v.z);
    }
    __device__ __forceinline__ static uint4 pack(const double (&x)[E]) {
        return make_uint4((unsigned)__double2loint(x[0]), (unsigned)__double2hiint(x[0]),
                          (unsigned)__double2loint(x[1]), (unsigned)__double2hiint(x[1]));
    }
};

template <typename T, int BW, int RPT, int NT>
__global__ void __launch_bounds__(NT)
gje_panel_cluster_kernel(int n, int k, int b, int RB, const T *__restrict__ A, T *__restrict__ X,
                         int *__restrict__ ipiv, int *__restrict__ moved, int *__restrict__ nmoved,
                         int *__restrict__ info, typename Prec<T>::acc *__restrict__ Tglob,
                         typename Prec<T>::acc *__restrict__ Pg, double *__restrict__ ldet)
{
    namespace cg = cooperative_groups;
    using Acc = typename Prec<T>::acc;
    constexpr int NW = NT / 32;                                // warps per CTA
    cg::cluster_group cl = cg::this_cluster();
    const int q = (int)cl.block_rank(), NC = (int)cl.num_blocks();
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int R = n - k;
    const int g0 = q * RB, nloc = max(0, min(RB, R - g0));
    constexpr int PW = 2 * BW + 4;                             // cand row, row j, |cand|, row index (16B-aligned rows)
    __shared__ __align__(16) Acc pub[2][PW];
    __shared__ __align__(16) Acc inbox[2][16][PW];             // pushed by every CTA of the cluster
    __shared__ Acc redv[32];
    __shared__ int redi[32];
    __shared__ int pivl[32];
    __shared__ int sflag;
    __shared__ Acc Ptop[32][33];
    __shared__ __align__(16) Acc Lw[32 * 32], Tw[32 * 32];
#ifdef LYAP_PANEL_PROF
    const long long t_start = clock64();
#endif
    Acc row[RPT][BW];
    constexpr int VE = Vec16<T>::E;
    // full panels with 16-byte aligned rows: each row as BW / VE vector loads (scalar 2-byte
    // loads of 32 strided rows per warp instruction made the load phase L1-bound)
    const bool vec = (b == BW) && ((long)n * sizeof(T)) % 16 == 0 && ((long)k * sizeof(T)) % 16 == 0;
#pragma unroll
    for (int h = 0; h < RPT; h++) {
        const int r = RPT * tid + h;
        const T *src = A + (long)(k + g0 + r) * n + k;
        if (vec) {
            if (r < nloc) {
                uint4 v[BW / VE];
#pragma unroll
                for (int u = 0; u < BW / VE; u++) v[u] = reinterpret_cast<const uint4 *>(src)[u];
#pragma unroll
                for (int u = 0; u < BW / VE; u++) {
                    Acc o[VE];
                    Vec16<T>::unpack(v[u], o);
#pragma unroll
                    for (int e = 0; e < VE; e++) row[h][u * VE + e] = o[e];
                }
            } else {
#pragma unroll
                for (int c = 0; c < BW; c++) row[h][c] = Acc(0);
            }
        } else {
#pragma unroll
            for (int c = 0; c < BW; c++) row[h][c] = (r < nloc && c < b) ? to_acc<T>(src[c]) : Acc(0);
        }
    }
    if (tid == 0) sflag = 0;
#ifdef LYAP_PANEL_PROF
    const long long t_loaded = clock64();
    long long pt[6] = {0, 0, 0, 0, 0, 0}, tl = clock64();
#define PPROF(i) do { if (q == 0 && tid == 0) { long long t_ = clock64(); pt[i] += t_ - tl; tl = t_; } } while (0)
#else
#define PPROF(i) do { } while (0)
#endif
    // columns unrolled: every register index and every (c > j) test is a compile-time constant
#pragma unroll
    for (int j = 0; j < BW; j++) {
        if (j >= b) break;
        const int buf = j & 1;
        // ---- local candidate: max |P[r][j]|, panel row >= j, lowest row on ties.  Rows
        // increase with (thread, slot), warp and CTA, so "lowest slot holding the maximum"
        // is the lowest row (the single-CTA tie rule).
        Acc bv = Acc(-1); int bi = R;
#pragma unroll
        for (int h = 0; h < RPT; h++) {
            const int r = RPT * tid + h, gi = g0 + r;
            if (r < nloc && gi >= j) argmax_merge(bv, bi, fabs(row[h][j]), gi);
        }
        warp_argmax<Acc>(bv, bi, lane);
        if (lane == 0) { redv[wid] = bv; redi[wid] = bi; }
        PPROF(0);
        __syncthreads();
        PPROF(1);
        bv = lane < NW ? redv[lane] : Acc(-1);
        bi = lane < NW ? redi[lane] : R;
        warp_argmax<Acc>(bv, bi, lane);                        // every lane needs the CTA winner
        if (tid == 0) { pub[buf][2 * BW] = bv; pub[buf][2 * BW + 1] = Acc(bi); }
#pragma unroll
        for (int h = 0; h < RPT; h++) {
            const int r = RPT * tid + h, gi = g0 + r;
            const bool own_c = r < nloc && gi == bi, own_j = r < nloc && gi == j;
            if (__any_sync(0xffffffffu, own_c || own_j)) {            // one warp (or two) per CTA
                if (own_c) row_store<Acc, BW>(row[h], &pub[buf][0]);
                if (own_j) row_store<Acc, BW>(row[h], &pub[buf][BW]);
            }
        }
        __syncthreads();
        PPROF(2);
        // ---- push this CTA's candidate (and row j) into every CTA's inbox
        for (int r = wid; r < NC; r += NW) {                   // warp r (mod NW) -> CTA r
            Acc *dst = cl.map_shared_rank(&inbox[buf][q][0], r);
            for (int e = lane; e < PW; e += 32) dst[e] = pub[buf][e];
        }
        cl.sync();
        PPROF(3);
        // ---- global winner from the local inbox
        Acc gbv = Acc(-1); int gbi = R;
        if (lane < NC) { gbv = inbox[buf][lane][2 * BW]; gbi = (int)inbox[buf][lane][2 * BW + 1]; }
        warp_argmax<Acc>(gbv, gbi, lane);
        const int pr = gbi < R ? gbi : j;                      // empty column: no swap (info is set)
        const Acc *pvp = &inbox[buf][pr / RB][0];
        const Acc *rjp = &inbox[buf][j / RB][BW];
        if (tid == 0) {
            pivl[j] = pr;
            if (!(gbv > Acc(0)) && sflag == 0) sflag = k + j + 1;
        }
        const Acc d = pvp[j];
        const Acc inv = (d != Acc(0)) ? Acc(1) / d : Acc(0);
        PPROF(4);
#pragma unroll
        for (int h = 0; h < RPT; h++) {
            const int r = RPT * tid + h, gi = g0 + r;
            const bool is_j = r < nloc && gi == j && pr != j, is_p = r < nloc && gi == pr && gi > j;
            if (__any_sync(0xffffffffu, is_j || is_p)) {
                if (is_j) row_load<Acc, BW>(row[h], pvp);
                if (is_p) row_load<Acc, BW>(row[h], rjp);
            }
            if (r < nloc && gi > j && d != Acc(0)) {
                const Acc l = row[h][j] * inv;
                row[h][j] = l;
#pragma unroll
                for (int c = j + 1; c < BW; c++) row[h][c] = fma(-l, pvp[c], row[h][c]);
            }
        }
        PPROF(5);
    }
#ifdef LYAP_PANEL_PROF
    const long long t_loop = clock64();
    if (q == 0 && tid == 0 && (k == 0 || k == 2048))
        printf("panel k=%d R=%d NC=%d cycles/col: argmax %lld bar1 %lld winner+pub+bar2 %lld push+csync %lld "
               "select %lld elim %lld | load %lld loop %lld\n", k, R, NC, pt[0] / b, pt[1] / b, pt[2] / b, pt[3] / b, pt[4] / b, pt[5] / b,
               t_loaded - t_start, t_loop - t_loaded);
#endif
    // ---- rows below the block: their multipliers (in Acc precision) go to Pg, and
    // gje_xabove_kernel (the whole GPU) forms X = -L21 L11^{-1} there
#pragma unroll
    for (int h = 0; h < RPT; h++) {
        const int r = RPT * tid + h, gi = g0 + r;
        if (r >= nloc || gi < b) continue;
        Acc *pr = Pg + (long)gi * BW;
        if constexpr (sizeof(Acc) == 4) {
#pragma unroll
            for (int c = 0; c < BW; c += 4)
                *reinterpret_cast<float4 *>(pr + c) = make_float4(row[h][c], row[h][c + 1], row[h][c + 2], row[h][c + 3]);
        } else {
#pragma unroll
            for (int c = 0; c < BW; c += 2) *reinterpret_cast<double2 *>(pr + c) = make_double2(row[h][c], row[h][c + 1]);
        }
    }
    // ---- Linv = L11^{-1}, Uinv = U11^{-1}, T = Uinv Linv on CTA 0 (owns panel rows 0..b-1);
    // same recurrences and summation order as the single-CTA kernel, loops unrolled
#pragma unroll
    for (int h = 0; h < RPT; h++) {
        const int r = RPT * tid + h;
        if (q == 0 && r < b)
#pragma unroll
            for (int c = 0; c < BW; c++) if (c < b) Ptop[r][c] = row[h][c];
    }
    __syncthreads();
    if (q == 0) {
        Acc *Uw = Tw;
        if (tid < b) {
            const int c = tid;
            for (int i = 0; i < b; i++) {
                Acc sacc = (i == c) ? Acc(1) : Acc(0);
#pragma unroll
                for (int t = 0; t < BW; t++)
                    if (t >= c && t < i) sacc = fma(-Ptop[i][t], Lw[t * 32 + c], sacc);
                Lw[i * 32 + c] = (i < c) ? Acc(0) : sacc;
            }
        } else if (tid >= 32 && tid < 32 + b) {
            const int c = tid - 32;
            for (int i = b - 1; i >= 0; i--) {
                Acc sacc = (i == c) ? Acc(1) : Acc(0);
#pragma unroll
                for (int t = BW - 1; t >= 1; t--)                // descending: x_{i+1}, the newest, enters last
                    if (t >= i + 1 && t <= c) sacc = fma(-Ptop[i][t], Uw[t * 32 + c], sacc);
                Uw[i * 32 + c] = (i > c) ? Acc(0) : sacc * (Acc(1) / Ptop[i][i]);   // reciprocal: off the chain
            }
        } else if (tid >= 64 && tid < 96) {
            // moved rows: replay the transpositions on the candidate positions (one warp)
            __shared__ int cand[64], src[64];
            __shared__ int ncand;
            const int ln = tid - 64;
            cand[ln] = ln; src[ln] = ln;
            if (ln == 0) ncand = b;
            __syncwarp();
            for (int j = 0; j < b; j++) {
                const int pj = pivl[j];
                const int nc0 = ncand;
                const unsigned hit0 = __ballot_sync(0xffffffffu, ln < nc0 && cand[ln] == pj);
                const unsigned hit1 = __ballot_sync(0xffffffffu, ln + 32 < nc0 && cand[ln + 32] == pj);
                int ip = hit0 ? __ffs(hit0) - 1 : (hit1 ? 32 + __ffs(hit1) - 1 : -1);
                if (ip < 0) {
                    ip = nc0;
                    if (ln == 0) { cand[ip] = pj; src[ip] = pj; ncand = nc0 + 1; }
                }
                __syncwarp();
                if (ln == 0) { const int t = src[j]; src[j] = src[ip]; src[ip] = t; }
                __syncwarp();
            }
            if (ln == 0) {
                int mm = 0;
                for (int t = 0; t < ncand; t++)
                    if (src[t] != cand[t]) { moved[2 * mm] = cand[t]; moved[2 * mm + 1] = src[t]; mm++; }
                *nmoved = mm;
                for (int j = 0; j < b; j++) ipiv[k + j] = k + pivl[j];
                if (sflag && *info == 0) *info = sflag;
                double sl = 0.0;                 // log|det| contribution (U's diagonal)
                for (int j = 0; j < b; j++) sl += log(fabs((double)Ptop[j][j]));
                ldet[k] = sl;
            }
        }
        __syncthreads();
        constexpr int RT = (32 + NW - 1) / NW;                   // rows of T per thread
        Acc tval[RT];
#pragma unroll
        for (int hh = 0; hh < RT; hh++) tval[hh] = Acc(0);
        const int ti = tid / 32, tc = tid % 32;
#pragma unroll
        for (int hh = 0; hh < RT; hh++)
            if (ti + NW * hh < b && tc < b)
#pragma unroll
                for (int t = 0; t < BW; t++)
                    if (t < b) tval[hh] = fma(Uw[(ti + NW * hh) * 32 + t], Lw[t * 32 + tc], tval[hh]);
        __syncthreads();
        for (int hh = 0; hh < RT; hh++)
            if (ti + NW * hh < b && tc < b) Tw[(ti + NW * hh) * 32 + tc] = tval[hh];
        __syncthreads();
#ifdef LYAP_PANEL_PROF
        const long long t_tail1 = clock64();
#endif
        // block rows: X = T; T and Linv to global for gje_xabove_kernel (rows above: -A T,
        // rows below: -L21 Linv)
        if (tid < b) {
            T *xr = X + (long)(k + tid) * b;
            for (int c = 0; c < b; c++) xr[c] = from_acc<T>(Tw[tid * 32 + c]);
        }
        for (int e = tid; e < 32 * 32; e += NT) { Tglob[e] = Tw[e]; Tglob[32 * 32 + e] = Lw[e]; }
#ifdef LYAP_PANEL_PROF
        __syncthreads();
        if (tid == 0 && (k == 0 || k == 2048))
            printf("panel tail k=%d: T %lld X block rows + publish %lld\n", k, t_tail1 - t_loop, clock64() - t_tail1);
#endif
    }
    cl.sync();                                                 // shared memory stays valid for remote readers
}

// gather moved source rows (full width) and their rowperm entries into tmp
template <typename T>
__global__ void gje_gather_kernel(int n, int k, int c0, int c1, const T *__restrict__ A, const int *__restrict__ moved,
                                  const int *__restrict__ nmoved, T *__restrict__ tmp,
                                  const int *__restrict__ rowperm, int *__restrict__ tmp_perm)
{
    int m = *nmoved;
    int t = blockIdx.y;
    if (t >= m) return;
    int src = k + moved[2 * t + 1];
    for (int c = c0 + blockIdx.x * blockDim.x + threadIdx.x; c < c1; c += gridDim.x * blockDim.x)
        tmp[(long)t * n + c] = A[(long)src * n + c];
    if (blockIdx.x == 0 && threadIdx.x == 0) tmp_perm[t] = rowperm[src];
}

// scatter moved rows, build B = pivot rows with B[:, panel] = I, zero pivot rows
// and the panel columns of A, for the columns [c0, c1) (all n, or the outer block of
// the two-level scheme).  O(b n) work: blockIdx.y < b are the block rows, the next
// 2b the moved-row slots, the rest zero the panel columns of all other rows.
template <typename T>
__global__ void gje_prep_kernel(int n, int k, int b, int c0, int c1, T *__restrict__ A,
                                const int *__restrict__ moved, const int *__restrict__ nmoved,
                                const T *__restrict__ tmp, const int *__restrict__ tmp_perm,
                                int *__restrict__ rowperm, T *__restrict__ B)
{
    const int m = *nmoved;
    const T zero = from_acc<T>(0), one = from_acc<T>(1);
    const int ty = blockIdx.y;
    const int cx = blockIdx.x * blockDim.x + threadIdx.x, sx = gridDim.x * blockDim.x;
    if (ty < b) {                                        // block row: B column, then zero
        const int local = ty;
        if (local >= n - k) return;
        const long i = k + local;
        int slot = -1;
        for (int t = 0; t < m; t++) if (moved[2 * t] == local) { slot = t; break; }
        for (int c = c0 + cx; c < c1; c += sx) {
            const bool panel_col = (c >= k && c < k + b);
            const T v = (slot >= 0) ? tmp[(long)slot * n + c] : A[i * n + c];
            B[(long)c * b + local] = panel_col ? ((c - k == local) ? one : zero) : v;   // Bt: n x b
            A[i * n + c] = zero;
        }
        if (slot >= 0 && cx == 0) rowperm[i] = tmp_perm[slot];
    } else if (ty < 3 * b) {                             // moved row below the block
        const int t = ty - b;
        if (t >= m) return;
        const int local = moved[2 * t];
        if (local < b) return;
        const long i = k + local;
        for (int c = c0 + cx; c < c1; c += sx) {
            const bool panel_col = (c >= k && c < k + b);
            A[i * n + c] = panel_col ? zero : tmp[(long)t * n + c];
        }
        if (cx == 0) rowperm[i] = tmp_perm[t];
    } else {                                             // panel columns of the other rows
        const long tot = (long)n * b;
        const long stride = (long)(gridDim.y - 3 * b) * sx;
        for (long e = (long)(ty - 3 * b) * sx + cx; e < tot; e += stride) {
            const long i = e / b;
            const int c = (int)(e - i * b);
            if (i >= k && i < k + b) continue;
            A[i * n + k + c] = zero;
        }
    }
}

// Two-level scheme, outer step for the block columns [K0, K0+nb): the inner steps
// transformed only the block columns; the other columns ("rest") now receive the
// block's row interchanges (the composite of the transpositions ipiv[K0..K0+nb) in
// order), then B_outer = the pivot rows' rest entries (n x nb, K-major for the GEMM)
// and the pivot rows' rest entries are zeroed.

// (1) composite permutation of the block in O(n) parallel work: with invprev = the inverse of rowperm
// before the block and rowperm after it, position i (>= K0) now holds the row that was at
// src = invprev[rowperm[i]].  The (dst, src) list order is irrelevant (each dst once);
// slot_of[y] = list index of pivot row K0 + y (or -1), for the scatter.
__global__ void gje_inv_snapshot_kernel(int n, const int *__restrict__ rowperm, int *__restrict__ invprev)
{
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) invprev[rowperm[i]] = i;
}
__global__ void gje_outer_perm2_kernel(int n, int K0, int nb, const int *__restrict__ rowperm,
                                       const int *__restrict__ invprev, int *__restrict__ omoved,
                                       int *__restrict__ onmoved, int *__restrict__ slot_of)
{
    for (int i = K0 + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int src = invprev[rowperm[i]];
        if (src != i) {
            const int t = atomicAdd(onmoved, 1);
            omoved[2 * t] = i;
            omoved[2 * t + 1] = src;
            if (i < K0 + nb) slot_of[i - K0] = t;
        }
    }
}

// (2) gather the moved source rows' rest entries
template <typename T>
__global__ void gje_outer_gather_kernel(int n, int K0, int nb, const T *__restrict__ A, const int *__restrict__ omoved,
                                        const int *__restrict__ onmoved, T *__restrict__ tmp2)
{
    const int t = blockIdx.y;
    if (t >= *onmoved) return;
    const long src = omoved[2 * t + 1];
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n - nb; e += gridDim.x * blockDim.x) {
        const int c = e < K0 ? e : e + nb;
        tmp2[(long)t * n + c] = A[src * n + c];
    }
}

// (3) scatter moved rows below the block; pivot rows -> B_outer (transposed through
// shared memory so both sides are coalesced) and zero
template <typename T>
__global__ void __launch_bounds__(256)
gje_outer_scatter_kernel(int n, int K0, int nb, T *__restrict__ A, const int *__restrict__ omoved,
                         const int *__restrict__ onmoved, const T *__restrict__ tmp2, T *__restrict__ Bo,
                         const int *__restrict__ slot_of, int moved_part)
{
    const int m = *onmoved;
    const int nrest = n - nb;
    // two launches: moved_part = 0 transposes the pivot rows (grid.y = 1), moved_part = 1
    // writes moved row blockIdx.y (a narrow grid.x: most of the 2 nb slots are real rows)
    if (!moved_part) {
        // pivot rows: tile of 32 rest columns x nb rows
        __shared__ T tile[32][33];
        __shared__ int slot[GJE_NB];
        for (int y = threadIdx.x; y < nb; y += blockDim.x) slot[y] = slot_of[y];
        __syncthreads();
        const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;     // 32 x 8
        for (int e0 = blockIdx.x * 32; e0 < nrest; e0 += gridDim.x * 32) {
            for (int y0 = 0; y0 < nb; y0 += 32) {
                for (int yy = ty; yy < 32; yy += 8) {
                    const int y = y0 + yy, e = e0 + tx;
                    T v = from_acc<T>(0);
                    if (y < nb && e < nrest) {
                        const int c = e < K0 ? e : e + nb;
                        const long row = K0 + y;
                        v = slot[y] >= 0 ? tmp2[(long)slot[y] * n + c] : A[row * n + c];
                        A[row * n + c] = from_acc<T>(0);
                    }
                    tile[yy][tx] = v;
                }
                __syncthreads();
                for (int cc = ty; cc < 32; cc += 8) {
                    const int e = e0 + cc, y = y0 + tx;
                    if (e < nrest && y < nb) {
                        const int c = e < K0 ? e : e + nb;
                        Bo[(long)c * nb + y] = tile[tx][cc];
                    }
                }
                __syncthreads();
            }
        }
    } else {
        const int t = blockIdx.y;
        if (t >= m) return;
        const int dst = omoved[2 * t];
        if (dst < K0 + nb) return;                               // pivot rows handled above
        for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nrest; e += gridDim.x * blockDim.x) {
            const int c = e < K0 ? e : e + nb;
            A[(long)dst * n + c] = tmp2[(long)t * n + c];
        }
    }
}

__global__ void iota_kernel(int n, int *p) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = i;
}
__global__ void invperm_kernel(int n, const int *rowperm, int *invperm) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        invperm[rowperm[i]] = i;
}

template <typename T>
__global__ void col_gather_kernel(int n, const T *__restrict__ G, const int *__restrict__ invperm, T *__restrict__ out)
{
    for (long i = blockIdx.y; i < n; i += gridDim.y)
        for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x)
            out[i * n + c] = G[i * n + invperm[c]];
}

// ------------------------------------------------------------------ driver
int gje_panel_width(int prec) { return prec == LYAP_FP64 ? 16 : 32; }

size_t gje_panel_smem(int n, int prec, int b, int R, bool *use_smem) {
    size_t acc = (prec == LYAP_FP64) ? 8 : 4;
    size_t head = acc * (2 * 32 * 32 + 32) + sizeof(int) * (32 + 32 + 4);
    size_t need = head + acc * (size_t)R * b;
    *use_smem = need <= 220 * 1024;
    return *use_smem ? need : head;
}

int GjeWork::alloc(int n_, int prec_) {
    n = n_; prec = prec_;
    int b = gje_panel_width(prec);
    size_t es = elem_size(prec);
    size_t acc = (prec == LYAP_FP64) ? 8 : 4;
    LYAP_CUDA_TRY(cudaMalloc(&X, es * (size_t)n * b));
    LYAP_CUDA_TRY(cudaMalloc(&B, es * (size_t)n * b));
    LYAP_CUDA_TRY(cudaMalloc(&tmp, es * (size_t)n * 2 * b));
    LYAP_CUDA_TRY(cudaMalloc(&Pglob, acc * (size_t)n * b));
    LYAP_CUDA_TRY(cudaMalloc(&Tg, acc * 2 * 32 * 32));   // T, then Linv
    if ((prec == LYAP_FP16 || prec == LYAP_BF16 || prec == LYAP_FP32) && n % 8 == 0 && n >= 2 * GJE_NB) {
        LYAP_CUDA_TRY(cudaMalloc(&Bo, es * (size_t)n * GJE_NB_MAX));
        LYAP_CUDA_TRY(cudaMalloc(&tmp2, es * (size_t)n * 2 * GJE_NB));
        LYAP_CUDA_TRY(cudaMalloc(&oints, sizeof(int) * (5 * GJE_NB + 8 + (size_t)n)));
        int lo_p = 0, hi_p = 0;
        cudaDeviceGetStreamPriorityRange(&lo_p, &hi_p);
        LYAP_CUDA_TRY(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, hi_p));
        LYAP_CUDA_TRY(cudaEventCreateWithFlags(&ev_a, cudaEventDisableTiming));
        LYAP_CUDA_TRY(cudaEventCreateWithFlags(&ev_b, cudaEventDisableTiming));
        omoved = oints; onmoved = oints + 4 * GJE_NB; slot_of = onmoved + 4; invprev = slot_of + GJE_NB;
    }
    LYAP_CUDA_TRY(cudaMalloc(&ints, sizeof(int) * (size_t)(4 * n + 4 * b + 8)));
    LYAP_CUDA_TRY(cudaMalloc(&ldet, sizeof(double) * (size_t)n));
    ipiv = ints; rowperm = ipiv + n; invperm = rowperm + n; moved = invperm + n;
    nmoved = moved + 4 * b; info = nmoved + 1; tmp_perm = info + 1;
    return LYAP_OK;
}

void GjeWork::release() {
    cudaFree(X); cudaFree(B); cudaFree(tmp); cudaFree(Pglob); cudaFree(Tg); cudaFree(Bo); cudaFree(tmp2);
    cudaFree(ints); cudaFree(oints); cudaFree(ldet);
    if (side) { cudaStreamSynchronize(side); cudaStreamDestroy(side); side = nullptr; }
    if (ev_a) { cudaEventDestroy(ev_a); ev_a = nullptr; }
    if (ev_b) { cudaEventDestroy(ev_b); ev_b = nullptr; }
    X = B = tmp = nullptr; Pglob = Tg = Bo = tmp2 = nullptr;
    ints = oints = omoved = onmoved = slot_of = invprev = nullptr;
}

// X rows above the panel: X[i, :] = -A[i, k:k+b] T for i < k, and rows below the block
// (cluster panel): X[k+gi, :] = -P[gi, :] Linv with the multipliers P the panel left in Pg
// (Acc precision, ld BW) and Linv = Tglob[1024..].  One thread per row: the row's b
// entries in registers, T / Linv rows as 16-byte shared broadcasts, 16-byte stores; per
// element the summation order is the panel's (t ascending from 0).
template <typename T>
__global__ void __launch_bounds__(128)
gje_xabove_kernel(int n, int k, int b, int R, const T *__restrict__ A, const typename Prec<T>::acc *__restrict__ Tglob,
                  const typename Prec<T>::acc *__restrict__ Pg, T *__restrict__ X)
{
    using Acc = typename Prec<T>::acc;
    constexpr int BW = std::is_same<T, double>::value ? 16 : 32;
    constexpr int VE = Vec16<T>::E;
    __shared__ __align__(16) Acc TL[2][32 * 32];               // T, Linv
    for (int e = threadIdx.x; e < 2 * 32 * 32; e += blockDim.x) TL[e >> 10][e & 1023] = Tglob[e];
    __syncthreads();
    const int tot = k + (R > b ? R - b : 0);
    const bool full = (b == BW);
    const bool vecA = full && ((long)n * sizeof(T)) % 16 == 0 && ((long)k * sizeof(T)) % 16 == 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += gridDim.x * blockDim.x) {
        Acc a[BW];
        const Acc *M;
        T *xr;
        if (i < k) {
            const T *src = A + (long)i * n + k;
            if (vecA) {
#pragma unroll
                for (int u = 0; u < BW / VE; u++) {
                    Acc o[VE];
                    Vec16<T>::unpack(reinterpret_cast<const uint4 *>(src)[u], o);
#pragma unroll
                    for (int e = 0; e < VE; e++) a[u * VE + e] = o[e];
                }
            } else {
#pragma unroll
                for (int t = 0; t < BW; t++) a[t] = (t < b) ? to_acc<T>(src[t]) : Acc(0);
            }
            M = TL[0];
            xr = X + (long)i * b;
        } else {
            const int gi = b + (i - k);
            const Acc *src = Pg + (long)gi * BW;
#pragma unroll
            for (int t = 0; t < BW; t++) a[t] = (t < b) ? src[t] : Acc(0);
            M = TL[1];
            xr = X + (long)(k + gi) * b;
        }
        if (full) {
#pragma unroll
            for (int c0 = 0; c0 < BW; c0 += VE) {
                Acc acc[VE];
#pragma unroll
                for (int e = 0; e < VE; e++) acc[e] = Acc(0);
#pragma unroll
                for (int t = 0; t < BW; t++) {
                    const Acc m = -a[t];
#pragma unroll
                    for (int e = 0; e < VE; e++) acc[e] = fma(m, M[t * 32 + c0 + e], acc[e]);
                }
                reinterpret_cast<uint4 *>(xr)[c0 / VE] = Vec16<T>::pack(acc);
            }
        } else {
            for (int c = 0; c < b; c++) {
                Acc sacc = Acc(0);
#pragma unroll
                for (int t = 0; t < BW; t++) if (t < b) sacc = fma(-a[t], M[t * 32 + c], sacc);
                xr[c] = from_acc<T>(sacc);
            }
        }
    }
}

// panel rows per CTA and cluster size: about 512 rows per CTA (one per thread), at
// least b rows on CTA 0, up to 16 CTAs (non-portable cluster size) for tall panels
template <typename T>
static int gje_panel_launch(cudaStream_t s, int n, int k, int b, T *A, GjeWork &w)
{
    using Acc = typename Prec<T>::acc;
    constexpr int BW = std::is_same<T, double>::value ? 16 : 32;
    const int R = n - k;
    // NTh threads per CTA, one panel row per thread (two when the cluster is full): 512 is
    // measured faster up to ~8K panel rows, 1024 (fewer CTAs in the cluster) above
    const int NTh = (R > 8192 && !env_flag("LYAP_GJE_512")) ? 1024 : 512;
    int nc = std::max(1, std::min(16, ceil_div(R, NTh)));
    if (const char *e = getenv("LYAP_GJE_NC")) nc = std::max(1, std::min(16, atoi(e)));
    const int RB = std::max(b, ceil_div(R, nc));
    nc = ceil_div(R, RB);
    if (RB > 2 * NTh || b > BW || env_flag("LYAP_GJE_1CTA")) {
        bool use_smem;
        size_t sm = gje_panel_smem(n, Prec<T>::code, b, R, &use_smem);
        // one-time setup (function-local static: thread-safe initialisation)
        static const bool attr1 = [] {
            cudaFuncSetAttribute(gje_panel_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
            return true;
        }();
        (void)attr1;
        gje_panel_kernel<T><<<1, 1024, sm, s>>>(n, k, b, A, (T *)w.X, w.ipiv, w.moved, w.nmoved, w.info,
                                                (Acc *)w.Pglob, use_smem ? 1 : 0, w.ldet);
        return launched();
    }
    void (*kern)(int, int, int, int, const T *, T *, int *, int *, int *, int *, Acc *, Acc *, double *);
    if (NTh == 1024) kern = (RB > 1024) ? gje_panel_cluster_kernel<T, BW, 2, 1024> : gje_panel_cluster_kernel<T, BW, 1, 1024>;
    else kern = (RB > 512) ? gje_panel_cluster_kernel<T, BW, 2, 512> : gje_panel_cluster_kernel<T, BW, 1, 512>;
    // one-time setup (function-local static: thread-safe initialisation)
    static const bool attr = [] {
        cudaFuncSetAttribute(gje_panel_cluster_kernel<T, BW, 1, 1024>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaFuncSetAttribute(gje_panel_cluster_kernel<T, BW, 2, 1024>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaFuncSetAttribute(gje_panel_cluster_kernel<T, BW, 1, 512>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaFuncSetAttribute(gje_panel_cluster_kernel<T, BW, 2, 512>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        return true;
    }();
    (void)attr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nc, 1, 1);
    cfg.blockDim = dim3(NTh, 1, 1);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = nc;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    LYAP_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, n, k, b, RB, (const T *)A, (T *)w.X, w.ipiv, w.moved, w.nmoved,
                                     w.info, (Acc *)w.Tg, (Acc *)w.Pglob, w.ldet));
    LYAP_TRY(launched());
    const int rows = k + std::max(0, R - b);                 // above the panel + below the block
    if (rows > 0)
        gje_xabove_kernel<T><<<std::min(ceil_div(rows, 128), 1184), 128, 0, s>>>(n, k, b, R, (const T *)A, (const Acc *)w.Tg,
                                                                               (const Acc *)w.Pglob, (T *)w.X);
    return launched();
}

// C (M x N, row-major, ld ldc) += A (M x K, row-major) B^T (B: N x K row-major) for the
// two-level sweep: tcgen05 for the 16-bit types, the 128 x 128 SIMT kernel for fp32.
template <typename T>
static int outer_gemm(cudaStream_t s, int M, int N, int K, const T *A, long lda, const T *B, long ldb, T *C,
                      long ldc, int cap = 0)
{
    if constexpr (std::is_same<T, float>::value)
        return gemm_strided<float, float, float, float>(s, M, N, K, 1.0f, A, lda, 1, B, 1, ldb, 1.0f, C, ldc, 1);
    else {
        // the rank-32 steps as in gje_ip.cu (same kernel: the two sweeps stay bitwise equal)
        if (K == 32 && lda == 32 && ldb == 32 && rank32_update_ok(Prec<T>::code, N, A, B, C, ldc))
            return rank32_update(s, Prec<T>::code, M, N, A, B, C, ldc);
        return tc_gemm(s, Prec<T>::code, M, N, K, 1.0f, A, lda, B, ldb, 1.0f, C, ldc, 0, cap);
    }
}

template <typename T>
static int gje_invert_t(cudaStream_t s, int n, T *A, GjeWork &w)
{
    using Acc = typename Prec<T>::acc;
    const int b0 = gje_panel_width(Prec<T>::code);
    LYAP_CUDA_TRY(cudaMemsetAsync(w.info, 0, sizeof(int), s));
    LYAP_CUDA_TRY(cudaMemsetAsync(w.ldet, 0, sizeof(double) * (size_t)n, s));
    iota_kernel<<<ceil_div(n, 256), 256, 0, s>>>(n, w.rowperm);
    LYAP_TRY(launched());
    // two-level blocking for the 16-bit types and fp32: inner 32-wide steps restricted to an
    // outer block of NB columns, then one rank-NB update of the rest (tcgen05 / SIMT fp32)
    constexpr bool half_t = std::is_same<T, __half>::value || std::is_same<T, __nv_bfloat16>::value;
    constexpr bool f32_t = std::is_same<T, float>::value;
    const bool two_level = (half_t || f32_t) && !(half_t && use_simt_gemm()) && n % 8 == 0 && n >= 2 * GJE_NB &&
                           w.Bo != nullptr && !env_flag("LYAP_GJE_1LEVEL");
    const int NBo = two_level ? GJE_NB : n;
    // look-ahead (two-level only): the inner steps (pivot panels) of block K0+NB run on the
    // high-priority side stream P while the main stream finishes the outer update of block
    // K0; the next block's columns are updated first so P can start early.
    // Opt-in (LYAP_GJE_LOOKAHEAD=1): with outer blocks of 512 it measured no faster than the
    // serial order at n = 16384 (74.2 ms either way) and occasionally much slower (one run
    // in ~12 at 270 ms: the 16-CTA panel cluster cannot always be placed beside the capped
    // persistent GEMM, so it waits for the whole update).
    const bool ahead = two_level && w.side != nullptr && env_flag("LYAP_GJE_LOOKAHEAD");
    cudaStream_t P = ahead ? w.side : s;
    if (ahead) {
        LYAP_CUDA_TRY(cudaEventRecord(w.ev_a, s));
        LYAP_CUDA_TRY(cudaStreamWaitEvent(P, w.ev_a, 0));
    }
    for (int K0 = 0; K0 < n; K0 += NBo) {
        const int nbk = std::min(NBo, n - K0);
        if (two_level && n - nbk > 0) {
            gje_inv_snapshot_kernel<<<std::min(ceil_div(n, 256), 592), 256, 0, P>>>(n, w.rowperm, w.invprev);
            LYAP_TRY(launched());
        }
        const int c0 = two_level ? K0 : 0, c1 = two_level ? K0 + nbk : n;
        for (int k = K0; k < K0 + nbk; k += b0) {
            const int b = std::min(b0, K0 + nbk - k);
            {
                // algorithmic work: panel LU ~ (n-k) b^2 flops + multiplier block X 2 n b^2
                KTimer kt(KC_GJE_PANEL, P, (double)(n - k) * b * b + 2.0 * n * b * b,
                          (double)sizeof(T) * ((double)(n - k) * b + (double)n * b));
                LYAP_TRY(gje_panel_launch<T>(P, n, k, b, A, w));
            }
            LYAP_TRY(launched());
            dim3 gg(ceil_div(c1 - c0, 256) < 8 ? ceil_div(c1 - c0, 256) : 8, 2 * b);
            gje_gather_kernel<T><<<gg, 256, 0, P>>>(n, k, c0, c1, A, w.moved, w.nmoved, (T *)w.tmp, w.rowperm,
                                                    w.tmp_perm);
            LYAP_TRY(launched());
            dim3 gp(std::min(ceil_div(c1 - c0, 256), 8), 3 * b + std::min(ceil_div((long)n * b, 8 * 256), 512));
            gje_prep_kernel<T><<<gp, 256, 0, P>>>(n, k, b, c0, c1, A, w.moved, w.nmoved, (const T *)w.tmp,
                                                  w.tmp_perm, w.rowperm, (T *)w.B);
            LYAP_TRY(launched());
            {
                KTimer kt(KC_GJE_UPDATE, P);
                if (two_level)
                    LYAP_TRY(outer_gemm<T>(P, n, nbk, b, (const T *)w.X, b, (const T *)w.B + (size_t)K0 * b, b, A + K0, n));
                else
                    LYAP_TRY(gemm_update(P, n, b, (const T *)w.X, (const T *)w.B, A));
            }
        }
        if (ahead) {
            LYAP_CUDA_TRY(cudaEventRecord(w.ev_b, P));             // inner steps of this block done
            LYAP_CUDA_TRY(cudaStreamWaitEvent(s, w.ev_b, 0));
        }
        if (two_level && n - nbk > 0) {
            LYAP_CUDA_TRY(cudaMemsetAsync(w.onmoved, 0, sizeof(int), s));
            LYAP_CUDA_TRY(cudaMemsetAsync(w.slot_of, 0xFF, sizeof(int) * GJE_NB, s));
            gje_outer_perm2_kernel<<<std::min(ceil_div(n - K0, 256), 592), 256, 0, s>>>(n, K0, nbk, w.rowperm, w.invprev,
                                                                                      w.omoved, w.onmoved, w.slot_of);
            LYAP_TRY(launched());
            // moved rows: one CTA row per list slot, 8 CTAs across the columns (the grid is
            // sized for the 2 nb possible slots; unused slots exit at once)
            const int gx = std::min(ceil_div(n - nbk, 256), 8);
            gje_outer_gather_kernel<T><<<dim3(gx, 2 * nbk), 256, 0, s>>>(n, K0, nbk, A, w.omoved, w.onmoved,
                                                                       (T *)w.tmp2);
            LYAP_TRY(launched());
            gje_outer_scatter_kernel<T><<<dim3(std::min(ceil_div(n - nbk, 32), 592), 1), 256, 0, s>>>(
                n, K0, nbk, A, w.omoved, w.onmoved, (const T *)w.tmp2, (T *)w.Bo, w.slot_of, 0);
            LYAP_TRY(launched());
            gje_outer_scatter_kernel<T><<<dim3(gx, 2 * nbk), 256, 0, s>>>(
                n, K0, nbk, A, w.omoved, w.onmoved, (const T *)w.tmp2, (T *)w.Bo, w.slot_of, 1);
            LYAP_TRY(launched());
            KTimer kt(KC_GJE_UPDATE, s);
            // A[:, rest] += X_outer B_outer, X_outer = the block columns (ld n); the next
            // block's columns first, then (look-ahead) the side stream may start on them
            const int cr = K0 + nbk;
            const int cn = ahead ? std::min(n, cr + NBo) : cr;
            if (ahead && cn > cr) {
                LYAP_TRY(outer_gemm<T>(s, n, cn - cr, nbk, A + K0, n, (const T *)w.Bo + (size_t)cr * nbk, nbk, A + cr, n));
                LYAP_CUDA_TRY(cudaEventRecord(w.ev_a, s));
                LYAP_CUDA_TRY(cudaStreamWaitEvent(P, w.ev_a, 0));
            }
            // with look-ahead, leave SMs for the pivot-panel cluster running concurrently on P
            const int cap = ahead ? 148 - 16 : 0;
            if (K0 > 0)
                LYAP_TRY(outer_gemm<T>(s, n, K0, nbk, A + K0, n, (const T *)w.Bo, nbk, A, n, cap));
            if (cn < n)
                LYAP_TRY(outer_gemm<T>(s, n, n - cn, nbk, A + K0, n, (const T *)w.Bo + (size_t)cn * nbk, nbk, A + cn, n,
                                       cap));
        }
    }
    invperm_kernel<<<ceil_div(n, 256), 256, 0, s>>>(n, w.rowperm, w.invperm);
    return launched();
}

// A += X (n x b, row-major) * B (b x n, row-major); fp32 (fp64) accumulation.
template <typename T>
int gemm_update(cudaStream_t s, int n, int b, const T *X, const T *B, T *A)
{
    using Acc = typename Prec<T>::acc;
    // B holds the pivot rows transposed (Bt, n x b row-major): A += X Bt^T
    if constexpr (std::is_same<T, __half>::value || std::is_same<T, __nv_bfloat16>::value) {
        if (!use_simt_gemm() && b == 32 && rank32_update_ok(Prec<T>::code, n, X, B, A, n))
            return rank32_update(s, Prec<T>::code, n, n, X, B, A, n);
        if (!use_simt_gemm() && b % 8 == 0)     // TMA rows must be 16-byte multiples
            return tc_gemm(s, Prec<T>::code, n, n, b, 1.0f, X, b, B, b, 1.0f, A, n, 0);
    }
    return gemm_strided<T, T, T, Acc>(s, n, n, b, Acc(1), X, b, 1, B, 1, b, Acc(1), A, n, 1);
}
template int gemm_update<double>(cudaStream_t, int, int, const double *, const double *, double *);
template int gemm_update<float>(cudaStream_t, int, int, const float *, const float *, float *);
template int gemm_update<__half>(cudaStream_t, int, int, const __half *, const __half *, __half *);
template int gemm_update<__nv_bfloat16>(cudaStream_t, int, int, const __nv_bfloat16 *, const __nv_bfloat16 *, __nv_bfloat16 *);

int gje_invert(cudaStream_t s, int n, int prec, void *A, GjeWork &w)
{
    switch (prec) {
        case LYAP_FP64: return gje_invert_t<double>(s, n, (double *)A, w);
        case LYAP_FP32: return gje_invert_t<float>(s, n, (float *)A, w);
        case LYAP_FP16: return gje_invert_t<__half>(s, n, (__half *)A, w);
        case LYAP_BF16: return gje_invert_t<__nv_bfloat16>(s, n, (__nv_bfloat16 *)A, w);
    }
    return LYAP_ERR_ARG;
}

int col_gather(cudaStream_t s, int n, int prec, const void *G, const int *invperm, void *out)
{
    dim3 g(ceil_div(n, 256) < 8 ? ceil_div(n, 256) : 8, n < 8192 ? n : 8192);
    switch (prec) {
        case LYAP_FP64: col_gather_kernel<double><<<g, 256, 0, s>>>(n, (const double *)G, invperm, (double *)out); break;
        case LYAP_FP32: col_gather_kernel<float><<<g, 256, 0, s>>>(n, (const float *)G, invperm, (float *)out); break;
        case LYAP_FP16: col_gather_kernel<__half><<<g, 256, 0, s>>>(n, (const __half *)G, invperm, (__half *)out); break;
        case LYAP_BF16: col_gather_kernel<__nv_bfloat16><<<g, 256, 0, s>>>(n, (const __nv_bfloat16 *)G, invperm, (__nv_bfloat16 *)out); break;
        default: return LYAP_ERR_ARG;
    }
    return launched();
}

}  // namespace lyap

// ------------------------------------------------------------------ C ABI
extern "C" int lyap_invert(int n, int prec, void *A, int *ipiv, void *stream)
{
    using namespace lyap;
    if (n <= 0 || A == nullptr || prec < 0 || prec > 3) return LYAP_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    GjeWork w;
    LYAP_TRY(w.alloc(n, prec));
    void *out = nullptr;
    int rc = LYAP_OK;
    if (cudaMalloc(&out, elem_size(prec) * (size_t)n * n) != cudaSuccess) { w.release(); return LYAP_ERR_CUDA; }
    if (gje_ip_eligible(n, prec, w)) {
        rc = gje_ip_invert(s, n, prec, A, out, w);
        if (rc == LYAP_OK) rc = col_gather(s, n, prec, out, w.invperm, A);
    } else {
        rc = gje_invert(s, n, prec, A, w);
        if (rc == LYAP_OK) rc = col_gather(s, n, prec, A, w.invperm, out);
        if (rc == LYAP_OK && cudaMemcpyAsync(A, out, elem_size(prec) * (size_t)n * n, cudaMemcpyDeviceToDevice, s) != cudaSuccess) rc = LYAP_ERR_CUDA;
    }
    if (rc == LYAP_OK && ipiv && cudaMemcpyAsync(ipiv, w.ipiv, sizeof(int) * n, cudaMemcpyDeviceToDevice, s) != cudaSuccess) rc = LYAP_ERR_CUDA;
    int info = 0;
    if (rc == LYAP_OK && cudaMemcpyAsync(&info, w.info, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess) rc = LYAP_ERR_CUDA;
    if (cudaStreamSynchronize(s) != cudaSuccess) rc = LYAP_ERR_CUDA;
    cudaFree(out);
    w.release();
    if (rc == LYAP_OK && info != 0) rc = LYAP_ERR_SINGULAR;
    return rc;
}
