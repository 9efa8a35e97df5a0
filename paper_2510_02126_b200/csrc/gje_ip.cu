// gje_ip.cu -- blocked Gauss-Jordan inversion with IMPLICIT partial pivoting for the
// Newton step A_k = (mu A_{k-1} + mu^{-1} A_{k-1}^{-1})/2 (PAPER.md Eq. newton-lyapu1 l.1125),
// 16-bit and fp32 storage, two-level blocking (gje.cu holds the row-swapping sweep that the
// fp64 path, ragged orders and small matrices use; both choose the same pivots and perform
// the same arithmetic on every matrix element, so their results are bitwise equal).
//
// Rows never move.  Physical row r carries its logical position pos[r] (the position
// LU with partial pivoting would have swapped it to): pos < k are finished pivot rows,
// pos >= k are still active.  A "row interchange" exchanges two positions in registers;
// the pivot search breaks ties by the lowest logical position, which is LAPACK's rule.
// With that the sweep needs no gather / scatter of moved rows at either blocking level,
// and one panel kernel per 32 columns does everything except the rank-32 update GEMM:
//
//   panel kernel (one cluster of up to 16 CTAs, one matrix row per thread, ALL n rows):
//     * 32 pivot steps.  Per step each warp leaves its best candidate (row + key) in
//       shared memory, one CTA barrier, one warp per destination CTA picks the CTA's
//       winner and pushes it into every CTA's inbox with st.async (completion counted on
//       the destination's mbarrier: no cluster barrier, no fence), every thread waits on
//       its own CTA's mbarrier, picks the cluster winner from the inbox and eliminates its
//       row.  The pushed pivot row is row j of the block's LU factors, so every CTA
//       collects L11/U11 as a by-product;
//     * every CTA forms Linv, Uinv, T = U11^{-1} L11^{-1} (redundantly: no exchange);
//     * every thread exports its row's multipliers (active rows) or panel entries (finished
//       rows) in fp32, CTA 0 exports T and Linv;
//     * the cluster copies the 32 pivot rows' block columns into B (K-major for the update,
//       B[:, panel] = I) and zeroes them;
//   then A[:, block] += X B with X = [-a T ; T ; -l Linv] formed tile by tile inside the
//   rank-32 update kernel (rank_update.cu; fp32 storage: X in the panel or by gje_ip_x_kernel,
//   update on the SIMT GEMM).
// After the 8 panels of an outer block of 256 columns, one kernel moves the 256 pivot rows'
// remaining entries into B_outer and the tensor cores (tcgen05) apply the rank-256 update; the
// next block's panels run beside it on a second stream (look-ahead).  At the end M_phys holds
// A^{-1}[pos[r], piv(c)] = M_phys[r, c]; a row-gathering copy writes G[i, :] = M_phys[piv(i), :],
// the layout the Newton update and the Z-side consume (A^{-1}[i][l] = G[i][invperm[l]],
// rowperm = piv, invperm = pos).
#include <cooperative_groups.h>
#include "common.cuh"
#include "gemm_simt.cuh"
#include "lyap_internal.h"
#include "ktimer.h"
#include "ptx.cuh"

namespace lyap {

namespace {

constexpr int BW = 32;                 // panel width
constexpr int SLOTW = 36;              // candidate record: 32 row entries, key, ~pos, physical row, pad (144 B)

__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
// 16-byte asynchronous store into a (remote) CTA's shared memory; the bytes are counted on
// that CTA's mbarrier (both addresses shared::cluster)
__device__ __forceinline__ void st_async_v4(uint32_t dst, const float4 &v, uint32_t mbar) {
    asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];"
                 :: "r"(dst), "r"(__float_as_uint(v.x)), "r"(__float_as_uint(v.y)), "r"(__float_as_uint(v.z)),
                    "r"(__float_as_uint(v.w)), "r"(mbar) : "memory");
}

// (key, npos) lexicographic maximum over the lanes with `in`; returns the winning lane
// (keys: 0 = no candidate; npos = ~position, so the lowest position wins ties)
__device__ __forceinline__ int warp_pick(unsigned key, unsigned npos) {
    const unsigned mx = __reduce_max_sync(0xffffffffu, key);
    unsigned who = __ballot_sync(0xffffffffu, key == mx);
    if (who & (who - 1)) {                                       // tie (rare): lowest position
        const unsigned pk = (key == mx) ? npos : 0u;
        const unsigned mp = __reduce_max_sync(0xffffffffu, pk);
        who = __ballot_sync(0xffffffffu, key == mx && pk == mp);
    }
    return __ffs(who) - 1;
}

template <typename T> struct Ld16;
template <> struct Ld16<__half> {
    static constexpr int E = 8;
    __device__ __forceinline__ static void unpack(const uint4 &v, float *o) {
        const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; i++) {
            o[2 * i] = __half2float(__ushort_as_half((unsigned short)(w[i] & 0xffffu)));
            o[2 * i + 1] = __half2float(__ushort_as_half((unsigned short)(w[i] >> 16)));
        }
    }
    __device__ __forceinline__ static uint4 pack(const float *x) {
        unsigned w[4];
#pragma unroll
        for (int i = 0; i < 4; i++)
            w[i] = (unsigned)__half_as_ushort(__float2half_rn(x[2 * i])) |
                   ((unsigned)__half_as_ushort(__float2half_rn(x[2 * i + 1])) << 16);
        return make_uint4(w[0], w[1], w[2], w[3]);
    }
};
template <> struct Ld16<__nv_bfloat16> {
    static constexpr int E = 8;
    __device__ __forceinline__ static void unpack(const uint4 &v, float *o) {
        const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; i++) {
            o[2 * i] = __uint_as_float(w[i] << 16);
            o[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
        }
    }
    __device__ __forceinline__ static uint4 pack(const float *x) {
        unsigned w[4];
#pragma unroll
        for (int i = 0; i < 4; i++)
            w[i] = (unsigned)__bfloat16_as_ushort(__float2bfloat16_rn(x[2 * i])) |
                   ((unsigned)__bfloat16_as_ushort(__float2bfloat16_rn(x[2 * i + 1])) << 16);
        return make_uint4(w[0], w[1], w[2], w[3]);
    }
};
template <> struct Ld16<float> {
    static constexpr int E = 4;
    __device__ __forceinline__ static void unpack(const uint4 &v, float *o) {
        o[0] = __uint_as_float(v.x); o[1] = __uint_as_float(v.y); o[2] = __uint_as_float(v.z); o[3] = __uint_as_float(v.w);
    }
    __device__ __forceinline__ static uint4 pack(const float *x) {
        return make_uint4(__float_as_uint(x[0]), __float_as_uint(x[1]), __float_as_uint(x[2]), __float_as_uint(x[3]));
    }
};

// explicit shared-memory accesses by 32-bit address: the column loop keeps its addresses in
// registers (generic pointers made ptxas recompute the cluster window base, an S2R, per access)
__device__ __forceinline__ void sts128(uint32_t a, float x, float y, float z, float w) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" :: "r"(a), "f"(x), "f"(y), "f"(z), "f"(w) : "memory");
}
__device__ __forceinline__ void sts32(uint32_t a, float x) {
    asm volatile("st.shared.f32 [%0], %1;" :: "r"(a), "f"(x) : "memory");
}
__device__ __forceinline__ float4 lds128(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ uint2 lds64u(uint32_t a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void mbar_expect_tx_a(uint32_t a, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_a(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" :: "r"(a), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_s2c(uint32_t dst_cluster, uint32_t src_cta, uint32_t bytes, uint32_t mbar_cluster) {
    asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(dst_cluster), "r"(src_cta), "r"(bytes), "r"(mbar_cluster) : "memory");
}

// Panel of the block columns [k, k+32) inside the outer block [K0, K0+nbk); see the header.
// pos_g[r]: logical position of physical row r (in/out); piv[i]: physical row at position i.
//
// Register layout: an active row keeps only its not yet eliminated entries, shifted so that
// the current column j is element 0 (row[c] = a_{r, k+j+c}; elements beyond 31-j are dead).
// The elimination of step j writes row[c-1] = row[c] - l u_c in place, so the column loop is
// rolled (runtime j) with compile-time register indices: the body stays in the instruction
// cache (a fully unrolled loop executes every instruction once, from a cold cache).  The
// multipliers l_{r,j} go to the thread's column of Lsm (shared memory), which finished rows
// fill with their panel entries at the start: the X phase reads both from there.
// XOUT: the X rows are formed by gje_ip_x_kernel on the whole GPU (large n: one panel row per
// thread on 16 SMs makes n x 32 x 32 multiply-adds a long tail); the panel then only exports
// the active rows' multipliers (Pg), T and Linv (Tg).
template <typename T, int NT, int RPT, bool XOUT>
__global__ void __launch_bounds__(NT)
gje_ip_panel_kernel(int n, int k, int K0, int nbk, T *__restrict__ A, T *__restrict__ X, T *__restrict__ B,
                    int *__restrict__ pos_g, int *__restrict__ piv, int *__restrict__ ipiv, int *__restrict__ info,
                    double *__restrict__ ldet, float *__restrict__ Pg, float *__restrict__ Tg)
{
    constexpr int NW = NT / 32;
    constexpr int VE = Ld16<T>::E;
    constexpr int LS = NT * RPT + 1;                             // Lsm row stride (odd: conflict-free both ways)
    constexpr int RB = NT * RPT;                                 // rows per CTA
    uint32_t q, NC;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(q));
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(NC));
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

    extern __shared__ __align__(16) float Lsm[];                 // [32][LS] multipliers / finished rows
    __shared__ __align__(16) float slot[2][NW][SLOTW];          // per-warp candidates (double buffered)
    __shared__ __align__(16) float inbox[2][16][SLOTW];         // one record per source CTA
    __shared__ __align__(8) uint64_t mbar[3];                    // two column buffers, L11 exchange
    __shared__ __align__(16) float PU[32][32];                   // U11 (row j = pivot row of step j, from column j)
    __shared__ __align__(128) float PL[32][32];                  // L11, strictly lower (copied in by the rows' owners)
    __shared__ __align__(128) float PLs[32][32];                 // staging of this CTA's rows of L11
    __shared__ __align__(16) float Lw[32 * 32], Tw[32 * 32];
    __shared__ float rdiag[32];
    __shared__ int pivl[32], pivphys[32];
    __shared__ int sflag;

#ifdef LYAP_PANEL_PROF
    long long tp[10]; int tpn = 0;
#define IPPROF() do { if (tid == 0 && q == 0) tp[tpn++] = clock64(); } while (0)
#else
#define IPPROF() do { } while (0)
#endif
    IPPROF();
    // programmatic dependent launch: the next kernel of the stream may set up beside this one
    // (it waits for this grid's completion before it reads or writes anything)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (tid == 0) {
        ptx::mbar_init(&mbar[0], 1);
        ptx::mbar_init(&mbar[1], 1);
        ptx::mbar_init(&mbar[2], 1);
        ptx::fence_mbar_init();
        ptx::mbar_arrive_expect_tx(&mbar[2], 32 * 32 * 4);       // 32 rows of L11, 128 bytes each
        sflag = 0;
    }
    // the cluster barrier that publishes the mbarrier initialisation is split: arrive here, wait
    // after the row loads (their latency hides it)
    __syncthreads();
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    // (programmatic dependent launch: barrier setup above overlaps the previous kernel's tail)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // rows: thread tid of CTA q owns physical rows q RB + RPT tid + h
    float row[RPT][BW];
    int pos[RPT];
    const int r0 = (int)q * RB + RPT * tid;
#pragma unroll
    for (int h = 0; h < RPT; h++) {
        const int r = r0 + h;
        if (r < n) {
            const uint4 *src = reinterpret_cast<const uint4 *>(A + (long)r * n + k);
            uint4 v[BW / VE];
#pragma unroll
            for (int u = 0; u < BW / VE; u++) v[u] = src[u];
#pragma unroll
            for (int u = 0; u < BW / VE; u++) Ld16<T>::unpack(v[u], &row[h][u * VE]);
            pos[h] = pos_g[r];
        } else {
#pragma unroll
            for (int c = 0; c < BW; c++) row[h][c] = 0.f;
            pos[h] = -1;                                         // never a candidate, never eliminated
        }
        if (!XOUT && pos[h] < k) {
#pragma unroll
            for (int c = 0; c < BW; c++) Lsm[c * LS + h * NT + tid] = row[h][c];
        }
    }
    IPPROF();
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");   // barriers initialised cluster-wide
    IPPROF();

    // loop-invariant shared addresses (buffer 0; buffer 1 at a constant offset)
    const uint32_t a_slot = ptx::smem_addr(&slot[0][0][0]);
    const uint32_t a_inbox = ptx::smem_addr(&inbox[0][0][0]);
    const uint32_t a_mbar = ptx::smem_addr(&mbar[0]);
    const uint32_t a_lsm = ptx::smem_addr(&Lsm[0]);
    constexpr uint32_t SLOT_B = NW * SLOTW * 4, INBOX_B = 16 * SLOTW * 4;
    const uint32_t a_myslot = a_slot + (uint32_t)wid * SLOTW * 4;
    // pusher warp w (and w + NW, ...): remote inbox slot of this CTA and remote barrier, per destination
    constexpr int ND = (16 + NW - 1) / NW;
    uint32_t r_inbox[ND], r_mbar[ND];
#pragma unroll
    for (int i = 0; i < ND; i++) {
        const int dc = wid + i * NW;
        r_inbox[i] = mapa(a_inbox + (uint32_t)(((int)q * SLOTW + (lane < SLOTW / 4 ? lane : 0) * 4) * 4), (uint32_t)(dc < (int)NC ? dc : 0));
        r_mbar[i] = mapa(a_mbar, (uint32_t)(dc < (int)NC ? dc : 0));
    }
    // LATE (512-thread CTAs): only the warps' keys go to shared memory before the barrier and
    // the CTA's winning warp stages and pushes its record afterwards -- every store in flight at
    // a __syncthreads costs ~5 cycles on the SM, nine STS.128 per warp 400-1300 cycles per
    // column.  With 8 warps the early staging is cheaper than the longer chain (measured: 1690 vs
    // 1960 cycles per column at n = 1024; 2430 vs 2350 at n = 16384 with 16 warps x 2 rows).
#ifdef LYAP_IP_LATE_ALL
    constexpr bool LATE = true;
#else
    constexpr bool LATE = NT >= 512;
#endif
    // LATE: lane -> (destination CTA, 16-byte chunk) tasks of the winning warp
    constexpr int NTASK = (16 * (SLOTW / 4) + 31) / 32;          // 144 tasks at 16 CTAs: 5 per lane
    uint32_t t_inbox[LATE ? NTASK : 1], t_mbar[LATE ? NTASK : 1], t_chunk[LATE ? NTASK : 1];
    if constexpr (LATE) {
#pragma unroll
        for (int i = 0; i < NTASK; i++) {
            const int task = lane + 32 * i, dc = task / (SLOTW / 4), ch = task - dc * (SLOTW / 4);
            const uint32_t d = (uint32_t)(dc < (int)NC ? dc : 0);
            t_chunk[i] = (uint32_t)ch * 16u;
            t_inbox[i] = mapa(a_inbox + (uint32_t)((int)q * SLOTW * 4) + (uint32_t)ch * 16u, d);
            t_mbar[i] = mapa(a_mbar, d);
        }
    }
    const uint32_t tx_bytes = NC * SLOTW * 4;

#pragma unroll 1
    for (int j = 0; j < BW; j++) {
        const uint32_t buf = (uint32_t)j & 1u;
        const int lp = k + j;                                    // the position this step fills
        if (tid == NT - 32) mbar_expect_tx_a(a_mbar + buf * 8u, tx_bytes);
        // ---- this thread's candidate, then the warp's: largest |a_rj| among active rows,
        // lowest position on ties.  key >= 1 for every active row (0 and NaN rank lowest).
        unsigned key = 0u, npos = 0u;
        int hsel = 0;
#pragma unroll
        for (int h = 0; h < RPT; h++) {
            const float v = fabsf(row[h][0]);
            const bool act = pos[h] >= lp;
            const unsigned kk = act ? ((v > 0.f) ? __float_as_uint(v) + 1u : 1u) : 0u;
            const unsigned pp = act ? ~(unsigned)pos[h] : 0u;
            if (kk > key || (kk == key && pp > npos)) { key = kk; npos = pp; hsel = h; }
        }
        if constexpr (LATE) {
            // every thread's reciprocal before the barrier (beside the reductions), so the
            // division is not on the chain after it
            float rinv_h[RPT];
#pragma unroll
            for (int h = 0; h < RPT; h++) rinv_h[h] = (row[h][0] != 0.f) ? 1.f / row[h][0] : 0.f;
            const int wl = warp_pick(key, npos);                 // the warp's best lane
            const uint32_t sa = a_myslot + buf * SLOT_B;
            if (lane == wl) sts128(sa + BW * 4, __uint_as_float(key), __uint_as_float(npos), 0.f, 0.f);
            __syncthreads();
            uint2 m2 = make_uint2(0u, 0u);
            if (lane < NW) m2 = lds64u(a_slot + buf * SLOT_B + (uint32_t)lane * SLOTW * 4 + BW * 4);
            const int ws = warp_pick(m2.x, m2.y);                // the CTA's best warp
            if (wid == ws) {
                if (lane == wl) {
#pragma unroll
                    for (int h = 0; h < RPT; h++)
                        if (h == hsel) {
#pragma unroll
                            for (int c = 0; c < BW; c += 4) sts128(sa + c * 4, row[h][c], row[h][c + 1], row[h][c + 2], row[h][c + 3]);
                            sts128(sa + BW * 4, __uint_as_float(key), __uint_as_float(npos), __int_as_float(r0 + h), rinv_h[h]);
                        }
                }
                __syncwarp();
#pragma unroll
                for (int i = 0; i < NTASK; i++)
                    if (lane + 32 * i < (int)NC * (SLOTW / 4))
                        st_async_v4(t_inbox[i] + buf * INBOX_B, lds128(sa + t_chunk[i]), t_mbar[i] + buf * 8u);
            }
        } else {
        {
            const unsigned mx = __reduce_max_sync(0xffffffffu, key);
            const uint32_t sa = a_myslot + buf * SLOT_B;
            if (mx == 0u) {                                      // no active row in this warp: key only
                if (lane == 0) sts128(sa + BW * 4, 0.f, 0.f, 0.f, 0.f);
            } else {
                unsigned who = __ballot_sync(0xffffffffu, key == mx);
                if (who & (who - 1)) {                           // tie (rare): lowest position
                    const unsigned pk = (key == mx) ? npos : 0u;
                    const unsigned mp = __reduce_max_sync(0xffffffffu, pk);
                    who = __ballot_sync(0xffffffffu, key == mx && pk == mp);
                }
                if (lane == __ffs(who) - 1) {
#pragma unroll
                    for (int h = 0; h < RPT; h++)
                        if (h == hsel) {
                            // the candidate's reciprocal travels with it
                            const float rinv = (row[h][0] != 0.f) ? 1.f / row[h][0] : 0.f;
#pragma unroll
                            for (int c = 0; c < BW; c += 4) sts128(sa + c * 4, row[h][c], row[h][c + 1], row[h][c + 2], row[h][c + 3]);
                            sts128(sa + BW * 4, __uint_as_float(key), __uint_as_float(npos), __int_as_float(r0 + h), rinv);
                        }
                }
            }
        }
        __syncthreads();
        // ---- warp w < NC: the CTA's winner goes to the inbox of CTA w (w + NW, ...)
        if (wid < (int)NC) {
            uint2 m2 = make_uint2(0u, 0u);
            if (lane < NW) m2 = lds64u(a_slot + buf * SLOT_B + (uint32_t)lane * SLOTW * 4 + BW * 4);
            const int ws = warp_pick(m2.x, m2.y);
            if (lane < SLOTW / 4) {
                const float4 v = lds128(a_slot + buf * SLOT_B + (uint32_t)ws * SLOTW * 4 + (uint32_t)lane * 16);
#pragma unroll
                for (int i = 0; i < ND; i++)
                    if (wid + i * NW < (int)NC) st_async_v4(r_inbox[i] + buf * INBOX_B, v, r_mbar[i] + buf * 8u);
            }
        }
        }
        mbar_wait_a(a_mbar + buf * 8u, (uint32_t)((j >> 1) & 1));
        // ---- cluster winner (every warp, from its CTA's inbox)
        uint2 m3 = make_uint2(0u, 0u);
        if (lane < (int)NC) m3 = lds64u(a_inbox + buf * INBOX_B + (uint32_t)lane * SLOTW * 4 + BW * 4);
        const int cs = warp_pick(m3.x, m3.y);
        const uint32_t a_prow = a_inbox + buf * INBOX_B + (uint32_t)cs * SLOTW * 4;
        const float4 meta = lds128(a_prow + BW * 4);            // key, ~pos, physical row, 1 / pivot
        const int pr = (int)~__float_as_uint(meta.y);
        const float inv = meta.w;                                // (d != 0) ? 1 / d : 0, from the row's owner
        float l[RPT];
        bool el[RPT];
#pragma unroll
        for (int h = 0; h < RPT; h++) {
            int p = pos[h];
            p = (p == pr) ? lp : ((p == lp) ? pr : p);           // the interchange, on positions only
            pos[h] = p;
            el[h] = p > lp;
            l[h] = row[h][0] * inv;
            if (el[h]) sts32(a_lsm + (uint32_t)((j * LS + h * NT + tid) * 4), l[h]);
        }
        // ---- elimination: row[c-1] = row[c] - l u_c.  Entries beyond 31-j are dead (their
        // values are never read), so the groups run unconditionally: columns 1..15 of the
        // window always, 16..31 while j < 16 -- one uniform branch per step (branches cost
        // more than the wasted multiply-adds on this latency chain).
#pragma unroll
        for (int half = 0; half < 2; half++) {
            if (half == 1 && j >= 16) break;
            float4 pv[4];
#pragma unroll
            for (int g = 0; g < 4; g++) pv[g] = lds128(a_prow + (uint32_t)(half * 4 + g) * 16);
#pragma unroll
            for (int g = 0; g < 4; g++) {
                const int G = half * 4 + g;
#pragma unroll
                for (int h = 0; h < RPT; h++)
                    if (el[h]) {
                        if (G > 0) row[h][4 * G - 1] = fmaf(-l[h], pv[g].x, row[h][4 * G]);
                        row[h][4 * G + 0] = fmaf(-l[h], pv[g].y, row[h][4 * G + 1]);
                        row[h][4 * G + 1] = fmaf(-l[h], pv[g].z, row[h][4 * G + 2]);
                        row[h][4 * G + 2] = fmaf(-l[h], pv[g].w, row[h][4 * G + 3]);
                    }
            }
        }
        if (wid == NW - 1) {                                     // bookkeeping: row j of U11 (off the chain)
            if (j + lane < BW) PU[j][j + lane] = inbox[buf][cs][lane];
            if (lane == 0) {
                pivl[j] = pr;
                pivphys[j] = __float_as_int(meta.z);
                rdiag[j] = inv;
                if (inv == 0.f && sflag == 0) sflag = lp + 1;
            }
        }
    }
    IPPROF();
    __syncthreads();                                             // pivphys complete
    // ---- L11: the CTA owning pivot row j stages l_{j, t < j} and copies it to every CTA's PL[j]
    for (int j = wid; j < BW; j += NW) {
        const int local = pivphys[j] - (int)q * RB;
        if (local < 0 || local >= RB) continue;                  // (warp-uniform)
        const int ot = local / RPT, oh = local - ot * RPT;
        PLs[j][lane] = (lane < j) ? Lsm[lane * LS + oh * NT + ot] : 0.f;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane < (int)NC)
            bulk_s2c(mapa(ptx::smem_addr(&PL[j][0]), (uint32_t)lane), ptx::smem_addr(&PLs[j][0]), 128u, mapa(a_mbar + 16u, (uint32_t)lane));
    }
    ptx::mbar_wait(&mbar[2], 0u);
    // all 32 rows of L11 are here: tell the cluster (the matching wait is at the kernel's end)
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    IPPROF();

    // ---- Linv = L11^{-1} (warp 0), Uinv = U11^{-1} (warp 1): column c in the registers of
    // lane c; T = Uinv Linv (all threads).  Summation order as in gje.cu's panels.
    {
        float *Uw = Tw;
        if (wid == 0) {
            const int c = lane;
            float x[32];
#pragma unroll
            for (int i = 0; i < 32; i++) {
                float s = (i == c) ? 1.f : 0.f;
#pragma unroll
                for (int t = 0; t < i; t++) s = fmaf(-PL[i][t], x[t], s);
                x[i] = s;
                Lw[i * 32 + c] = s;
            }
        } else if (wid == 1) {
            const int c = lane;
            float x[32];
#pragma unroll
            for (int i = 31; i >= 0; i--) {
                float s = (i == c) ? 1.f : 0.f;
#pragma unroll
                for (int t = 31; t > i; t--) s = fmaf(-PU[i][t], x[t], s);
                x[i] = (i > c) ? 0.f : s * rdiag[i];
                Uw[i * 32 + c] = x[i];
            }
        } else if (wid == 2 && q == 0) {
            // log|det| contribution (U's diagonal): one fp64 log per lane, summed in order
            const double lg = log(fabs((double)PU[lane][lane]));
            double sl = 0.0;
            for (int j = 0; j < 32; j++) sl += __shfl_sync(0xffffffffu, lg, j);
            piv[k + lane] = pivphys[lane];
            ipiv[k + lane] = pivl[lane];
            if (lane == 0) {
                ldet[k] = sl;
                if (sflag && *info == 0) *info = sflag;
            }
        }
        __syncthreads();
        constexpr int RT = (32 + NW - 1) / NW;
        float tval[RT];
        const int ti = tid / 32, tc = tid % 32;
#pragma unroll
        for (int hh = 0; hh < RT; hh++) {
            tval[hh] = 0.f;
            if (ti + NW * hh < 32)
#pragma unroll
                for (int t = 0; t < BW; t++) tval[hh] = fmaf(Uw[(ti + NW * hh) * 32 + t], Lw[t * 32 + tc], tval[hh]);
        }
        __syncthreads();
#pragma unroll
        for (int hh = 0; hh < RT; hh++)
            if (ti + NW * hh < 32) Tw[(ti + NW * hh) * 32 + tc] = tval[hh];
        __syncthreads();
    }

    IPPROF();
    if constexpr (XOUT) {
        // ---- export: multipliers (active rows), panel entries (finished rows), positions, T and
        // Linv: the X rows are formed by the fused update kernel (or gje_ip_x_kernel).  The rows
        // leave through the warp: finished rows first put their entries into their Lsm column,
        // then lane t writes element t of one row at a time -- 128 contiguous bytes per store
        // instruction (a thread writing its own row touches 32 sectors per instruction: 10 K
        // cycles per panel at n = 16384 against ~4 K this way).
        if constexpr (NT >= 512 || RPT >= 2) {
#pragma unroll
            for (int h = 0; h < RPT; h++) {
                const int r = r0 + h;
                if (r < n) {
                    pos_g[r] = pos[h];
                    if (pos[h] < k) {
#pragma unroll
                        for (int c = 0; c < BW; c++) Lsm[c * LS + h * NT + tid] = row[h][c];
                    }
                }
            }
            __syncwarp();
#pragma unroll
            for (int h = 0; h < RPT; h++) {
#pragma unroll 4
                for (int src = 0; src < 32; src++) {
                    const int ps = __shfl_sync(0xffffffffu, pos[h], src);
                    const int rs = (int)q * RB + RPT * (tid - lane + src) + h;
                    if (rs < n && (ps < k || ps >= k + BW))        // (pivot rows: X = a row of T, nothing to export)
                        Pg[(long)rs * BW + lane] = Lsm[lane * LS + h * NT + (tid - lane + src)];
                }
            }
        } else {
            // 256-thread CTAs: every thread writes its own row (fewer rows per SM: measured equal or
            // slightly faster than the cooperative form, 1.35 vs 1.37 ms per inversion at n = 1024)
#pragma unroll
            for (int h = 0; h < RPT; h++) {
                const int r = r0 + h;
                if (r >= n) continue;
                const int p = pos[h];
                pos_g[r] = p;
                float4 *dst = reinterpret_cast<float4 *>(Pg + (long)r * BW);
                if (p >= k + BW) {
                    const float *lc = &Lsm[h * NT + tid];
#pragma unroll
                    for (int c = 0; c < BW; c += 4) dst[c / 4] = make_float4(lc[c * LS], lc[(c + 1) * LS], lc[(c + 2) * LS], lc[(c + 3) * LS]);
                } else if (p < k) {
#pragma unroll
                    for (int c = 0; c < BW; c += 4) dst[c / 4] = make_float4(row[h][c], row[h][c + 1], row[h][c + 2], row[h][c + 3]);
                }
            }
        }
        if (q == 0)
            for (int e = tid; e < 32 * 32; e += NT) { Tg[e] = Tw[e]; Tg[32 * 32 + e] = Lw[e]; }
    } else {
        // ---- X rows (u_s), panel entries of A zeroed, positions written back
#pragma unroll
        for (int h = 0; h < RPT; h++) {
            const int r = r0 + h;
            if (r >= n) continue;
            const int p = pos[h];
            pos_g[r] = p;
            uint4 *xr = reinterpret_cast<uint4 *>(X + (long)r * BW);
            uint4 *ar = reinterpret_cast<uint4 *>(A + (long)r * n + k);
            if (p >= k && p < k + BW) {
                const float *tr = &Tw[(p - k) * 32];
#pragma unroll
                for (int c0 = 0; c0 < BW; c0 += VE) xr[c0 / VE] = Ld16<T>::pack(tr + c0);
            } else {
                const float *M = (p < k) ? Tw : Lw;
                const float *lc = &Lsm[h * NT + tid];
#pragma unroll
                for (int c0 = 0; c0 < BW; c0 += 8) {
                    float acc[8];
#pragma unroll
                    for (int e = 0; e < 8; e++) acc[e] = 0.f;
#pragma unroll 8
                    for (int t = 0; t < BW; t++) {
                        const float m = -lc[t * LS];
                        const float4 m0 = *reinterpret_cast<const float4 *>(M + t * 32 + c0);
                        const float4 m1 = *reinterpret_cast<const float4 *>(M + t * 32 + c0 + 4);
                        acc[0] = fmaf(m, m0.x, acc[0]); acc[1] = fmaf(m, m0.y, acc[1]);
                        acc[2] = fmaf(m, m0.z, acc[2]); acc[3] = fmaf(m, m0.w, acc[3]);
                        acc[4] = fmaf(m, m1.x, acc[4]); acc[5] = fmaf(m, m1.y, acc[5]);
                        acc[6] = fmaf(m, m1.z, acc[6]); acc[7] = fmaf(m, m1.w, acc[7]);
                    }
                    if constexpr (VE == 8) xr[c0 / 8] = Ld16<T>::pack(acc);
                    else { xr[c0 / 4] = Ld16<T>::pack(acc); xr[c0 / 4 + 1] = Ld16<T>::pack(acc + 4); }
                }
            }
#pragma unroll
            for (int u = 0; u < BW / VE; u++) ar[u] = make_uint4(0u, 0u, 0u, 0u);
        }
    }

    IPPROF();
    // ---- B = the pivot rows' block columns (K-major: B[c][t]), B[:, panel] = I; rows zeroed.
    // One warp per group of VE columns: lane t loads 16 bytes of pivot row t, then VE stores of
    // 64 contiguous bytes (the 32 t of one column) per warp.
    {
        const int ngroups = nbk / VE;
        const long prow_off = (long)pivphys[lane] * n;
        for (int gidx = (int)q * NW + wid; gidx < ngroups; gidx += (int)NC * NW) {
            const int col0 = K0 + gidx * VE;
            uint4 *ap = reinterpret_cast<uint4 *>(A + prow_off + col0);
            float v[VE];
            if (col0 >= k && col0 < k + BW) {
#pragma unroll
                for (int e = 0; e < VE; e++) v[e] = (col0 + e - k == lane) ? 1.f : 0.f;
            } else {
                Ld16<T>::unpack(*ap, v);
            }
            *ap = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
            for (int e = 0; e < VE; e++) B[(long)(col0 + e) * BW + lane] = from_acc<T>(v[e]);
        }
    }
    // no CTA leaves while a peer may not yet have received its L11 rows (the copies read this
    // CTA's staging buffer): every CTA arrived once it held all 32 rows, long ago by now
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
#ifdef LYAP_PANEL_PROF
    IPPROF();
    if (tid == 0 && q == 0 && (k == 0 || k == 544))
        printf("ip panel k=%d n=%d NC=%d NT=%d RPT=%d cycles: load %lld csync %lld loop %lld (%lld/col) Lxchg %lld T %lld X %lld B %lld\n",
               k, n, (int)NC, NT, RPT, tp[1] - tp[0], tp[2] - tp[1], tp[3] - tp[2], (tp[3] - tp[2]) / 32, tp[4] - tp[3],
               tp[5] - tp[4], tp[6] - tp[5], tp[7] - tp[6]);
#endif
}

// X rows for the panel [k, k+32) (XOUT panels): finished rows -a T (a = the row's panel
// entries, still in A), pivot rows T, active rows -l Linv (l from Pg); panel entries of A
// zeroed.  One thread per row; per element the summation order of the in-panel X phase.
template <typename T>
__global__ void __launch_bounds__(128)
gje_ip_x_kernel(int n, int k, T *__restrict__ A, const int *__restrict__ pos_g, const float *__restrict__ Pg,
                const float *__restrict__ Tg, T *__restrict__ X)
{
    constexpr int VE = Ld16<T>::E;
    __shared__ __align__(16) float TL[2][32 * 32];               // T, Linv
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int e = threadIdx.x; e < 2 * 32 * 32; e += blockDim.x) TL[e >> 10][e & 1023] = Tg[e];
    __syncthreads();
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        const int p = pos_g[r];
        uint4 *xr = reinterpret_cast<uint4 *>(X + (long)r * BW);
        uint4 *ar = reinterpret_cast<uint4 *>(A + (long)r * n + k);
        if (p >= k && p < k + BW) {
            const float *tr = &TL[0][(p - k) * 32];
#pragma unroll
            for (int c0 = 0; c0 < BW; c0 += VE) xr[c0 / VE] = Ld16<T>::pack(tr + c0);
        } else {
            float a[BW];
            const float *M;
            if (p < k) {
#pragma unroll
                for (int u = 0; u < BW / VE; u++) Ld16<T>::unpack(ar[u], &a[u * VE]);
                M = TL[0];
            } else {
                const float4 *src = reinterpret_cast<const float4 *>(Pg + (long)r * BW);
#pragma unroll
                for (int u = 0; u < BW / 4; u++) { const float4 v = src[u]; a[4 * u] = v.x; a[4 * u + 1] = v.y; a[4 * u + 2] = v.z; a[4 * u + 3] = v.w; }
                M = TL[1];
            }
#pragma unroll
            for (int c0 = 0; c0 < BW; c0 += 8) {
                float acc[8];
#pragma unroll
                for (int e = 0; e < 8; e++) acc[e] = 0.f;
#pragma unroll
                for (int t = 0; t < BW; t++) {
                    const float m = -a[t];
                    const float4 m0 = *reinterpret_cast<const float4 *>(M + t * 32 + c0);
                    const float4 m1 = *reinterpret_cast<const float4 *>(M + t * 32 + c0 + 4);
                    acc[0] = fmaf(m, m0.x, acc[0]); acc[1] = fmaf(m, m0.y, acc[1]);
                    acc[2] = fmaf(m, m0.z, acc[2]); acc[3] = fmaf(m, m0.w, acc[3]);
                    acc[4] = fmaf(m, m1.x, acc[4]); acc[5] = fmaf(m, m1.y, acc[5]);
                    acc[6] = fmaf(m, m1.z, acc[6]); acc[7] = fmaf(m, m1.w, acc[7]);
                }
                if constexpr (VE == 8) xr[c0 / 8] = Ld16<T>::pack(acc);
                else { xr[c0 / 4] = Ld16<T>::pack(acc); xr[c0 / 4 + 1] = Ld16<T>::pack(acc + 4); }
            }
        }
#pragma unroll
        for (int u = 0; u < BW / VE; u++) ar[u] = make_uint4(0u, 0u, 0u, 0u);
    }
}

// Outer step: the nb pivot rows' entries outside the block columns go to Bo (K-major:
// Bo[c][y]) and are zeroed.  One CTA per tile of 64 columns x 128 pivot rows: 16-byte loads
// along the rows, transposed through shared memory, 16-byte stores along y.
template <typename T>
__global__ void __launch_bounds__(256)
gje_ip_outer_prep_kernel(int n, int K0, int nb, int eb, int ee, T *__restrict__ A, const int *__restrict__ piv,
                         T *__restrict__ Bo)
{
    constexpr int VE = 16 / (int)sizeof(T);                       // elements per 16-byte vector
    constexpr int TC = 64, TR = 128;                              // tile: columns x pivot rows
    __shared__ T tile[TR][TC + VE];                               // row stride keeps 16-byte alignment
    __shared__ int prow[TR];
    // rest columns [eb, ee) (indices that skip the block), eb a multiple of 64
    const int nrest = ee;
    const int e0 = eb + blockIdx.x * TC, y0 = blockIdx.y * TR;
    for (int y = threadIdx.x; y < TR; y += blockDim.x) prow[y] = (y0 + y < nb) ? piv[K0 + y0 + y] : -1;
    __syncthreads();
    // rest column e -> matrix column c (the block columns are skipped); K0 and nb are
    // multiples of VE, so a vector never straddles the block
    constexpr int CV = TC / VE;                                   // vectors per tile row
    constexpr int NI = TR * CV / 256;                             // vectors per thread: all loads first
    static_assert(TR * CV % 256 == 0, "tile / block size");
    uint4 v[NI];
    uint4 *ap[NI];
#pragma unroll
    for (int i = 0; i < NI; i++) {
        const int idx = threadIdx.x + i * 256, yy = idx / CV, cv = idx - yy * CV, e = e0 + cv * VE;
        ap[i] = nullptr;
        v[i] = make_uint4(0u, 0u, 0u, 0u);
        if (prow[yy] >= 0 && e < nrest) {
            const int c = e < K0 ? e : e + nb;
            ap[i] = reinterpret_cast<uint4 *>(A + (long)prow[yy] * n + c);
            v[i] = *ap[i];
        }
    }
#pragma unroll
    for (int i = 0; i < NI; i++) {
        const int idx = threadIdx.x + i * 256, yy = idx / CV, cv = idx - yy * CV;
        if (ap[i]) *ap[i] = make_uint4(0u, 0u, 0u, 0u);
        *reinterpret_cast<uint4 *>(&tile[yy][cv * VE]) = v[i];
    }
    __syncthreads();
    constexpr int YV = TR / VE;                                   // y-vectors per tile column
    for (int idx = threadIdx.x; idx < TC * YV; idx += blockDim.x) {
        const int cc = idx / YV, yv = idx - cc * YV, e = e0 + cc, y = y0 + yv * VE;
        if (e < nrest && y < nb) {
            alignas(16) T o[VE];
#pragma unroll
            for (int u = 0; u < VE; u++) o[u] = tile[yv * VE + u][cc];
            const int c = e < K0 ? e : e + nb;
            *reinterpret_cast<uint4 *>(Bo + (long)c * nb + y) = *reinterpret_cast<const uint4 *>(o);
        }
    }
}

// G[i, :] = M[piv[i], :] (16-byte vectors), invperm from rowperm = piv
template <typename T>
__global__ void __launch_bounds__(256)
gje_ip_finish_kernel(int n, const T *__restrict__ M, const int *__restrict__ piv, T *__restrict__ G)
{
    constexpr int VE = 16 / sizeof(T);
    const int nv = n / VE;
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        const uint4 *src = reinterpret_cast<const uint4 *>(M + (long)piv[i] * n);
        uint4 *dst = reinterpret_cast<uint4 *>(G + (long)i * n);
        for (int v = threadIdx.x; v < nv; v += blockDim.x) dst[v] = src[v];
    }
}

__global__ void iota2_kernel(int n, int *a, int *b) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) { a[i] = i; b[i] = i; }
}

template <typename T>
int ip_gemm(cudaStream_t s, int M, int N, int K, const T *A, long lda, const T *B, long ldb, T *C, long ldc, int cap = 0,
            bool pdl = false)
{
    if constexpr (std::is_same<T, float>::value)
        return gemm_strided<float, float, float, float>(s, M, N, K, 1.0f, A, lda, 1, B, 1, ldb, 1.0f, C, ldc, 1);
    else {
        if (K == 32 && lda == 32 && ldb == 32 && rank32_update_ok(Prec<T>::code, N, A, B, C, ldc))
            return rank32_update(s, Prec<T>::code, M, N, A, B, C, ldc, pdl);
        return tc_gemm(s, Prec<T>::code, M, N, K, 1.0f, A, lda, B, ldb, 1.0f, C, ldc, 0, cap, pdl);
    }
}

template <typename T, int NT, int RPT, bool XOUT>
int panel_launch(cudaStream_t s, int n, int k, int K0, int nbk, T *A, GjeWork &w, bool xkernel)
{
    auto kern = gje_ip_panel_kernel<T, NT, RPT, XOUT>;
    constexpr int dsm = 32 * (NT * RPT + 1) * (int)sizeof(float);     // Lsm
    static const bool attr = [] {
        cudaFuncSetAttribute(gje_ip_panel_kernel<T, NT, RPT, XOUT>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaFuncSetAttribute(gje_ip_panel_kernel<T, NT, RPT, XOUT>, cudaFuncAttributeMaxDynamicSharedMemorySize, dsm);
        return true;
    }();
    (void)attr;
    const int nc = ceil_div(n, NT * RPT);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nc, 1, 1);
    cfg.blockDim = dim3(NT, 1, 1);
    cfg.dynamicSmemBytes = dsm;
    cfg.stream = s;
    // programmatic dependent launch of the step's three kernels: 3 % at n <= 4096; above, the
    // early-resident CTAs of the next kernel take SMs from the look-ahead update (n = 16384:
    // 60.8 against 46.4 ms per inversion), so it is off there
    const bool pdl = n <= 4096 && !env_flag("LYAP_GJE_NO_PDL");
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = nc;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 2 : 1;
    LYAP_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, n, k, K0, nbk, A, (T *)w.X, (T *)w.B, w.invperm, w.rowperm, w.ipiv,
                                     w.info, w.ldet, (float *)w.Pglob, (float *)w.Tg));
    LYAP_TRY(launched());
    if (XOUT && xkernel) {
        cudaLaunchConfig_t cx = {};
        cx.gridDim = dim3(std::min(ceil_div(n, 128), 592)); cx.blockDim = dim3(128); cx.stream = s;
        cx.attrs = at + 1; cx.numAttrs = pdl ? 1 : 0;
        LYAP_CUDA_TRY(cudaLaunchKernelEx(&cx, gje_ip_x_kernel<T>, n, k, A, (const int *)w.invperm, (const float *)w.Pglob,
                                         (const float *)w.Tg, (T *)w.X));
        LYAP_TRY(launched());
    }
    return LYAP_OK;
}

template <typename T>
int gje_ip_invert_t(cudaStream_t s, int n, T *A, T *G, GjeWork &w)
{
    LYAP_CUDA_TRY(cudaMemsetAsync(w.info, 0, sizeof(int), s));
    LYAP_CUDA_TRY(cudaMemsetAsync(w.ldet, 0, sizeof(double) * (size_t)n, s));
    iota2_kernel<<<ceil_div(n, 256), 256, 0, s>>>(n, w.rowperm, w.invperm);
    LYAP_TRY(launched());
    // threads per CTA: the cluster has at most 16 CTAs; LYAP_GJE_IP_NT overrides (tuning)
    // (measured at n = 16384: 512 threads x 2 rows 2430 cycles per column, 1024 x 1 3440)
    // (n = 8192: 256 threads x 2 rows 14.9 ms per inversion, 512 x 1 16.8: the column time follows the
    // warps per CTA; n = 16384: 512 x 2 40.5 ms, 256 x 4 42.7, 1024 x 1 slower still)
    int nt = n <= 8192 ? 256 : 512, rpt = n <= 4096 ? 1 : 2;
    if (const char *e = getenv("LYAP_GJE_IP_NT")) nt = atoi(e);
    if (const char *e = getenv("LYAP_GJE_IP_RPT")) rpt = atoi(e);
    if (nt == 128) rpt = 2;
    if (ceil_div(n, nt * rpt) > 16) { nt = n <= 8192 ? 512 : 1024; rpt = 1; }
    // outer block: GJE_NB columns (w.Bo holds n x GJE_NB_MAX; LYAP_GJE_IP_NB for tuning)
    int NB = GJE_NB;
    if (const char *e = getenv("LYAP_GJE_IP_NB")) NB = std::max(64, std::min(GJE_NB_MAX, atoi(e) / 32 * 32));
    const bool xout = !env_flag("LYAP_GJE_IP_XIN");             // 512-thread panels: X rows by the separate kernel
    // 16-bit storage: the X rows are formed inside the rank-32 update kernel (rank_update.cu)
    constexpr bool half_t = !std::is_same<T, float>::value;
    // (measured: n = 1024 1.43 -> 1.35 ms per inversion, 3072 4.50 -> 4.36, 8192 18.6 -> 17.0, 16384
    // 45.4 -> 43.9; with the full 16-CTA cluster of 256-thread CTAs (n = 4096) the X phase on the
    // panel's 16 SMs is as fast, 6.21 vs 6.25 ms: in-panel there)
    const bool fused = half_t && n % 8 == 0 && !(n > 3584 && n <= 4096) && !env_flag("LYAP_GJE_NO_FUSEX") &&
                       !env_flag("LYAP_NO_RANK32");
    const bool xk = !fused;
    // Look-ahead: the panels and rank-32 updates of block K0 + NB run on the high-priority
    // stream P while the main stream applies the rest of block K0's rank-NB update.  Order on
    // the main stream: B_outer, the update of the NEXT block's columns (then P may start), the
    // update of all other columns as one CTA per tile -- SMs come free tile by tile, so P's
    // cluster launches are not locked out.  The two streams touch disjoint columns of A.
    // (Measured at n = 16384: 58.6 ms per inversion without look-ahead, 49.6 with; the rest
    // update in 16 column chunks, chunk i released with panel i as a persistent GEMM capped at
    // 132 CTAs: 50.9; capped persistent GEMMs of 64 / 100 / 132 CTAs for the whole rest: 57.)
    const bool ahead = w.side != nullptr && n >= 4 * NB && !env_flag("LYAP_GJE_NO_LOOKAHEAD");
    cudaStream_t P = ahead ? w.side : s;
    if (ahead) {
        LYAP_CUDA_TRY(cudaEventRecord(w.ev_a, s));
        LYAP_CUDA_TRY(cudaStreamWaitEvent(P, w.ev_a, 0));
    }
    for (int K0 = 0; K0 < n; K0 += NB) {
        const int nbk = std::min(NB, n - K0);
        for (int k = K0; k < K0 + nbk; k += BW) {
            {
                KTimer kt(KC_GJE_PANEL, P, (double)(n - k) * BW * BW + 2.0 * n * BW * BW,
                          (double)sizeof(T) * ((double)n * BW + (double)n * BW));
                if (nt == 128) LYAP_TRY(panel_launch<T, 128, 2, false>(P, n, k, K0, nbk, A, w, xk));
                else if (nt == 256 && rpt == 1 && fused) LYAP_TRY(panel_launch<T, 256, 1, true>(P, n, k, K0, nbk, A, w, xk));
                else if (nt == 256 && rpt == 1) LYAP_TRY(panel_launch<T, 256, 1, false>(P, n, k, K0, nbk, A, w, xk));
                else if (nt == 256 && fused) LYAP_TRY(panel_launch<T, 256, 2, true>(P, n, k, K0, nbk, A, w, xk));
                else if (nt == 256) LYAP_TRY(panel_launch<T, 256, 2, false>(P, n, k, K0, nbk, A, w, xk));
                else if (nt == 512 && rpt == 1 && !xout) LYAP_TRY(panel_launch<T, 512, 1, false>(P, n, k, K0, nbk, A, w, xk));
                else if (nt == 512 && rpt == 1) LYAP_TRY(panel_launch<T, 512, 1, true>(P, n, k, K0, nbk, A, w, xk));
                else if (nt == 512) LYAP_TRY(panel_launch<T, 512, 2, true>(P, n, k, K0, nbk, A, w, xk));
                else LYAP_TRY(panel_launch<T, 1024, 1, true>(P, n, k, K0, nbk, A, w, xk));
            }
            KTimer kt(KC_GJE_UPDATE, P);
            const bool pdl = n <= 4096 && !env_flag("LYAP_GJE_NO_PDL");
            const bool xexp = !(nt == 128 || (nt == 512 && rpt == 1 && !xout));   // panel exported
            if (fused && xexp)
                LYAP_TRY(rank32_fused_update(P, Prec<T>::code, n, nbk, k, K0, (const float *)w.Pglob, (const float *)w.Tg,
                                             w.invperm, (const T *)w.B + (size_t)K0 * BW, A + K0, n, pdl));
            else
                LYAP_TRY(ip_gemm<T>(P, n, nbk, BW, (const T *)w.X, BW, (const T *)w.B + (size_t)K0 * BW, BW, A + K0, n, 0, pdl));
        }
        if (ahead) {
            LYAP_CUDA_TRY(cudaEventRecord(w.ev_b, P));             // inner steps of this block done
            LYAP_CUDA_TRY(cudaStreamWaitEvent(s, w.ev_b, 0));
        }
        if (n - nbk > 0) {
            // B_outer in rest-column indices e (e < K0: column e, else column e + nbk)
            auto prep = [&](int eb, int ee) -> int {
                if (ee <= eb) return LYAP_OK;
                gje_ip_outer_prep_kernel<T><<<dim3(ceil_div(ee - eb, 64), ceil_div(nbk, 128)), 256, 0, s>>>(
                    n, K0, nbk, eb, ee, A, w.rowperm, (T *)w.Bo);
                return launched();
            };
            KTimer kt(KC_GJE_UPDATE, s);
            const int cr = K0 + nbk;
            const int cn = ahead ? std::min(n, cr + NB) : cr;
            if (ahead && cn > cr) {
                // the next block's columns first (B_outer for them, their update), then P may start;
                // the other columns' B_outer and update run beside P
                LYAP_TRY(prep(K0, K0 + (cn - cr)));
                LYAP_TRY(ip_gemm<T>(s, n, cn - cr, nbk, A + K0, n, (const T *)w.Bo + (size_t)cr * nbk, nbk, A + cr, n));
                LYAP_CUDA_TRY(cudaEventRecord(w.ev_a, s));
                LYAP_CUDA_TRY(cudaStreamWaitEvent(P, w.ev_a, 0));
                LYAP_TRY(prep(0, K0));
                LYAP_TRY(prep(K0 + (cn - cr), n - nbk));
            } else {
                LYAP_TRY(prep(0, n - nbk));
            }
            int cap = (ahead && cn > cr) ? -1 : 0;
            if (const char *e = getenv("LYAP_GJE_LA_CAP")) cap = (ahead && cn > cr) ? atoi(e) : 0;   // tuning
            if (K0 > 0) LYAP_TRY(ip_gemm<T>(s, n, K0, nbk, A + K0, n, (const T *)w.Bo, nbk, A, n, cap));
            if (cn < n) LYAP_TRY(ip_gemm<T>(s, n, n - cn, nbk, A + K0, n, (const T *)w.Bo + (size_t)cn * nbk, nbk, A + cn, n, cap));
        }
    }
    gje_ip_finish_kernel<T><<<std::min(n, 148 * 8), 256, 0, s>>>(n, A, w.rowperm, G);
    return launched();
}

}  // namespace

// The implicit-pivoting sweep serves 16-bit and fp32 storage with n a multiple of 32 and at
// least two outer blocks, up to 16 CTAs x 1024 rows; LYAP_GJE_SWAP=1 forces gje.cu's sweep.
bool gje_ip_eligible(int n, int prec, const GjeWork &w)
{
    if (prec == LYAP_FP64 || w.Bo == nullptr) return false;
    if ((prec == LYAP_FP16 || prec == LYAP_BF16) && use_simt_gemm()) return false;
    if (n % 32 != 0 || n < 2 * GJE_NB || n > 16 * 1024) return false;
    return !env_flag("LYAP_GJE_SWAP");
}

// A (n x n, u_s, destroyed) -> G = the sweep's result in gje.cu's layout; w.rowperm / invperm /
// ipiv / ldet / info as gje_invert leaves them.
int gje_ip_invert(cudaStream_t s, int n, int prec, void *A, void *G, GjeWork &w)
{
    switch (prec) {
        case LYAP_FP32: return gje_ip_invert_t<float>(s, n, (float *)A, (float *)G, w);
        case LYAP_FP16: return gje_ip_invert_t<__half>(s, n, (__half *)A, (__half *)G, w);
        case LYAP_BF16: return gje_ip_invert_t<__nv_bfloat16>(s, n, (__nv_bfloat16 *)A, (__nv_bfloat16 *)G, w);
    }
    return LYAP_ERR_ARG;
}

}  // namespace lyap
