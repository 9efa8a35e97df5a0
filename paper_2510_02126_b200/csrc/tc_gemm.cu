// tc_gemm.cu -- 5th-generation tensor-core GEMM for the 16-bit solver precisions:
//     C = alpha * A * B^T + beta * C,  A (M x K) and B (N x K) row-major ("K-major"),
//     bf16 or fp16 operands, fp32 accumulation in TMEM, C in the same 16-bit type
//     (row-major or column-major output).
// Used for the Gauss-Jordan rank-b update of the inversion (Eq. newton-lyapu1,
// A_{k-1}^{-1}) and for the Z-side products A_{k-1}^{-1} Z_{k-1} (Alg. 3/4 line 4).
//
// One CTA per 128 x 128 output tile, 4 warps:
//   warp 0 (one elected lane)  TMA producer: 64-wide K blocks of A and B into a
//                              4-stage shared-memory ring (128B swizzle), mbarrier
//                              full/empty pipeline;
//   warp 1 (one elected lane)  issues tcgen05.mma.cta_group::1.kind::f16 (M=128,
//                              N=128, K=16) into a 128-column fp32 TMEM accumulator,
//                              tcgen05.commit releases each smem stage;
//   warps 0-3                  epilogue: tcgen05.ld 32x32b (each thread one row),
//                              alpha/beta blend with C staged through the idle
//                              pipeline shared memory, row-coalesced 16-bit stores.
#include <cuda.h>
#include <cuda_runtime.h>
#include "common.cuh"
#include "lyap_internal.h"
#include "ktimer.h"

namespace lyap {

namespace tc {
constexpr int BM = 128, BN = 128, BK = 64, STAGES = 4;
constexpr int A_STAGE = BM * BK * 2, B_STAGE = BN * BK * 2;          // bytes
constexpr int C_STAGE = BM * BN * 2;                                 // C tile (TMA epilogue)
constexpr int SMEM = STAGES * (A_STAGE + B_STAGE) + C_STAGE + 1024 + 256;   // + alignment + barriers
// pipeline depth by K: short-K updates (the Gauss-Jordan rank-b steps) keep the
// shared-memory footprint small so 2-3 CTAs share an SM and overlap their epilogues
__host__ __device__ constexpr int smem_bytes(int ns) { return ns * (A_STAGE + B_STAGE) + C_STAGE + 1024 + 256; }
inline int stages_for(int nk) { return nk <= 2 ? nk : (nk <= 4 ? 2 : STAGES); }

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" :: "r"(smem_u32(b)), "r"(phase) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
        :: "r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1) : "memory");
}
// the same with an L2 eviction policy (streaming C tiles of the look-ahead update must not push
// the next block's columns, which the concurrent panels read, out of the L2)
__device__ __forceinline__ uint64_t l2_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void tma_load_2d_hint(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;"
        :: "r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(pol) : "memory");
}
__device__ __forceinline__ void tma_store_2d_hint(const CUtensorMap *map, const void *src, int c0, int c1, uint64_t pol) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3}], [%1], %4;"
                 :: "l"(map), "r"(smem_u32(src)), "r"(c0), "r"(c1), "l"(pol) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap *map, const void *src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];"
                 :: "l"(map), "r"(smem_u32(src)), "r"(c0), "r"(c1) : "memory");
}
// K-major, 128B-swizzled canonical layout: 8-row x 128-byte atoms, atoms 1024 B apart.
__device__ __forceinline__ uint64_t smem_desc(const void *p) {
    uint64_t a = smem_u32(p);
    return ((a & 0x3FFFFull) >> 4) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" :: "r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t addr, float *v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; i++) v[i] = __uint_as_float(r[i]);
}
}  // namespace tc

template <typename T>
__global__ void __launch_bounds__(128, 3)
tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const __grid_constant__ CUtensorMap tmC, int M, int N, int K, float alpha, float beta,
               T *__restrict__ C, long ldc, int colmajor, int ctma, int ns, int cstream)
{
    using namespace tc;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *base = (unsigned char *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    unsigned char *sA = base;
    unsigned char *sB = base + ns * A_STAGE;
    unsigned char *sC = sB + ns * B_STAGE;                  // 1024-aligned (stage sizes are)
    uint64_t *full = (uint64_t *)(sC + C_STAGE);
    uint64_t *empty = full + ns;
    uint64_t *done = empty + ns;
    uint64_t *cbar = done + 1;
    uint32_t *tmem_slot = (uint32_t *)(cbar + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int nk = (K + BK - 1) / BK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < ns; s++) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], 1); }
        tc::mbar_init(done, 1);
        tc::mbar_init(cbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" :: "l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" :: "l"(&tmB) : "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"(tc::smem_u32(tmem_slot)), "r"(BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;
    // programmatic dependent launch: the setup above overlaps the previous kernel's tail;
    // every thread waits here before touching its inputs / outputs (a no-op otherwise)
    asm volatile("griddepcontrol.wait;" ::: "memory");

    if (warp == 0 && lane == 0) {
        // ---------------- TMA producer (the C tile first when it is blended in)
        if (ctma && beta != 0.f) {
            tc::mbar_expect_tx(cbar, C_STAGE);
            for (int w = 0; w < 4; w++)
                for (int hh = 0; hh < 2; hh++)
                    if (cstream) tc::tma_load_2d_hint(sC + (w * 2 + hh) * 4096, &tmC, cbar, n0 + 64 * hh, m0 + 32 * w, tc::l2_evict_first());
                    else tc::tma_load_2d(sC + (w * 2 + hh) * 4096, &tmC, cbar, n0 + 64 * hh, m0 + 32 * w);
        }
        for (int kb = 0; kb < nk; kb++) {
            const int s = kb % ns;
            if (kb >= ns) tc::mbar_wait(&empty[s], ((kb / ns) - 1) & 1);
            tc::mbar_expect_tx(&full[s], A_STAGE + B_STAGE);
            tc::tma_load_2d(sA + s * A_STAGE, &tmA, &full[s], kb * BK, m0);
            tc::tma_load_2d(sB + s * B_STAGE, &tmB, &full[s], kb * BK, n0);
        }
    } else if (warp == 1 && lane == 0) {
        // ---------------- MMA issuer
        const uint32_t fmt = std::is_same<T, __nv_bfloat16>::value ? 1u : 0u;
        const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(BN >> 3) << 17) |
                               ((uint32_t)(BM >> 4) << 24);
        for (int kb = 0; kb < nk; kb++) {
            const int s = kb % ns;
            tc::mbar_wait(&full[s], (kb / ns) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint64_t da = tc::smem_desc(sA + s * A_STAGE), db = tc::smem_desc(sB + s * B_STAGE);
#pragma unroll
            for (int k = 0; k < BK / 16; k++)   // +32 bytes along K = +2 in the start-address field
                tc::mma_f16(tmem, da + 2 * k, db + 2 * k, idesc, (kb > 0 || k > 0) ? 1u : 0u);
            tc::mma_commit(&empty[s]);
        }
        tc::mma_commit(done);
    }
    // ---------------- epilogue (all 4 warps): thread = one accumulator row
    tc::mbar_wait(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int row = m0 + warp * 32 + lane;
    if (colmajor) {
        // consecutive lanes = consecutive rows = consecutive addresses: coalesced as is
        for (int c0 = 0; c0 < BN; c0 += 16) {
            float v[16];
            tc::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
            if (row < M) {
#pragma unroll
                for (int i = 0; i < 16; i++) {
                    const int col = n0 + c0 + i;
                    if (col < N) {
                        T *cp = C + (long)col * ldc + row;
                        float r = alpha * v[i];
                        if (beta != 0.f) r = fmaf(beta, to_f<T>(*cp), r);
                        *cp = from_f<T>(r);
                    }
                }
            }
        }
    } else if (ctma) {
        // row-major C through TMA: the warp's 32 x 128 tile is two 32 x 64 boxes in
        // 128B-swizzled shared memory (16-byte chunk j of row r at chunk j ^ (r & 7)),
        // loaded by the producer before the main loop and stored back by TMA.
        if (beta != 0.f) tc::mbar_wait(cbar, 0);
        unsigned char *wbox = sC + warp * 2 * 4096;
        for (int c0 = 0; c0 < BN; c0 += 16) {
            float v[16];
            tc::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
            unsigned char *rowp = wbox + (c0 >> 6) * 4096 + lane * 128;
            const int j0 = (c0 & 63) >> 3;
            uint4 *p0 = reinterpret_cast<uint4 *>(rowp + (((j0) ^ (lane & 7)) << 4));
            uint4 *p1 = reinterpret_cast<uint4 *>(rowp + (((j0 + 1) ^ (lane & 7)) << 4));
            alignas(16) T o[16];
            if (beta != 0.f) {
                alignas(16) T ci[16];
                *reinterpret_cast<uint4 *>(ci) = *p0;
                *reinterpret_cast<uint4 *>(ci + 8) = *p1;
#pragma unroll
                for (int i = 0; i < 16; i++) o[i] = from_f<T>(fmaf(beta, to_f<T>(ci[i]), alpha * v[i]));
            } else {
#pragma unroll
                for (int i = 0; i < 16; i++) o[i] = from_f<T>(alpha * v[i]);
            }
            *p0 = *reinterpret_cast<const uint4 *>(o);
            *p1 = *reinterpret_cast<const uint4 *>(o + 8);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
            if (cstream) {
                const uint64_t pol = tc::l2_evict_first();
                tc::tma_store_2d_hint(&tmC, wbox, n0, m0 + 32 * warp, pol);
                tc::tma_store_2d_hint(&tmC, wbox + 4096, n0 + 64, m0 + 32 * warp, pol);
            } else {
                tc::tma_store_2d(&tmC, wbox, n0, m0 + 32 * warp);
                tc::tma_store_2d(&tmC, wbox + 4096, n0 + 64, m0 + 32 * warp);
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        __syncwarp();
    } else {
        // generic row-major fallback (unaligned C): one element per access
        for (int c0 = 0; c0 < BN; c0 += 16) {
            float v[16];
            tc::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
            if (row < M) {
#pragma unroll
                for (int i = 0; i < 16; i++) {
                    const int col = n0 + c0 + i;
                    if (col < N) {
                        T *cp = C + (long)row * ldc + col;
                        float r = alpha * v[i];
                        if (beta != 0.f) r = fmaf(beta, to_f<T>(*cp), r);
                        *cp = from_f<T>(r);
                    }
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(BN));
}

// ---------------------------------------------------------------- persistent variant
// One CTA per SM loops over 128 x 128 output tiles (row-major C via TMA); warp-specialised:
//   warp 0 (one lane)  TMA producer: the C tile of the tile (when blended) into one of two
//                      C buffers, then the K blocks into the 4-stage A/B ring;
//   warp 1 (one lane)  tcgen05.mma issuer into one of two TMEM accumulators (256 columns);
//   warps 2-5          epilogue: TMEM -> registers -> blend with C in 128B-swizzled shared
//                      memory -> TMA store; it frees the accumulator as soon as it has been
//                      read, so the MMAs of tile i+1 overlap the epilogue of tile i.
// Barriers: full/empty (A/B ring), acc_full/acc_empty (accumulators), c_full/c_empty (C).
namespace tc {
constexpr int PSTAGES = 4, PTHREADS = 192;
constexpr int PSMEM = PSTAGES * (A_STAGE + B_STAGE) + 2 * C_STAGE + 1024 + 512;
}  // namespace tc

template <typename T>
__global__ void __launch_bounds__(tc::PTHREADS, 1)
tc_gemm_persistent_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                          const __grid_constant__ CUtensorMap tmC, int M, int N, int K, float alpha, float beta)
{
    using namespace tc;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *base = (unsigned char *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    unsigned char *sA = base;
    unsigned char *sB = sA + PSTAGES * A_STAGE;
    unsigned char *sC = sB + PSTAGES * B_STAGE;                 // 2 x C_STAGE
    uint64_t *full = (uint64_t *)(sC + 2 * C_STAGE);
    uint64_t *empty = full + PSTAGES;
    uint64_t *acc_full = empty + PSTAGES;
    uint64_t *acc_empty = acc_full + 2;
    uint64_t *c_full = acc_empty + 2;
    uint64_t *c_empty = c_full + 2;
    uint32_t *tmem_slot = (uint32_t *)(c_empty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tiles_n = (N + BN - 1) / BN, tiles = tiles_n * ((M + BM - 1) / BM);
    const int nk = (K + BK - 1) / BK;
    const bool blend = (beta != 0.f);
    // one wave of CTAs: the next kernel of the stream may set up beside this one (PDL)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0) {
        for (int i = 0; i < PSTAGES; i++) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
        for (int i = 0; i < 2; i++) {
            mbar_init(&acc_full[i], 1);
            mbar_init(&acc_empty[i], 4);            // one arrival per epilogue warp
            mbar_init(&c_full[i], 1);
            mbar_init(&c_empty[i], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" :: "l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" :: "l"(&tmB) : "memory");
        asm volatile("prefetch.tensormap [%0];" :: "l"(&tmC) : "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"(smem_u32(tmem_slot)), "r"(2 * BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;
    // programmatic dependent launch: the setup above overlaps the previous kernel's tail;
    // every thread waits here before touching its inputs / outputs (a no-op otherwise)
    asm volatile("griddepcontrol.wait;" ::: "memory");

    if (warp == 0) {
        if (lane == 0) {
            int kc = 0;
            for (int t = blockIdx.x, i = 0; t < tiles; t += gridDim.x, i++) {
                const int m0 = (t / tiles_n) * BM, n0 = (t % tiles_n) * BN, ab = i & 1;
                if (blend) {
                    if (i >= 2) mbar_wait(&c_empty[ab], ((i >> 1) - 1) & 1);
                    mbar_expect_tx(&c_full[ab], C_STAGE);
                    for (int w = 0; w < 4; w++)
                        for (int hh = 0; hh < 2; hh++)
                            tma_load_2d(sC + ab * C_STAGE + (w * 2 + hh) * 4096, &tmC, &c_full[ab], n0 + 64 * hh,
                                        m0 + 32 * w);
                }
                for (int kb = 0; kb < nk; kb++, kc++) {
                    const int st = kc % PSTAGES;
                    if (kc >= PSTAGES) mbar_wait(&empty[st], ((kc / PSTAGES) - 1) & 1);
                    mbar_expect_tx(&full[st], A_STAGE + B_STAGE);
                    tma_load_2d(sA + st * A_STAGE, &tmA, &full[st], kb * BK, m0);
                    tma_load_2d(sB + st * B_STAGE, &tmB, &full[st], kb * BK, n0);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t fmt = std::is_same<T, __nv_bfloat16>::value ? 1u : 0u;
            const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(BN >> 3) << 17) |
                                   ((uint32_t)(BM >> 4) << 24);
            int kc = 0;
            for (int t = blockIdx.x, i = 0; t < tiles; t += gridDim.x, i++) {
                const int ab = i & 1;
                if (i >= 2) mbar_wait(&acc_empty[ab], ((i >> 1) - 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t acc = tmem + (uint32_t)(ab * BN);
                for (int kb = 0; kb < nk; kb++, kc++) {
                    const int st = kc % PSTAGES;
                    mbar_wait(&full[st], (kc / PSTAGES) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint64_t da = smem_desc(sA + st * A_STAGE), db = smem_desc(sB + st * B_STAGE);
#pragma unroll
                    for (int k = 0; k < BK / 16; k++)
                        mma_f16(acc, da + 2 * k, db + 2 * k, idesc, (kb > 0 || k > 0) ? 1u : 0u);
                    mma_commit(&empty[st]);
                }
                mma_commit(&acc_full[ab]);
            }
        }
    } else {
        // ---- epilogue warps 2..5; TMEM lane quarter = warp % 4
        const int q4 = warp & 3;
        for (int t = blockIdx.x, i = 0; t < tiles; t += gridDim.x, i++) {
            const int m0 = (t / tiles_n) * BM, n0 = (t % tiles_n) * BN, ab = i & 1;
            unsigned char *wbox = sC + ab * C_STAGE + q4 * 2 * 4096;
            if (!blend && i >= 2) {
                // the previous TMA store out of this buffer must have read it
                if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                __syncwarp();
            }
            mbar_wait(&acc_full[ab], (i >> 1) & 1);
            if (blend) mbar_wait(&c_full[ab], (i >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            for (int c0 = 0; c0 < BN; c0 += 16) {
                float v[16];
                tmem_ld16(tmem + (uint32_t)(ab * BN) + ((uint32_t)(q4 * 32) << 16) + (uint32_t)c0, v);
                unsigned char *rowp = wbox + (c0 >> 6) * 4096 + lane * 128;
                const int j0 = (c0 & 63) >> 3;
                uint4 *p0 = reinterpret_cast<uint4 *>(rowp + (((j0) ^ (lane & 7)) << 4));
                uint4 *p1 = reinterpret_cast<uint4 *>(rowp + (((j0 + 1) ^ (lane & 7)) << 4));
                alignas(16) T o[16];
                if (blend) {
                    alignas(16) T ci[16];
                    *reinterpret_cast<uint4 *>(ci) = *p0;
                    *reinterpret_cast<uint4 *>(ci + 8) = *p1;
#pragma unroll
                    for (int e = 0; e < 16; e++) o[e] = from_f<T>(fmaf(beta, to_f<T>(ci[e]), alpha * v[e]));
                } else {
#pragma unroll
                    for (int e = 0; e < 16; e++) o[e] = from_f<T>(alpha * v[e]);
                }
                *p0 = *reinterpret_cast<const uint4 *>(o);
                *p1 = *reinterpret_cast<const uint4 *>(o + 8);
            }
            // accumulator read: let the MMA warp reuse it
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[ab]);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                tma_store_2d(&tmC, wbox, n0, m0 + 32 * q4);
                tma_store_2d(&tmC, wbox + 4096, n0 + 64, m0 + 32 * q4);
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                if (blend) {
                    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    mbar_arrive(&c_empty[ab]);
                }
            }
            __syncwarp();
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        __syncwarp();
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(2 * BN));
}

// ---------------------------------------------------------------- host side
namespace {
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = []() -> EncodeTiledFn {         // thread-safe one-time lookup
        cudaDriverEntryPointQueryResult q;
        void *p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return (EncodeTiledFn)p;
        return nullptr;
    }();
    return fn;
}
// rows x cols row-major 16-bit matrix with leading dimension ld (elements); box = 64 x box_rows
int make_map(CUtensorMap *m, const void *ptr, int prec, long rows, long cols, long ld, int box_rows) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return LYAP_ERR_CUDA;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(m, prec == LYAP_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2,
                    const_cast<void *>(ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);      // out-of-bounds elements read as zero
    return r == CUDA_SUCCESS ? LYAP_OK : LYAP_ERR_ARG;
}
}  // namespace

// C = alpha * A (M x K, ld lda) * B^T (B: N x K, ld ldb) + beta * C  (C ld ldc, row- or column-major)
namespace {
template <typename... KArgs, typename... Args>
int launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl, Args... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid; cfg.blockDim = block; cfg.dynamicSmemBytes = smem; cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at; cfg.numAttrs = pdl ? 1 : 0;
    LYAP_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, KArgs(args)...));
    return LYAP_OK;
}
}  // namespace

int tc_gemm(cudaStream_t s, int prec, int M, int N, int K, float alpha, const void *A, long lda, const void *B,
            long ldb, float beta, void *C, long ldc, int colmajor, int max_ctas, bool pdl)
{
    if (M <= 0 || N <= 0 || K <= 0) return LYAP_OK;
    if (prec != LYAP_BF16 && prec != LYAP_FP16) return LYAP_ERR_ARG;
    if ((lda * 2) % 16 || (ldb * 2) % 16 || ((uintptr_t)A % 16) || ((uintptr_t)B % 16)) return LYAP_ERR_ARG;
    CUtensorMap ma, mb, mc;
    LYAP_TRY(make_map(&ma, A, prec, M, K, lda, tc::BM));
    LYAP_TRY(make_map(&mb, B, prec, N, K, ldb, tc::BN));
    // TMA epilogue for row-major C with 16-byte aligned rows
    const int ctma = (!colmajor && (ldc * 2) % 16 == 0 && ((uintptr_t)C % 16) == 0 && !env_flag("LYAP_TC_NO_CTMA"))
                         ? 1 : 0;
    if (ctma) LYAP_TRY(make_map(&mc, C, prec, M, N, ldc, 32));
    else mc = ma;
    dim3 grid(ceil_div(N, tc::BN), ceil_div(M, tc::BM));
    const int ns = tc::stages_for(ceil_div(K, tc::BK));
    const int smem = tc::smem_bytes(ns);
    // one-time attribute setup; a function-local static is initialised thread-safely, and
    // nsm is published only after every attribute is set (concurrent solver handles)
    static const int nsm = [] {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(tc_gemm_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::SMEM);
        cudaFuncSetAttribute(tc_gemm_kernel<__half>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::SMEM);
        cudaFuncSetAttribute(tc_gemm_persistent_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::PSMEM);
        cudaFuncSetAttribute(tc_gemm_persistent_kernel<__half>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::PSMEM);
        return v;
    }();
    // the look-ahead's rest update (max_ctas < 0) streams its C tiles through the L2 (evict first)
    const int cstream = (max_ctas < 0 && ctma && !env_flag("LYAP_TC_NO_CHINT")) ? 1 : 0;
    KTimer kt(KC_TCGEMM, s, 2.0 * M * N * K, 2.0 * ((double)M * K + (double)N * K + (beta != 0.f ? 2.0 : 1.0) * M * N));
    const int tiles = (int)(grid.x * grid.y);
    // max_ctas < 0: one CTA per tile (SMs come free tile by tile, so a concurrent
    // high-priority cluster launch is not locked out for the whole product)
    if (ctma && tiles >= nsm && max_ctas >= 0 && !env_flag("LYAP_TC_NONPERSISTENT")) {
        const int g = std::min(tiles, max_ctas > 0 ? std::min(max_ctas, nsm) : nsm);
        if (prec == LYAP_BF16)
            LYAP_TRY(launch_pdl(tc_gemm_persistent_kernel<__nv_bfloat16>, dim3(g), dim3(tc::PTHREADS), tc::PSMEM, s, pdl, ma, mb, mc,
                                M, N, K, alpha, beta));
        else
            LYAP_TRY(launch_pdl(tc_gemm_persistent_kernel<__half>, dim3(g), dim3(tc::PTHREADS), tc::PSMEM, s, pdl, ma, mb, mc, M, N,
                                K, alpha, beta));
        return launched();
    }
    if (prec == LYAP_BF16)
        tc_gemm_kernel<__nv_bfloat16><<<grid, 128, smem, s>>>(ma, mb, mc, M, N, K, alpha, beta,
                                                               (__nv_bfloat16 *)C, ldc, colmajor, ctma, ns, cstream);
    else
        tc_gemm_kernel<__half><<<grid, 128, smem, s>>>(ma, mb, mc, M, N, K, alpha, beta, (__half *)C, ldc,
                                                       colmajor, ctma, ns, cstream);
    return launched();
}

}  // namespace lyap

// standalone entry for tests: C = alpha A B^T + beta C (row-major C, 16-bit types)
extern "C" int lyap_tc_gemm(int prec, int M, int N, int K, float alpha, const void *A, long lda, const void *B,
                            long ldb, float beta, void *C, long ldc, void *stream)
{
    int rc = lyap::tc_gemm((cudaStream_t)stream, prec, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, 0);
    if (rc == LYAP_OK && cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) rc = LYAP_ERR_CUDA;
    return rc;
}
