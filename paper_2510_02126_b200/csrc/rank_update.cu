// rank_update.cu -- the rank-32 update of the Gauss-Jordan sweep's inner steps,
//     C (M x N, row-major, ld ldc) += X (M x 32, row-major) * Bt^T   (Bt: N x 32, row-major),
// for 16-bit storage with fp32 accumulation (the inversion of the Newton
// step; north_star: trailing update accumulating in fp32).
//
// With K = 32 the product is pure streaming: 2 M N element reads + writes of C against
// 64 flops per element, far below the tensor ridge.  The persistent tcgen05 kernel
// (tc_gemm.cu) spends its time in per-tile TMA -> MMA -> TMEM -> epilogue latency at this
// depth (13 us for n x 512 at n = 16384, 32 MB of traffic) and needs a whole SM per CTA, so it
// also waits for SMs while the look-ahead update runs.  This kernel keeps the operands in
// registers / shared memory and C tiles in flight by 16-byte cp.async: 64 x 128 tiles, 128
// threads, ~26 KB of shared memory (several CTAs per SM, co-resident with other kernels),
// warp-level mma.sync m16n8k16 (tensor cores; the rate is irrelevant here).
// Rounding order as the tcgen05 epilogue: the 32 products accumulate from zero in fp32, then
// C_old is added and the sum is rounded once.
#include "common.cuh"
#include "lyap_internal.h"

namespace lyap {

namespace {

constexpr int RU_TM = 64, RU_TN = 128, RU_K = 32;
constexpr int RU_CLD = RU_TN + 8;        // C tile row stride (elements): 16-byte aligned, conflict-free fragments
constexpr int RU_BLD = RU_K + 8;         // Bt tile row stride

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(gmem) : "memory");
}

template <typename T> struct Mma;
template <> struct Mma<__nv_bfloat16> {
    __device__ __forceinline__ static void run(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
    }
    __device__ __forceinline__ static float lo(uint32_t w) { return __uint_as_float(w << 16); }
    __device__ __forceinline__ static float hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
    __device__ __forceinline__ static uint32_t pack(float x, float y) {
        return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(x)) | ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(y)) << 16);
    }
};
template <> struct Mma<__half> {
    __device__ __forceinline__ static void run(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
    }
    __device__ __forceinline__ static float lo(uint32_t w) { return __half2float(__ushort_as_half((unsigned short)(w & 0xffffu))); }
    __device__ __forceinline__ static float hi(uint32_t w) { return __half2float(__ushort_as_half((unsigned short)(w >> 16))); }
    __device__ __forceinline__ static uint32_t pack(float x, float y) {
        return (uint32_t)__half_as_ushort(__float2half_rn(x)) | ((uint32_t)__half_as_ushort(__float2half_rn(y)) << 16);
    }
};

// grid (ceil(N / 128), ceil(M / 64)); N a multiple of 8, rows of C 16-byte aligned
template <typename T>
__global__ void __launch_bounds__(128)
rank32_update_kernel(int M, int N, const T *__restrict__ X, const T *__restrict__ Bt, T *__restrict__ C, long ldc)
{
    __shared__ __align__(16) T Cs[RU_TM][RU_CLD];
    __shared__ __align__(16) T Bs[RU_TN][RU_BLD];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int m0 = blockIdx.y * RU_TM, n0 = blockIdx.x * RU_TN;
    // programmatic dependent launch (a no-op without the launch attribute)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // ---- C tile and Bt tile by 16-byte asynchronous copies (all in flight at once)
    for (int v = tid; v < RU_TM * (RU_TN / 8); v += 128) {
        const int r = v / (RU_TN / 8), cv = v - r * (RU_TN / 8);
        if (m0 + r < M && n0 + cv * 8 < N) cp_async16(&Cs[r][cv * 8], C + (long)(m0 + r) * ldc + n0 + cv * 8);
    }
    for (int v = tid; v < RU_TN * (RU_K / 8); v += 128) {
        const int r = v / (RU_K / 8), cv = v - r * (RU_K / 8);
        if (n0 + r < N) cp_async16(&Bs[r][cv * 8], Bt + (long)(n0 + r) * RU_K + cv * 8);
        else *reinterpret_cast<uint4 *>(&Bs[r][cv * 8]) = make_uint4(0u, 0u, 0u, 0u);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    // ---- X fragments of this warp's 16 rows straight from global memory (L2 resident)
    const int g = lane >> 2, t = lane & 3;
    const int r0 = m0 + warp * 16;
    uint32_t a[2][4];
#pragma unroll
    for (int ks = 0; ks < 2; ks++) {
#pragma unroll
        for (int h = 0; h < 4; h++) {
            const int row = r0 + g + (h & 1) * 8, col = ks * 16 + 2 * t + (h >> 1) * 8;
            a[ks][h] = (row < M) ? *reinterpret_cast<const uint32_t *>(X + (long)row * RU_K + col) : 0u;
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    // ---- per n-tile of 8 columns: two MMAs from zero, add the old C, round, back into the tile
#pragma unroll 4
    for (int nt = 0; nt < RU_TN / 8; nt++) {
        float d[4] = {0.f, 0.f, 0.f, 0.f};
        const T *bp = &Bs[nt * 8 + g][2 * t];
#pragma unroll
        for (int ks = 0; ks < 2; ks++) {
            const uint32_t b0 = *reinterpret_cast<const uint32_t *>(bp + ks * 16);
            const uint32_t b1 = *reinterpret_cast<const uint32_t *>(bp + ks * 16 + 8);
            Mma<T>::run(d, a[ks], b0, b1);
        }
        uint32_t *c0 = reinterpret_cast<uint32_t *>(&Cs[warp * 16 + g][nt * 8 + 2 * t]);
        uint32_t *c1 = reinterpret_cast<uint32_t *>(&Cs[warp * 16 + g + 8][nt * 8 + 2 * t]);
        const uint32_t o0 = *c0, o1 = *c1;
        *c0 = Mma<T>::pack(Mma<T>::lo(o0) + d[0], Mma<T>::hi(o0) + d[1]);
        *c1 = Mma<T>::pack(Mma<T>::lo(o1) + d[2], Mma<T>::hi(o1) + d[3]);
    }
    __syncthreads();
    for (int v = tid; v < RU_TM * (RU_TN / 8); v += 128) {
        const int r = v / (RU_TN / 8), cv = v - r * (RU_TN / 8);
        if (m0 + r < M && n0 + cv * 8 < N)
            *reinterpret_cast<uint4 *>(C + (long)(m0 + r) * ldc + n0 + cv * 8) = *reinterpret_cast<const uint4 *>(&Cs[r][cv * 8]);
    }
}

// The same update with the X tile formed in the kernel (implicit-pivoting sweep, gje_ip.cu):
//   X[r, :] = -P[r, :] M,  M = T for finished rows (pos[r] < k), Linv for active rows
//   (pos[r] >= k + 32), and X[r, :] = T[pos[r] - k, :] for the panel's pivot rows,
// P (fp32, n x 32) = the panel kernel's export (finished rows: their panel entries, active rows:
// their multipliers), TL = T then Linv (fp32, 32 x 32 each).  Per element the summation order
// and the single rounding to u_s of gje_ip_x_kernel, so the result is bitwise the same as with
// a separate X kernel -- without its launch, its n x 32 round trip through memory and its 9 us
// on the critical path of every 32 columns.  C is A[:, K0 : K0 + N]; its panel columns
// [k, k + 32) count as zero on input (B is the identity there: they receive X itself).
// Each 64-row X tile is formed once per 128-column tile (four times for a 512-column block):
// 512 multiply-adds per thread, two threads per row.
template <typename T>
__global__ void __launch_bounds__(128)
rank32_fused_kernel(int M, int N, int k, int K0, const float *__restrict__ P, const float *__restrict__ TL,
                    const int *__restrict__ pos, const T *__restrict__ Bt, T *__restrict__ C, long ldc)
{
    __shared__ __align__(16) T Cs[RU_TM][RU_CLD];
    __shared__ __align__(16) T Bs[RU_TN][RU_BLD];
    __shared__ __align__(16) T Xs[RU_TM][RU_BLD];
    __shared__ __align__(16) float Ms[2][32 * 32];               // T, Linv
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int m0 = blockIdx.y * RU_TM, n0 = blockIdx.x * RU_TN;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int v = tid; v < RU_TM * (RU_TN / 8); v += 128) {
        const int r = v / (RU_TN / 8), cv = v - r * (RU_TN / 8);
        if (m0 + r < M && n0 + cv * 8 < N) cp_async16(&Cs[r][cv * 8], C + (long)(m0 + r) * ldc + n0 + cv * 8);
    }
    for (int v = tid; v < RU_TN * (RU_K / 8); v += 128) {
        const int r = v / (RU_K / 8), cv = v - r * (RU_K / 8);
        if (n0 + r < N) cp_async16(&Bs[r][cv * 8], Bt + (long)(n0 + r) * RU_K + cv * 8);
        else *reinterpret_cast<uint4 *>(&Bs[r][cv * 8]) = make_uint4(0u, 0u, 0u, 0u);
    }
    for (int v = tid; v < 2 * 32 * 32 / 4; v += 128) cp_async16(&Ms[0][0] + v * 4, TL + v * 4);
    asm volatile("cp.async.commit_group;" ::: "memory");
    // ---- this thread's half row of X: row tid / 2, columns 16 (tid & 1) .. + 15
    const int xr = tid >> 1, c0 = (tid & 1) * 16, row = m0 + xr;
    float pr[32];
    int p = -1;
    if (row < M) {
        p = pos[row];
        const float4 *src = reinterpret_cast<const float4 *>(P + (long)row * 32);
#pragma unroll
        for (int u = 0; u < 8; u++) { const float4 v = src[u]; pr[4 * u] = v.x; pr[4 * u + 1] = v.y; pr[4 * u + 2] = v.z; pr[4 * u + 3] = v.w; }
    } else {
#pragma unroll
        for (int u = 0; u < 32; u++) pr[u] = 0.f;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    {
        float acc[16];
        if (p >= k && p < k + 32) {
            const float *tr = &Ms[0][(p - k) * 32 + c0];
#pragma unroll
            for (int e = 0; e < 16; e++) acc[e] = tr[e];
        } else {
            const float *Mm = (p < k) ? Ms[0] : Ms[1];
#pragma unroll
            for (int e = 0; e < 16; e++) acc[e] = 0.f;
#pragma unroll
            for (int t = 0; t < 32; t++) {
                const float m = -pr[t];
#pragma unroll
                for (int e4 = 0; e4 < 16; e4 += 4) {
                    const float4 mv = *reinterpret_cast<const float4 *>(Mm + t * 32 + c0 + e4);
                    acc[e4 + 0] = fmaf(m, mv.x, acc[e4 + 0]);
                    acc[e4 + 1] = fmaf(m, mv.y, acc[e4 + 1]);
                    acc[e4 + 2] = fmaf(m, mv.z, acc[e4 + 2]);
                    acc[e4 + 3] = fmaf(m, mv.w, acc[e4 + 3]);
                }
            }
        }
        uint32_t w[8];
#pragma unroll
        for (int e = 0; e < 8; e++) w[e] = Mma<T>::pack(acc[2 * e], acc[2 * e + 1]);
        *reinterpret_cast<uint4 *>(&Xs[xr][c0]) = make_uint4(w[0], w[1], w[2], w[3]);
        *reinterpret_cast<uint4 *>(&Xs[xr][c0 + 8]) = make_uint4(w[4], w[5], w[6], w[7]);
    }
    __syncthreads();
    const int g = lane >> 2, t = lane & 3;
    uint32_t a[2][4];
#pragma unroll
    for (int ks = 0; ks < 2; ks++)
#pragma unroll
        for (int h = 0; h < 4; h++)
            a[ks][h] = *reinterpret_cast<const uint32_t *>(&Xs[warp * 16 + g + (h & 1) * 8][ks * 16 + 2 * t + (h >> 1) * 8]);
    const int pc0 = k - K0 - n0;                                 // panel columns inside this tile: [pc0, pc0 + 32)
#pragma unroll 4
    for (int nt = 0; nt < RU_TN / 8; nt++) {
        float d[4] = {0.f, 0.f, 0.f, 0.f};
        const T *bp = &Bs[nt * 8 + g][2 * t];
#pragma unroll
        for (int ks = 0; ks < 2; ks++) {
            const uint32_t b0 = *reinterpret_cast<const uint32_t *>(bp + ks * 16);
            const uint32_t b1 = *reinterpret_cast<const uint32_t *>(bp + ks * 16 + 8);
            Mma<T>::run(d, a[ks], b0, b1);
        }
        uint32_t *q0 = reinterpret_cast<uint32_t *>(&Cs[warp * 16 + g][nt * 8 + 2 * t]);
        uint32_t *q1 = reinterpret_cast<uint32_t *>(&Cs[warp * 16 + g + 8][nt * 8 + 2 * t]);
        const bool pan = nt * 8 >= pc0 && nt * 8 < pc0 + 32;     // (an n-tile is inside the panel or outside)
        const uint32_t o0 = pan ? 0u : *q0, o1 = pan ? 0u : *q1;
        *q0 = Mma<T>::pack(Mma<T>::lo(o0) + d[0], Mma<T>::hi(o0) + d[1]);
        *q1 = Mma<T>::pack(Mma<T>::lo(o1) + d[2], Mma<T>::hi(o1) + d[3]);
    }
    __syncthreads();
    for (int v = tid; v < RU_TM * (RU_TN / 8); v += 128) {
        const int r = v / (RU_TN / 8), cv = v - r * (RU_TN / 8);
        if (m0 + r < M && n0 + cv * 8 < N)
            *reinterpret_cast<uint4 *>(C + (long)(m0 + r) * ldc + n0 + cv * 8) = *reinterpret_cast<const uint4 *>(&Cs[r][cv * 8]);
    }
}

}  // namespace

int rank32_fused_update(cudaStream_t s, int prec, int M, int N, int k, int K0, const float *P, const float *TL,
                        const int *pos, const void *Bt, void *C, long ldc, bool pdl)
{
    if (M <= 0 || N <= 0) return LYAP_OK;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ceil_div(N, RU_TN), ceil_div(M, RU_TM));
    cfg.blockDim = dim3(128);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    if (prec == LYAP_BF16)
        LYAP_CUDA_TRY(cudaLaunchKernelEx(&cfg, rank32_fused_kernel<__nv_bfloat16>, M, N, k, K0, P, TL, pos,
                                         (const __nv_bfloat16 *)Bt, (__nv_bfloat16 *)C, ldc));
    else
        LYAP_CUDA_TRY(cudaLaunchKernelEx(&cfg, rank32_fused_kernel<__half>, M, N, k, K0, P, TL, pos, (const __half *)Bt,
                                         (__half *)C, ldc));
    return launched();
}

bool rank32_update_ok(int prec, int N, const void *X, const void *Bt, const void *C, long ldc)
{
    return (prec == LYAP_FP16 || prec == LYAP_BF16) && N % 8 == 0 && (ldc * 2) % 16 == 0 && ((uintptr_t)C % 16) == 0 &&
           ((uintptr_t)X % 16) == 0 && ((uintptr_t)Bt % 16) == 0 && !env_flag("LYAP_NO_RANK32");
}

int rank32_update(cudaStream_t s, int prec, int M, int N, const void *X, const void *Bt, void *C, long ldc, bool pdl)
{
    if (M <= 0 || N <= 0) return LYAP_OK;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ceil_div(N, RU_TN), ceil_div(M, RU_TM));
    cfg.blockDim = dim3(128);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    if (prec == LYAP_BF16)
        LYAP_CUDA_TRY(cudaLaunchKernelEx(&cfg, rank32_update_kernel<__nv_bfloat16>, M, N, (const __nv_bfloat16 *)X,
                                         (const __nv_bfloat16 *)Bt, (__nv_bfloat16 *)C, ldc));
    else
        LYAP_CUDA_TRY(cudaLaunchKernelEx(&cfg, rank32_update_kernel<__half>, M, N, (const __half *)X, (const __half *)Bt,
                                         (__half *)C, ldc));
    return launched();
}

}  // namespace lyap
