// Latency probes for the Gauss-Jordan panel's per-column chain (sm_100a): redux.sync, ballot,
// __syncthreads, IEEE division, st.async -> mbarrier round trips (own CTA / remote CTA).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) { uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o; }
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" :: "r"(smem_addr(b)), "r"(parity) : "memory");
}
__global__ void __cluster_dims__(2, 1, 1) probe(long long *out, float dd)
{
    __shared__ __align__(16) float box[64];
    __shared__ __align__(8) uint64_t mb[2];
    __shared__ float sm[1024];
    uint32_t q; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(q));
    const int tid = threadIdx.x, lane = tid & 31;
    if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_addr(&mb[0]))); asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_addr(&mb[1])));
                    asm volatile("fence.mbarrier_init.release.cluster;"); }
    for (int i = tid; i < 1024; i += blockDim.x) sm[i] = (float)((i * 7 + 1) % 1024);
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    const int N = 64;
    long long t0, t1;
    // 1. redux chain
    unsigned x = tid * 2654435761u;
    t0 = clock64();
    for (int i = 0; i < N; i++) x = __reduce_max_sync(0xffffffffu, x ^ (unsigned)i) + lane;
    t1 = clock64();
    if (tid == 0 && q == 0) out[0] = (t1 - t0) / N;
    // 2. ballot + ffs chain
    t0 = clock64();
    for (int i = 0; i < N; i++) { unsigned b = __ballot_sync(0xffffffffu, (x & 1u) == 0u); x += __ffs(b) + i; }
    t1 = clock64();
    if (tid == 0 && q == 0) out[1] = (t1 - t0) / N;
    // 3. __syncthreads (all warps), with one LDS dependent on it
    float acc = 0.f;
    t0 = clock64();
    for (int i = 0; i < N; i++) { sm[tid] = acc; __syncthreads(); acc += sm[(tid + 32) % blockDim.x]; }
    t1 = clock64();
    if (tid == 0 && q == 0) out[2] = (t1 - t0) / N;
    // 4. division chain
    float d = dd;
    t0 = clock64();
    for (int i = 0; i < N; i++) d = 1.f / d + 0.5f;
    t1 = clock64();
    if (tid == 0 && q == 0) out[3] = (t1 - t0) / N;
    // 5. LDS pointer chase
    int idx = lane;
    t0 = clock64();
    for (int i = 0; i < N; i++) idx = (int)sm[idx];
    t1 = clock64();
    if (tid == 0 && q == 0) out[4] = (t1 - t0) / N;
    __syncthreads();
    // 6. st.async to own CTA + mbarrier wait round trip (warp 0 only)
    if (tid < 32) {
        t0 = clock64();
        for (int i = 0; i < N; i++) {
            if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_addr(&mb[0])), "r"(16) : "memory");
            if (lane == 0) {
                uint32_t dst = mapa(smem_addr(&box[0]), q), m = mapa(smem_addr(&mb[0]), q);
                asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1,%2,%3,%4}, [%5];" :: "r"(dst), "r"(i), "r"(i), "r"(i), "r"(i), "r"(m) : "memory");
            }
            mbar_wait(&mb[0], i & 1);
            acc += box[0];
        }
        t1 = clock64();
        if (tid == 0 && q == 0) out[5] = (t1 - t0) / N;
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    // 7. ping-pong between the two CTAs: one-way latency = round trip / 2
    if (tid < 32) {
        t0 = clock64();
        for (int i = 0; i < N; i++) {
            if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_addr(&mb[1])), "r"(16) : "memory");
            if (q == 0) {
                if (lane == 0) { uint32_t dst = mapa(smem_addr(&box[4]), 1), m = mapa(smem_addr(&mb[1]), 1);
                    asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1,%2,%3,%4}, [%5];" :: "r"(dst), "r"(i), "r"(i), "r"(i), "r"(i), "r"(m) : "memory"); }
                mbar_wait(&mb[1], i & 1);
            } else {
                mbar_wait(&mb[1], i & 1);
                if (lane == 0) { uint32_t dst = mapa(smem_addr(&box[4]), 0), m = mapa(smem_addr(&mb[1]), 0);
                    asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1,%2,%3,%4}, [%5];" :: "r"(dst), "r"(i), "r"(i), "r"(i), "r"(i), "r"(m) : "memory"); }
            }
            acc += box[4];
        }
        t1 = clock64();
        if (tid == 0 && q == 0) out[6] = (t1 - t0) / N / 2;
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    // 8. cluster barrier
    t0 = clock64();
    for (int i = 0; i < N; i++) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    t1 = clock64();
    if (tid == 0 && q == 0) out[7] = (t1 - t0) / N;
    if (acc == 12345.f && x == 77 && d == 3.f && idx == 5) out[15] = 1;
}
int main()
{
    long long *o; cudaMalloc(&o, 16 * sizeof(long long)); cudaMemset(o, 0, 128);
    for (int nt : {32, 256, 1024}) {
        probe<<<2, nt>>>(o, 1.37f);
        long long h[16]; cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
        printf("nt=%4d: redux %lld  ballot+ffs %lld  syncthreads+LDS %lld  div %lld  LDS %lld  st.async self %lld  remote one-way %lld  cluster barrier %lld  (%s)\n",
               nt, h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
