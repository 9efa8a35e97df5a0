// DSMEM push throughput into ONE destination CTA / mbarrier: N x st.async.v4 (16 B each, one
// complete_tx per store) against bulk shared->shared::cluster copies (one complete_tx per copy).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) { uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o; }
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" :: "r"(smem_addr(b)), "r"(parity) : "memory");
}
#define CSYNC() asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory")
// every CTA pushes `per` 16-byte stores (or one bulk copy of 16*per bytes) to EVERY CTA; all wait for all
__global__ void probe(long long *out, int per, int bulk)
{
    __shared__ __align__(128) float box[16][64];   // per source CTA 256 B
    __shared__ __align__(128) float src[64];
    __shared__ __align__(8) uint64_t mb;
    uint32_t q, NC; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(q)); asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(NC));
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_addr(&mb))); asm volatile("fence.mbarrier_init.release.cluster;"); }
    if (tid < 64) src[tid] = tid;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    CSYNC();
    const int N = 32;
    long long t0 = clock64();
    for (int i = 0; i < N; i++) {
        if (tid == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_addr(&mb)), "r"(NC * per * 16) : "memory");
        if (wid < (int)NC) {           // warp w -> CTA w
            uint32_t m = mapa(smem_addr(&mb), wid);
            if (!bulk) {
                if (lane < per) {
                    uint32_t dst = mapa(smem_addr(&box[q][lane * 4]), wid);
                    asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1,%2,%3,%4}, [%5];" :: "r"(dst), "r"(i), "r"(i), "r"(i), "r"(i), "r"(m) : "memory");
                }
            } else if (lane == 0) {
                uint32_t dst = mapa(smem_addr(&box[q][0]), wid);
                asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(dst), "r"(smem_addr(&src[0])), "r"(per * 16), "r"(m) : "memory");
            }
        }
        mbar_wait(&mb, i & 1);
    }
    long long t1 = clock64();
    if (tid == 0 && q == 0) out[0] = (t1 - t0) / N;
    CSYNC();
}
int main()
{
    long long *o; cudaMalloc(&o, 64);
    cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int nc : {2, 4, 8, 16}) for (int bulk : {0, 1}) for (int per : {1, 4, 9, 16}) {
        cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(nc); cfg.blockDim = dim3(512);
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = nc; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, probe, o, per, bulk);
        long long h; cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
        printf("NC=%2d %s per-source %2d x16B: %5lld cycles per all-to-all round (%s)\n", nc, bulk ? "bulk " : "stas ", per, h, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
