// Micro-benchmark: cost of a thread-block-cluster barrier, of __syncthreads, and of a
// DSMEM load round trip on B200 (sizes 1..16 CTAs, 512 threads).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_clsync(int iters, long long *out) {
    cg::cluster_group cl = cg::this_cluster();
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) cl.sync();
    long long t1 = clock64();
    if (threadIdx.x == 0 && cl.block_rank() == 0) out[0] = (t1 - t0) / iters;
}
__global__ void k_bar(int iters, long long *out) {
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (t1 - t0) / iters;
}
__global__ void k_dsmem(int iters, long long *out) {
    cg::cluster_group cl = cg::this_cluster();
    __shared__ double buf[64];
    if (threadIdx.x < 64) buf[threadIdx.x] = threadIdx.x;
    cl.sync();
    const unsigned nb = cl.num_blocks();
    double acc = 0;
    long long t0 = clock64();
    if (threadIdx.x == 0) {
        for (int i = 0; i < iters; i++) {
            const double *r = cl.map_shared_rank(buf, (cl.block_rank() + 1) % nb);
            acc += r[(i + (int)acc) & 63];        // dependent chain
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && cl.block_rank() == 0) { out[2] = (t1 - t0) / iters; out[3] = (long long)acc; }
    cl.sync();
}
// barrier + DSMEM gather pattern of one panel column: arrive/wait + 8 remote loads
__global__ void k_pattern(int iters, long long *out) {
    cg::cluster_group cl = cg::this_cluster();
    __shared__ double buf[2][64];
    const unsigned nb = cl.num_blocks();
    double acc = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        if (threadIdx.x < 32) buf[i & 1][threadIdx.x] = acc + i;
        __syncthreads();
        cl.sync();
        if (threadIdx.x < 32) {
            double v = 0;
            if ((threadIdx.x & 31) < (int)nb) v = cl.map_shared_rank(buf[i & 1], threadIdx.x)[threadIdx.x];
            for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            acc += v * 1e-9;
        }
        __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && cl.block_rank() == 0) { out[4] = (t1 - t0) / iters; out[5] = (long long)acc; }
    cl.sync();
}

template <typename K>
void run(K kern, int nb, int iters, long long *d) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nb); cfg.blockDim = dim3(512);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = nb; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, iters, d);
    if (e != cudaSuccess) printf("launch error %s\n", cudaGetErrorString(e));
    cudaDeviceSynchronize();
}

int main() {
    long long *d, h[8];
    cudaMalloc(&d, 64);
    for (int nb : {1, 2, 4, 8, 16}) {
        run(k_clsync, nb, 2000, d);
        run(k_bar, nb, 2000, d);
        run(k_dsmem, nb, 2000, d);
        run(k_pattern, nb, 2000, d);
        cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
        printf("cluster %2d x 512 thr: cluster.sync %5lld clk  __syncthreads %4lld clk  dsmem load %4lld clk  "
               "column pattern %5lld clk\n", nb, h[0], h[1], h[2], h[4]);
    }
    return 0;
}
