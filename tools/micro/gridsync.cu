// microbenchmark: cost of cooperative-groups grid.sync() on this GPU
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int iters, int *x) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; i++) { if (threadIdx.x == 0) atomicAdd(x, 1); g.sync(); }
}
// hand-rolled barrier: sense-reversing counter
__global__ void k2(int iters, unsigned *bar, int *x) {
    volatile unsigned *vb = bar;
    unsigned nb = gridDim.x;
    for (int i = 0; i < iters; i++) {
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned target = (i + 1) * nb;
            __threadfence();
            atomicAdd(bar, 1);
            while (vb[0] < target) { }
            __threadfence();
        }
        __syncthreads();
    }
}
// flag-array barrier: every CTA publishes its own sequence number (one release store, no
// atomic), warp 0 of every CTA polls all flags (acquire loads), one __syncthreads each side
__global__ void k3(int iters, unsigned *flags) {
    const unsigned nb = gridDim.x;
    for (int i = 0; i < iters; i++) {
        __syncthreads();
        if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(flags + blockIdx.x * 32), "r"(i + 1) : "memory");
        if (threadIdx.x < 32) {
            for (unsigned b = threadIdx.x; b < nb; b += 32) {
                unsigned v;
                do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + b * 32) : "memory"); } while (v < (unsigned)(i + 1));
            }
        }
        __syncthreads();
    }
}
int main() {
    int *x; unsigned *bar; cudaMalloc(&x, 4); cudaMalloc(&bar, 4);
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    for (int grid : {16, 64, 148}) {
        int iters = 2000;
        void *args[] = {&iters, &x};
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaLaunchCooperativeKernel((void*)k, grid, 256, args, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k, grid, 256, args, 0, 0);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        cudaMemset(bar, 0, 4);
        void *args2[] = {&iters, &bar, &x};
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k2, grid, 256, args2, 0, 0);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms2; cudaEventElapsedTime(&ms2, a, b);
        unsigned *fl; cudaMalloc(&fl, 4 * 32 * 256); cudaMemset(fl, 0, 4 * 32 * 256);
        void *args3[] = {&iters, &fl};
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k3, grid, 256, args3, 0, 0);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms3; cudaEventElapsedTime(&ms3, a, b);
        printf("grid %d: cg grid.sync %.3f us, custom barrier %.3f us, flag array %.3f us (err %s)\n", grid, ms * 1e3 / iters, ms2 * 1e3 / iters, ms3 * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    }
}
