// cost of k STS.128 by one lane per warp immediately before __syncthreads (the barrier drains stores)
#include <cstdio>
#include <cuda_runtime.h>
template <int K>
__global__ void probe(long long *out)
{
    __shared__ __align__(16) float buf[32][K * 4 + 4];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    float acc = tid;
    const int N = 64;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < N; i++) {
        if (lane == (i & 31)) {
#pragma unroll
            for (int c = 0; c < K; c++) *reinterpret_cast<float4 *>(&buf[wid][c * 4]) = make_float4(acc, acc + 1, acc + 2, acc + 3);
        }
        __syncthreads();
        acc += buf[(wid + 1) % (blockDim.x / 32)][(i & 3)];
    }
    long long t1 = clock64();
    if (tid == 0) out[0] = (t1 - t0) / N;
    if (acc == 1234.5f) out[1] = 1;
}
int main()
{
    long long *o; cudaMalloc(&o, 64);
    long long h;
    for (int nt : {256, 1024}) {
        probe<1><<<1, nt>>>(o); cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost); printf("nt=%d K=1: %lld cycles/iter\n", nt, h);
        probe<3><<<1, nt>>>(o); cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost); printf("nt=%d K=3: %lld cycles/iter\n", nt, h);
        probe<9><<<1, nt>>>(o); cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost); printf("nt=%d K=9: %lld cycles/iter\n", nt, h);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
