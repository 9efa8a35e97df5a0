// common.cuh -- shared device/host helpers of the B200 Lyapunov IR library.
// Product code only (no oracle code is shared).
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <algorithm>
#include "../../include/lyap_ir.h"

namespace lyap {

extern std::atomic<int64_t> g_launches;

#define LYAP_CUDA_TRY(expr)                                                        \
    do {                                                                           \
        cudaError_t _e = (expr);                                                   \
        if (_e != cudaSuccess) {                                                   \
            fprintf(stderr, "lyap: CUDA error %s at %s:%d\n", cudaGetErrorString(_e), \
                    __FILE__, __LINE__);                                           \
            return LYAP_ERR_CUDA;                                                  \
        }                                                                          \
    } while (0)

#define LYAP_TRY(...)                  \
    do {                               \
        int _r = (__VA_ARGS__);        \
        if (_r != LYAP_OK) return _r;  \
    } while (0)

// Count a launch and check for launch errors.  LYAP_SYNC_DEBUG=1 synchronises after every
// launch and names the launch site of an asynchronous fault (debugging only).
inline int launched(const char *file = __builtin_FILE(), int line = __builtin_LINE()) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    static const bool sync_dbg = [] { const char *v = getenv("LYAP_SYNC_DEBUG"); return v && v[0] == '1'; }();
    if (e == cudaSuccess && sync_dbg) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        fprintf(stderr, "lyap: launch error %s (launch at %s:%d)\n", cudaGetErrorString(e), file, line);
        return LYAP_ERR_CUDA;
    }
    return LYAP_OK;
}

inline int ceil_div(long a, long b) { return (int)((a + b - 1) / b); }

// debugging switches read once per process (LYAP_QR_1CTA=1 etc.)
inline bool env_flag(const char *name) {
    const char *e = getenv(name);
    return e && e[0] && e[0] != '0';
}

// ---------------------------------------------------------------- precision
template <typename T> struct Prec;
template <> struct Prec<double>        { using acc = double; static constexpr int code = LYAP_FP64; static constexpr int t = 53; };
template <> struct Prec<float>         { using acc = float;  static constexpr int code = LYAP_FP32; static constexpr int t = 24; };
template <> struct Prec<__half>        { using acc = float;  static constexpr int code = LYAP_FP16; static constexpr int t = 11; };
template <> struct Prec<__nv_bfloat16> { using acc = float;  static constexpr int code = LYAP_BF16; static constexpr int t = 8; };

__host__ __device__ inline double unit_roundoff(int prec) {
    return prec == LYAP_FP64 ? 0x1p-53 : prec == LYAP_FP32 ? 0x1p-24 : prec == LYAP_FP16 ? 0x1p-11 : 0x1p-8;
}
inline size_t elem_size(int prec) { return prec == LYAP_FP64 ? 8 : prec == LYAP_FP32 ? 4 : 2; }

template <typename T> __device__ __forceinline__ float  to_f(T x);
template <> __device__ __forceinline__ float to_f<float>(float x) { return x; }
template <> __device__ __forceinline__ float to_f<__half>(__half x) { return __half2float(x); }
template <> __device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }

template <typename T> __device__ __forceinline__ double to_d(T x) { return (double)to_f<T>(x); }
template <> __device__ __forceinline__ double to_d<double>(double x) { return x; }

template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ __half from_f<__half>(float x) { return __float2half_rn(x); }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }
template <> __device__ __forceinline__ double from_f<double>(float x) { return (double)x; }

template <typename T> __device__ __forceinline__ T from_d(double x);
template <> __device__ __forceinline__ double from_d<double>(double x) { return x; }
template <> __device__ __forceinline__ float from_d<float>(double x) { return __double2float_rn(x); }
template <> __device__ __forceinline__ __half from_d<__half>(double x) { return __double2half(x); }
template <> __device__ __forceinline__ __nv_bfloat16 from_d<__nv_bfloat16>(double x) { return __double2bfloat16(x); }

// Accumulator conversions: acc is float for 16/32-bit storage, double for fp64.
template <typename T> __device__ __forceinline__ typename Prec<T>::acc to_acc(T x);
template <> __device__ __forceinline__ double to_acc<double>(double x) { return x; }
template <> __device__ __forceinline__ float to_acc<float>(float x) { return x; }
template <> __device__ __forceinline__ float to_acc<__half>(__half x) { return __half2float(x); }
template <> __device__ __forceinline__ float to_acc<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }

template <typename T> __device__ __forceinline__ T from_acc(typename Prec<T>::acc x);
template <> __device__ __forceinline__ double from_acc<double>(double x) { return x; }
template <> __device__ __forceinline__ float from_acc<float>(float x) { return x; }
template <> __device__ __forceinline__ __half from_acc<__half>(float x) { return __float2half_rn(x); }
template <> __device__ __forceinline__ __nv_bfloat16 from_acc<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

// Round a double to precision `prec` and back (value semantics of storing in prec).
__device__ __forceinline__ double round_to(double x, int prec) {
    switch (prec) {
        case LYAP_FP32: return (double)__double2float_rn(x);
        case LYAP_FP16: return (double)__half2float(__double2half(x));
        case LYAP_BF16: return (double)__bfloat162float(__double2bfloat16(x));
        default: return x;
    }
}

// ---------------------------------------------------------------- reductions
template <typename V>
__device__ __forceinline__ V warp_sum(V v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
template <typename V>
__device__ __forceinline__ V warp_max(V v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block-wide sum; every thread gets the result.  `sh` needs 32 slots.
template <typename V>
__device__ V block_sum(V v, V *sh) {
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    V t = (threadIdx.x < (unsigned)nw) ? sh[threadIdx.x] : V(0);
    if (w == 0) t = warp_sum(t);
    if (threadIdx.x == 0) sh[0] = t;
    __syncthreads();
    V r = sh[0];
    __syncthreads();
    return r;
}
template <typename V>
__device__ V block_max(V v, V *sh) {
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_max(v);
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    V t = (threadIdx.x < (unsigned)nw) ? sh[threadIdx.x] : V(0);
    if (w == 0) t = warp_max(t);
    if (threadIdx.x == 0) sh[0] = t;
    __syncthreads();
    V r = sh[0];
    __syncthreads();
    return r;
}

// atomicMax on non-negative doubles via their ordered bit patterns.
__device__ __forceinline__ void atomic_max_nonneg(double *addr, double v) {
    atomicMax(reinterpret_cast<unsigned long long *>(addr), (unsigned long long)__double_as_longlong(v));
}

}  // namespace lyap
