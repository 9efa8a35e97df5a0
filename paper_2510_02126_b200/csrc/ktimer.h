// ktimer.h -- kernel classes that bench.py can time with CUDA events.
#pragma once
#include <cuda_runtime.h>

namespace lyap {

enum KernelClass {
    KC_GJE_UPDATE = 0,   // rank-b update GEMM of the Gauss-Jordan inversion
    KC_GJE_PANEL = 1,    // pivoted panel factorization
    KC_ZSIDE_GEMM = 2,   // A_k^{-1} Z_k products
    KC_JACOBI = 3,       // fp64 symmetric eigensolver
    KC_QR = 4,           // fp64 Householder QR
    KC_RESID_GEMM = 5,   // fp64 A Z of the residual factor
    KC_NEWTON_UPDATE = 6,// fused Newton averaging update
    KC_DGEMM = 7,        // fp64 DMMA GEMM kernel (all fp64 products)
    KC_TCGEMM = 8,       // tcgen05 16-bit GEMM kernel
    KC_QR_PANEL = 9,     // Householder panel kernel
    KC_TRIDIAG = 10,     // cooperative tridiagonalisation kernel
    KC_WY = 11,          // fused compact-WY block-reflector application
    KC_RRQR = 12         // column-pivoted QR of RankTruncChol
};

void ktimer_begin(int cls, cudaStream_t s);
void ktimer_end(int cls, cudaStream_t s);
void ktimer_work(int cls, double flops, double bytes);   // algorithmic work of one timed launch

struct KTimer {
    int c;
    cudaStream_t s;
    KTimer(int cls, cudaStream_t st) : c(cls), s(st) { ktimer_begin(c, s); }
    KTimer(int cls, cudaStream_t st, double flops, double bytes) : c(cls), s(st) {
        ktimer_begin(c, s);
        ktimer_work(c, flops, bytes);
    }
    ~KTimer() { ktimer_end(c, s); }
};

}  // namespace lyap
