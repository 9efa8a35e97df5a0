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
    KC_NEWTON_UPDATE = 6 // fused Newton averaging update
};

void ktimer_begin(int cls, cudaStream_t s);
void ktimer_end(int cls, cudaStream_t s);

struct KTimer {
    int c;
    cudaStream_t s;
    KTimer(int cls, cudaStream_t st) : c(cls), s(st) { ktimer_begin(c, s); }
    ~KTimer() { ktimer_end(c, s); }
};

}  // namespace lyap
