// gje.cu -- blocked in-place inversion A <- A^{-1} for the Newton step
// A_k = (mu A_{k-1} + mu^{-1} A_{k-1}^{-1})/2 (PAPER.md Eq. newton-lyapu1 l.1125).
//
// Algorithm: blocked Gauss-Jordan elimination with partial pivoting.  Each
// block step k (panel width b) is
//   1. panel kernel (one CTA): LU with partial pivoting of the panel
//      A[k:n, k:k+b] (warp-shuffle argmax pivot search), inversion of the
//      b x b pivot block T = A11^{-1}, and the multiplier block
//      X = [-A[0:k,panel] T ; T ; -L21 L11^{-1}]            (n x b)
//   2. row-swap / prep kernels: apply the pivot rows to all n columns, copy
//      the pivot rows to B (b x n) with B[:, panel] = I, zero the pivot rows
//      and the panel columns of A,
//   3. rank-b update A += X B (n x n x b GEMM, fp32 accumulation for 16-bit
//      storage).
// After the last step A holds (PA)^{-1} = A^{-1} P^T, i.e. A^{-1}[:, rowperm[i]]
// = A[:, i]; the caller gathers columns with invperm.  The pivot sequence is
// exactly that of LU with partial pivoting (the rows below the block see the
// same Schur complement as right-looking LU).
#include "common.cuh"
#include "gemm_simt.cuh"
#include "lyap_internal.h"
#include "ktimer.h"

namespace lyap {

// -------------------------------------------------------------------- panel
template <typename Acc>
struct ArgMax { Acc v; int i; };

template <typename Acc>
__device__ __forceinline__ void argmax_merge(Acc &v, int &i, Acc v2, int i2) {
    if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
}

template <typename T>
__global__ void __launch_bounds__(1024)
gje_panel_kernel(int n, int k, int b, T *__restrict__ A, T *__restrict__ X,
                 int *__restrict__ ipiv, int *__restrict__ moved, int *__restrict__ nmoved,
                 int *__restrict__ info, typename Prec<T>::acc *__restrict__ Pglob, int use_smem)
{
    using Acc = typename Prec<T>::acc;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int R = n - k;
    const int tid = threadIdx.x, nt = blockDim.x;
    Acc *Lw = reinterpret_cast<Acc *>(smem_raw);              // b*b : Linv
    Acc *Tw = Lw + 32 * 32;                                    // b*b : T = A11^{-1}
    Acc *redv = Tw + 32 * 32;                                  // 32
    int *redi = reinterpret_cast<int *>(redv + 32);            // 32
    int *pivl = redi + 32;                                     // 32 local pivots
    int *sflag = pivl + 32;                                    // 1
    Acc *P = use_smem ? reinterpret_cast<Acc *>(sflag + 4) : Pglob;   // R*b (row-major, ld b)

    for (int idx = tid; idx < R * b; idx += nt) {
        const int r = idx / b, c = idx - r * b;
        P[idx] = to_acc<T>(A[(long)(k + r) * n + k + c]);
    }
    if (tid == 0) *sflag = 0;
    __syncthreads();

    for (int j = 0; j < b; j++) {
        // ---- pivot search: max |P[r][j]|, r >= j, lowest index on ties
        Acc bv = Acc(-1); int bi = R;
        for (int r = j + tid; r < R; r += nt) {
            Acc v = fabs(P[(long)r * b + j]);
            argmax_merge(bv, bi, v, r);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            Acc v2 = __shfl_xor_sync(0xffffffffu, bv, o);
            int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
            argmax_merge(bv, bi, v2, i2);
        }
        if ((tid & 31) == 0) { redv[tid >> 5] = bv; redi[tid >> 5] = bi; }
        __syncthreads();
        if (tid < 32) {
            int nw = nt >> 5;
            bv = tid < nw ? redv[tid] : Acc(-1);
            bi = tid < nw ? redi[tid] : R;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                Acc v2 = __shfl_xor_sync(0xffffffffu, bv, o);
                int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
                argmax_merge(bv, bi, v2, i2);
            }
            int p = bi;
            if (tid == 0) {
                pivl[j] = p;
                if (!(bv > Acc(0))) {            // zero (or nan) pivot column
                    if (*sflag == 0) *sflag = k + j + 1;
                }
            }
            // swap rows j and p (one warp, b <= 32 columns)
            if (p != j && tid < b) {
                Acc t = P[(long)j * b + tid];
                P[(long)j * b + tid] = P[(long)p * b + tid];
                P[(long)p * b + tid] = t;
            }
        }
        __syncthreads();
        const Acc d = P[(long)j * b + j];
        if (d != Acc(0)) {
            const Acc inv = Acc(1) / d;
            for (int r = j + 1 + tid; r < R; r += nt) {
                Acc *row = P + (long)r * b;
                Acc l = row[j] * inv;
                row[j] = l;
                for (int c = j + 1; c < b; c++) row[c] = fma(-l, P[(long)j * b + c], row[c]);
            }
        }
        __syncthreads();
    }

    // ---- Linv = L11^{-1} (unit lower), Uinv = U11^{-1}; T = Uinv * Linv
    Acc *Uw = Tw;   // reuse T storage for Uinv first, then form T into Lw/Tw carefully
    if (tid < b) {
        int c = tid;
        // Linv column c
        for (int i = 0; i < b; i++) {
            Acc s = (i == c) ? Acc(1) : Acc(0);
            if (i > c)
                for (int t = c; t < i; t++) s = fma(-P[(long)i * b + t], Lw[t * 32 + c], s);
            Lw[i * 32 + c] = (i < c) ? Acc(0) : s;
        }
    } else if (tid >= 32 && tid < 32 + b) {
        int c = tid - 32;
        for (int i = b - 1; i >= 0; i--) {
            Acc s = (i == c) ? Acc(1) : Acc(0);
            if (i < c)
                for (int t = i + 1; t <= c; t++) s = fma(-P[(long)i * b + t], Uw[t * 32 + c], s);
            Uw[i * 32 + c] = (i > c) ? Acc(0) : s / P[(long)i * b + i];
        }
    }
    __syncthreads();
    // T = Uinv * Linv, computed into registers then stored over Uw
    Acc tval = Acc(0);
    int ti = tid / 32, tc = tid % 32;
    if (ti < b && tc < b)
        for (int t = 0; t < b; t++) tval = fma(Uw[ti * 32 + t], Lw[t * 32 + tc], tval);
    __syncthreads();
    if (ti < b && tc < b) Tw[ti * 32 + tc] = tval;
    __syncthreads();

    // ---- X rows
    for (int idx = tid; idx < n * b; idx += nt) {
        const int i = idx / b, c = idx - i * b;
        Acc s = Acc(0);
        if (i >= k && i < k + b) {
            s = Tw[(i - k) * 32 + c];
        } else if (i >= k + b) {
            const Acc *row = P + (i - k) * b;
            for (int t = 0; t < b; t++) s = fma(-row[t], Lw[t * 32 + c], s);
        } else {
            const T *arow = A + (long)i * n + k;
            for (int t = 0; t < b; t++) s = fma(-to_acc<T>(arow[t]), Tw[t * 32 + c], s);
        }
        X[idx] = from_acc<T>(s);
    }
    // ---- pivots and the list of moved rows (dst local pos, src local row)
    if (tid == 0) {
        for (int j = 0; j < b; j++) ipiv[k + j] = k + pivl[j];
        if (*sflag && *info == 0) *info = *sflag;
        // replay the transpositions on a small position map of candidates
        int cand[64], src[64], nc = 0;
        for (int j = 0; j < b; j++) { cand[nc] = j; src[nc] = j; nc++; }
        for (int j = 0; j < b; j++) {
            int p = pivl[j];
            int ip = -1;
            for (int t = 0; t < nc; t++) if (cand[t] == p) { ip = t; break; }
            if (ip < 0) { cand[nc] = p; src[nc] = p; ip = nc; nc++; }
            int ij = j;   // position j is always cand[j]
            int tmp = src[ij]; src[ij] = src[ip]; src[ip] = tmp;
        }
        int m = 0;
        for (int t = 0; t < nc; t++)
            if (src[t] != cand[t]) { moved[2 * m] = cand[t]; moved[2 * m + 1] = src[t]; m++; }
        *nmoved = m;
    }
}

// gather moved source rows (full width) and their rowperm entries into tmp
template <typename T>
__global__ void gje_gather_kernel(int n, int k, const T *__restrict__ A, const int *__restrict__ moved,
                                  const int *__restrict__ nmoved, T *__restrict__ tmp,
                                  const int *__restrict__ rowperm, int *__restrict__ tmp_perm)
{
    int m = *nmoved;
    int t = blockIdx.y;
    if (t >= m) return;
    int src = k + moved[2 * t + 1];
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x)
        tmp[(long)t * n + c] = A[(long)src * n + c];
    if (blockIdx.x == 0 && threadIdx.x == 0) tmp_perm[t] = rowperm[src];
}

// scatter moved rows, build B = pivot rows with B[:, panel] = I, zero pivot rows
// and the panel columns of A.
template <typename T>
__global__ void gje_prep_kernel(int n, int k, int b, T *__restrict__ A, const int *__restrict__ moved,
                                const int *__restrict__ nmoved, const T *__restrict__ tmp,
                                const int *__restrict__ tmp_perm, int *__restrict__ rowperm,
                                T *__restrict__ B)
{
    const int m = *nmoved;
    const T zero = from_acc<T>(0), one = from_acc<T>(1);
    // rows: blockIdx.y indexes rows 0..n-1
    for (long i = blockIdx.y; i < n; i += gridDim.y) {
        int local = (int)i - k;
        int slot = -1;
        if (local >= 0 && local < n - k)
            for (int t = 0; t < m; t++) if (moved[2 * t] == local) { slot = t; break; }
        const bool in_block = (local >= 0 && local < b);
        for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
            const bool panel_col = (c >= k && c < k + b);
            if (in_block) {
                T v = (slot >= 0) ? tmp[(long)slot * n + c] : A[i * n + c];
                B[(long)c * b + local] = panel_col ? ((c - k == local) ? one : zero) : v;   // Bt: n x b
                A[i * n + c] = zero;
            } else if (slot >= 0) {
                A[i * n + c] = panel_col ? zero : tmp[(long)slot * n + c];
            } else if (panel_col) {
                A[i * n + c] = zero;
            }
        }
        if (slot >= 0 && blockIdx.x == 0 && threadIdx.x == 0) rowperm[i] = tmp_perm[slot];
    }
}

__global__ void iota_kernel(int n, int *p) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = i;
}
__global__ void invperm_kernel(int n, const int *rowperm, int *invperm) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        invperm[rowperm[i]] = i;
}

template <typename T>
__global__ void col_gather_kernel(int n, const T *__restrict__ G, const int *__restrict__ invperm, T *__restrict__ out)
{
    for (long i = blockIdx.y; i < n; i += gridDim.y)
        for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x)
            out[i * n + c] = G[i * n + invperm[c]];
}

// ------------------------------------------------------------------ driver
int gje_panel_width(int prec) { return prec == LYAP_FP64 ? 16 : 32; }

size_t gje_panel_smem(int n, int prec, int b, int R, bool *use_smem) {
    size_t acc = (prec == LYAP_FP64) ? 8 : 4;
    size_t head = acc * (2 * 32 * 32 + 32) + sizeof(int) * (32 + 32 + 4);
    size_t need = head + acc * (size_t)R * b;
    *use_smem = need <= 220 * 1024;
    return *use_smem ? need : head;
}

int GjeWork::alloc(int n_, int prec_) {
    n = n_; prec = prec_;
    int b = gje_panel_width(prec);
    size_t es = elem_size(prec);
    size_t acc = (prec == LYAP_FP64) ? 8 : 4;
    LYAP_CUDA_TRY(cudaMalloc(&X, es * (size_t)n * b));
    LYAP_CUDA_TRY(cudaMalloc(&B, es * (size_t)n * b));
    LYAP_CUDA_TRY(cudaMalloc(&tmp, es * (size_t)n * 2 * b));
    LYAP_CUDA_TRY(cudaMalloc(&Pglob, acc * (size_t)n * b));
    LYAP_CUDA_TRY(cudaMalloc(&ints, sizeof(int) * (size_t)(4 * n + 4 * b + 8)));
    ipiv = ints; rowperm = ipiv + n; invperm = rowperm + n; moved = invperm + n;
    nmoved = moved + 4 * b; info = nmoved + 1; tmp_perm = info + 1;
    return LYAP_OK;
}

void GjeWork::release() {
    cudaFree(X); cudaFree(B); cudaFree(tmp); cudaFree(Pglob); cudaFree(ints);
    X = B = tmp = nullptr; Pglob = nullptr; ints = nullptr;
}

template <typename T>
static int gje_invert_t(cudaStream_t s, int n, T *A, GjeWork &w)
{
    using Acc = typename Prec<T>::acc;
    const int b0 = gje_panel_width(Prec<T>::code);
    LYAP_CUDA_TRY(cudaMemsetAsync(w.info, 0, sizeof(int), s));
    iota_kernel<<<ceil_div(n, 256), 256, 0, s>>>(n, w.rowperm);
    LYAP_TRY(launched());
    for (int k = 0; k < n; k += b0) {
        int b = (n - k < b0) ? n - k : b0;
        bool use_smem;
        size_t sm = gje_panel_smem(n, Prec<T>::code, b, n - k, &use_smem);
        static bool attr_set = false;
        if (!attr_set) {
            LYAP_CUDA_TRY(cudaFuncSetAttribute(gje_panel_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
            attr_set = true;
        }
        {
            KTimer kt(KC_GJE_PANEL, s);
            gje_panel_kernel<T><<<1, 1024, sm, s>>>(n, k, b, A, (T *)w.X, w.ipiv + 0, w.moved, w.nmoved,
                                                    w.info, (Acc *)w.Pglob, use_smem ? 1 : 0);
        }
        LYAP_TRY(launched());
        dim3 gg(ceil_div(n, 256) < 8 ? ceil_div(n, 256) : 8, 2 * b);
        gje_gather_kernel<T><<<gg, 256, 0, s>>>(n, k, A, w.moved, w.nmoved, (T *)w.tmp, w.rowperm, w.tmp_perm);
        LYAP_TRY(launched());
        dim3 gp(ceil_div(n, 256) < 4 ? ceil_div(n, 256) : 4, n < 4096 ? n : 4096);
        gje_prep_kernel<T><<<gp, 256, 0, s>>>(n, k, b, A, w.moved, w.nmoved, (const T *)w.tmp, w.tmp_perm,
                                              w.rowperm, (T *)w.B);
        LYAP_TRY(launched());
        {
            KTimer kt(KC_GJE_UPDATE, s);
            LYAP_TRY(gemm_update(s, n, b, (const T *)w.X, (const T *)w.B, A));
        }
    }
    invperm_kernel<<<ceil_div(n, 256), 256, 0, s>>>(n, w.rowperm, w.invperm);
    return launched();
}

// A += X (n x b, row-major) * B (b x n, row-major); fp32 (fp64) accumulation.
template <typename T>
int gemm_update(cudaStream_t s, int n, int b, const T *X, const T *B, T *A)
{
    using Acc = typename Prec<T>::acc;
    // B holds the pivot rows transposed (Bt, n x b row-major): A += X Bt^T
    if constexpr (std::is_same<T, __half>::value || std::is_same<T, __nv_bfloat16>::value) {
        if (!use_simt_gemm() && b % 8 == 0)     // TMA rows must be 16-byte multiples
            return tc_gemm(s, Prec<T>::code, n, n, b, 1.0f, X, b, B, b, 1.0f, A, n, 0);
    }
    return gemm_strided<T, T, T, Acc>(s, n, n, b, Acc(1), X, b, 1, B, 1, b, Acc(1), A, n, 1);
}
template int gemm_update<double>(cudaStream_t, int, int, const double *, const double *, double *);
template int gemm_update<float>(cudaStream_t, int, int, const float *, const float *, float *);
template int gemm_update<__half>(cudaStream_t, int, int, const __half *, const __half *, __half *);
template int gemm_update<__nv_bfloat16>(cudaStream_t, int, int, const __nv_bfloat16 *, const __nv_bfloat16 *, __nv_bfloat16 *);

int gje_invert(cudaStream_t s, int n, int prec, void *A, GjeWork &w)
{
    switch (prec) {
        case LYAP_FP64: return gje_invert_t<double>(s, n, (double *)A, w);
        case LYAP_FP32: return gje_invert_t<float>(s, n, (float *)A, w);
        case LYAP_FP16: return gje_invert_t<__half>(s, n, (__half *)A, w);
        case LYAP_BF16: return gje_invert_t<__nv_bfloat16>(s, n, (__nv_bfloat16 *)A, w);
    }
    return LYAP_ERR_ARG;
}

int col_gather(cudaStream_t s, int n, int prec, const void *G, const int *invperm, void *out)
{
    dim3 g(ceil_div(n, 256) < 8 ? ceil_div(n, 256) : 8, n < 8192 ? n : 8192);
    switch (prec) {
        case LYAP_FP64: col_gather_kernel<double><<<g, 256, 0, s>>>(n, (const double *)G, invperm, (double *)out); break;
        case LYAP_FP32: col_gather_kernel<float><<<g, 256, 0, s>>>(n, (const float *)G, invperm, (float *)out); break;
        case LYAP_FP16: col_gather_kernel<__half><<<g, 256, 0, s>>>(n, (const __half *)G, invperm, (__half *)out); break;
        case LYAP_BF16: col_gather_kernel<__nv_bfloat16><<<g, 256, 0, s>>>(n, (const __nv_bfloat16 *)G, invperm, (__nv_bfloat16 *)out); break;
        default: return LYAP_ERR_ARG;
    }
    return launched();
}

}  // namespace lyap

// ------------------------------------------------------------------ C ABI
extern "C" int lyap_invert(int n, int prec, void *A, int *ipiv, void *stream)
{
    using namespace lyap;
    if (n <= 0 || A == nullptr || prec < 0 || prec > 3) return LYAP_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    GjeWork w;
    LYAP_TRY(w.alloc(n, prec));
    void *out = nullptr;
    int rc = LYAP_OK;
    if (cudaMalloc(&out, elem_size(prec) * (size_t)n * n) != cudaSuccess) { w.release(); return LYAP_ERR_CUDA; }
    rc = gje_invert(s, n, prec, A, w);
    if (rc == LYAP_OK) rc = col_gather(s, n, prec, A, w.invperm, out);
    if (rc == LYAP_OK && cudaMemcpyAsync(A, out, elem_size(prec) * (size_t)n * n, cudaMemcpyDeviceToDevice, s) != cudaSuccess) rc = LYAP_ERR_CUDA;
    if (rc == LYAP_OK && ipiv && cudaMemcpyAsync(ipiv, w.ipiv, sizeof(int) * n, cudaMemcpyDeviceToDevice, s) != cudaSuccess) rc = LYAP_ERR_CUDA;
    int info = 0;
    if (rc == LYAP_OK && cudaMemcpyAsync(&info, w.info, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess) rc = LYAP_ERR_CUDA;
    if (cudaStreamSynchronize(s) != cudaSuccess) rc = LYAP_ERR_CUDA;
    cudaFree(out);
    w.release();
    if (rc == LYAP_OK && info != 0) rc = LYAP_ERR_SINGULAR;
    return rc;
}
