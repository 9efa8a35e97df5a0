// ir.cu -- host orchestration of the mixed-precision IR solver (PAPER.md
// Algorithms 1-4, Fragments 1-4) on one GPU, and the C ABI of include/lyap_ir.h.
//
// The handle owns all device workspace, sized once at creation for order n
// and factor width cmax:
//   A-side  : A_k, A_{k+1}, W (n x n in u_s) and the cached inverse sequence
//             A_0^{-1}, A_1^{-1}, ... (Section 3.4 "store the sequence of
//             computed matrix inverses"; on B200 the cache lives in HBM, e.g.
//             512 MB per fp16 inverse at n = 16384)
//   Z-side  : Z_k in u_s (column-major, appended in place), Y_k in fp64
//   fp64    : F = [Z, AZ, L], Householder / Jacobi / RRQR workspaces.
// Host decisions (Newton termination, ranks after truncation, IR stopping)
// read a few device scalars per step; every arithmetic step runs in this
// library's kernels.
#include <cmath>
#include <cstring>
#include <vector>
#include <algorithm>
#include "common.cuh"
#include "gemm_simt.cuh"
#include "lyap_internal.h"
#include "newton_kernels.h"
#include "ktimer.h"

namespace lyap { std::atomic<int64_t> g_launches{0}; }

using namespace lyap;

struct lyap_ir_ctx {
    int n = 0, cmax = 0, us = 0, mmax = 64;
    int PF = 0, PZ = 0, PW = 0;
    lyap_ir_options opt{};
    cudaStream_t s = nullptr;
    size_t es = 0;
    // A side
    void *Ak = nullptr, *An = nullptr, *W = nullptr;
    std::vector<void *> inv;   // cached Gauss-Jordan results G_k (u_s, column-permuted, 2^e-scaled)
    std::vector<int *> perms;  // per cached step: rowperm (n) and invperm (n) of the inversion
    std::vector<int> iexp;     // per cached step: range-scaling exponent e_k
    int ksteps = 0;
    std::vector<double> mu, delta, infn;
    GjeWork gje;
    QrWork qr;
    EigWork eig;
    RrqrWork rrqr;
    double *scal = nullptr, *part = nullptr, *hscal = nullptr;
    int *ibuf = nullptr;       // selection indices (3 lists of PW) + counts
    // Z side (u_s)
    void *Zt = nullptr;        // n x PZ
    double *Yc = nullptr, *Yn = nullptr;   // PZ x PZ
    // fp64 work
    double *Zd = nullptr, *Zd2 = nullptr;  // n x PW
    double *F = nullptr, *U = nullptr;     // n x PW
    double *Tm = nullptr, *Nm = nullptr, *TN = nullptr, *Hm = nullptr, *Vm = nullptr, *Vs = nullptr;  // PW x PW
    double *wv = nullptr;                  // PW
    // IR state (fp64)
    double *Zsol[2] = {nullptr, nullptr};  // n x PW
    double *Ysol[2] = {nullptr, nullptr};  // PW x PW
    double *Ld = nullptr, *Lm = nullptr;   // n x PW
    double *Sd = nullptr;                  // PW x PW
    double *Zdel = nullptr, *Zdel2 = nullptr;  // n x PZ
    double *Ydel = nullptr;                // PZ x PZ
    // host-path staging
    double *hA = nullptr, *hL = nullptr, *hS = nullptr, *hZ = nullptr, *hY = nullptr;
    cudaEvent_t ev[8];
    double t_newton = 0, t_res = 0, t_upd = 0;
    bool zorth = false;        // leading factor columns are orthonormal (set by the IR loop)
    bool y_diag = false;       // the Newton inner factor Y_k is diagonal (zside)
    bool ysol_diag = false;    // the solution's Y (and the correction's Y_d) are diagonal
};

namespace {

bool verbose() {
    static int v = -1;
    if (v < 0) { const char *e = getenv("LYAP_VERBOSE"); v = (e && e[0] == '1') ? 1 : 0; }
    return v == 1;
}

int cap_fail(int line, long need, long have) {
    fprintf(stderr, "lyap: capacity exceeded at ir.cu:%d (need %ld, have %ld); raise max_cols\n", line, need, have);
    return LYAP_ERR_CAPACITY;
}

int dmalloc(void **p, size_t bytes) {
    if (cudaMalloc(p, bytes > 0 ? bytes : 16) != cudaSuccess) return LYAP_ERR_CUDA;
    return LYAP_OK;
}
template <typename P> int dalloc(P **p, size_t count) { return dmalloc((void **)p, sizeof(P) * count); }

int sync_read(lyap_ir_ctx *h, void *dst, const void *src, size_t bytes) {
    LYAP_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, h->s));
    LYAP_CUDA_TRY(cudaStreamSynchronize(h->s));
    return LYAP_OK;
}

// C (n x c, col-major) = A_j^{-1} Z (Z n x c, col-major, u_s).  The cache holds the
// Gauss-Jordan result G_j as computed (A_j^{-1}[i][l] = 2^{-e_j} G_j[i][invperm_j[l]]), so
// A_j^{-1} Z = 2^{-e_j} G_j Z' with Z'[t] = Z[rowperm_j[t]]: one row gather of Z (n c
// elements) replaces an n^2 un-permuted copy of the inverse in the Newton update.
int zside_gemm(lyap_ir_ctx *h, int j, const void *Z, void *Out, int c) {
    const int n = h->n;
    const void *G = h->inv[j];
    LYAP_TRY(nk_row_gather(h->s, h->us, n, c, Z, h->perms[j], h->W));
    const void *Zp = h->W;
    const double alpha = std::ldexp(1.0, -h->iexp[j]);
    if ((h->us == LYAP_BF16 || h->us == LYAP_FP16) && !use_simt_gemm() && n % 8 == 0)
        // Out (n x c, column-major) = G (n x n, row-major = K-major) * Z', Z'^T rows K-major
        return tc_gemm(h->s, h->us, n, c, n, (float)alpha, G, n, Zp, n, 0.0f, Out, n, 1);
    switch (h->us) {
        case LYAP_FP64:
            return gemm_strided<double, double, double, double>(h->s, n, c, n, alpha, (const double *)G, n, 1,
                                                                (const double *)Zp, 1, n, 0.0, (double *)Out, 1, n);
        case LYAP_FP32:
            return gemm_strided<float, float, float, float>(h->s, n, c, n, (float)alpha, (const float *)G, n, 1,
                                                            (const float *)Zp, 1, n, 0.0f, (float *)Out, 1, n);
        case LYAP_FP16:
            return gemm_strided<__half, __half, __half, float>(h->s, n, c, n, (float)alpha, (const __half *)G, n, 1,
                                                               (const __half *)Zp, 1, n, 0.0f, (__half *)Out, 1, n);
        case LYAP_BF16:
            return gemm_strided<__nv_bfloat16, __nv_bfloat16, __nv_bfloat16, float>(
                h->s, n, c, n, (float)alpha, (const __nv_bfloat16 *)G, n, 1, (const __nv_bfloat16 *)Zp, 1, n, 0.0f,
                (__nv_bfloat16 *)Out, 1, n);
    }
    return LYAP_ERR_ARG;
}

// ------------------------------------------------------------------ A side
int aseq_compute(lyap_ir_ctx *h, const double *A) {
    const int n = h->n, us = h->us;
    cudaStream_t s = h->s;
    const long nn = (long)n * n;
    LYAP_TRY(nk_cast(s, us, n, A, h->Ak, h->part, h->scal + SC_RED));
    LYAP_TRY(nk_roll(s, h->scal));
    const double tauN = 10.0 * std::sqrt((double)n * unit_roundoff(us));
    int scaling_on = h->opt.scaling, countdown = -1, in_region = 0;
    double dprev = INFINITY;
    h->mu.clear(); h->delta.clear(); h->infn.clear();
    h->ksteps = 0;
    for (int it = 1; it <= h->opt.kmax; it++) {
        if ((int)h->inv.size() < it) {
            void *p = nullptr;
            LYAP_TRY(dmalloc(&p, h->es * nn));
            h->inv.push_back(p);
            int *pp = nullptr;
            LYAP_TRY(dalloc(&pp, 2 * (size_t)n));
            h->perms.push_back(pp);
        }
        if ((int)h->iexp.size() < it) h->iexp.push_back(0);
        // W = 2^{-e} A_k goes straight into the cache slot and is inverted in place there
        // (the Newton update then streams A_k and G in and A_{k+1} out: three n^2 streams)
        // (the implicit-pivoting sweep works in the free A_{k+1} buffer and writes its result,
        // rows back in order, into the slot)
        void *G = h->inv[it - 1];
        if (gje_ip_eligible(n, us, h->gje)) {
            LYAP_TRY(nk_scale(s, us, nn, h->Ak, h->An, h->scal));
            LYAP_TRY(gje_ip_invert(s, n, us, h->An, G, h->gje));
        } else {
            LYAP_TRY(nk_scale(s, us, nn, h->Ak, G, h->scal));
            LYAP_TRY(gje_invert(s, n, us, G, h->gje));
        }
        // mu_k: Frobenius-norm scaling (opt.scaling = 1, the paper's choice l.1406) or
        // determinantal scaling |det A_k|^{-1/n} (opt.scaling = 2, l.1139)
        if (h->opt.scaling == 2) LYAP_TRY(nk_mu_det(s, n, h->gje.ldet, h->scal, scaling_on));
        else LYAP_TRY(nk_mu(s, us, n, G, h->part, h->scal, scaling_on));
        LYAP_TRY(nk_update(s, us, n, h->Ak, G, h->gje.invperm, h->An, nullptr, h->scal, h->part));
        LYAP_CUDA_TRY(cudaMemcpyAsync(h->perms[it - 1], h->gje.rowperm, sizeof(int) * (size_t)n,
                                      cudaMemcpyDeviceToDevice, s));
        LYAP_CUDA_TRY(cudaMemcpyAsync(h->perms[it - 1] + n, h->gje.invperm, sizeof(int) * (size_t)n,
                                      cudaMemcpyDeviceToDevice, s));
        LYAP_TRY(nk_roll(s, h->scal));
        int info = 0;
        LYAP_CUDA_TRY(cudaMemcpyAsync(&info, h->gje.info, sizeof(int), cudaMemcpyDeviceToHost, s));
        LYAP_TRY(sync_read(h, h->hscal, h->scal, sizeof(double) * SC_COUNT));
        if (info != 0) return LYAP_ERR_SINGULAR;
        const double *sc = h->hscal;
        h->iexp[it - 1] = (int)sc[SC_EXP];
        double delta = std::sqrt(sc[SC_RED + 0]) / std::sqrt(sc[SC_RED + 1]);
        double inf = sc[SC_RED + 2];
        if (!std::isfinite(sc[SC_RED + 3]) || !std::isfinite(delta)) return LYAP_ERR_OVERFLOW;
        h->mu.push_back(sc[SC_MU]);
        h->delta.push_back(delta);
        h->infn.push_back(inf);
        std::swap(h->Ak, h->An);
        h->ksteps = it;
        const int region_step = in_region;
        if (delta < 1e-2) { scaling_on = 0; in_region = 1; }
        if (countdown < 0) {
            bool trig = inf <= tauN;
            if (region_step && delta > dprev / 2.0) trig = true;
            if (trig) {
                countdown = h->opt.extra;
                if (countdown == 0) break;
            }
        } else {
            countdown--;
            if (countdown == 0) break;
        }
        dprev = delta;
    }
    return LYAP_OK;
}

// ------------------------------------------------------------------ truncations
// RankTruncLdlt (l.1295-1304) on Zt (u_s, n x c) / Yc (fp64, ld PZ); in place.
int trunc_ldlt(lyap_ir_ctx *h, int c, int *cnew) {
    const int n = h->n;
    cudaStream_t s = h->s;
    const int k = std::min(n, c);
    LYAP_TRY(nk_to_f64(s, h->us, (long)n * c, h->Zt, h->Zd, 1.0));
    LYAP_TRY(qr_f64(s, n, c, h->Zd, h->U, h->Tm, h->qr));
    // T Y T^T; Y is diagonal whenever the inner factor was (every correction equation and
    // any diagonal user S): then T Y is a column scaling (bitwise the same products)
    if (h->y_diag) LYAP_TRY(nk_scale_cols(s, k, c, h->Tm, k, h->Yc, h->PZ, h->TN, k));
    else LYAP_TRY(dgemm_cm(s, false, false, k, c, c, 1.0, h->Tm, k, h->Yc, h->PZ, 0.0, h->TN, k));
    LYAP_TRY(dgemm_cm(s, false, true, k, k, c, 1.0, h->TN, k, h->Tm, k, 0.0, h->Hm, k));
    LYAP_TRY(syev_f64(s, k, h->Hm, h->wv, h->Vm, h->eig));
    LYAP_TRY(nk_select(s, k, h->wv, unit_roundoff(h->us), 1, h->ibuf, h->ibuf + 3 * h->PW));
    int r = 0;
    LYAP_TRY(sync_read(h, &r, h->ibuf + 3 * h->PW, sizeof(int)));
    LYAP_TRY(nk_gather_cols(s, k, r, h->Vm, k, h->ibuf, h->wv, 0, h->Vs, k));
    LYAP_TRY(dgemm_cm(s, false, false, n, r, k, 1.0, h->U, n, h->Vs, k, 0.0, h->Zd, n));
    LYAP_TRY(nk_from_f64(s, h->us, (long)n * r, h->Zd, h->Zt));
    LYAP_TRY(nk_diag_from_sel(s, r, h->wv, h->ibuf, h->us, h->Yc, h->PZ));
    *cnew = r;
    return LYAP_OK;
}

int trunc_chol(lyap_ir_ctx *h, int c, int *cnew) {
    const int n = h->n;
    cudaStream_t s = h->s;
    LYAP_TRY(nk_to_f64(s, h->us, (long)n * c, h->Zt, h->Zd, 1.0));
    int r = 0;
    LYAP_TRY(rank_trunc_chol_f64(s, n, c, h->Zd, std::sqrt(unit_roundoff(h->us)), h->us, h->Zd2, &r, h->rrqr));
    LYAP_TRY(nk_from_f64(s, h->us, (long)n * r, h->Zd2, h->Zt));
    *cnew = r;
    return LYAP_OK;
}

// is the m x m device matrix S diagonal? (read back; m is the small inner dimension)
int is_diag_dev(lyap_ir_ctx *h, const double *S, int m, bool *out) {
    std::vector<double> hs((size_t)m * m);
    LYAP_TRY(sync_read(h, hs.data(), S, sizeof(double) * hs.size()));
    bool d = true;
    for (int j = 0; j < m && d; j++)
        for (int i = 0; i < m; i++)
            if (i != j && hs[i + (size_t)j * m] != 0.0) { d = false; break; }
    *out = d;
    return LYAP_OK;
}

// ------------------------------------------------------------------ Z side
// Algorithm 4 (ldlt) / Algorithm 3 on the cached A-sequence.  Output fp64
// Zout (n x c, ld n) and, for LDL^T, Yout (c x c, ld ldy).
int zside(lyap_ir_ctx *h, bool ldlt, const double *L, int m, const double *S, double *Zout, double *Yout,
          int ldy, int *cout, bool s_diag) {
    const int n = h->n, us = h->us;
    h->y_diag = ldlt && s_diag;             // Y_k stays diagonal through blkdiag scaling and truncation
    cudaStream_t s = h->s;
    if (m > h->PZ / 2) return LYAP_ERR_CAPACITY;
    LYAP_TRY(nk_load_factor(s, us, (long)n * m, L, h->Zt, h->scal, SC_EL));
    if (ldlt) LYAP_TRY(nk_load_inner(s, us, m, S, h->Yc, h->PZ, h->scal, SC_ES));
    int c = m;
    const double rho_n = h->opt.rho * n;
    const char *Zbytes = (const char *)h->Zt;
    for (int j = 0; j < h->ksteps; j++) {
        if (2 * c > h->PZ) return cap_fail(__LINE__, 2 * c, h->PZ);
        const double mu = h->mu[j];
        {
            KTimer kt(KC_ZSIDE_GEMM, s);
            LYAP_TRY(zside_gemm(h, j, h->Zt, (void *)(Zbytes + h->es * (size_t)n * c), c));
        }
        if (ldlt) {
            LYAP_TRY(nk_y_blkdiag(s, c, h->Yc, h->PZ, h->Yn, h->PZ, mu / 2.0, 1.0 / (2.0 * mu), us));
            std::swap(h->Yc, h->Yn);
        } else {
            LYAP_TRY(nk_chol_scale(s, us, (long)n * c, h->Zt, std::sqrt(mu / 2.0), 1.0 / std::sqrt(2.0 * mu)));
        }
        c *= 2;
        if ((double)c > rho_n) {
            int r = 0;
            if (ldlt) LYAP_TRY(trunc_ldlt(h, c, &r));
            else LYAP_TRY(trunc_chol(h, c, &r));
            if (verbose()) fprintf(stderr, "lyap:   newton step %d: truncate %d -> %d\n", j, c, r);
            c = r;
        }
    }
    LYAP_TRY(nk_finish_factor(s, us, (long)n * c, h->Zt, Zout, ldlt ? 1.0 : 1.0 / std::sqrt(2.0), h->scal, SC_EL));
    if (ldlt) {
        LYAP_TRY(sync_read(h, h->hscal, h->scal, sizeof(double) * SC_COUNT));
        double f = std::ldexp(1.0, (int)h->hscal[SC_ES] - 1);    // Y = Y_k / 2, undo 2^{-e} range scaling
        LYAP_TRY(nk_copy_block(s, c, c, h->Yc, h->PZ, Yout, ldy, f));
    }
    *cout = c;
    return LYAP_OK;
}

// ------------------------------------------------------------------ fragments
// F = [Z, A Z, L]; returns p = 2c + m
int build_F(lyap_ir_ctx *h, const double *A, const double *L, int m, int c, const double *Z) {
    const int n = h->n;
    cudaStream_t s = h->s;
    LYAP_TRY(nk_copy_block(s, n, c, Z, n, h->F, n, 1.0));
    {
        KTimer kt(KC_RESID_GEMM, s, 2.0 * n * (double)n * c, 8.0 * ((double)n * n + 2.0 * n * c));
        LYAP_TRY(gemm_strided<double, double, double, double>(s, n, c, n, 1.0, A, n, 1, Z, 1, n, 0.0,
                                                              h->F + (size_t)n * c, 1, n));
    }
    LYAP_TRY(nk_copy_block(s, n, m, L, n, h->F + (size_t)n * 2 * c, n, 1.0));
    return LYAP_OK;
}

// Fragment 3 (ldlt, Y != null, S != null) / Fragment 1 (Y == null).
// Outputs: ldlt: Ld (n x r), Sd (r x r, ld r) ; chol: Ld = L+ (n x rp), Lm = L- (n x rm)
// Thin QR of h->F (n x p) into h->U (n x k), h->Tm (k x p).  When the leading c
// columns are known to be orthonormal (Z = V Theta_t from a previous solution
// update), the QR is [Z, Q2] with R = [[I, Rz], [0, R2]]: the remaining columns are
// projected out of span(Z) twice (block classical Gram-Schmidt with
// reorthogonalisation) and only those are Householder-factorised.  The thin QR
// with non-negative diag(R) is unique, so this equals the Householder result up
// to rounding.
int thin_qr_F(lyap_ir_ctx *h, int p, int c_orth) {
    const int n = h->n;
    cudaStream_t s = h->s;
    const int c = c_orth, q = p - c;
    // fast path with ample room (p <= n/2: the projected block is rarely rank deficient
    // there; near convergence [Z, AZ, L] is numerically rank deficient and the unpivoted
    // Householder completion would not stay orthogonal to Z); the result is verified
    if (!h->zorth || c <= 0 || q <= 0 || 2 * p > n || env_flag("LYAP_NO_BCGS"))
        return qr_f64(s, n, p, h->F, h->U, h->Tm, h->qr);
    const double *Z = h->F;
    double *B = h->F + (size_t)n * c;
    double *X1 = h->TN, *X2 = h->Hm, *R2 = h->Vs;
    LYAP_TRY(nk_copy_block(s, n, q, B, n, h->Zd2, n, 1.0));   // keep B for the fallback
    LYAP_TRY(dgemm_cm(s, true, false, c, q, n, 1.0, Z, n, B, n, 0.0, X1, c));
    LYAP_TRY(dgemm_cm(s, false, false, n, q, c, -1.0, Z, n, X1, c, 1.0, B, n));
    LYAP_TRY(dgemm_cm(s, true, false, c, q, n, 1.0, Z, n, B, n, 0.0, X2, c));
    LYAP_TRY(dgemm_cm(s, false, false, n, q, c, -1.0, Z, n, X2, c, 1.0, B, n));
    LYAP_TRY(nk_axpy(s, (long)c * q, 1.0, X2, X1));          // Rz = X1 + X2
    const int k2 = std::min(n - c, q);
    LYAP_TRY(qr_f64(s, n, q, B, h->U + (size_t)n * c, R2, h->qr));
    // checks: |diag(R2)| range (a near-zero pivot leaves an arbitrary Householder
    // completion column) and ||Z^T Q2||_F (the completion must stay orthogonal to Z)
    LYAP_TRY(nk_diag_range(s, k2, R2, k2, h->scal + SC_TR));
    LYAP_TRY(dgemm_cm(s, true, false, c, k2, n, 1.0, Z, n, h->U + (size_t)n * c, n, 0.0, X2, c));
    LYAP_TRY(nk_sumsq(s, (long)c * k2, X2, h->scal + SC_ORTH));
    LYAP_TRY(sync_read(h, h->hscal, h->scal, sizeof(double) * SC_COUNT));
    const double dmin = h->hscal[SC_TR], dmax = h->hscal[SC_TR + 1], e2 = h->hscal[SC_ORTH];
    if (!(dmin >= 1e-6 * dmax) || !(e2 <= 1e-24)) {
        if (verbose()) fprintf(stderr, "lyap:   BCGS fast path rejected (dmin/dmax %.2e, ||Z^T Q2|| %.2e)\n",
                               dmax > 0 ? dmin / dmax : 0.0, std::sqrt(e2));
        LYAP_TRY(nk_copy_block(s, n, q, h->Zd2, n, B, n, 1.0));
        return qr_f64(s, n, p, h->F, h->U, h->Tm, h->qr);
    }
    LYAP_TRY(nk_copy_block(s, n, c, Z, n, h->U, n, 1.0));
    return nk_assemble_T(s, c, q, k2, X1, R2, h->Tm);
}

int res_fac(lyap_ir_ctx *h, const double *A, const double *L, int m, const double *S, int c, const double *Z,
            const double *Y, int ldy, double eta_r, double *Ld, double *Sd, int *r, double *Lm, int *rm,
            double *resF) {
    const int n = h->n;
    cudaStream_t s = h->s;
    const int p = 2 * c + m;
    if (p > h->PW) return cap_fail(__LINE__, p, h->PW);
    const int k = std::min(n, p);
    LYAP_TRY(build_F(h, A, L, m, c, Z));
    LYAP_TRY(thin_qr_F(h, p, c));
    // H = T N T^T with N = [[0, Y, 0], [Y, 0, 0], [0, 0, S]] (Y = I for Cholesky, S = I
    // if absent): H = G + G^T + T3 S T3^T, G = T1 Y T2^T with T = [T1 T2 T3] -- the
    // structure of N saves two thirds of the dense T N T^T products
    {
        const double *T1 = h->Tm, *T2 = h->Tm + (size_t)k * c, *T3 = h->Tm + (size_t)2 * k * c;
        const double *W = T1;
        if (Y) {
            LYAP_TRY(dgemm_cm(s, false, false, k, c, c, 1.0, T1, k, Y, ldy, 0.0, h->TN, k));
            W = h->TN;
        }
        LYAP_TRY(dgemm_cm(s, false, true, k, k, c, 1.0, W, k, T2, k, 0.0, h->Hm, k));
        LYAP_TRY(nk_sym_add(s, k, h->Hm, k));
        const double *W3 = T3;
        if (Y && S) {
            double *w3 = h->TN + (size_t)k * c;
            LYAP_TRY(dgemm_cm(s, false, false, k, m, m, 1.0, T3, k, S, m, 0.0, w3, k));
            W3 = w3;
        }
        LYAP_TRY(dgemm_cm(s, false, true, k, k, m, 1.0, W3, k, T3, k, 1.0, h->Hm, k));
    }
    LYAP_TRY(syev_f64(s, k, h->Hm, h->wv, h->Vm, h->eig));
    LYAP_TRY(nk_sumsq(s, k, h->wv, h->scal + SC_TR));
    int *cnt = h->ibuf + 3 * h->PW;
    if (Y) {
        LYAP_TRY(nk_select(s, k, h->wv, eta_r, 0, h->ibuf, cnt));
    } else {
        LYAP_TRY(nk_select(s, k, h->wv, eta_r, 2, h->ibuf, cnt));
        LYAP_TRY(nk_select(s, k, h->wv, eta_r, 3, h->ibuf + h->PW, cnt + 1));
    }
    int counts[2] = {0, 0};
    LYAP_CUDA_TRY(cudaMemcpyAsync(counts, cnt, sizeof(int) * 2, cudaMemcpyDeviceToHost, s));
    LYAP_TRY(sync_read(h, h->hscal, h->scal, sizeof(double) * SC_COUNT));
    *resF = std::sqrt(h->hscal[SC_TR]);
    if (Y) {
        int rr = counts[0];
        LYAP_TRY(nk_gather_cols(s, k, rr, h->Vm, k, h->ibuf, h->wv, 0, h->Vs, k));
        LYAP_TRY(dgemm_cm(s, false, false, n, rr, k, 1.0, h->U, n, h->Vs, k, 0.0, Ld, n));
        LYAP_TRY(nk_diag_from_sel(s, rr, h->wv, h->ibuf, LYAP_FP64, Sd, rr));
        *r = rr;
    } else {
        int rp = counts[0], rmm = counts[1];
        LYAP_TRY(nk_gather_cols(s, k, rp, h->Vm, k, h->ibuf, h->wv, 1, h->Vs, k));
        LYAP_TRY(dgemm_cm(s, false, false, n, rp, k, 1.0, h->U, n, h->Vs, k, 0.0, Ld, n));
        LYAP_TRY(nk_gather_cols(s, k, rmm, h->Vm, k, h->ibuf + h->PW, h->wv, 2, h->Vs, k));
        LYAP_TRY(dgemm_cm(s, false, false, n, rmm, k, 1.0, h->U, n, h->Vs, k, 0.0, Lm, n));
        *r = rp;
        *rm = rmm;
    }
    return LYAP_OK;
}

// Fragment 4 (Y != null) / Fragment 2 (Y == null: G = [Z, Zp, Zm], J = blkdiag(I, I, -I)).
int sol_upt(lyap_ir_ctx *h, int c, const double *Z, const double *Y, int ldy, int cd, const double *Zd,
            const double *Yd, int ldyd, int cm, const double *Zm, double eta_s, double *Zn, double *Yn, int ldyn,
            int *r) {
    const int n = h->n;
    cudaStream_t s = h->s;
    const int p = c + cd + cm;
    if (p > h->PW) return cap_fail(__LINE__, p, h->PW);
    const int k = std::min(n, p);
    LYAP_TRY(nk_copy_block(s, n, c, Z, n, h->F, n, 1.0));
    LYAP_TRY(nk_copy_block(s, n, cd, Zd, n, h->F + (size_t)n * c, n, 1.0));
    if (cm > 0) LYAP_TRY(nk_copy_block(s, n, cm, Zm, n, h->F + (size_t)n * (c + cd), n, 1.0));
    LYAP_TRY(thin_qr_F(h, p, c));
    if (Y) LYAP_TRY(nk_build_blkdiag(s, c, cd, Y, ldy, Yd, ldyd, 0, h->Nm));
    else LYAP_TRY(nk_build_blkdiag(s, c + cd, cm, nullptr, 0, nullptr, 0, 0, h->Nm));
    // N diagonal (the signature J, or blkdiag of diagonal Y, Y_d): T N is a column scaling
    if (!Y || h->ysol_diag) LYAP_TRY(nk_scale_cols(s, k, p, h->Tm, k, h->Nm, p, h->TN, k));
    else LYAP_TRY(dgemm_cm(s, false, false, k, p, p, 1.0, h->Tm, k, h->Nm, p, 0.0, h->TN, k));
    LYAP_TRY(dgemm_cm(s, false, true, k, k, p, 1.0, h->TN, k, h->Tm, k, 0.0, h->Hm, k));
    LYAP_TRY(syev_f64(s, k, h->Hm, h->wv, h->Vm, h->eig));
    int *cnt = h->ibuf + 3 * h->PW;
    LYAP_TRY(nk_select(s, k, h->wv, eta_s, 2, h->ibuf, cnt));
    int rr = 0;
    LYAP_TRY(sync_read(h, &rr, cnt, sizeof(int)));
    LYAP_TRY(nk_gather_cols(s, k, rr, h->Vm, k, h->ibuf, h->wv, Y ? 0 : 1, h->Vs, k));
    LYAP_TRY(dgemm_cm(s, false, false, n, rr, k, 1.0, h->U, n, h->Vs, k, 0.0, Zn, n));
    if (Y) LYAP_TRY(nk_diag_from_sel(s, rr, h->wv, h->ibuf, LYAP_FP64, Yn, ldyn));
    *r = rr;
    return LYAP_OK;
}

// ||Z Y Z^T||_F^2 = tr((Z^T Z Y)^2)   (Y == null: tr((Z^T Z)^2))
int implied_norm2(lyap_ir_ctx *h, int c, const double *Z, const double *Y, int ldy, double *out_host) {
    const int n = h->n;
    cudaStream_t s = h->s;
    if (c == 0) { *out_host = 0.0; return LYAP_OK; }
    LYAP_TRY(dgemm_cm(s, true, false, c, c, n, 1.0, Z, n, Z, n, 0.0, h->Hm, c));
    const double *P = h->Hm;
    if (Y) {
        LYAP_TRY(dgemm_cm(s, false, false, c, c, c, 1.0, h->Hm, c, Y, ldy, 0.0, h->TN, c));
        P = h->TN;
    }
    LYAP_TRY(nk_trace_prod(s, c, P, h->scal + SC_TR2));
    LYAP_TRY(sync_read(h, h->hscal, h->scal, sizeof(double) * SC_COUNT));
    *out_host = h->hscal[SC_TR2];
    return LYAP_OK;
}

float elapsed(cudaEvent_t a, cudaEvent_t b) { float ms = 0.f; cudaEventElapsedTime(&ms, a, b); return ms; }

// Solver precision u_s per solve (the paper's problem statement passes u_s with the
// equation): a different u_s than the handle's current one re-allocates the u_s-typed
// buffers (A_k, A_{k+1}, W, Z_k, the Gauss-Jordan workspace) and drops the inverse cache.
int set_precision(lyap_ir_ctx *h, int us) {
    if (us < 0 || us == h->us) return LYAP_OK;
    if (us > 3) return LYAP_ERR_ARG;
    LYAP_CUDA_TRY(cudaStreamSynchronize(h->s));
    for (void *p : {h->Ak, h->An, h->W, h->Zt}) cudaFree(p);
    for (void *p : h->inv) cudaFree(p);
    for (int *p : h->perms) cudaFree(p);
    h->inv.clear();
    h->perms.clear();
    h->iexp.clear();
    h->ksteps = 0;
    h->Ak = h->An = h->W = h->Zt = nullptr;
    h->gje.release();
    h->gje = GjeWork();
    h->us = us;
    h->es = elem_size(us);
    const size_t nn = (size_t)h->n * h->n;
    LYAP_TRY(dmalloc(&h->Ak, h->es * nn));
    LYAP_TRY(dmalloc(&h->An, h->es * nn));
    LYAP_TRY(dmalloc(&h->W, h->es * (size_t)h->n * h->PZ));
    LYAP_TRY(dmalloc(&h->Zt, h->es * (size_t)h->n * h->PZ));
    return h->gje.alloc(h->n, us);
}

int ir_solve(lyap_ir_ctx *h, const double *A, const double *L, int m, const double *S, int ur, double tol,
             int maxit, double *Zout, double *Yout, int *rank_out, lyap_ir_report *rep) {
    const int n = h->n;
    cudaStream_t s = h->s;
    const bool ldlt = (S != nullptr);
    lyap_ir_report R;
    std::memset(&R, 0, sizeof(R));
    if (ur != LYAP_FP64) return LYAP_ERR_ARG;
    if (m <= 0 || m > h->mmax) return LYAP_ERR_ARG;
    double tn = 0, tr = 0, tu = 0;
    LYAP_CUDA_TRY(cudaEventRecord(h->ev[0], s));
    // ---- initial solve (Algorithm 1/2 line 1)
    int rc = aseq_compute(h, A);
    R.inversions = h->ksteps;
    R.newton_steps = h->ksteps;
    R.newton_flops = 2.0 * (double)n * n * n * h->ksteps;
    int cur = 0, c = 0;
    if (rc != LYAP_OK) {
        R.status = LYAP_STATUS_SOLVER_FAILED;
        if (rep) *rep = R;
        *rank_out = 0;
        return (rc == LYAP_ERR_CUDA) ? rc : LYAP_OK;
    }
    bool s_diag = false;
    if (ldlt) LYAP_TRY(is_diag_dev(h, S, m, &s_diag));
    LYAP_TRY(zside(h, ldlt, L, m, S, h->Zsol[cur], h->Ysol[cur], h->PW, &c, s_diag));
    h->ysol_diag = s_diag;                  // afterwards every update produces a diagonal Y
    R.newton_calls = 1;
    LYAP_CUDA_TRY(cudaEventRecord(h->ev[1], s));
    LYAP_CUDA_TRY(cudaEventSynchronize(h->ev[1]));
    tn += elapsed(h->ev[0], h->ev[1]);
    // ---- norms for Eq. res-fac-sol
    double nA2 = 0, nW2 = 0;
    LYAP_TRY(nk_sumsq(s, (long)n * n, A, h->scal + SC_TR));
    LYAP_TRY(sync_read(h, h->hscal, h->scal, sizeof(double) * SC_COUNT));
    nA2 = h->hscal[SC_TR];
    if (ldlt) {
        LYAP_TRY(dgemm_cm(s, true, false, m, m, n, 1.0, L, n, L, n, 0.0, h->Hm, m));
        LYAP_TRY(dgemm_cm(s, false, false, m, m, m, 1.0, h->Hm, m, S, m, 0.0, h->TN, m));
        LYAP_TRY(nk_trace_prod(s, m, h->TN, h->scal + SC_TR2));
        LYAP_TRY(sync_read(h, h->hscal, h->scal, sizeof(double) * SC_COUNT));
        nW2 = h->hscal[SC_TR2];
    } else {
        LYAP_TRY(implied_norm2(h, m, L, nullptr, 0, &nW2));
    }
    const double nA = std::sqrt(nA2), nW = std::sqrt(std::max(nW2, 0.0));
    int stagn = 0;
    double prev_rel = 0.0;     // previous relative residual (theta_i, Eq. it-early-terminate l.1413)
    R.status = LYAP_STATUS_MAXSTEPS;
    for (int i = 1;; i++) {
        LYAP_CUDA_TRY(cudaEventRecord(h->ev[2], s));
        double resF = 0.0;
        int r = 0, rmm = 0;
        h->zorth = (i >= 2);       // Z_i = V_{i-1} Theta_t has orthonormal columns after an update
        LYAP_TRY(res_fac(h, A, L, m, S, c, h->Zsol[cur], ldlt ? h->Ysol[cur] : nullptr, h->PW, h->opt.eta_r,
                         h->Ld, h->Sd, &r, h->Lm, &rmm, &resF));
        double nX2 = 0;
        LYAP_TRY(implied_norm2(h, c, h->Zsol[cur], ldlt ? h->Ysol[cur] : nullptr, h->PW, &nX2));
        LYAP_CUDA_TRY(cudaEventRecord(h->ev[3], s));
        LYAP_CUDA_TRY(cudaEventSynchronize(h->ev[3]));
        tr += elapsed(h->ev[2], h->ev[3]);
        const double rel = resF / (nW + 2.0 * std::sqrt(std::max(nX2, 0.0)) * nA);
        if (R.nres < LYAP_MAX_REPORT) { R.res[R.nres] = rel; R.ranks[R.nres] = c; }
        R.nres++;
        R.final_res = rel;
        bool stop = false;
        if (rel <= tol) { R.status = LYAP_STATUS_CONVERGED; stop = true; }
        else if (i >= 2) {
            double theta = rel / prev_rel;
            stagn = (theta > 0.9) ? stagn + 1 : 0;
            if (stagn >= 2) { R.status = LYAP_STATUS_STAGNATED; stop = true; }
        }
        prev_rel = rel;
        if (!stop && i > maxit) { R.status = LYAP_STATUS_MAXSTEPS; stop = true; }
        if (stop) break;
        // ---- correction equation(s) at u_s (cached A-sequence)
        LYAP_CUDA_TRY(cudaEventRecord(h->ev[4], s));
        if (!h->opt.cache) {
            rc = aseq_compute(h, A);
            R.inversions += h->ksteps;
            R.newton_flops += 2.0 * (double)n * n * n * h->ksteps;
            if (rc != LYAP_OK) { R.status = LYAP_STATUS_SOLVER_FAILED; break; }
        }
        int cd = 0, cm = 0;
        // a factor outgrowing the handle's capacity ends the refinement with the last
        // iterate (LYAP_STATUS_CAPACITY) instead of an error
        int rcz = LYAP_OK;
        if (ldlt) {
            rcz = zside(h, true, h->Ld, r, h->Sd, h->Zdel, h->Ydel, h->PZ, &cd, true);   // Sd diagonal
        } else {
            if (r > 0) rcz = zside(h, false, h->Ld, r, nullptr, h->Zdel, nullptr, 0, &cd, false);
            if (rcz == LYAP_OK && rmm > 0) rcz = zside(h, false, h->Lm, rmm, nullptr, h->Zdel2, nullptr, 0, &cm, false);
        }
        if (rcz == LYAP_ERR_CAPACITY) { R.status = LYAP_STATUS_CAPACITY; break; }
        LYAP_TRY(rcz);
        R.newton_calls++;
        LYAP_CUDA_TRY(cudaEventRecord(h->ev[5], s));
        // ---- solution update at u_c = fp64
        int cn = 0;
        const int nxt = 1 - cur;
        const int rcu = sol_upt(h, c, h->Zsol[cur], ldlt ? h->Ysol[cur] : nullptr, h->PW, cd, h->Zdel,
                                ldlt ? h->Ydel : nullptr, h->PZ, cm, h->Zdel2, h->opt.eta_s, h->Zsol[nxt],
                                h->Ysol[nxt], h->PW, &cn);
        if (rcu == LYAP_ERR_CAPACITY) { R.status = LYAP_STATUS_CAPACITY; break; }
        LYAP_TRY(rcu);
        LYAP_CUDA_TRY(cudaEventRecord(h->ev[6], s));
        LYAP_CUDA_TRY(cudaEventSynchronize(h->ev[6]));
        tn += elapsed(h->ev[4], h->ev[5]);
        tu += elapsed(h->ev[5], h->ev[6]);
        if (2 * cn + m > h->PW || cn > h->cmax) {
            // the update is valid but the next residual (or the output) would not fit:
            // keep the last verified iterate
            R.status = LYAP_STATUS_CAPACITY;
            if (verbose()) fprintf(stderr, "lyap: stop at step %d: rank %d exceeds the capacity\n", i, cn);
            break;
        }
        h->ysol_diag = true;                // the update's Y is diag(selected eigenvalues)
        cur = nxt;
        c = cn;
        R.steps = i;
        if (verbose())
            fprintf(stderr, "lyap: step %d rel=%.3e c=%d r=%d rm=%d cd=%d cm=%d -> %d\n", i, rel, c, r, rmm, cd,
                    cm, cn);
    }
    h->zorth = false;
    LYAP_CUDA_TRY(cudaEventRecord(h->ev[7], s));
    LYAP_CUDA_TRY(cudaEventSynchronize(h->ev[7]));
    if (c > h->cmax) return cap_fail(__LINE__, c, h->cmax);
    LYAP_CUDA_TRY(cudaMemcpyAsync(Zout, h->Zsol[cur], sizeof(double) * (size_t)n * c, cudaMemcpyDeviceToDevice, s));
    if (ldlt && Yout) LYAP_TRY(nk_copy_block(s, c, c, h->Ysol[cur], h->PW, Yout, h->cmax, 1.0));
    LYAP_CUDA_TRY(cudaStreamSynchronize(s));
    R.rank = c;
    R.newton_ms = tn; R.residual_ms = tr; R.update_ms = tu;
    R.total_ms = elapsed(h->ev[0], h->ev[7]);
    *rank_out = c;
    if (rep) *rep = R;
    return LYAP_OK;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

void lyap_ir_default_options(lyap_ir_options *o) {
    o->kmax = 50;
    o->scaling = 1;
    o->extra = 1;
    o->rho = 0.1;
    o->eta_r = 1e-4;
    o->eta_s = 10.0 * 0x1p-53;
    o->cache = 1;
    o->newton_cols = 0;
    o->work_cols = 0;
}

int64_t lyap_launch_count(void) { return g_launches.load(); }

int lyap_ir_create(lyap_ir_handle *out, int n, int cmax, int us, const lyap_ir_options *opt, void *stream) {
    if (!out || n <= 0 || cmax <= 0 || us < 0 || us > 3) return LYAP_ERR_ARG;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return LYAP_ERR_CUDA;
    lyap_ir_ctx *h = new lyap_ir_ctx();
    h->n = n; h->cmax = cmax; h->us = us;
    if (opt) h->opt = *opt; else lyap_ir_default_options(&h->opt);
    h->s = (cudaStream_t)stream;
    h->es = elem_size(us);
    const int rho_n = (int)std::ceil(h->opt.rho * n);
    h->PF = 2 * cmax + h->mmax;
    h->PZ = h->opt.newton_cols > 0 ? h->opt.newton_cols : 2 * std::max(h->PF, rho_n) + 16;
    h->PW = h->opt.work_cols > 0 ? std::max(h->opt.work_cols, h->PF) : h->PF + h->PZ;
    const size_t nn = (size_t)n * n;
    int rc = LYAP_OK;
    auto A = [&](int r) { if (rc == LYAP_OK) rc = r; };
    A(dmalloc(&h->Ak, h->es * nn));
    A(dmalloc(&h->An, h->es * nn));
    A(dmalloc(&h->W, h->es * (size_t)n * h->PZ));      // row-gathered Z' of the Z-side product
    A(h->gje.alloc(n, us));
    A(h->qr.alloc(n, h->PW));
    A(h->eig.alloc(std::min(n, h->PW)));
    A(h->rrqr.alloc(n, h->PZ));
    A(dalloc(&h->scal, SC_COUNT));
    A(dalloc(&h->part, 4 * (size_t)n + 16));
    A(dalloc(&h->ibuf, 3 * (size_t)h->PW + 8));
    A(dmalloc(&h->Zt, h->es * (size_t)n * h->PZ));
    A(dalloc(&h->Yc, (size_t)h->PZ * h->PZ));
    A(dalloc(&h->Yn, (size_t)h->PZ * h->PZ));
    A(dalloc(&h->Zd, (size_t)n * h->PW));
    A(dalloc(&h->Zd2, (size_t)n * h->PW));
    A(dalloc(&h->F, (size_t)n * h->PW));
    A(dalloc(&h->U, (size_t)n * h->PW));
    for (double **p : {&h->Tm, &h->Nm, &h->TN, &h->Hm, &h->Vm, &h->Vs}) A(dalloc(p, (size_t)h->PW * h->PW));
    A(dalloc(&h->wv, (size_t)h->PW));
    for (int i = 0; i < 2; i++) {
        A(dalloc(&h->Zsol[i], (size_t)n * h->PW));
        A(dalloc(&h->Ysol[i], (size_t)h->PW * h->PW));
    }
    A(dalloc(&h->Ld, (size_t)n * h->PW));
    A(dalloc(&h->Lm, (size_t)n * h->PW));
    A(dalloc(&h->Sd, (size_t)h->PW * h->PW));
    A(dalloc(&h->Zdel, (size_t)n * h->PZ));
    A(dalloc(&h->Zdel2, (size_t)n * h->PZ));
    A(dalloc(&h->Ydel, (size_t)h->PZ * h->PZ));
    if (rc == LYAP_OK && cudaMallocHost(&h->hscal, sizeof(double) * SC_COUNT) != cudaSuccess) rc = LYAP_ERR_CUDA;
    for (int i = 0; i < 8 && rc == LYAP_OK; i++)
        if (cudaEventCreate(&h->ev[i]) != cudaSuccess) rc = LYAP_ERR_CUDA;
    if (rc != LYAP_OK) { lyap_ir_destroy(h); return rc; }
    *out = h;
    return LYAP_OK;
}

int lyap_ir_destroy(lyap_ir_handle h) {
    if (!h) return LYAP_OK;
    cudaStreamSynchronize(h->s);
    for (void *p : {h->Ak, h->An, h->W, h->Zt}) cudaFree(p);
    for (void *p : h->inv) cudaFree(p);
    for (int *p : h->perms) cudaFree(p);
    h->gje.release(); h->qr.release(); h->eig.release(); h->rrqr.release();
    for (void *p : {(void *)h->scal, (void *)h->part, (void *)h->ibuf, (void *)h->Yc, (void *)h->Yn, (void *)h->Zd,
                    (void *)h->Zd2, (void *)h->F, (void *)h->U, (void *)h->Tm, (void *)h->Nm, (void *)h->TN,
                    (void *)h->Hm, (void *)h->Vm, (void *)h->Vs, (void *)h->wv, (void *)h->Zsol[0],
                    (void *)h->Zsol[1], (void *)h->Ysol[0], (void *)h->Ysol[1], (void *)h->Ld, (void *)h->Lm,
                    (void *)h->Sd, (void *)h->Zdel, (void *)h->Zdel2, (void *)h->Ydel, (void *)h->hA,
                    (void *)h->hL, (void *)h->hS, (void *)h->hZ, (void *)h->hY})
        if (p) cudaFree(p);
    if (h->hscal) cudaFreeHost(h->hscal);
    for (int i = 0; i < 8; i++) if (h->ev[i]) cudaEventDestroy(h->ev[i]);
    delete h;
    return LYAP_OK;
}

int lyap_ir_solve(lyap_ir_handle h, const double *A, const double *L, int m, const double *S, int us, int ur,
                  double tol, int maxit, double *Z, double *Y, int *rank, lyap_ir_report *rep) {
    if (!h || !A || !L || !Z || !rank || us > 3) return LYAP_ERR_ARG;
    LYAP_TRY(set_precision(h, us));
    return ir_solve(h, A, L, m, S, ur, tol, maxit, Z, Y, rank, rep);
}

int lyap_ir_solve_host(lyap_ir_handle h, const double *A, const double *L, int m, const double *S, int us,
                       int ur, double tol, int maxit, double *Z, double *Y, int *rank, lyap_ir_report *rep) {
    if (!h || !A || !L || !Z || !rank || m <= 0 || m > h->mmax || us > 3) return LYAP_ERR_ARG;
    LYAP_TRY(set_precision(h, us));
    const int n = h->n;
    if (!h->hA) {
        LYAP_TRY(dalloc(&h->hA, (size_t)n * n));
        LYAP_TRY(dalloc(&h->hL, (size_t)n * h->mmax));
        LYAP_TRY(dalloc(&h->hS, (size_t)h->mmax * h->mmax));
        LYAP_TRY(dalloc(&h->hZ, (size_t)n * h->cmax));
        LYAP_TRY(dalloc(&h->hY, (size_t)h->cmax * h->cmax));
    }
    cudaStream_t s = h->s;
    LYAP_CUDA_TRY(cudaMemcpyAsync(h->hA, A, sizeof(double) * (size_t)n * n, cudaMemcpyHostToDevice, s));
    LYAP_CUDA_TRY(cudaMemcpyAsync(h->hL, L, sizeof(double) * (size_t)n * m, cudaMemcpyHostToDevice, s));
    if (S) LYAP_CUDA_TRY(cudaMemcpyAsync(h->hS, S, sizeof(double) * (size_t)m * m, cudaMemcpyHostToDevice, s));
    int rc = ir_solve(h, h->hA, h->hL, m, S ? h->hS : nullptr, ur, tol, maxit, h->hZ, S ? h->hY : nullptr, rank, rep);
    if (rc != LYAP_OK) return rc;
    LYAP_CUDA_TRY(cudaMemcpyAsync(Z, h->hZ, sizeof(double) * (size_t)n * (*rank), cudaMemcpyDeviceToHost, s));
    if (S && Y) LYAP_CUDA_TRY(cudaMemcpyAsync(Y, h->hY, sizeof(double) * (size_t)h->cmax * (*rank), cudaMemcpyDeviceToHost, s));
    LYAP_CUDA_TRY(cudaStreamSynchronize(s));
    return LYAP_OK;
}

int lyap_newton_aseq(lyap_ir_handle h, const double *A, int *steps, double *mu, double *delta, double *infnorm) {
    if (!h || !A || !steps) return LYAP_ERR_ARG;
    int rc = aseq_compute(h, A);
    *steps = h->ksteps;
    for (int j = 0; j < h->ksteps; j++) {
        if (mu) mu[j] = h->mu[j];
        if (delta) delta[j] = h->delta[j];
        if (infnorm) infnorm[j] = h->infn[j];
    }
    return rc;
}

int lyap_newton_get_inverse(lyap_ir_handle h, int j, void *out) {
    if (!h || !out || j < 0 || j >= h->ksteps) return LYAP_ERR_ARG;
    // A_j^{-1}[i][l] = 2^{-e_j} G_j[i][invperm_j[l]]
    LYAP_TRY(col_gather(h->s, h->n, h->us, h->inv[j], h->perms[j] + h->n, out));
    LYAP_TRY(nk_ldexp(h->s, h->us, (long)h->n * h->n, out, -h->iexp[j]));
    LYAP_CUDA_TRY(cudaStreamSynchronize(h->s));
    return LYAP_OK;
}

int lyap_newton_z(lyap_ir_handle h, int ldlt, const double *L, int m, const double *S, double *Z, double *Y, int *c) {
    if (!h || !L || !Z || !c || (ldlt && (!S || !Y))) return LYAP_ERR_ARG;
    bool s_diag = false;
    if (ldlt) LYAP_TRY(is_diag_dev(h, S, m, &s_diag));
    int rc = zside(h, ldlt != 0, L, m, S, Z, Y, h->cmax, c, s_diag);
    if (rc == LYAP_OK) LYAP_CUDA_TRY(cudaStreamSynchronize(h->s));
    return rc;
}

int lyap_rank_trunc_ldlt(int n, int c, const double *Z, const double *Y, int prec, double *Zout, double *Yout,
                         int *k, void *stream) {
    if (n <= 0 || c <= 0 || !Z || !Y || !Zout || !Yout || !k) return LYAP_ERR_ARG;
    lyap_ir_handle h = nullptr;
    lyap_ir_options o;
    lyap_ir_default_options(&o);
    o.rho = 0.0;
    int rc = lyap_ir_create(&h, n, std::max(1, c / 2 + 1), prec, &o, stream);
    if (rc != LYAP_OK) return rc;
    if (c > h->PZ) { lyap_ir_destroy(h); return LYAP_ERR_CAPACITY; }
    cudaStream_t s = h->s;
    rc = nk_from_f64(s, prec, (long)n * c, Z, h->Zt);
    if (rc == LYAP_OK) rc = nk_copy_block(s, c, c, Y, c, h->Yc, h->PZ, 1.0);
    int r = 0;
    if (rc == LYAP_OK) rc = trunc_ldlt(h, c, &r);
    if (rc == LYAP_OK) rc = nk_to_f64(s, prec, (long)n * r, h->Zt, Zout, 1.0);
    if (rc == LYAP_OK) rc = nk_copy_block(s, r, r, h->Yc, h->PZ, Yout, r, 1.0);
    if (cudaStreamSynchronize(s) != cudaSuccess) rc = LYAP_ERR_CUDA;
    *k = r;
    lyap_ir_destroy(h);
    return rc;
}

int lyap_res_fac_ldlt(lyap_ir_handle h, const double *A, const double *L, int m, const double *S, int c,
                      const double *Z, const double *Y, double eta_r, double *Ld, double *Sd, int *r, double *resF) {
    if (!h || !A || !L || !S || !Z || !Y || !Ld || !Sd || !r || !resF) return LYAP_ERR_ARG;
    int rm = 0;
    int rc = res_fac(h, A, L, m, S, c, Z, Y, c, eta_r, Ld, Sd, r, nullptr, &rm, resF);
    if (rc == LYAP_OK) LYAP_CUDA_TRY(cudaStreamSynchronize(h->s));
    return rc;
}

int lyap_res_fac_chol(lyap_ir_handle h, const double *A, const double *L, int m, int c, const double *Z,
                      double eta_r, double *Lp, int *rp, double *Lm, int *rm, double *resF) {
    if (!h || !A || !L || !Z || !Lp || !Lm || !rp || !rm || !resF) return LYAP_ERR_ARG;
    int rc = res_fac(h, A, L, m, nullptr, c, Z, nullptr, 0, eta_r, Lp, nullptr, rp, Lm, rm, resF);
    if (rc == LYAP_OK) LYAP_CUDA_TRY(cudaStreamSynchronize(h->s));
    return rc;
}

int lyap_sol_upt_ldlt(lyap_ir_handle h, int c, const double *Z, const double *Y, int cd, const double *Zd,
                      const double *Yd, double eta_s, double *Zn, double *Yn, int *r) {
    if (!h || !Z || !Y || !Zd || !Yd || !Zn || !Yn || !r) return LYAP_ERR_ARG;
    bool d1 = false, d2 = false;
    LYAP_TRY(is_diag_dev(h, Y, c, &d1));
    LYAP_TRY(is_diag_dev(h, Yd, cd, &d2));
    h->ysol_diag = d1 && d2;
    int rc = sol_upt(h, c, Z, Y, c, cd, Zd, Yd, cd, 0, nullptr, eta_s, Zn, Yn, c + cd, r);
    if (rc == LYAP_OK) LYAP_CUDA_TRY(cudaStreamSynchronize(h->s));
    return rc;
}

int lyap_sol_upt_chol(lyap_ir_handle h, int c, const double *Z, int cp, const double *Zp, int cm, const double *Zm,
                      double eta_s, double *Zn, int *r) {
    if (!h || !Z || !Zp || !Zn || !r || (cm > 0 && !Zm)) return LYAP_ERR_ARG;
    int rc = sol_upt(h, c, Z, nullptr, 0, cp, Zp, nullptr, 0, cm, Zm, eta_s, Zn, nullptr, 0, r);
    if (rc == LYAP_OK) LYAP_CUDA_TRY(cudaStreamSynchronize(h->s));
    return rc;
}

}  // extern "C"
