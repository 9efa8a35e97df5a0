"""Pins of the CPU oracle against things other than itself (-m "not gpu").

Each test names what fixes the expected value: a PAPER.md table or equation,
a closed form, an independent library routine, or brute force.
"""
import os

import numpy as np
import pytest
import scipy.linalg as sla

import problems as P

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- precision
def _table1():
    rows = {}
    for line in open(os.path.join(GOLD, "table1_precisions.txt")):
        if line.startswith("#") or not line.strip():
            continue
        name, t, e, u, xmin, xmax = line.split()
        lg = [float(v.split("e")[0]) for v in (u, xmin, xmax)]
        ex = [int(v.split("e")[1]) for v in (u, xmin, xmax)]
        import math
        rows[name] = (int(t), int(e)) + tuple(math.log10(a) + b for a, b in zip(lg, ex))
    return rows


def _same3(x, ref):
    """Equal to three significant figures (the table rounds or truncates the 4th digit).
    Compared in log10 so that 1.80e308 (above DBL_MAX when parsed) is handled."""
    import math
    return abs(math.log10(x) - ref) < math.log10(1.005)


def test_table1_constants(orc):
    """PAPER.md Table 1: u, x_min, x_max to three significant figures."""
    for name, (t, e, u, xmin, xmax) in _table1().items():
        assert _same3(orc.unit_roundoff(name), u), name
        assert _same3(orc.xmin(name), xmin), name
        assert _same3(orc.xmax(name), xmax), name
        assert orc.unit_roundoff(name) == 2.0 ** (-t)


def _boundary_values():
    vals = []
    for name in ["fp16", "bf16", "fp32"]:
        t, e = _table1()[name][:2]
        emin = -(2 ** (e - 1)) + 2
        emax = 2 ** (e - 1) - 1
        xm = (2 - 2.0 ** (1 - t)) * 2.0 ** emax
        ulp_max = 2.0 ** (emax - t + 1)
        sub = 2.0 ** (emin - t + 1)
        vals += [2.0 ** emin, 2.0 ** emin * (1 - 2.0 ** -t), sub, sub / 2, sub * 1.5, sub * 0.75,
                 xm, xm + ulp_max / 2, xm + ulp_max / 2 * (1 - 2 ** -20), xm * 1.5,
                 1 + 2.0 ** -t, 1 + 3 * 2.0 ** -t, 1 + 2.0 ** -t * (1 + 2 ** -30), 1 - 2.0 ** (-t - 1)]
    vals = np.array(vals)
    return np.concatenate([vals, -vals, [0.0, -0.0, np.inf, -np.inf]])


def test_fast_rounding_equals_definition(orc):
    """The fast bit-level path equals the frexp/nearbyint definition."""
    rng = np.random.default_rng(7)
    x = rng.standard_normal(20000) * np.exp(rng.uniform(-100, 100, 20000))
    x = np.concatenate([x, _boundary_values()])
    for p in ["fp16", "bf16", "fp32"]:
        fast = orc.round_(x, p)
        ref = np.array([orc.round_ref_scalar(v, p) for v in x])
        assert np.array_equal(fast, ref), p


def test_fp16_fp32_match_numpy(orc):
    """numpy's float64->float16/float32 conversions are correctly rounded (RNE, subnormals)."""
    rng = np.random.default_rng(8)
    x = rng.standard_normal(50000) * np.exp(rng.uniform(-25, 15, 50000))
    x = np.concatenate([x, _boundary_values()])
    with np.errstate(over="ignore"):
        assert np.array_equal(orc.round_(x, "fp16"), x.astype(np.float16).astype(np.float64))
        assert np.array_equal(orc.round_(x, "fp32"), x.astype(np.float32).astype(np.float64))


def test_bf16_matches_bit_rne_on_float32_values(orc):
    """bf16 = float32 with the 16 low bits rounded off (RNE); independent integer version."""
    rng = np.random.default_rng(9)
    f = (rng.standard_normal(50000) * np.exp(rng.uniform(-80, 80, 50000))).astype(np.float32)
    f = f[np.isfinite(f)]
    b = f.view(np.uint32).astype(np.uint64)
    lsb = (b >> 16) & 1
    r = ((b + 0x7FFF + lsb) & 0xFFFF0000).astype(np.uint32).view(np.float32).astype(np.float64)
    assert np.array_equal(orc.round_(f.astype(np.float64), "bf16"), r)


def test_spec_rounding_examples(orc):
    """Table 1 overflow threshold; below-half-ulp additions vanish."""
    assert orc.round_scalar(7.0e4, "fp16") == np.inf
    assert orc.round_scalar(1 + 2.0 ** -9, "bf16") == 1.0
    assert orc.round_scalar(65504.0, "fp16") == 65504.0
    assert orc.round_scalar(256.0 * 256.0, "fp16") == np.inf
    assert orc.round_scalar(0.1 + 0.2, "fp64") == 0.1 + 0.2
    assert np.isnan(orc.round_scalar(np.nan, "bf16"))


# ---------------------------------------------------------------- kernels
def test_gemm_fp64_and_emulated_fp16(orc):
    rng = np.random.default_rng(1)
    A = rng.standard_normal((7, 5))
    B = rng.standard_normal((5, 4))
    assert np.allclose(orc.gemm("fp64", A, B), A @ B, rtol=1e-14, atol=1e-14)
    assert np.allclose(orc.gemm("fp64", A.T, B, ta=True), A @ B, rtol=1e-14, atol=1e-14)
    assert np.allclose(orc.gemm("fp64", A, B.T, tb=True), A @ B, rtol=1e-14, atol=1e-14)
    # numpy float16 arithmetic rounds every + and * to fp16 (exact fp32 op, then RNE)
    A16 = A.astype(np.float16)
    B16 = B.astype(np.float16)
    ref = np.zeros((7, 4), dtype=np.float16)
    for i in range(7):
        for j in range(4):
            s = np.float16(A16[i, 0] * B16[0, j])
            for l in range(1, 5):
                s = np.float16(s + np.float16(A16[i, l] * B16[l, j]))
            ref[i, j] = s
    got = orc.gemm("fp16", A16.astype(np.float64), B16.astype(np.float64))
    assert np.array_equal(got, ref.astype(np.float64))


def test_getrf_pivots_match_lapack(orc):
    """Partial-pivoting pivot sequence = LAPACK dgetrf's (scipy.linalg.lu_factor)."""
    for seed in range(5):
        A = np.random.default_rng(seed).standard_normal((30, 30))
        LU, piv, info = orc.getrf("fp64", A)
        assert info == 0
        lu_ref, piv_ref = sla.lu_factor(A)
        assert np.array_equal(piv, piv_ref)
        assert np.allclose(LU, lu_ref, rtol=1e-10, atol=1e-12)


def test_getrf_ties_lowest_index_and_singular(orc):
    A = np.array([[1.0, 2.0], [-1.0, 3.0]])
    _, piv, info = orc.getrf("fp64", A)
    assert info == 0 and list(piv) == [0, 1]
    _, _, info = orc.getrf("fp64", np.array([[1.0, 1.0], [1.0, 1.0]]))
    assert info == 2
    _, _, info = orc.inverse("fp64", np.zeros((3, 3)))
    assert info == 1


def test_inverse_fp64_and_error_bound_low_precision(orc):
    rng = np.random.default_rng(3)
    n = 40
    A = rng.standard_normal((n, n)) + n ** 0.5 * np.eye(n)
    X, piv, info = orc.inverse("fp64", A)
    assert info == 0
    assert np.allclose(X, np.linalg.inv(A), rtol=1e-11, atol=1e-13)
    kappa = np.linalg.cond(A, "fro")
    for p in ["fp32", "fp16", "bf16"]:
        Ap = orc.round_(A, p)
        Xp, _, info = orc.inverse(p, Ap)
        assert info == 0
        err = np.linalg.norm(Ap @ Xp - np.eye(n)) / np.sqrt(n)
        assert err <= 100 * n * orc.unit_roundoff(p) * kappa, (p, err)
    assert np.array_equal(orc.inverse("fp64", np.diag([2.0, 4.0]))[0], np.diag([0.5, 0.25]))


def test_qr_householder(orc):
    rng = np.random.default_rng(4)
    for (m, n) in [(50, 6), (20, 20), (6, 9)]:
        A = rng.standard_normal((m, n))
        Q, R = orc.qr("fp64", A)
        k = min(m, n)
        assert np.allclose(Q.T @ Q, np.eye(k), atol=1e-14)
        assert np.allclose(Q @ R, A, atol=1e-13)
        assert np.all(np.diag(R) >= 0) and np.allclose(np.tril(R, -1), 0)
        Qn, Rn = np.linalg.qr(A)
        sgn = np.sign(np.diag(Rn))
        assert np.allclose(R, sgn[:, None] * Rn, atol=1e-12)
    Q, R = orc.qr("fp64", np.array([[3.0], [4.0]]))
    assert np.allclose(Q[:, 0], [0.6, 0.8]) and np.isclose(R[0, 0], 5.0)
    # rank deficient: duplicated column
    z = rng.standard_normal((10, 1))
    Q, R = orc.qr("fp64", np.hstack([z, z, rng.standard_normal((10, 1))]))
    assert abs(R[1, 1]) < 1e-14 * np.linalg.norm(z)


def test_syev_jacobi_matches_eigh(orc):
    rng = np.random.default_rng(5)
    for n in [1, 2, 8, 25]:
        B = rng.standard_normal((n, n))
        A = B + B.T
        w, V, _ = orc.syev("fp64", A)
        wr = np.linalg.eigvalsh(A)[::-1]
        assert np.allclose(w, wr, atol=1e-13 * np.abs(wr).max())
        assert np.allclose(V @ np.diag(w) @ V.T, A, atol=1e-12 * np.linalg.norm(A))
        assert np.allclose(V.T @ V, np.eye(n), atol=1e-13)
    w, V, _ = orc.syev("fp64", np.array([[0.0, 1.0], [1.0, 0.0]]))
    assert np.allclose(w, [1, -1])
    w, V, _ = orc.syev("fp64", np.diag([5.0, 1.0]))
    assert np.allclose(w, [5, 1]) and np.allclose(np.abs(V), np.eye(2))


def test_rank_trunc_chol(orc):
    rng = np.random.default_rng(6)
    z = rng.standard_normal((20, 1))
    Zt = orc.rank_trunc_chol("fp64", np.hstack([z, z]))
    assert Zt.shape[1] == 1
    assert np.allclose(Zt @ Zt.T, 2 * z @ z.T, atol=1e-13 * 2 * (z ** 2).sum())
    Zt = orc.rank_trunc_chol("fp64", np.eye(3))
    assert Zt.shape[1] == 3 and np.allclose(Zt @ Zt.T, np.eye(3))
    # 4 dominant directions + 1e-12 noise: rank count equals the SVD's at the same threshold
    n, c = 40, 12
    Z = rng.standard_normal((n, 4)) @ rng.standard_normal((4, c)) + 1e-12 * rng.standard_normal((n, c))
    Zt = orc.rank_trunc_chol("fp64", Z, 1e-8)
    s = np.linalg.svd(Z, compute_uv=False)
    assert Zt.shape[1] == int(np.sum(s > 1e-8 * s[0])) == 4
    G, Gt = Z @ Z.T, Zt @ Zt.T
    assert np.linalg.norm(G - Gt) <= 2e-8 * np.linalg.norm(Z, 2) * np.linalg.norm(Z)


def test_rank_trunc_ldlt(orc):
    rng = np.random.default_rng(7)
    z = rng.standard_normal((15, 1))
    Zt, Yt = orc.rank_trunc_ldlt("fp64", np.hstack([z, z]), np.diag([1.0, -1.0]))
    # exact cancellation: the implied product is zero up to rounding (a relative
    # threshold cannot tell rounding noise from signal when everything is noise)
    assert np.linalg.norm(Zt @ Yt @ Zt.T) <= 1e-14 * (z ** 2).sum()
    Z = rng.standard_normal((30, 10))
    Y = np.diag(rng.uniform(-1, 1, 10))
    Zt, Yt = orc.rank_trunc_ldlt("fp64", Z, Y)
    X = Z @ Y @ Z.T
    assert np.linalg.norm(Zt @ Yt @ Zt.T - X) <= 1e-12 * np.linalg.norm(X)
    assert np.allclose(Yt, np.diag(np.diag(Yt)))


# ---------------------------------------------------------------- brute force
def test_kron_closed_form_diagonal(orc):
    """Diagonal A: X_ij = -W_ij / (a_i + a_j) (exact solution of Eq. eq:lyap)."""
    p = P.diagonal_problem(12, 3, 0)
    a = p.meta["a"]
    W = p.W()
    X = orc.kron_solve(p.A, W)
    Xc = -W / (a[:, None] + a[None, :])
    assert np.allclose(X, Xc, rtol=1e-13, atol=1e-15)
    assert np.allclose(orc.kron_solve(-np.eye(2), np.eye(2)), np.eye(2) / 2)
    assert np.isclose(orc.kron_solve(np.array([[-2.0]]), np.array([[4.0]]))[0, 0], 1.0)


def test_kron_matches_bartels_stewart(orc):
    for seed in range(3):
        p = P.random_stable(9, 2, seed)
        W = p.W()
        X = orc.kron_solve(p.A, W)
        Xs = sla.solve_continuous_lyapunov(p.A, -W)
        assert np.linalg.norm(X - Xs) <= 1e-12 * np.linalg.norm(Xs)
        assert orc.rel_residual_explicit(p.A, X, W) < 1e-14


# ---------------------------------------------------------------- Newton
def test_newton_closed_forms(orc):
    Z, q = orc.newton_chol("fp64", -np.eye(2), np.array([[1.0], [0.0]]))
    assert np.allclose(Z @ Z.T, np.diag([0.5, 0.0]))
    Z, Y, q = orc.newton_ldlt("fp64", -np.eye(2), np.array([[1.0], [0.0]]), np.array([[-1.0]]))
    assert np.allclose(Z @ Y @ Z.T, np.diag([-0.5, 0.0]))
    Z, q = orc.newton_chol("fp64", np.array([[-3.0]]), np.array([[2.0]]))
    assert np.isclose((Z @ Z.T)[0, 0], 4.0 / 6.0)


def test_newton_vs_kron_and_stopping_contract(orc):
    """Algorithms 3/4 in fp64 vs Eq. lyap-ls; ||A_k+I||_inf <= 10 sqrt(n u), then `extra` more
    steps (l.1312 says two; reading R-EXTRA defaults to one, both are checked)."""
    for seed in range(4):
        p = P.random_stable(8, 2, seed)
        W = p.W()
        X = orc.kron_solve(p.A, W)
        Z, q = orc.newton_chol("fp64", p.A, p.L)
        assert np.linalg.norm(Z @ Z.T - X) <= 1e-10 * np.linalg.norm(X)
        Z2, Y2, q2 = orc.newton_ldlt("fp64", p.A, p.L)
        assert np.linalg.norm(Z2 @ Y2 @ Z2.T - X) <= 1e-10 * np.linalg.norm(X)
        tau = 10 * np.sqrt(8 * orc.unit_roundoff("fp64"))
        first = next(j for j, v in enumerate(q.inf) if v <= tau)
        assert q.steps == first + 1 + 1 and q.inf[-1] <= tau
        q2 = orc.aseq("fp64", p.A, extra=2)
        assert q2.steps == first + 1 + 2


def test_newton_scaling_invariance(orc):
    p = P.random_stable(20, 2, 11, shift=0.2)
    Zs, qs = orc.newton_chol("fp64", p.A, p.L, scaling=True)
    Zu, qu = orc.newton_chol("fp64", p.A, p.L, scaling=False)
    Xs, Xu = Zs @ Zs.T, Zu @ Zu.T
    assert np.linalg.norm(Xs - Xu) <= 1e-10 * np.linalg.norm(Xu)
    assert qs.steps <= 2 * qu.steps


def test_inverse_cache_prefix_identity(orc):
    """Section 3.4: the A-side sequence is independent of the right-hand side."""
    p = P.random_stable(12, 3, 2)
    q1 = orc.aseq("fp16", p.A)
    q2 = orc.aseq("fp16", p.A)
    assert q1.steps == q2.steps
    for a, b in zip(q1.inverses, q2.inverses):
        assert np.array_equal(a, b)
    r1 = orc.ir_ldlt(p.A, p.L, us="fp16", cache=True)
    r0 = orc.ir_ldlt(p.A, p.L, us="fp16", cache=False)
    assert np.array_equal(r1.Z, r0.Z) and r1.steps == r0.steps
    assert r1.inversions == q1.steps and r0.inversions == q1.steps * r0.newton_calls


# ---------------------------------------------------------------- fragments
def test_fragment_residual_norm_identity(orc):
    """sqrt(sum lambda_j^2) of H_i equals the explicitly formed ||R||_F (l.311)."""
    rng = np.random.default_rng(12)
    for seed in range(4):
        p = P.random_stable(12, 2, seed)
        Z = rng.standard_normal((12, 5))
        Y = np.diag(rng.uniform(0.1, 1, 5))
        X = Z @ Y @ Z.T
        R = p.A @ X + X @ p.A.T + p.W()
        Ld, Sd, resF = orc.res_fac_ldlt("fp64", p.A, p.L, np.eye(2), Z, Y, eta_r=0.0)
        assert np.isclose(resF, np.linalg.norm(R), rtol=1e-10)
        assert np.allclose(Ld @ Sd @ Ld.T, R, atol=1e-11 * np.linalg.norm(R))
        Lp, Lm, resF2 = orc.res_fac_chol("fp64", p.A, p.L, Z, eta_r=0.0)
        Xc = Z @ Z.T
        Rc = p.A @ Xc + Xc @ p.A.T + p.W()
        assert np.isclose(resF2, np.linalg.norm(Rc), rtol=1e-10)
        assert np.allclose(Lp @ Lp.T - Lm @ Lm.T, Rc, atol=1e-11 * np.linalg.norm(Rc))


def test_fragment_solution_update_is_psd_projection(orc):
    """Fragments 2/4 = projection of X_i + X_i^+ - X_i^- onto the PSD cone (l.249-251)."""
    rng = np.random.default_rng(13)
    n = 20
    Z = rng.standard_normal((n, 4))
    Zp = rng.standard_normal((n, 2))
    Zm = 1.5 * rng.standard_normal((n, 3))
    Xbp = Z @ Z.T + Zp @ Zp.T - Zm @ Zm.T
    w, V = np.linalg.eigh(Xbp)
    Xproj = (V * np.maximum(w, 0)) @ V.T
    Zn = orc.sol_upt_chol("fp64", Z, Zp, Zm, eta_s=1e-15)
    assert np.linalg.norm(Zn @ Zn.T - Xproj) <= 1e-11 * np.linalg.norm(Xproj)
    Zn, Yn = orc.sol_upt_ldlt("fp64", Z, np.eye(4), np.hstack([Zp, Zm]),
                              np.diag([1.0] * 2 + [-1.0] * 3), eta_s=1e-15)
    assert np.linalg.norm(Zn @ Yn @ Zn.T - Xproj) <= 1e-11 * np.linalg.norm(Xproj)
    # X_i + X^+ - X_i = X^+
    Zn = orc.sol_upt_chol("fp64", Z, Zp, Z, eta_s=1e-15)
    assert np.linalg.norm(Zn @ Zn.T - Zp @ Zp.T) <= 1e-12 * np.linalg.norm(Zp @ Zp.T)


# ---------------------------------------------------------------- IR
@pytest.mark.parametrize("seed", range(10))
def test_ir_fp64_equals_kron(orc, seed):
    """Acceptance 1: all-fp64 IR reproduces the Kronecker solution."""
    rng = np.random.default_rng(100 + seed)
    n = int(rng.choice([4, 6, 8, 10]))
    m = int(rng.choice([1, 2, 3]))
    p = P.random_stable(n, m, seed)
    W = p.W()
    X = orc.kron_solve(p.A, W)
    r = orc.ir_chol(p.A, p.L, us="fp64", tol=1e-14)
    Xc = r.Z @ r.Z.T
    assert orc.rel_residual_explicit(p.A, Xc, W) <= 1e-13
    assert np.linalg.norm(Xc - X) <= 1e-10 * np.linalg.norm(X)
    S = np.diag(rng.uniform(0.5, 2, m))
    W2 = p.L @ S @ p.L.T
    X2 = orc.kron_solve(p.A, W2)
    r2 = orc.ir_ldlt(p.A, p.L, S, us="fp64", tol=1e-14)
    Xl = r2.Z @ r2.Y @ r2.Z.T
    assert orc.rel_residual_explicit(p.A, Xl, W2) <= 1e-13
    assert np.linalg.norm(Xl - X2) <= 1e-10 * np.linalg.norm(X2)


@pytest.mark.parametrize("us", ["fp32", "fp16", "bf16"])
def test_ir_low_precision_solver_reaches_fp64(orc, us):
    """Table 2 (l.1078) / Theorems 2.1-2.2: u_s in {fp32, fp16, bf16}, u_r = u_c = fp64 gives an
    fp64-level residual for kappa well below 1/u_s."""
    p = P.random_stable(10, 2, 21)
    W = p.W()
    X = orc.kron_solve(p.A, W)
    for r, Xr in [(orc.ir_chol(p.A, p.L, us=us), None), (orc.ir_ldlt(p.A, p.L, us=us), None)]:
        Xr = r.Z @ (r.Y if r.Y is not None else np.eye(r.Z.shape[1])) @ r.Z.T
        assert r.status == "converged", r
        assert orc.rel_residual_explicit(p.A, Xr, W) <= 1e-13
        assert np.linalg.norm(Xr - X) <= 1e-10 * np.linalg.norm(X)
        assert np.allclose(Xr, Xr.T, atol=1e-14 * np.linalg.norm(Xr))
        assert np.linalg.eigvalsh(Xr).min() >= -1e-12 * np.linalg.norm(Xr)
        # residual reduction each step before convergence (Theorem 2.1 behaviour)
        assert all(b < a for a, b in zip(r.res, r.res[1:]))


def test_table3_newton_counts(orc):
    """PAPER.md Table 3 (l.1449-1506, golden/table3_alpha_n100.txt): the per-call Newton counts alpha
    of the n=100 Cholesky block for u_s in {bf16, fp32, fp64} are reproduced exactly by the
    A-side of Algorithms 3/4 with Frobenius scaling, the delta-rules of Section 4 and one
    extra iteration (reading R-EXTRA)."""
    for line in open(os.path.join(GOLD, "table3_alpha_n100.txt")):
        if line.startswith("#") or not line.strip():
            continue
        cond, q, a16, a32, a64 = line.split()
        p = P.paper_synthetic(100, 3, float(q), seed=0)
        got = [orc.aseq(us, p.A).steps for us in ("bf16", "fp32", "fp64")]
        assert got == [int(a16), int(a32), int(a64)], (cond, got)


def test_ir_iteration_trend_table3(orc):
    """Acceptance 4 (Table 3 pattern, l.1449-1506): total Newton iterations grow and the per-call count
    shrinks as u_s is lowered (paper_synthetic n=100, q=0.5)."""
    p = P.paper_synthetic(100, 3, 0.5, seed=0)
    tot, mx = {}, {}
    for us in ["fp64", "fp32", "bf16"]:
        r = orc.ir_chol(p.A, p.L, us=us)
        assert r.status == "converged"
        assert r.final_res <= 1e-13
        tot[us], mx[us] = r.newton_total, r.newton_max
    assert tot["bf16"] >= tot["fp32"] >= tot["fp64"]
    assert mx["bf16"] <= mx["fp32"] <= mx["fp64"]


def test_ir_relative_residual_matches_explicit(orc):
    """The reported relative residual (fragment eigenvalues) equals Eq. res-fac-sol formed
    explicitly in fp64."""
    p = P.random_stable(12, 2, 5)
    r = orc.ir_ldlt(p.A, p.L, us="bf16", imax=2, tol=0.0)
    # res of the returned iterate is the last reported one
    X = r.Z @ r.Y @ r.Z.T
    assert np.isclose(r.final_res, orc.rel_residual_explicit(p.A, X, p.W()), rtol=1e-4)


def test_ir_bf16_ill_conditioned_reports_failure(orc):
    """Acceptance 3: an ill-conditioned bf16 run reports non-convergence, no crash."""
    p = P.paper_synthetic(40, 3, 3.5, seed=1)
    r = orc.ir_chol(p.A, p.L, us="bf16", imax=6)
    assert r.status in ("converged", "stagnated", "max_steps", "solver_failure")


def test_cfg0_converges(orc):
    """configs[0]: n=64 Cholesky fp16 solver, tol 1e-14, at most 10 IR steps."""
    p = P.cfg0()
    r = orc.ir_chol(p.A, p.L, us="fp16", tol=1e-14, imax=10)
    assert r.status == "converged" and r.steps <= 10
    X = r.Z @ r.Z.T
    assert orc.rel_residual_explicit(p.A, X, p.W()) <= 1e-13


# ---------------------------------------------------------------- generators
def test_generators():
    p = P.cfg0()
    ev = np.sort(np.linalg.eigvalsh(p.A))
    assert np.allclose(ev, np.sort(-np.logspace(0, 2, 64)), rtol=1e-12)
    p1 = P.cfg1(n=64)
    K = p1.A + (p1.A + p1.A.T) * 0  # noqa
    sym = (p1.A + p1.A.T) / 2
    assert np.linalg.eigvalsh(sym).max() <= -1 + 1e-10
    assert np.all(np.diag(p1.S) >= 0.5) and np.all(np.diag(p1.S) <= 2)
    Acd = P.convection_diffusion(8, 10.0)
    assert np.isclose(np.linalg.norm(Acd), 1.0)
    assert np.linalg.eigvalsh((Acd + Acd.T) / 2).max() < 0
    V = P.sine_orthogonal(9)
    assert np.allclose(V @ V, np.eye(9), atol=1e-14)
    ps = P.paper_synthetic(5, 2, 2.0, 0)
    assert np.allclose(np.sort(np.linalg.eigvalsh(ps.A)), np.sort(-np.logspace(0, 2, 5)))
    q = P.cfg4_member(70, n=64)
    assert q.meta["kappa"] == 100.0
    assert np.allclose(np.sort(np.linalg.eigvals(q.A).real), np.sort(-np.logspace(0, 2, 64)), rtol=1e-8)
    a = P.cfg1(seed=3, n=32).A
    b = P.cfg1(seed=3, n=32).A
    assert np.array_equal(a, b)


# ---------------------------------------------------------------- determinantal scaling
def test_logdet_triangular_closed_form(orc):
    """log|det| from the LU pivots equals sum log|d_i| for a triangular matrix (|det| is
    invariant under the row interchanges) and numpy's slogdet for a general one."""
    rng = np.random.default_rng(21)
    d = rng.uniform(0.5, 3.0, 12) * np.sign(rng.standard_normal(12))
    T = np.triu(rng.standard_normal((12, 12)), 1) * 0.1 + np.diag(d)
    _, _, info, ld = orc.inverse_logdet("fp64", T.T)
    assert info == 0
    assert np.isclose(ld, np.sum(np.log(np.abs(d))), rtol=0, atol=1e-13)
    G = rng.standard_normal((30, 30))
    _, _, _, ld2 = orc.inverse_logdet("fp64", G)
    assert np.isclose(ld2, np.linalg.slogdet(G)[1], rtol=1e-13)


def test_determinantal_scaling_closed_forms(orc):
    """mu_0 = |det A|^{-1/n}: for A = -c I, mu_0 = 1/c and A_1 = -I
    exactly (one Newton step lands on the sign); for a triangular A, the product of the
    diagonal.  The scaled iteration still converges to -I on a nonnormal stable matrix."""
    q = orc.aseq("fp64", -4.0 * np.eye(8), scaling="det")
    assert np.isclose(q.mu[0], 0.25, rtol=1e-15)
    assert q.inf[0] <= 1e-15                              # ||A_1 + I||_inf = 0
    rng = np.random.default_rng(22)
    d = -rng.uniform(0.5, 4.0, 10)
    T = np.tril(rng.standard_normal((10, 10)), -1) * 0.2 + np.diag(d)
    q = orc.aseq("fp64", T, scaling="det")
    assert np.isclose(q.mu[0], np.exp(-np.mean(np.log(np.abs(d)))), rtol=1e-13)
    p = P.random_stable(25, 2, 3)
    q = orc.aseq("fp64", p.A, scaling="det")
    assert q.converged and q.inf[-1] <= 10 * np.sqrt(25 * 2.0 ** -53)
