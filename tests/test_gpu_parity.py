"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle (-m gpu).

Tolerances:
  * integer / index work (pivots, ranks, step counts): bit-exact;
  * fp64 kernels (QR, Jacobi, fragments, fp64 inversion): 1e-10..1e-12 relative;
  * low-precision inversion: element-wise against the oracle's tc model (tests/test_gpu_inversion.py);
  * full IR: ||X - X_oracle||_F / ||X_oracle||_F <= 1e-10, final normwise residual
    <= 1e-13, identical IR step counts (BASELINE.json north_star).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import problems as P  # noqa: E402


@pytest.fixture(scope="module")
def gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests (no CPU fallback exists)")
    import paper_2510_02126_b200 as G
    G.lib()
    return G


def cuda(x, dt=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(x), dtype=dt, device="cuda")


def colmajor(x):
    """(rows, cols) numpy -> CUDA tensor holding the column-major layout (shape (cols, rows))."""
    return cuda(np.ascontiguousarray(np.asarray(x).T))


# ------------------------------------------------------------------ inversion
@pytest.mark.parametrize("n", [1, 37, 100, 301, 1100, 2100])
def test_invert_fp64_pivots_bitexact(gpu, orc, n):
    rng = np.random.default_rng(n)
    A = rng.standard_normal((n, n))
    X = cuda(A)
    ipiv = torch.zeros(n, dtype=torch.int32, device="cuda")
    gpu.invert(X, ipiv)
    _, piv_ref, info = orc.getrf("fp64", A)
    assert info == 0
    assert np.array_equal(ipiv.cpu().numpy(), piv_ref)
    Xr, _, _ = orc.inverse("fp64", A)
    err = np.linalg.norm(X.cpu().numpy() - Xr) / np.linalg.norm(Xr)
    assert err <= 1e-12 * np.linalg.cond(A)


def test_invert_singular_reports(gpu):
    X = cuda(np.ones((5, 5)))
    with pytest.raises(gpu.LyapError):
        gpu.invert(X)


# ------------------------------------------------------------------ fp64 kernels
@pytest.mark.parametrize("m,n", [(500, 37), (64, 64), (20, 30), (1, 1), (1030, 17)])
def test_qr_parity(gpu, orc, m, n):
    A = np.random.default_rng(m * 31 + n).standard_normal((m, n))
    Qt, Rt = gpu.qr(colmajor(A))
    Q, R = Qt.T.cpu().numpy(), Rt.T.cpu().numpy()
    Qo, Ro = orc.qr("fp64", A)
    assert np.allclose(Q, Qo, atol=1e-11) and np.allclose(R, Ro, atol=1e-11 * np.abs(Ro).max())


@pytest.mark.parametrize("m,n", [(5000, 700), (9000, 300)])
def test_qr_parity_two_level(gpu, orc, m, n):
    """Two-level blocking (outer blocks of 256 applied by DMMA GEMMs, ragged last block);
    m = 9000 > 16 x 256 rows: the grid-cooperative register panel."""
    A = np.random.default_rng(m + n).standard_normal((m, n))
    Qt, Rt = gpu.qr(colmajor(A))
    Q, R = Qt.T.cpu().numpy(), Rt.T.cpu().numpy()
    Qo, Ro = orc.qr("fp64", A)
    assert np.allclose(Q, Qo, atol=1e-11) and np.allclose(R, Ro, atol=1e-11 * np.abs(Ro).max())


@pytest.mark.parametrize("m,n", [(16384, 1100), (40000, 64)])
def test_qr_large_properties(gpu, m, n):
    """configs[3]-size thin QR: Q^T Q = I, Q R = A, R upper triangular with diag(R) >= 0
    (the unique thin QR), checked in fp64 on the device."""
    g = torch.Generator(device="cuda").manual_seed(m)
    At = torch.randn((n, m), dtype=torch.float64, device="cuda", generator=g)
    At[n // 2] = At[0] + 1e-9 * At[n // 2]                        # a nearly dependent column
    Qt, Rt = gpu.qr(At)
    Q, R = Qt.T, Rt.T
    k = min(m, n)
    assert torch.linalg.norm(Q.T @ Q - torch.eye(k, dtype=torch.float64, device="cuda")) <= 1e-13 * k
    assert torch.linalg.norm(Q @ R - At.T) <= 1e-14 * torch.linalg.norm(At) * np.sqrt(n)
    assert torch.count_nonzero(torch.tril(R, -1)) == 0
    assert bool((torch.diagonal(R) >= 0).all())


@pytest.mark.parametrize("n", [1, 2, 17, 64, 131])
def test_syev_parity(gpu, orc, n):
    B = np.random.default_rng(n).standard_normal((n, n))
    A = B + B.T
    w, V = gpu.syev(cuda(A))
    wo, Vo, _ = orc.syev("fp64", A)
    scale = np.abs(wo).max()
    assert np.allclose(w.cpu().numpy(), wo, atol=1e-12 * scale)
    assert np.allclose(V.cpu().numpy(), Vo, atol=1e-9)


def _eig_checks(A, w, V, tol=1e-12):
    n = A.shape[0]
    scale = max(np.abs(np.linalg.eigvalsh(A)).max(), 1e-300)
    wr = np.linalg.eigvalsh(A)[::-1]
    assert np.allclose(w, wr, atol=tol * scale * max(1, n / 100))
    assert np.linalg.norm(V.T @ V - np.eye(n)) <= tol * n
    assert np.linalg.norm(A @ V - V * w[None, :]) <= tol * scale * n


@pytest.mark.parametrize("n", [33, 64, 131, 300, 700, 1100, 2100])
def test_syevd_random(gpu, n):
    """Tridiagonalisation + divide-and-conquer path (n > 32) against numpy eigh and
    the defining identities A V = V diag(w), V^T V = I."""
    B = np.random.default_rng(n + 5).standard_normal((n, n))
    A = B + B.T
    w, V = gpu.syev(cuda(A))
    _eig_checks(A, w.cpu().numpy(), V.cpu().numpy())


@pytest.mark.parametrize("kind", ["graded", "clustered", "lowrank", "indefinite_pm"])
def test_syevd_hard_spectra(gpu, kind):
    """Spectra like the IR's kernel matrices: eigenvalues spanning 15 decades, clusters,
    exact zero blocks (heavy deflation), and +/- pairs."""
    n = 257
    rng = np.random.default_rng(9)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    if kind == "graded":
        lam = np.sign(rng.standard_normal(n)) * 10.0 ** (-15 * rng.uniform(0, 1, n))
    elif kind == "clustered":
        lam = np.repeat([1.0, 1e-3, -2.0, 5e-9], [60, 70, 60, 67]) * (1 + 1e-14 * rng.standard_normal(n))
    elif kind == "lowrank":
        lam = np.zeros(n)
        lam[:10] = rng.uniform(1, 2, 10)
    else:
        x = rng.uniform(0.1, 1, n // 2)
        lam = np.concatenate([x, -x, [0.5]])
    A = (Q * lam[None, :]) @ Q.T
    A = (A + A.T) / 2
    w, V = gpu.syev(cuda(A))
    _eig_checks(A, w.cpu().numpy(), V.cpu().numpy(), tol=1e-12)


@pytest.mark.parametrize("n,c,r", [(700, 300, 25), (3000, 700, 6), (2500, 900, 60), (1500, 1300, 90)])
def test_rank_trunc_chol_parity_sizes(gpu, orc, n, c, r):
    """Register-resident (c <= 512) and streamed (c > 512, up to four CTAs per SM) QRCP
    variants and the grid-size rule, against the oracle's RRQR (decaying spectrum)."""
    rng = np.random.default_rng(n + c)
    sv = np.logspace(0, -8, r)
    Z = (rng.standard_normal((n, r)) * sv[None, :]) @ rng.standard_normal((r, c)) + 1e-12 * rng.standard_normal((n, c))
    tol = np.sqrt(orc.unit_roundoff("fp16"))
    Zg = gpu.rank_trunc_chol(colmajor(Z), tol, "fp64").cpu().numpy()
    Zo = orc.rank_trunc_chol("fp64", Z, tol)
    assert Zg.shape == Zo.shape
    assert np.allclose(Zg, Zo, atol=1e-10 * np.abs(Zo).max())


@pytest.mark.parametrize("n,c,r", [(700, 300, 25), (3000, 700, 120), (1500, 1300, 90), (2000, 64, 40)])
def test_rank_trunc_chol_blocked_parity(gpu, orc, n, c, r, monkeypatch):
    """Blocked QRCP (xLAQPS scheme: blocks of 32 pivots, read-only GEMV per step, DMMA
    trailing update per block, early block end on norm cancellation) against the oracle's
    unblocked RRQR: same rank, same factor."""
    monkeypatch.setenv("LYAP_RRQR_BLOCKED", "1")
    rng = np.random.default_rng(n + 3 * c)
    sv = np.logspace(0, -7, r)
    Z = (rng.standard_normal((n, r)) * sv[None, :]) @ rng.standard_normal((r, c)) + 1e-12 * rng.standard_normal((n, c))
    tol = np.sqrt(orc.unit_roundoff("fp32"))
    Zg = gpu.rank_trunc_chol(colmajor(Z), tol, "fp64").cpu().numpy()
    Zo = orc.rank_trunc_chol("fp64", Z, tol)
    assert Zg.shape == Zo.shape
    assert np.allclose(Zg, Zo, atol=1e-10 * np.abs(Zo).max())


@pytest.mark.slow
def test_rank_trunc_chol_blocked_large(gpu, monkeypatch):
    """configs[3]-size truncation (n = 16384, c = 3000, blocked path by default): the kept
    factor reproduces Z Z^T to the RankTruncChol bound (l.1256-1266, reading R-RRQR:
    ||Z Z^T - Zk Zk^T||_2 <= 2 ||S|| ||Z|| + ||S||^2 with ||S|| <= sqrt(u) |r11|), and the
    blocked and unblocked paths keep the same rank."""
    g = torch.Generator(device="cuda").manual_seed(5)
    n, c, r = 16384, 3000, 700
    sv = torch.logspace(0, -6, r, dtype=torch.float64, device="cuda")
    Zt = ((torch.randn(n, r, dtype=torch.float64, device="cuda", generator=g) * sv) @
          torch.randn(r, c, dtype=torch.float64, device="cuda", generator=g)).T.contiguous()
    tol = 2.0 ** -12
    Zb = gpu.rank_trunc_chol(Zt, tol, "fp64")
    monkeypatch.setenv("LYAP_RRQR_BLOCKED", "0")
    Zu = gpu.rank_trunc_chol(Zt, tol, "fp64")
    assert Zb.shape == Zu.shape
    Z = Zt.T

    def norm2(apply, dim, its=60):
        """2-norm of a symmetric operator by power iteration (converged to a few digits)."""
        x = torch.randn(dim, dtype=torch.float64, device="cuda", generator=g)
        lam = 0.0
        for _ in range(its):
            y = apply(x)
            lam = torch.linalg.norm(y).item()
            x = y / lam
        return lam

    nZ2 = norm2(lambda x: Z.T @ (Z @ x), c)                       # ||Z||_2^2
    nD = norm2(lambda x: Z @ (Z.T @ x) - Zb @ (Zb.T @ x), n)       # ||Z Z^T - Zk Zk^T||_2
    # ||S||_F <= tol |r11| <= tol ||Z||_2
    assert nD <= (2 * tol + tol ** 2) * nZ2 * 1.05
    assert torch.linalg.norm(Zb - Zu) <= 1e-9 * torch.linalg.norm(Zu)


def test_rank_trunc_chol_parity(gpu, orc):
    rng = np.random.default_rng(3)
    n, c = 200, 40
    Z = rng.standard_normal((n, 6)) @ rng.standard_normal((6, c)) + 1e-9 * rng.standard_normal((n, c))
    tol = np.sqrt(orc.unit_roundoff("fp16"))
    Zg = gpu.rank_trunc_chol(colmajor(Z), tol, "fp64").cpu().numpy()
    Zo = orc.rank_trunc_chol("fp64", Z, tol)
    assert Zg.shape == Zo.shape
    assert np.allclose(Zg, Zo, atol=1e-10 * np.abs(Zo).max())


def test_rank_trunc_ldlt_parity(gpu, orc):
    rng = np.random.default_rng(4)
    n, c = 150, 24
    Z = rng.standard_normal((n, c))
    Y = np.diag(rng.uniform(-1, 1, c)) * np.array([10.0 ** -(i % 8) for i in range(c)])
    Zg, Yg = gpu.rank_trunc_ldlt(colmajor(Z), cuda(Y), "fp64")
    Zo, Yo = orc.rank_trunc_ldlt("fp64", Z, Y)
    assert Zg.shape[1] == Zo.shape[1]
    Xg = Zg.cpu().numpy() @ Yg.cpu().numpy() @ Zg.cpu().numpy().T
    Xo = Zo @ Yo @ Zo.T
    assert np.linalg.norm(Xg - Xo) <= 1e-11 * np.linalg.norm(Xo)


# ------------------------------------------------------------------ Newton
@pytest.mark.parametrize("us", ["fp64", "fp32", "fp16", "bf16"])
@pytest.mark.parametrize("n", [100, 128])
def test_newton_aseq_counts(gpu, orc, us, n):
    """The A-side step count (an integer decided by floats) matches the oracle's.  n = 128
    takes the row-staged 16-byte Newton update in every precision, n = 100 the element-wise
    one for fp16/bf16."""
    p = P.paper_synthetic(n, 3, 1.0, seed=0)
    s = gpu.Solver(n, us=us, max_cols=64)
    out = s.newton_aseq(cuda(p.A))
    q = orc.aseq(us, p.A)
    assert out["steps"] == q.steps
    rt = 1e-12 if us == "fp64" else 50 * orc.unit_roundoff(us)
    assert np.allclose(out["mu"], q.mu, rtol=rt)


@pytest.mark.parametrize("us", ["fp64", "fp32", "fp16", "bf16"])
@pytest.mark.parametrize("n", [100, 128])
def test_newton_determinantal_scaling(gpu, orc, us, n):
    """Determinantal scaling mu_k = |det A_k|^{-1/n} (l.1139; log|det| from the Gauss-Jordan
    pivots): step count and mu_k against the oracle (tc model)."""
    p = P.paper_synthetic(n, 3, 1.5, seed=1)
    s = gpu.Solver(n, us=us, max_cols=64, scaling=2)
    out = s.newton_aseq(cuda(p.A))
    with orc.model("tc"):
        q = orc.aseq(us, p.A, scaling="det")
    assert out["steps"] == q.steps
    rt = 1e-12 if us == "fp64" else 50 * orc.unit_roundoff(us)
    assert np.allclose(out["mu"], q.mu, rtol=rt)
    assert out["inf"][-1] <= 10 * np.sqrt(n * orc.unit_roundoff(us))


def test_ir_determinantal_scaling_converges(gpu, orc):
    """A full IR solve with the determinantal scaling (configs[0], fp16 solver) reaches the
    fp64 solution and agrees with the oracle run with the same scaling."""
    p = P.cfg0()
    s = gpu.Solver(p.n, us="fp16", max_cols=128, scaling=2)
    res = s.solve(cuda(p.A), colmajor(p.L), None, tol=1e-14, maxit=10)
    with orc.model("tc"):
        ro = orc.ir_chol(p.A, p.L, us="fp16", tol=1e-14, imax=10, scaling="det")
    assert res.report["status"] == ro.status == "converged"
    assert res.report["steps"] == ro.steps
    Xg, Xo = _X(res.Z, None), _X(ro.Z, None)
    assert np.linalg.norm(Xg - Xo) <= 1e-10 * np.linalg.norm(Xo)


@pytest.mark.parametrize("ldlt", [False, True])
def test_newton_solve_vs_kron(gpu, orc, ldlt):
    p = P.random_stable(30, 2, 5)
    W = p.W() if not ldlt else p.L @ np.diag([1.0, -0.5]) @ p.L.T
    X = orc.kron_solve(p.A, W)
    s = gpu.Solver(30, us="fp64", max_cols=64)
    s.newton_aseq(cuda(p.A))
    if ldlt:
        Z, Y = s.newton_z(colmajor(p.L), cuda(np.diag([1.0, -0.5])))
        Xg = (Z @ Y @ Z.T).cpu().numpy()
    else:
        Z, _ = s.newton_z(colmajor(p.L))
        Xg = (Z @ Z.T).cpu().numpy()
    assert np.linalg.norm(Xg - X) <= 1e-10 * np.linalg.norm(X)


# ------------------------------------------------------------------ fragments
def test_fragments_parity(gpu, orc):
    rng = np.random.default_rng(11)
    p = P.random_stable(60, 3, 2)
    S = np.diag([1.0, 0.5, 2.0])
    Z = rng.standard_normal((60, 7))
    Y = np.diag(rng.uniform(0.1, 1, 7))
    s = gpu.Solver(60, us="fp64", max_cols=64)
    Ld, Sd, resF = s.res_fac_ldlt(cuda(p.A), colmajor(p.L), cuda(S), colmajor(Z), cuda(Y), eta_r=1e-4)
    Lo, So, resFo = orc.res_fac_ldlt("fp64", p.A, p.L, S, Z, Y, eta_r=1e-4)
    assert Ld.shape[1] == Lo.shape[1]
    assert np.isclose(resF, resFo, rtol=1e-12)
    Rg = (Ld @ Sd @ Ld.T).cpu().numpy()
    assert np.linalg.norm(Rg - Lo @ So @ Lo.T) <= 1e-11 * np.linalg.norm(Lo @ So @ Lo.T)
    Lp, Lm, resF2 = s.res_fac_chol(cuda(p.A), colmajor(p.L), colmajor(Z), eta_r=1e-4)
    Lpo, Lmo, resF2o = orc.res_fac_chol("fp64", p.A, p.L, Z, eta_r=1e-4)
    assert (Lp.shape[1], Lm.shape[1]) == (Lpo.shape[1], Lmo.shape[1])
    assert np.isclose(resF2, resF2o, rtol=1e-12)
    Rc = (Lp @ Lp.T - Lm @ Lm.T).cpu().numpy()
    Rco = Lpo @ Lpo.T - Lmo @ Lmo.T
    assert np.linalg.norm(Rc - Rco) <= 1e-11 * np.linalg.norm(Rco)
    # solution updates
    Zd = rng.standard_normal((60, 4))
    Yd = np.diag([1.0, -0.2, 0.3, -1e-3])
    Zn, Yn = s.sol_upt_ldlt(colmajor(Z), cuda(Y), colmajor(Zd), cuda(Yd))
    Zno, Yno = orc.sol_upt_ldlt("fp64", Z, Y, Zd, Yd, 10 * 2.0 ** -53)
    assert Zn.shape[1] == Zno.shape[1]
    Xn, Xno = (Zn @ Yn @ Zn.T).cpu().numpy(), Zno @ Yno @ Zno.T
    assert np.linalg.norm(Xn - Xno) <= 1e-11 * np.linalg.norm(Xno)
    Zp, Zm = rng.standard_normal((60, 3)), 0.1 * rng.standard_normal((60, 2))
    Zc = s.sol_upt_chol(colmajor(Z), colmajor(Zp), colmajor(Zm)).cpu().numpy()
    Zco = orc.sol_upt_chol("fp64", Z, Zp, Zm, 10 * 2.0 ** -53)
    assert Zc.shape[1] == Zco.shape[1]
    assert np.linalg.norm(Zc @ Zc.T - Zco @ Zco.T) <= 1e-11 * np.linalg.norm(Zco @ Zco.T)


# ------------------------------------------------------------------ full IR
def _X(Z, Y):
    Z = Z.cpu().numpy() if hasattr(Z, "cpu") else Z
    if Y is None:
        return Z @ Z.T
    Y = Y.cpu().numpy() if hasattr(Y, "cpu") else Y
    return Z @ Y @ Z.T


def _ir_parity(gpu, orc, p, us, ldlt, tol=1e-14, maxit=20, max_cols=256):
    s = gpu.Solver(p.n, us=us, max_cols=max_cols)
    S = p.S if ldlt else None
    res = s.solve(cuda(p.A), colmajor(p.L), cuda(S) if ldlt else None, tol=tol, maxit=maxit)
    # the GPU computes u_s products/inversions on tensor-core arithmetic (u_s operands,
    # fp32 accumulation): compare with the oracle's "tc" model (reading R-TC)
    with orc.model("tc"):
        if ldlt:
            ro = orc.ir_ldlt(p.A, p.L, S, us=us, tol=tol, imax=maxit)
        else:
            ro = orc.ir_chol(p.A, p.L, us=us, tol=tol, imax=maxit)
    Xg, Xo = _X(res.Z, res.Y), _X(ro.Z, ro.Y)
    W = p.W()
    # a reference independent of both precision models: the fp64 Bartels-Stewart solution
    # (scipy), whose error is within kappa_Lyap x eps of the exact X
    import scipy.linalg as sla
    Xbs = sla.solve_continuous_lyapunov(p.A, -W)
    if res.report["status"] == "converged":
        assert np.linalg.norm(Xg - Xbs) <= 1e-10 * np.linalg.norm(Xbs)
    return res, ro, Xg, Xo, W


@pytest.mark.parametrize("us", ["fp16", "bf16", "fp32"])
def test_ir_cfg0_parity(gpu, orc, us):
    """configs[0]: n=64 Cholesky-type, fp16 solver, tol 1e-14, <= 10 IR steps."""
    p = P.cfg0()
    res, ro, Xg, Xo, W = _ir_parity(gpu, orc, p, us, ldlt=False, maxit=10)
    assert res.report["status"] == ro.status == "converged"
    assert res.report["steps"] == ro.steps
    assert res.report["newton_steps"] == ro.newton_max
    assert orc.rel_residual_explicit(p.A, Xg, W) <= 1e-13
    assert np.linalg.norm(Xg - Xo) <= 1e-10 * np.linalg.norm(Xo)


@pytest.mark.parametrize("us", ["fp16", "bf16"])
def test_ir_ldlt_parity_small(gpu, orc, us):
    p = P.cfg1(seed=5, n=96, m=3)
    res, ro, Xg, Xo, W = _ir_parity(gpu, orc, p, us, ldlt=True)
    assert res.report["status"] == ro.status == "converged"
    assert res.report["steps"] == ro.steps
    assert orc.rel_residual_explicit(p.A, Xg, W) <= 1e-13
    assert np.linalg.norm(Xg - Xo) <= 1e-10 * np.linalg.norm(Xo)


def test_ir_ragged_and_indefinite_S(gpu, orc):
    """n not a multiple of the panel width, m = 1 and a non-identity inner factor (W must be
    PSD for the projected IR; indefinite S is covered by the Newton test)."""
    p = P.random_stable(39, 2, 9)
    S = np.diag([1.0, 0.3])
    s = gpu.Solver(39, us="fp16", max_cols=64)
    res = s.solve(cuda(p.A), colmajor(p.L), cuda(S), tol=1e-14)
    X = orc.kron_solve(p.A, p.L @ S @ p.L.T)
    Xg = _X(res.Z, res.Y)
    assert np.linalg.norm(Xg - X) <= 1e-10 * np.linalg.norm(X)
    p1 = P.random_stable(33, 1, 10)
    s1 = gpu.Solver(33, us="bf16", max_cols=64)
    r1 = s1.solve(cuda(p1.A), colmajor(p1.L), None, tol=1e-14)
    X1 = orc.kron_solve(p1.A, p1.W())
    assert np.linalg.norm(_X(r1.Z, None) - X1) <= 1e-10 * np.linalg.norm(X1)


def test_host_path_equals_device_path(gpu, orc):
    p = P.cfg0()
    s = gpu.Solver(p.n, us="fp16", max_cols=128)
    rd = s.solve(cuda(p.A), colmajor(p.L), None, tol=1e-14, maxit=10)
    Zh, Yh, rep = s.solve_host(p.A, np.ascontiguousarray(p.L.T), None, tol=1e-14, maxit=10)
    assert rep["steps"] == rd.report["steps"]
    assert np.array_equal(Zh, rd.Z.cpu().numpy())


@pytest.mark.slow
def test_ir_cfg1_full_size(gpu, orc):
    """configs[1] at full size (n=1024, LDL^T, bf16): the oracle's IR (emulated bf16)
    and the GPU path agree."""
    p = P.cfg1()
    res, ro, Xg, Xo, W = _ir_parity(gpu, orc, p, "bf16", ldlt=True, maxit=30, max_cols=640)
    assert res.report["status"] == ro.status
    assert res.report["steps"] == ro.steps
    assert orc.rel_residual_explicit(p.A, Xg, W) <= 1e-13
    assert np.linalg.norm(Xg - Xo) <= 1e-10 * np.linalg.norm(Xo)


def test_ir_capacity_stop_returns_last_iterate(gpu, orc):
    """A factor outgrowing max_cols ends the refinement with status "capacity" and the
    last verified iterate (not an error): its explicit residual matches the reported one."""
    p = P.cfg0()
    s = gpu.Solver(p.n, us="fp16", max_cols=40)
    res = s.solve(cuda(p.A), colmajor(p.L), None, tol=1e-14, maxit=10)
    rep = res.report
    assert rep["status"] in ("capacity", "converged")
    if rep["status"] == "capacity":
        Xg = _X(res.Z, res.Y)
        r_exp = orc.rel_residual_explicit(p.A, Xg, p.W())
        assert np.isfinite(r_exp) and r_exp <= 10 * rep["res"][0]


def test_solver_precision_per_solve(gpu):
    """u_s is an argument of lyap_ir_solve (the paper's problem statement): one handle
    solving with fp16, then bf16, then fp32, then fp16 again reproduces, bit for bit, the
    solves of handles created for each precision."""
    p = P.cfg0()
    A, L = cuda(p.A), colmajor(p.L)
    s = gpu.Solver(p.n, us="fp16", max_cols=128)
    for us in ("fp16", "bf16", "fp32", "fp16"):
        r = s.solve(A, L, None, tol=1e-14, maxit=10, us=us)
        ref = gpu.Solver(p.n, us=us, max_cols=128).solve(A, L, None, tol=1e-14, maxit=10)
        assert r.report["steps"] == ref.report["steps"]
        assert torch.equal(r.Z, ref.Z), us


def test_solve_argument_validation(gpu):
    """Mistyped or mis-shaped arguments raise before reaching the C ABI."""
    p = P.cfg0()
    s = gpu.Solver(p.n, us="fp16", max_cols=128)
    A, L = cuda(p.A), colmajor(p.L)
    with pytest.raises(gpu.LyapError):
        s.solve(A.float(), L)
    with pytest.raises(gpu.LyapError):
        s.solve(A[:-1], L)
    with pytest.raises(gpu.LyapError):
        s.solve(A, L[:, :-1].contiguous())
    with pytest.raises(gpu.LyapError):
        s.solve(A, L, cuda(np.eye(3)))
