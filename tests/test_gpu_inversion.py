"""Low-precision inversion parity (-m gpu): every Gauss-Jordan variant the solver runs --
one-CTA panel (n <= 301), 512- and 1024-thread cluster panels, one-level and two-level
(outer blocks of 512, ragged last block) sweeps, the non-persistent and persistent
tcgen05 updates, the look-ahead stream -- element by element against the oracle's
tc model (u_s operands and results, fp32 accumulation; reading R-TC), and the n = 4096 /
16384 configurations by their fp64 backward error on sampled columns.

Bound (Eq. newton-lyapu1 l.1125 needs A^{-1} at precision u_s): two inversions of the
same u_s matrix that both carry forward errors of order u_s kappa_2(A) differ by
||X_gpu - X_tc||_F / ||X_tc||_F <= C_INV u_s kappa_2(A).  C_INV is set from the measured
ratios; every case asserts that the bound is < 0.5, so a
zero or garbage inverse fails.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import problems as P  # noqa: E402

C_INV = 1.0          # measured max 0.40 (bf16, one-level sweep, n = 1288)
C_BWD = 0.1          # sampled backward error / u_s: measured max 0.016 (configs[2], configs[3])
TDT = {"fp16": torch.float16, "bf16": torch.bfloat16, "fp32": torch.float32}


@pytest.fixture(scope="module")
def gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests (no CPU fallback exists)")
    import paper_2510_02126_b200 as G
    G.lib()
    return G


def _test_matrix(n, kappa, seed):
    """Nonsymmetric Hurwitz test matrix with kappa_2 = kappa: -(Q diag(lambda) Q^T) + K,
    lambda log-spaced in [1, kappa], K skew (the configs[1] recipe), scaled by 1/max|a|."""
    rng = np.random.default_rng(seed)
    Q = P.haar_orthogonal(n, rng)
    lam = np.logspace(0, np.log10(kappa), n)
    G = np.triu(rng.normal(0.0, 0.1, (n, n)), 1)
    A = -(Q * lam[None, :]) @ Q.T + (G - G.T)
    return A / np.abs(A).max()


def _gpu_inverse(gpu, A, us, ipiv=None):
    X = torch.as_tensor(A, dtype=torch.float64, device="cuda").to(TDT[us]).contiguous()
    gpu.invert(X, ipiv)
    return X.double().cpu().numpy()


@pytest.mark.parametrize("us,kappa", [("fp16", 64.0), ("bf16", 16.0), ("fp32", 1e4)])
@pytest.mark.parametrize("n", [130, 1024, 1288, 2048])
def test_invert_vs_oracle_tc(gpu, orc, us, kappa, n):
    """n = 130: one-CTA panel, one level; 1024: cluster panels, two outer blocks; 1288 =
    512 + 512 + 264: ragged outer block; 2048: four outer blocks, persistent tcgen05 update."""
    if us == "fp32" and n > 1288:
        pytest.skip("fp32 covered up to the ragged two-level case (oracle time)")
    A = orc.round_(_test_matrix(n, kappa, seed=n), us)
    k2 = np.linalg.cond(A, 2)
    u = orc.unit_roundoff(us)
    bound = C_INV * u * k2
    assert bound < 0.5, "vacuous bound"
    Xg = _gpu_inverse(gpu, A, us)
    with orc.model("tc"):
        Xo, _, info = orc.inverse(us, A)
    assert info == 0
    err = np.linalg.norm(Xg - Xo) / np.linalg.norm(Xo)
    print(f"inv {us} n={n}: |X_gpu - X_tc|/|X_tc| = {err:.3e} = {err / (u * k2):.3f} u kappa_2")
    assert err <= bound


@pytest.mark.parametrize("us", ["fp16", "bf16"])
def test_invert_lookahead_vs_oracle_tc(gpu, orc, us, monkeypatch):
    """Opt-in look-ahead stream of the two-level sweep (LYAP_GJE_LOOKAHEAD=1) and the
    one-level sweep (LYAP_GJE_1LEVEL=1) against the same oracle inverse."""
    n, kappa = 1288, (64.0 if us == "fp16" else 16.0)
    A = orc.round_(_test_matrix(n, kappa, seed=7), us)
    k2 = np.linalg.cond(A, 2)
    u = orc.unit_roundoff(us)
    with orc.model("tc"):
        Xo, _, _ = orc.inverse(us, A)
    for env in ("LYAP_GJE_LOOKAHEAD", "LYAP_GJE_1LEVEL"):
        monkeypatch.setenv(env, "1")
        Xg = _gpu_inverse(gpu, A, us)
        monkeypatch.delenv(env)
        err = np.linalg.norm(Xg - Xo) / np.linalg.norm(Xo)
        print(f"{env} {us}: {err / (u * k2):.3f} u kappa_2")
        assert err <= C_INV * u * k2 < 0.5


def _sampled_backward_error(A_dev, X_dev, cols):
    """||A X(:, cols) - I(:, cols)||_F / (||A||_F ||X(:, cols)||_F) in fp64 on the device."""
    Xc = X_dev[:, cols].double()
    R = A_dev.double() @ Xc
    R[cols, torch.arange(len(cols), device=R.device)] -= 1.0
    return (torch.linalg.norm(R) / (torch.linalg.norm(A_dev.double()) * torch.linalg.norm(Xc))).item()


@pytest.mark.slow
@pytest.mark.parametrize("gen,n", [("cfg2", 4096), ("cfg3", 16384)])
def test_invert_large_backward_error(gpu, orc, gen, n):
    """configs[2]/[3] sizes (1024-thread cluster panels above 8192 panel rows, persistent
    tcgen05 update): fp64 normwise backward error on 96 sampled columns <= C_BWD u_s.  A is
    scaled by the power of two 2^-e with max|a_ij| in [1/2, 1) (reading R-RANGE) so that
    the inverse stays inside the fp16 range."""
    p = getattr(P, gen)()
    e = int(np.frexp(np.abs(p.A).max())[1])
    for us in ("fp16", "bf16"):
        A = torch.as_tensor(np.ldexp(p.A, -e), device="cuda").to(TDT[us]).contiguous()
        X = A.clone()
        gpu.invert(X)
        cols = torch.as_tensor(np.random.default_rng(1).choice(n, 96, replace=False), device="cuda")
        eta = _sampled_backward_error(A, X, cols)
        u = orc.unit_roundoff(us)
        print(f"{gen} {us}: sampled backward error {eta:.3e} = {eta / u:.3f} u_s")
        assert eta <= C_BWD * u


@pytest.mark.slow
def test_cfg3_aseq_cached_inverses_backward_error(gpu, orc):
    """Every cached inverse of the configs[3] fp16 A-sequence (Section 3.4 cache): the
    sequence A_{j+1} = (mu_j A_j + A_j^{-1} / mu_j) / 2 is rebuilt in fp64 from the cached
    inverses (A_0 = fl16(A)), and each A_j X_j = I is checked on sampled columns; the
    rebuilt A_j differs from the GPU's u_s iterate by O(u_s) (measured within C_BWD u_s)."""
    p = P.cfg3()
    n = p.n
    s = gpu.Solver(n, us="fp16", max_cols=64)
    A0 = torch.as_tensor(p.A, device="cuda")
    out = s.newton_aseq(A0)
    assert out["steps"] >= 2
    u = orc.unit_roundoff("fp16")
    cols = torch.as_tensor(np.random.default_rng(2).choice(n, 64, replace=False), device="cuda")
    Aj = A0.half().double()
    for j in range(out["steps"]):
        Xj = s.newton_inverse(j).double()
        eta = _sampled_backward_error(Aj, Xj, cols)
        print(f"cfg3 A_{j}: sampled backward error {eta / u:.3f} u_s, mu {out['mu'][j]:.4f}")
        assert eta <= C_BWD * u
        mu = out["mu"][j]
        Aj = ((mu * Aj + Xj / mu) / 2).half().double()
        del Xj


@pytest.mark.parametrize("us", ["fp64", "fp32", "fp16", "bf16"])
def test_newton_cached_inverses_vs_oracle(gpu, orc, us):
    """The Newton update's cache write (Section 3.4): every cached A_j^{-1} against the
    oracle's cached sequence, element by element (n = 128: the 16-byte vector path)."""
    n = 128
    pr = P.paper_synthetic(n, 3, 1.0, seed=0)
    s = gpu.Solver(n, us=us, max_cols=64)
    out = s.newton_aseq(torch.as_tensor(pr.A, device="cuda"))
    with orc.model("tc"):
        q = orc.aseq(us, pr.A)
    assert out["steps"] == q.steps
    u = orc.unit_roundoff(us)
    for j in range(q.steps):
        Xg = s.newton_inverse(j).double().cpu().numpy()
        Xo = q.inverses[j]
        err = np.linalg.norm(Xg - Xo) / np.linalg.norm(Xo)
        k2 = np.linalg.cond(Xo, 2)
        print(f"{us} cached inverse {j}: {err:.3e} = {err / (u * k2):.3f} u kappa_2")
        assert err <= max(2 * C_INV * u * k2 * (j + 1), 1e-13)   # measured max 5.4 (fp64, j = 4)
        assert err < 0.5


@pytest.mark.parametrize("us", ["fp16", "bf16", "fp32"])
@pytest.mark.parametrize("n", [1024, 2048, 4096])
def test_implicit_pivoting_equals_row_swapping(gpu, us, n, monkeypatch):
    """The implicit-pivoting sweep (gje_ip.cu: rows stay in place, positions are exchanged;
    cluster panel with st.async candidate pushes) against the row-swapping sweep (gje.cu,
    LYAP_GJE_SWAP=1): the same LU-with-partial-pivoting pivot sequence (ties by the lowest
    position) and the same arithmetic on every element, so the inverses are equal bit for
    bit (one inversion per Newton step; north_star: partial pivoting)."""
    A = torch.as_tensor(_test_matrix(n, 64.0, seed=5 * n), dtype=torch.float64, device="cuda").to(TDT[us]).contiguous()
    X2, p2 = A.clone(), torch.zeros(n, dtype=torch.int32, device="cuda")
    monkeypatch.setenv("LYAP_GJE_SWAP", "1")
    gpu.invert(X2, p2)
    monkeypatch.delenv("LYAP_GJE_SWAP", raising=False)
    # the look-ahead (two streams, n >= 2048) splits the rank-512 update by columns: the
    # tcgen05 products are unaffected, the fp32 SIMT product may split K differently for a
    # narrower column range (another summation order), so fp32 is bitwise only without it
    for ahead in (True, False):
        if ahead:
            monkeypatch.delenv("LYAP_GJE_NO_LOOKAHEAD", raising=False)
        else:
            monkeypatch.setenv("LYAP_GJE_NO_LOOKAHEAD", "1")
        for rep in range(2 if ahead else 1):                 # twice: stream races would show as differences
            X1, p1 = A.clone(), torch.zeros(n, dtype=torch.int32, device="cuda")
            gpu.invert(X1, p1)
            torch.cuda.synchronize()
            assert torch.equal(p1, p2)
            if us != "fp32" or not ahead:
                assert torch.equal(X1, X2)
            else:
                d = (X1.double() - X2.double()).norm() / X2.double().norm()
                assert float(d) < 1e-5
    res = (A.double() @ X1.double() - torch.eye(n, device="cuda", dtype=torch.float64)).norm() / n ** 0.5
    assert float(res) < 0.05


def test_implicit_pivoting_ties_and_zeros(gpu, monkeypatch):
    """A matrix with many equal-magnitude pivot candidates and exact zeros (the convection-
    diffusion stencil of configs[2], n = 32 x 32 grid): the tie rule (lowest logical position)
    must reproduce the row-swapping sweep's pivots exactly."""
    p = P.cfg2(g=32)
    A = torch.as_tensor(p.A, dtype=torch.float64, device="cuda")
    A = (A / A.abs().max()).to(torch.float16).contiguous()
    n = A.shape[0]
    X1, p1 = A.clone(), torch.zeros(n, dtype=torch.int32, device="cuda")
    monkeypatch.delenv("LYAP_GJE_SWAP", raising=False)
    gpu.invert(X1, p1)
    X2, p2 = A.clone(), torch.zeros(n, dtype=torch.int32, device="cuda")
    monkeypatch.setenv("LYAP_GJE_SWAP", "1")
    gpu.invert(X2, p2)
    torch.cuda.synchronize()
    assert torch.equal(p1, p2)
    assert torch.equal(X1, X2)
