"""configs[2] / configs[3] families and the stagnation path (-m gpu).

The full-size configs[2] (n = 4096) and configs[3] (n = 16384) are beyond the oracle, so
the GPU path is compared with the oracle (tc model, reading R-TC) on reduced grids of the
same recipes -- identical status, IR step count, Newton steps per call, and residual
history (Eq. res-fac-sol, l.1391) within a factor 2 per step -- and the full sizes are
checked by properties (explicit fp64 residual, status).  The stagnation path (PAPER.md
l.1413-1417, Table 3's "--" entries l.1449-1506) is compared on the paper's own
synthetic generator.
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


def cuda(x):
    return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")


def _X(Z, Y=None):
    Z = Z.cpu().numpy() if hasattr(Z, "cpu") else Z
    if Y is None:
        return Z @ Z.T
    Y = Y.cpu().numpy() if hasattr(Y, "cpu") else Y
    return Z @ Y @ Z.T


def _compare(gpu, orc, p, us, imax, ldlt=False, max_cols=512, chaotic=False):
    s = gpu.Solver(p.n, us=us, max_cols=max_cols)
    res = s.solve(cuda(p.A), cuda(p.L.T), cuda(p.S) if ldlt else None, tol=1e-14, maxit=imax)
    with orc.model("tc"):
        ro = (orc.ir_ldlt(p.A, p.L, p.S, us=us, tol=1e-14, imax=imax) if ldlt
              else orc.ir_chol(p.A, p.L, us=us, tol=1e-14, imax=imax))
    rep = res.report
    print(f"{p.name} {us}: gpu {rep['status']} {rep['steps']} {['%.2e' % r for r in rep['res']]}")
    print(f"{p.name} {us}: orc {ro.status} {ro.steps} {['%.2e' % r for r in ro.res]}")
    assert rep["status"] == ro.status
    if chaotic:
        return res, ro
    assert rep["steps"] == ro.steps
    assert rep["newton_steps"] == ro.newton_max
    rg, rr = np.array(rep["res"]), np.array(ro.res)
    assert len(rg) == len(rr)
    # residual history within a factor 2 per step while it is above the fp64 noise floor
    # of the residual formation itself (~1e-12: below it both runs are at tol within a
    # step, and the value is set by fp64 rounding, not by the method)
    above = np.maximum(rg, rr) > 1e-12
    assert np.all(np.abs(np.log2(rg[above] / rr[above])) <= 1.0), (rg, rr)
    return res, ro


@pytest.mark.parametrize("g,us", [(10, "fp16"), (12, "fp16"), (16, "fp16"), (10, "fp32"), (14, "fp32")])
def test_cfg2_family_parity(gpu, orc, g, us):
    """configs[2] recipe (convection 10, indicator patches) on g x g grids: the fp16 IR's
    contraction per step grows with the grid (0.02 at g = 10, 0.13 at g = 16: max_steps
    at i_max = 10) -- the trend that ends in stagnation at g = 64 (kappa u_s ~ 1, l.1518)."""
    p = P.cfg2(g=g)
    res, ro = _compare(gpu, orc, p, us, imax=10)
    if ro.status == "converged":
        Xg, Xo = _X(res.Z), _X(ro.Z)
        assert np.linalg.norm(Xg - Xo) <= 1e-10 * np.linalg.norm(Xo)
        assert orc.rel_residual_explicit(p.A, Xg, p.W()) <= 1e-13


@pytest.mark.parametrize("g,us", [(10, "fp16"), (12, "fp16"), (10, "fp32"), (12, "fp32")])
def test_cfg3_family_parity(gpu, orc, g, us):
    """configs[3] recipe (convection 50, Gaussian L) on g x g grids, fp16 and fp32 solvers."""
    p = P.cfg3(g=g)
    res, ro = _compare(gpu, orc, p, us, imax=10)
    assert ro.status == "converged"
    Xg, Xo = _X(res.Z), _X(ro.Z)
    assert np.linalg.norm(Xg - Xo) <= 1e-10 * np.linalg.norm(Xo)
    assert orc.rel_residual_explicit(p.A, Xg, p.W()) <= 1e-13


@pytest.mark.parametrize("index", [0, 64, 128, 192, 255])
def test_cfg4_member_parity(gpu, orc, index):
    """configs[4] recipe (A = V diag(-lambda) V^{-1}, kappa = 10^(1 + index // 64)) at a
    reduced order n = 128, fp16 solver, kappa = 1e1 .. 1e4.  Up to kappa = 1e3 (kappa u_s
    = 0.5) the GPU and the oracle's tc model agree step for step; at kappa = 1e4 (kappa u_s
    = 4.9) both converge to the same solution, but the contraction per IR step is set by
    rounding (the GPU rounds the Schur complement to u_s after every 32 columns, the tc
    oracle keeps it in fp32: first residual 1.2e-5 vs 0.8e-5) and the step counts may differ
    by one (reading R-STAG)."""
    p = P.cfg4_member(index, n=128)
    res, ro = _compare(gpu, orc, p, "fp16", imax=30, chaotic=(index >= 192))
    assert ro.status == "converged"
    if index >= 192:
        assert abs(res.report["steps"] - ro.steps) <= 1
    Xg, Xo = _X(res.Z), _X(ro.Z)
    assert np.linalg.norm(Xg - Xo) <= 1e-10 * np.linalg.norm(Xo)
    assert orc.rel_residual_explicit(p.A, Xg, p.W()) <= 1e-13


@pytest.mark.parametrize("kind", ["ldlt", "chol"])
def test_stagnation_path_parity(gpu, orc, kind):
    """PAPER.md Section 5.2 generator, n = 100, kappa ~ 10^3.5, bf16 solver: Table 3 prints
    "--" (failure) for both solver types, and neither the GPU nor the oracle converges (the
    residual never gets below 1e-4).  Here kappa u_s ~ 12: every iterate is
    rounding-dominated, so the step count, the residual values and even which stop rule
    ends the run (theta > 0.9 twice, l.1413-1417, or i_max) depend on the order of every
    rounding and are not comparable between two arithmetics (readings R-TC, R-STAG)."""
    p = P.paper_synthetic(100, 3, 3.5, seed=0, kind=kind)
    s = gpu.Solver(p.n, us="bf16", max_cols=512)
    res = s.solve(cuda(p.A), cuda(p.L.T), cuda(p.S) if kind == "ldlt" else None, tol=1e-14, maxit=50)
    with orc.model("tc"):
        ro = (orc.ir_ldlt(p.A, p.L, p.S, us="bf16", tol=1e-14, imax=50) if kind == "ldlt"
              else orc.ir_chol(p.A, p.L, us="bf16", tol=1e-14, imax=50))
    rep = res.report
    print(f"{kind}: gpu {rep['status']} {rep['steps']} {['%.2e' % r for r in rep['res']]}")
    print(f"{kind}: orc {ro.status} {ro.steps} {['%.2e' % r for r in ro.res]}")
    # no convergence on either side; the stop reason (theta rule or i_max, R-STAG) and the
    # step count are set by rounding-dominated residual oscillations
    fail = ("stagnated", "max_steps", "capacity")
    assert ro.status in fail and rep["status"] in fail
    assert min(rep["res"]) > 1e-4 and min(ro.res) > 1e-4


def _explicit_rel_residual_dev(A, Lt, Z, Y=None):
    """Eq. res-fac-sol in fp64 on the device (test-side check, n = 16384)."""
    X = Z @ (Y @ Z.T if Y is not None else Z.T)
    W = Lt.T @ Lt
    R = A @ X + X @ A.T + W
    return (torch.linalg.norm(R) / (torch.linalg.norm(W) + 2 * torch.linalg.norm(X) * torch.linalg.norm(A))).item()


@pytest.mark.slow
def test_cfg3_full_size(gpu):
    """configs[3] at full size (n = 16384, m = 16).  fp32 solver: converges, explicit fp64
    residual <= 1e-13.  fp16 solver: kappa(A) near 1/u_s -- the IR does not contract (the
    reduced-grid trend above), the run ends without convergence and the returned iterate's
    explicit residual equals the reported one."""
    p = P.cfg3()
    A, Lt = cuda(p.A), cuda(p.L.T)
    s = gpu.Solver(p.n, us="fp32", max_cols=6144, newton_cols=14336, work_cols=16384)
    r = s.solve(A, Lt, None, tol=1e-14, maxit=10)
    rep = r.report
    print("cfg3 fp32", {k: v for k, v in rep.items() if k != "ranks"})
    assert rep["status"] == "converged"
    assert _explicit_rel_residual_dev(A, Lt, r.Z) <= 1e-13
    del s, r
    s16 = gpu.Solver(p.n, us="fp16", max_cols=4096, newton_cols=8192, work_cols=10240)
    r16 = s16.solve(A, Lt, None, tol=1e-14, maxit=10)
    rep = r16.report
    print("cfg3 fp16", {k: v for k, v in rep.items() if k != "ranks"})
    assert rep["status"] != "converged"
    assert min(rep["res"]) > 1e-6
    assert np.isclose(_explicit_rel_residual_dev(A, Lt, r16.Z), rep["final_res"], rtol=1e-6)
