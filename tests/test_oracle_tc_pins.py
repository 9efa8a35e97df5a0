"""Pins of the oracle's "tc" precision model (reading R-TC) against
independent numpy float32 arithmetic (-m "not gpu").

The tc model is "u_s operands and results, fp32 accumulation" -- the arithmetic of
fp16/bf16 tensor cores that accumulate in fp32.  Every whole-IR
GPU parity test compares against it, so it is pinned here against references that
share nothing with oracle.c: numpy's IEEE float32 scalar arithmetic (every + - * /
correctly rounded to binary32), numpy's float16 conversion and an integer bf16
round-to-nearest-even on the float32 bit pattern.
"""
import numpy as np
import pytest

import problems as P


def _to_us(x32: np.ndarray, us: str) -> np.ndarray:
    """Round float32 values to u_s (fp16: numpy's conversion; bf16: integer RNE)."""
    x32 = np.asarray(x32, dtype=np.float32)
    if us == "fp16":
        return x32.astype(np.float16).astype(np.float64)
    b = x32.view(np.uint32).astype(np.uint64)
    lsb = (b >> 16) & 1
    r = ((b + 0x7FFF + lsb) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32).astype(np.float64)


def _operands(rng, shape, us):
    x = rng.standard_normal(shape).astype(np.float32)
    return _to_us(x, us)


@pytest.mark.parametrize("us", ["fp16", "bf16"])
@pytest.mark.parametrize("m,n,k", [(7, 5, 33), (4, 9, 1), (3, 3, 200)])
def test_tc_gemm_equals_float32_accumulation(orc, us, m, n, k):
    """orc_gemm under model("tc") == u_s operands, sequential float32 accumulation of
    float32-rounded products, one final rounding to u_s -- bit for bit."""
    rng = np.random.default_rng(m * 100 + n * 10 + k)
    A = _operands(rng, (m, k), us)
    B = _operands(rng, (k, n), us)
    A32, B32 = A.astype(np.float32), B.astype(np.float32)
    ref = np.zeros((m, n), dtype=np.float32)
    for i in range(m):
        for j in range(n):
            s = np.float32(A32[i, 0] * B32[0, j])
            for l in range(1, k):
                s = np.float32(s + np.float32(A32[i, l] * B32[l, j]))
            ref[i, j] = s
    with orc.model("tc"):
        got = orc.gemm(us, A, B)
    assert np.array_equal(got, _to_us(ref, us))
    # the chop model (every operation rounded to u_s) is a different arithmetic
    if k >= 33:
        assert not np.array_equal(orc.gemm(us, A, B), got)


def _lu_solve_float32(A64: np.ndarray):
    """Textbook LU with partial pivoting (largest |a|, lowest index on ties), then
    X(:, j) = U^{-1} L^{-1} P e_j column by column -- all in numpy float32 scalars."""
    n = A64.shape[0]
    A = A64.astype(np.float32).copy()
    piv = np.zeros(n, dtype=np.int32)
    for j in range(n):
        col = np.abs(A[j:, j])
        ip = j + int(np.argmax(col))          # argmax returns the first maximum
        piv[j] = ip
        if ip != j:
            A[[j, ip], :] = A[[ip, j], :]
        d = A[j, j]
        for i in range(j + 1, n):
            A[i, j] = np.float32(A[i, j] / d)
        for kk in range(j + 1, n):
            u = A[j, kk]
            for i in range(j + 1, n):
                A[i, kk] = np.float32(A[i, kk] - np.float32(A[i, j] * u))
    X = np.zeros((n, n), dtype=np.float32)
    for j in range(n):
        y = np.zeros(n, dtype=np.float32)
        y[j] = 1.0
        for i in range(n):
            if piv[i] != i:
                y[i], y[piv[i]] = y[piv[i]], y[i]
        for l in range(n):
            for i in range(l + 1, n):
                y[i] = np.float32(y[i] - np.float32(A[i, l] * y[l]))
        for l in range(n - 1, -1, -1):
            y[l] = np.float32(y[l] / A[l, l])
            for i in range(l):
                y[i] = np.float32(y[i] - np.float32(A[i, l] * y[l]))
        X[:, j] = y
    return X, piv


@pytest.mark.parametrize("us", ["fp16", "bf16"])
@pytest.mark.parametrize("n", [1, 5, 17, 24])
def test_tc_inverse_equals_float32_lu(orc, us, n):
    """orc_inverse under model("tc") == float32 LU + solve against I, rounded once to
    u_s; identical pivots.  Inputs are u_s values (A_k is stored in u_s)."""
    rng = np.random.default_rng(40 + n)
    A = _operands(rng, (n, n), us) + np.diag(_to_us(np.full(n, 0.25, np.float32), us))
    X32, piv32 = _lu_solve_float32(A)
    with orc.model("tc"):
        Xo, pivo, info = orc.inverse(us, A)
    assert info == 0
    assert np.array_equal(pivo, piv32)
    assert np.array_equal(Xo, _to_us(X32, us))


def test_tc_model_is_exact_for_fp32_and_fp64(orc):
    """For u_s in {fp32, fp64} the two models coincide (accumulation = u_s)."""
    rng = np.random.default_rng(5)
    A = rng.standard_normal((9, 9)) + 3 * np.eye(9)
    for us in ("fp32", "fp64"):
        Ar = orc.round_(A, us)
        X1, p1, _ = orc.inverse(us, Ar)
        with orc.model("tc"):
            X2, p2, _ = orc.inverse(us, Ar)
        assert np.array_equal(X1, X2) and np.array_equal(p1, p2)


@pytest.mark.parametrize("us", ["fp16", "bf16"])
def test_tc_ir_reaches_model_independent_solution(orc, us):
    """The tc-model IR on configs[0] (reduced n) converges to the fp64 Kronecker solution
    (Eq. lyap-ls, a model-independent reference) -- the model changes the path, not
    the limit (Table 2 semantics, l.1078)."""
    p = P.cfg0(n=24, m=2)
    X = orc.kron_solve(p.A, p.W())
    with orc.model("tc"):
        r = orc.ir_chol(p.A, p.L, us=us, tol=1e-14, imax=10)
    assert r.status == "converged"
    Xt = r.Z @ r.Z.T
    assert np.linalg.norm(Xt - X) <= 1e-11 * np.linalg.norm(X)
