"""CPU oracle for PAPER.md (arXiv 2510.02126) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It is
a ctypes binding to ``liblyaporacle.so`` (plain C, ``oracle/oracle.c``), which
shares no code with the CUDA product path.  All matrices cross the boundary as
column-major float64 arrays.

Parity status per function is recorded in DESIGN.md ("Oracle pins").
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

FP64, FP32, FP16, BF16 = 0, 1, 2, 3
PREC = {"fp64": FP64, "fp32": FP32, "fp16": FP16, "bf16": BF16}

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liblyaporacle.so")
_lib = None

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


def build() -> str:
    """Compile the oracle with make (plain C, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        src = os.path.join(_HERE, "oracle.c")
        if (not os.path.exists(_LIB_PATH)) or os.path.getmtime(src) > os.path.getmtime(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _declare(_lib)
    return _lib


class NewtonParams(C.Structure):
    _fields_ = [("kmax", C.c_int), ("scaling", C.c_int), ("extra", C.c_int), ("rho", C.c_double)]


class IRParams(C.Structure):
    _fields_ = [("us", C.c_int), ("ur", C.c_int), ("uc", C.c_int), ("tol", C.c_double),
                ("imax", C.c_int), ("eta_r", C.c_double), ("eta_s", C.c_double),
                ("newton", NewtonParams), ("cache", C.c_int)]


MAXREP = 128


class IRReport(C.Structure):
    _fields_ = [("steps", C.c_int), ("status", C.c_int), ("newton_calls", C.c_int),
                ("newton_total", C.c_int), ("newton_max", C.c_int), ("inversions", C.c_int),
                ("nres", C.c_int), ("res", C.c_double * MAXREP), ("rank", C.c_int * MAXREP),
                ("final_res", C.c_double)]


def _declare(L):
    L.orc_unit_roundoff.restype = C.c_double
    L.orc_unit_roundoff.argtypes = [C.c_int]
    L.orc_xmin.restype = C.c_double
    L.orc_xmin.argtypes = [C.c_int]
    L.orc_xmax.restype = C.c_double
    L.orc_xmax.argtypes = [C.c_int]
    L.orc_round.restype = C.c_double
    L.orc_round.argtypes = [C.c_double, C.c_int]
    L.orc_round_ref.restype = C.c_double
    L.orc_round_ref.argtypes = [C.c_double, C.c_int]
    L.orc_round_array.argtypes = [_dp, C.c_long, C.c_int]
    L.orc_gemm.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                           _dp, C.c_int, _dp, C.c_int, _dp, C.c_int]
    L.orc_getrf.restype = C.c_int
    L.orc_getrf.argtypes = [C.c_int, C.c_int, _dp, C.c_int, _ip]
    L.orc_inverse.restype = C.c_int
    L.orc_inverse.argtypes = [C.c_int, C.c_int, _dp, _dp, _ip]
    L.orc_inverse_ld.restype = C.c_int
    L.orc_inverse_ld.argtypes = [C.c_int, C.c_int, _dp, _dp, _ip, C.POINTER(C.c_double)]
    L.orc_qr.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp, _dp]
    L.orc_syev.restype = C.c_int
    L.orc_syev.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp]
    L.orc_rank_trunc_chol.restype = C.c_int
    L.orc_rank_trunc_chol.argtypes = [C.c_int, C.c_int, C.c_int, _dp, C.c_double, _dp]
    L.orc_rank_trunc_ldlt.restype = C.c_int
    L.orc_rank_trunc_ldlt.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, _dp]
    L.orc_aseq_compute.restype = C.c_void_p
    L.orc_aseq_compute.argtypes = [C.c_int, C.c_int, _dp, C.POINTER(NewtonParams), _ip]
    for nm, rt in [("orc_aseq_steps", C.c_int), ("orc_aseq_converged", C.c_int)]:
        getattr(L, nm).restype = rt
        getattr(L, nm).argtypes = [C.c_void_p]
    for nm in ["orc_aseq_mu", "orc_aseq_delta", "orc_aseq_inf"]:
        getattr(L, nm).restype = C.c_double
        getattr(L, nm).argtypes = [C.c_void_p, C.c_int]
    L.orc_aseq_inverse.restype = _dp
    L.orc_aseq_inverse.argtypes = [C.c_void_p, C.c_int]
    L.orc_aseq_pivots.restype = _ip
    L.orc_aseq_pivots.argtypes = [C.c_void_p, C.c_int]
    L.orc_aseq_free.argtypes = [C.c_void_p]
    L.orc_newton_ldlt_z.restype = C.c_int
    L.orc_newton_ldlt_z.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_int, _dp, _dp, C.c_double,
                                    C.POINTER(_dp), C.POINTER(_dp), _ip]
    L.orc_newton_chol_z.restype = C.c_int
    L.orc_newton_chol_z.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_int, _dp, C.c_double,
                                    C.POINTER(_dp), _ip]
    L.orc_res_fac_ldlt.restype = C.c_int
    L.orc_res_fac_ldlt.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, C.c_int, _dp, _dp,
                                   C.c_double, C.POINTER(_dp), C.POINTER(_dp), _dp]
    L.orc_sol_upt_ldlt.restype = C.c_int
    L.orc_sol_upt_ldlt.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp, C.c_int, _dp, _dp,
                                   C.c_double, C.POINTER(_dp), C.POINTER(_dp)]
    L.orc_res_fac_chol.restype = C.c_int
    L.orc_res_fac_chol.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp, C.c_int, _dp, C.c_double,
                                   C.POINTER(_dp), _ip, C.POINTER(_dp), _ip, _dp]
    L.orc_sol_upt_chol.restype = C.c_int
    L.orc_sol_upt_chol.argtypes = [C.c_int, C.c_int, C.c_int, _dp, C.c_int, _dp, C.c_int, _dp,
                                   C.c_double, C.POINTER(_dp)]
    L.orc_ir_ldlt.restype = C.c_int
    L.orc_ir_ldlt.argtypes = [C.POINTER(IRParams), C.c_int, C.c_int, _dp, _dp, _dp,
                              C.POINTER(_dp), C.POINTER(_dp), C.POINTER(IRReport)]
    L.orc_ir_chol.restype = C.c_int
    L.orc_ir_chol.argtypes = [C.POINTER(IRParams), C.c_int, C.c_int, _dp, _dp,
                              C.POINTER(_dp), C.POINTER(IRReport)]
    L.orc_form_x.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp]
    L.orc_rel_residual_explicit.restype = C.c_double
    L.orc_rel_residual_explicit.argtypes = [C.c_int, _dp, _dp, _dp]
    L.orc_kron_solve.restype = C.c_int
    L.orc_kron_solve.argtypes = [C.c_int, _dp, _dp, _dp]
    L.orc_free.argtypes = [C.c_void_p]
    L.orc_set_model.argtypes = [C.c_int]
    L.orc_get_model.restype = C.c_int


# ----------------------------------------------------------------- helpers
def _f(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _prec(p) -> int:
    return PREC[p] if isinstance(p, str) else int(p)


def _take(ptr, rows: int, cols: int) -> np.ndarray:
    """Copy a malloc'ed column-major block out and free it."""
    n = rows * cols
    if n > 0:
        out = np.ctypeslib.as_array(ptr, shape=(n,)).copy().reshape((cols, rows)).T.copy(order="F")
    else:
        out = np.zeros((rows, cols), order="F")
    lib().orc_free(C.cast(ptr, C.c_void_p))
    return out


# ----------------------------------------------------------------- API
MODELS = {"chop": 0, "tc": 1}


class model:
    """Context manager selecting the u_s precision model ("chop" or "tc")."""

    def __init__(self, name: str):
        self.name = name

    def __enter__(self):
        self.prev = lib().orc_get_model()
        lib().orc_set_model(MODELS[self.name])
        return self

    def __exit__(self, *exc):
        lib().orc_set_model(self.prev)
        return False


def unit_roundoff(p) -> float:
    return lib().orc_unit_roundoff(_prec(p))


def xmin(p) -> float:
    return lib().orc_xmin(_prec(p))


def xmax(p) -> float:
    return lib().orc_xmax(_prec(p))


def round_(x, p):
    a = np.array(x, dtype=np.float64, copy=True)
    flat = np.ascontiguousarray(a.reshape(-1))
    lib().orc_round_array(_p(flat), flat.size, _prec(p))
    return flat.reshape(a.shape)


def round_ref_scalar(x: float, p) -> float:
    return lib().orc_round_ref(float(x), _prec(p))


def round_scalar(x: float, p) -> float:
    return lib().orc_round(float(x), _prec(p))


def gemm(p, A, B, ta=False, tb=False):
    A, B = _f(A), _f(B)
    m = A.shape[1] if ta else A.shape[0]
    k = A.shape[0] if ta else A.shape[1]
    n = B.shape[0] if tb else B.shape[1]
    Cm = np.zeros((m, n), order="F")
    lib().orc_gemm(_prec(p), int(ta), int(tb), m, n, k, _p(A), A.shape[0], _p(B), B.shape[0],
                   _p(Cm), m)
    return Cm


def getrf(p, A):
    A = _f(A).copy(order="F")
    n = A.shape[0]
    piv = np.zeros(n, dtype=np.int32)
    info = lib().orc_getrf(_prec(p), n, _p(A), n, piv.ctypes.data_as(_ip))
    return A, piv, info


def inverse(p, A):
    A = _f(A)
    n = A.shape[0]
    X = np.zeros((n, n), order="F")
    piv = np.zeros(n, dtype=np.int32)
    info = lib().orc_inverse(_prec(p), n, _p(A), _p(X), piv.ctypes.data_as(_ip))
    return X, piv, info


def inverse_logdet(p, A):
    """(A^{-1}, pivots, info, log|det A|) from one LU with partial pivoting."""
    A = _f(A)
    n = A.shape[0]
    X = np.zeros((n, n), order="F")
    piv = np.zeros(n, dtype=np.int32)
    ld = C.c_double(0.0)
    info = lib().orc_inverse_ld(_prec(p), n, _p(A), _p(X), piv.ctypes.data_as(_ip), C.byref(ld))
    return X, piv, info, ld.value


def qr(p, A):
    A = _f(A)
    m, n = A.shape
    k = min(m, n)
    Q = np.zeros((m, k), order="F")
    R = np.zeros((k, n), order="F")
    lib().orc_qr(_prec(p), m, n, _p(A), _p(Q), _p(R))
    return Q, R


def syev(p, A):
    A = _f(A)
    n = A.shape[0]
    w = np.zeros(n)
    V = np.zeros((n, n), order="F")
    sweeps = lib().orc_syev(_prec(p), n, _p(A), _p(w), _p(V))
    return w, V, sweeps


def rank_trunc_chol(p, Z, tol_rel=None):
    Z = _f(Z)
    n, c = Z.shape
    if tol_rel is None:
        tol_rel = np.sqrt(unit_roundoff(p))
    out = np.zeros((n, max(c, 1)), order="F")
    k = lib().orc_rank_trunc_chol(_prec(p), n, c, _p(Z), float(tol_rel), _p(out))
    return out[:, :k].copy(order="F")


def rank_trunc_ldlt(p, Z, Y):
    Z, Y = _f(Z), _f(Y)
    n, c = Z.shape
    Zo = np.zeros((n, max(c, 1)), order="F")
    Yo = np.zeros((max(c, 1), max(c, 1)), order="F")
    k = lib().orc_rank_trunc_ldlt(_prec(p), n, c, _p(Z), _p(Y), _p(Zo), _p(Yo))
    Yk = np.ctypeslib.as_array(Yo.reshape(-1, order="F")[: k * k]).reshape((k, k), order="F")
    return Zo[:, :k].copy(order="F"), Yk.copy(order="F")


@dataclass
class ASeq:
    """Cached A-side Newton sequence (Section 3.4)."""
    steps: int
    converged: bool
    mu: list
    delta: list
    inf: list
    inverses: list = field(repr=False)
    pivots: list = field(repr=False)
    handle: int = field(repr=False, default=0)


SCALINGS = {"none": 0, "fro": 1, "det": 2}


def newton_params(kmax=50, scaling=True, extra=1, rho=0.1) -> NewtonParams:
    """scaling: False/"none" (mu = 1), True/"fro" (Frobenius norm, l.1406), "det"
    (|det A_k|^{-1/n}, l.1139)."""
    sc = SCALINGS[scaling] if isinstance(scaling, str) else int(scaling)
    return NewtonParams(kmax, sc, extra, rho)


def aseq(p, A, kmax=50, scaling=True, extra=1, keep=False):
    A = _f(A)
    n = A.shape[0]
    P = newton_params(kmax, scaling, extra)
    info = C.c_int(0)
    h = lib().orc_aseq_compute(_prec(p), n, _p(A), C.byref(P), C.byref(info))
    k = lib().orc_aseq_steps(h)
    res = ASeq(steps=k, converged=bool(lib().orc_aseq_converged(h)),
               mu=[lib().orc_aseq_mu(h, j) for j in range(k)],
               delta=[lib().orc_aseq_delta(h, j) for j in range(k)],
               inf=[lib().orc_aseq_inf(h, j) for j in range(k)],
               inverses=[np.ctypeslib.as_array(lib().orc_aseq_inverse(h, j), shape=(n * n,))
                         .reshape((n, n), order="F").copy(order="F") for j in range(k)],
               pivots=[np.ctypeslib.as_array(lib().orc_aseq_pivots(h, j), shape=(n,)).copy()
                       for j in range(k)])
    if info.value != 0:
        lib().orc_aseq_free(h)
        raise FloatingPointError(f"Newton A-sequence failed at precision {p}: info={info.value}")
    if keep:
        res.handle = h
    else:
        lib().orc_aseq_free(h)
    return res


def newton_ldlt(p, A, L, S=None, kmax=50, scaling=True, extra=1, rho=0.1):
    """Algorithm 4 at precision p; returns (Z, Y, ASeq)."""
    A, L = _f(A), _f(L)
    n, m = L.shape
    S = np.eye(m) if S is None else S
    S = _f(S)
    q = aseq(p, A, kmax, scaling, extra, keep=True)
    Zp, Yp, nt = _dp(), _dp(), C.c_int(0)
    c = lib().orc_newton_ldlt_z(_prec(p), q.handle, n, m, _p(L), _p(S), rho,
                                C.byref(Zp), C.byref(Yp), C.byref(nt))
    lib().orc_aseq_free(q.handle)
    q.handle = 0
    return _take(Zp, n, c), _take(Yp, c, c), q


def newton_chol(p, A, L, kmax=50, scaling=True, extra=1, rho=0.1):
    """Algorithm 3 at precision p; returns (Z, ASeq)."""
    A, L = _f(A), _f(L)
    n, m = L.shape
    q = aseq(p, A, kmax, scaling, extra, keep=True)
    Zp, nt = _dp(), C.c_int(0)
    c = lib().orc_newton_chol_z(_prec(p), q.handle, n, m, _p(L), rho, C.byref(Zp), C.byref(nt))
    lib().orc_aseq_free(q.handle)
    q.handle = 0
    return _take(Zp, n, c), q


def res_fac_ldlt(p, A, L, S, Z, Y, eta_r=1e-4):
    A, L, S, Z, Y = map(_f, (A, L, S, Z, Y))
    n, m = L.shape
    c = Z.shape[1]
    Lp, Sp, r = _dp(), _dp(), C.c_double(0)
    k = lib().orc_res_fac_ldlt(_prec(p), n, m, _p(A), _p(L), _p(S), c, _p(Z), _p(Y), eta_r,
                               C.byref(Lp), C.byref(Sp), C.byref(r))
    return _take(Lp, n, k), _take(Sp, k, k), r.value


def sol_upt_ldlt(p, Z, Y, Zd, Yd, eta_s):
    Z, Y, Zd, Yd = map(_f, (Z, Y, Zd, Yd))
    n, c = Z.shape
    cd = Zd.shape[1]
    Zp, Yp = _dp(), _dp()
    k = lib().orc_sol_upt_ldlt(_prec(p), n, c, _p(Z), _p(Y), cd, _p(Zd), _p(Yd), eta_s,
                               C.byref(Zp), C.byref(Yp))
    return _take(Zp, n, k), _take(Yp, k, k)


def res_fac_chol(p, A, L, Z, eta_r=1e-4):
    A, L, Z = map(_f, (A, L, Z))
    n, m = L.shape
    c = Z.shape[1]
    Lp, Lm, kp, km, r = _dp(), _dp(), C.c_int(0), C.c_int(0), C.c_double(0)
    lib().orc_res_fac_chol(_prec(p), n, m, _p(A), _p(L), c, _p(Z), eta_r, C.byref(Lp),
                           C.byref(kp), C.byref(Lm), C.byref(km), C.byref(r))
    return _take(Lp, n, kp.value), _take(Lm, n, km.value), r.value


def sol_upt_chol(p, Z, Zp_, Zm_, eta_s):
    Z, Zp_, Zm_ = map(_f, (Z, Zp_, Zm_))
    n, c = Z.shape
    out = _dp()
    k = lib().orc_sol_upt_chol(_prec(p), n, c, _p(Z), Zp_.shape[1], _p(Zp_), Zm_.shape[1],
                               _p(Zm_), eta_s, C.byref(out))
    return _take(out, n, k)


@dataclass
class IRResult:
    Z: np.ndarray
    Y: np.ndarray | None
    steps: int
    status: str
    newton_calls: int
    newton_total: int
    newton_max: int
    inversions: int
    res: list
    rank: list
    final_res: float


_STATUS = {0: "converged", 1: "stagnated", 2: "max_steps", 3: "solver_failure"}


def ir_params(us="fp16", ur="fp64", uc="fp64", tol=1e-14, imax=50, eta_r=1e-4, eta_s=None,
              kmax=50, scaling=True, extra=1, rho=0.1, cache=True) -> IRParams:
    # extra=1: reading R-EXTRA -- Tables 4-5's per-call counts alpha
    # match one iteration after the first step meeting Eq. newton-stop-tau.
    if eta_s is None:
        eta_s = 10 * unit_roundoff("fp64")        # eta_s = 10u
    return IRParams(_prec(us), _prec(ur), _prec(uc), tol, imax, eta_r, eta_s,
                    newton_params(kmax, scaling, extra, rho), int(cache))


def _result(Z, Y, rep) -> IRResult:
    nres = min(rep.nres, MAXREP)
    return IRResult(Z=Z, Y=Y, steps=rep.steps, status=_STATUS[rep.status],
                    newton_calls=rep.newton_calls, newton_total=rep.newton_total,
                    newton_max=rep.newton_max, inversions=rep.inversions,
                    res=[rep.res[i] for i in range(nres)], rank=[rep.rank[i] for i in range(nres)],
                    final_res=rep.final_res)


def ir_ldlt(A, L, S=None, **kw) -> IRResult:
    """Algorithm 2 with Algorithm 4 as solver."""
    A, L = _f(A), _f(L)
    n, m = L.shape
    S = _f(np.eye(m) if S is None else S)
    P = ir_params(**kw)
    rep = IRReport()
    Zp, Yp = _dp(), _dp()
    c = lib().orc_ir_ldlt(C.byref(P), n, m, _p(A), _p(L), _p(S), C.byref(Zp), C.byref(Yp),
                          C.byref(rep))
    return _result(_take(Zp, n, c), _take(Yp, c, c), rep)


def ir_chol(A, L, **kw) -> IRResult:
    """Algorithm 1 with Algorithm 3 as solver."""
    A, L = _f(A), _f(L)
    n, m = L.shape
    P = ir_params(**kw)
    rep = IRReport()
    Zp = _dp()
    c = lib().orc_ir_chol(C.byref(P), n, m, _p(A), _p(L), C.byref(Zp), C.byref(rep))
    return _result(_take(Zp, n, c), None, rep)


def form_x(Z, Y=None):
    Z = _f(Z)
    n, c = Z.shape
    X = np.zeros((n, n), order="F")
    Yf = _f(Y) if Y is not None else None
    lib().orc_form_x(n, c, _p(Z), _p(Yf) if Yf is not None else None, _p(X))
    return X


def rel_residual_explicit(A, X, W) -> float:
    A, X, W = map(_f, (A, X, W))
    return lib().orc_rel_residual_explicit(A.shape[0], _p(A), _p(X), _p(W))


def kron_solve(A, W):
    A, W = _f(A), _f(W)
    n = A.shape[0]
    X = np.zeros((n, n), order="F")
    info = lib().orc_kron_solve(n, _p(A), _p(W), _p(X))
    if info != 0:
        raise np.linalg.LinAlgError(f"kron_solve failed: {info}")
    return X
