"""B200-native mixed-precision iterative refinement for low-rank Lyapunov equations.

Thin ctypes binding over ``liblyapir.so`` (hand-written sm_100a CUDA kernels,
C ABI declared in ``include/lyap_ir.h``).  Only argument marshalling happens
here: torch provides device memory and the stream; every arithmetic step of
the solver runs in the library's kernels.  There is no CPU fallback: if the
shared library or a CUDA device is missing, every entry point raises.

Layout conventions (see include/lyap_ir.h): ``A`` is an (n, n) row-major
float64 tensor; tall factors (L, Z) are column-major, which this binding
represents as the contiguous transpose, i.e. a tensor ``Lt`` of shape (m, n)
with ``L = Lt.T``.  Small square matrices (S, Y) are symmetric here, so their
layout is immaterial.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

_HERE = os.path.dirname(os.path.abspath(__file__))
# LYAP_LIB: an instrumented build (tools/ profiling runs only); default the in-tree library
_LIB_PATH = os.environ.get("LYAP_LIB") or os.path.join(_HERE, "liblyapir.so")
_lib = None

FP64, FP32, FP16, BF16 = 0, 1, 2, 3
PREC = {"fp64": FP64, "fp32": FP32, "fp16": FP16, "bf16": BF16}
STATUS = {0: "converged", 1: "stagnated", 2: "max_steps", 3: "solver_failure", 4: "capacity"}
ERRORS = {-1: "invalid argument", -2: "CUDA error / no device", -3: "singular matrix",
          -4: "overflow in solver precision", -5: "capacity exceeded"}


class LyapError(RuntimeError):
    pass


class Options(C.Structure):
    _fields_ = [("kmax", C.c_int), ("scaling", C.c_int), ("extra", C.c_int), ("rho", C.c_double),
                ("eta_r", C.c_double), ("eta_s", C.c_double), ("cache", C.c_int),
                ("newton_cols", C.c_int), ("work_cols", C.c_int)]


MAXREP = 128


class Report(C.Structure):
    _fields_ = [("status", C.c_int), ("steps", C.c_int), ("newton_steps", C.c_int),
                ("newton_calls", C.c_int), ("inversions", C.c_int), ("rank", C.c_int), ("nres", C.c_int),
                ("res", C.c_double * MAXREP), ("ranks", C.c_int * MAXREP), ("final_res", C.c_double),
                ("newton_ms", C.c_double), ("residual_ms", C.c_double), ("update_ms", C.c_double),
                ("total_ms", C.c_double), ("newton_flops", C.c_double)]

    def as_dict(self) -> dict:
        k = min(self.nres, MAXREP)
        return dict(status=STATUS.get(self.status, str(self.status)), steps=self.steps,
                    newton_steps=self.newton_steps, newton_calls=self.newton_calls,
                    inversions=self.inversions, rank=self.rank, res=list(self.res[:k]),
                    ranks=list(self.ranks[:k]), final_res=self.final_res, newton_ms=self.newton_ms,
                    residual_ms=self.residual_ms, update_ms=self.update_ms, total_ms=self.total_ms,
                    newton_flops=self.newton_flops)


SYMBOLS = ["lyap_ir_default_options", "lyap_ir_create", "lyap_ir_destroy", "lyap_ir_solve",
           "lyap_ir_solve_host", "lyap_invert", "lyap_newton_aseq", "lyap_newton_get_inverse",
           "lyap_newton_z", "lyap_qr", "lyap_syev", "lyap_rank_trunc_chol", "lyap_rank_trunc_ldlt",
           "lyap_res_fac_ldlt", "lyap_res_fac_chol", "lyap_sol_upt_ldlt", "lyap_sol_upt_chol",
           "lyap_launch_count", "lyap_kernel_timing", "lyap_kernel_stats", "lyap_kernel_work", "lyap_tc_gemm"]

KERNEL_CLASSES = {"gje_update": 0, "gje_panel": 1, "zside_gemm": 2, "eig": 3, "qr": 4,
                  "resid_gemm": 5, "newton_update": 6, "dgemm": 7, "tc_gemm": 8, "qr_panel": 9,
                  "tridiag": 10, "wy_apply": 11, "rrqr": 12}


def library_path() -> str:
    return _LIB_PATH


def lib():
    """Load liblyapir.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise LyapError(f"{_LIB_PATH} is missing: run __graft_entry__.build() "
                            "(there is no CPU fallback)")
        L = C.CDLL(_LIB_PATH)
        vp, ip, dp = C.c_void_p, C.POINTER(C.c_int), C.c_void_p
        L.lyap_ir_default_options.argtypes = [C.POINTER(Options)]
        L.lyap_ir_default_options.restype = None
        L.lyap_ir_create.argtypes = [C.POINTER(vp), C.c_int, C.c_int, C.c_int, C.POINTER(Options), vp]
        L.lyap_ir_destroy.argtypes = [vp]
        L.lyap_ir_solve.argtypes = [vp, dp, dp, C.c_int, dp, C.c_int, C.c_int, C.c_double, C.c_int, dp, dp, ip,
                                    C.POINTER(Report)]
        L.lyap_ir_solve_host.argtypes = L.lyap_ir_solve.argtypes
        L.lyap_invert.argtypes = [C.c_int, C.c_int, vp, vp, vp]
        L.lyap_newton_aseq.argtypes = [vp, dp, ip, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                       C.POINTER(C.c_double)]
        L.lyap_newton_get_inverse.argtypes = [vp, C.c_int, vp]
        L.lyap_newton_z.argtypes = [vp, C.c_int, dp, C.c_int, dp, dp, dp, ip]
        L.lyap_qr.argtypes = [C.c_int, C.c_int, dp, dp, dp, vp]
        L.lyap_syev.argtypes = [C.c_int, dp, dp, dp, vp]
        L.lyap_rank_trunc_chol.argtypes = [C.c_int, C.c_int, dp, C.c_double, C.c_int, dp, ip, vp]
        L.lyap_rank_trunc_ldlt.argtypes = [C.c_int, C.c_int, dp, dp, C.c_int, dp, dp, ip, vp]
        L.lyap_res_fac_ldlt.argtypes = [vp, dp, dp, C.c_int, dp, C.c_int, dp, dp, C.c_double, dp, dp, ip,
                                        C.POINTER(C.c_double)]
        L.lyap_res_fac_chol.argtypes = [vp, dp, dp, C.c_int, C.c_int, dp, C.c_double, dp, ip, dp, ip,
                                        C.POINTER(C.c_double)]
        L.lyap_sol_upt_ldlt.argtypes = [vp, C.c_int, dp, dp, C.c_int, dp, dp, C.c_double, dp, dp, ip]
        L.lyap_sol_upt_chol.argtypes = [vp, C.c_int, dp, C.c_int, dp, C.c_int, dp, C.c_double, dp, ip]
        L.lyap_launch_count.restype = C.c_int64
        L.lyap_tc_gemm.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_float, vp, C.c_long, vp, C.c_long,
                                   C.c_float, vp, C.c_long, vp]
        L.lyap_tc_gemm.restype = C.c_int
        L.lyap_kernel_timing.argtypes = [C.c_int]
        L.lyap_kernel_stats.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_int64)]
        L.lyap_kernel_work.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double)]
        for s in SYMBOLS:
            if s not in ("lyap_ir_default_options", "lyap_launch_count"):
                getattr(L, s).restype = C.c_int
        _lib = L
    return _lib


def _check(rc: int, what: str):
    if rc != 0:
        raise LyapError(f"{what}: {ERRORS.get(rc, rc)}")


def _prec(p) -> int:
    return PREC[p] if isinstance(p, str) else int(p)


def _ptr(t) -> int | None:
    if t is None:
        return None
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.is_contiguous()):
        raise LyapError("expected a contiguous CUDA tensor")
    return t.data_ptr()


def _check_f64(name, t, shape, device=None):
    """Shape / dtype / device check of a solve argument (the C ABI reads exactly this
    many elements: a smaller or mistyped buffer would be read past its end)."""
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.is_contiguous()):
        raise LyapError(f"{name}: expected a contiguous CUDA tensor")
    if t.dtype != torch.float64:
        raise LyapError(f"{name}: expected float64, got {t.dtype}")
    if tuple(t.shape) != tuple(shape):
        raise LyapError(f"{name}: expected shape {tuple(shape)}, got {tuple(t.shape)}")
    if device is not None and t.device != device:
        raise LyapError(f"{name}: on {t.device}, expected {device}")


def _stream():
    import torch
    return torch.cuda.current_stream().cuda_stream


def launch_count() -> int:
    return int(lib().lyap_launch_count())


def kernel_timing(cls):
    """Start timing one kernel class (name or id; None disables)."""
    c = -1 if cls is None else (KERNEL_CLASSES[cls] if isinstance(cls, str) else int(cls))
    lib().lyap_kernel_timing(c)


def kernel_stats():
    """(device ms, timed launches, algorithmic flops, algorithmic bytes) since kernel_timing()."""
    ms, n = C.c_double(0), C.c_int64(0)
    fl, by = C.c_double(0), C.c_double(0)
    lib().lyap_kernel_stats(C.byref(ms), C.byref(n))
    lib().lyap_kernel_work(C.byref(fl), C.byref(by))
    return ms.value, n.value, fl.value, by.value


def default_options(**kw) -> Options:
    o = Options()
    lib().lyap_ir_default_options(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


@dataclass
class Result:
    Z: "object"          # (n, rank) view of the column-major factor
    Y: "object | None"   # (rank, rank) or None (Cholesky type)
    report: dict


class Solver:
    """Handle for one equation order n and solver precision us (PAPER.md Algorithms 1-4)."""

    def __init__(self, n: int, us="fp16", max_cols: int = 256, **options):
        import torch
        if not torch.cuda.is_available():
            raise LyapError("no CUDA device: the B200 path has no CPU fallback")
        self.n, self.us, self.max_cols = n, _prec(us), max_cols
        self.opt = default_options(**options)
        self.h = C.c_void_p()
        _check(lib().lyap_ir_create(C.byref(self.h), n, max_cols, self.us, C.byref(self.opt), _stream()),
               "lyap_ir_create")

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            lib().lyap_ir_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- full IR solve (device buffers)
    def solve(self, A, Lt, S=None, tol=1e-14, maxit=50, out=None, us=None) -> Result:
        """A: (n,n) fp64 CUDA; Lt: (m,n) fp64 CUDA (= L^T); S: (m,m) fp64 CUDA or None;
        us: solver precision for this solve (None: the handle's current one)."""
        import torch
        n, cm = self.n, self.max_cols
        m = Lt.shape[0] if isinstance(Lt, torch.Tensor) and Lt.dim() == 2 else -1
        _check_f64("A", A, (n, n))
        _check_f64("Lt", Lt, (m, n), A.device)
        if S is not None:
            _check_f64("S", S, (m, m), A.device)
        if out is None:
            Zt = torch.empty((cm, n), dtype=torch.float64, device=A.device)
            Yb = torch.zeros((cm, cm), dtype=torch.float64, device=A.device) if S is not None else None
        else:
            Zt, Yb = out
        rank = C.c_int(0)
        rep = Report()
        if us is not None:
            self.us = _prec(us)
        _check(lib().lyap_ir_solve(self.h, _ptr(A), _ptr(Lt), m, _ptr(S), self.us, FP64, tol, maxit, _ptr(Zt),
                                   _ptr(Yb), C.byref(rank), C.byref(rep)), "lyap_ir_solve")
        r = rank.value
        Y = Yb[:r, :r] if Yb is not None else None      # Yb is column-major cm x cm: Y[i,j] = Yb[j,i]
        return Result(Z=Zt[:r].T, Y=(Y.T if Y is not None else None), report=rep.as_dict())

    # ---- end-to-end with host (numpy) buffers
    def solve_host(self, A, Lt, S=None, tol=1e-14, maxit=50, us=None):
        import numpy as np
        n, cm = self.n, self.max_cols
        A = np.ascontiguousarray(A, dtype=np.float64)
        Lt = np.ascontiguousarray(Lt, dtype=np.float64)
        S = None if S is None else np.ascontiguousarray(S, dtype=np.float64)
        m = Lt.shape[0] if Lt.ndim == 2 else -1
        if A.shape != (n, n) or Lt.ndim != 2 or Lt.shape[1] != n or (S is not None and S.shape != (m, m)):
            raise LyapError(f"solve_host: expected A ({n},{n}), Lt (m,{n}), S (m,m); got "
                            f"{A.shape}, {Lt.shape}, {None if S is None else S.shape}")
        Zt = np.empty((cm, n), dtype=np.float64)
        Yb = np.zeros((cm, cm), dtype=np.float64) if S is not None else None
        rank = C.c_int(0)
        rep = Report()
        p = lambda a: None if a is None else a.ctypes.data
        if us is not None:
            self.us = _prec(us)
        _check(lib().lyap_ir_solve_host(self.h, p(A), p(Lt), Lt.shape[0], p(S), self.us, FP64, tol, maxit, p(Zt),
                                        p(Yb), C.byref(rank), C.byref(rep)), "lyap_ir_solve_host")
        r = rank.value
        return Zt[:r].T, (Yb[:r, :r].T if Yb is not None else None), rep.as_dict()

    # ---- steps of the hot path
    def newton_aseq(self, A):
        k = C.c_int(0)
        km = self.opt.kmax
        mu, de, inf = (C.c_double * km)(), (C.c_double * km)(), (C.c_double * km)()
        _check(lib().lyap_newton_aseq(self.h, _ptr(A), C.byref(k), mu, de, inf), "lyap_newton_aseq")
        s = k.value
        return dict(steps=s, mu=list(mu[:s]), delta=list(de[:s]), inf=list(inf[:s]))

    def newton_inverse(self, j: int):
        import torch
        dt = {FP64: torch.float64, FP32: torch.float32, FP16: torch.float16, BF16: torch.bfloat16}[self.us]
        out = torch.empty((self.n, self.n), dtype=dt, device="cuda")
        _check(lib().lyap_newton_get_inverse(self.h, j, _ptr(out)), "lyap_newton_get_inverse")
        return out

    def newton_z(self, Lt, S=None):
        import torch
        n, cm = self.n, self.max_cols
        Zt = torch.empty((cm, n), dtype=torch.float64, device="cuda")
        Yb = torch.zeros((cm, cm), dtype=torch.float64, device="cuda")
        c = C.c_int(0)
        _check(lib().lyap_newton_z(self.h, int(S is not None), _ptr(Lt), Lt.shape[0], _ptr(S), _ptr(Zt),
                                   _ptr(Yb), C.byref(c)), "lyap_newton_z")
        r = c.value
        return Zt[:r].T, (Yb[:r, :r].T if S is not None else None)

    def res_fac_ldlt(self, A, Lt, S, Zt, Y, eta_r=1e-4):
        import torch
        n, m, c = self.n, Lt.shape[0], Zt.shape[0]
        p = 2 * c + m
        Ld = torch.empty((p, n), dtype=torch.float64, device="cuda")
        Sd = torch.zeros((p * p,), dtype=torch.float64, device="cuda")
        r, resF = C.c_int(0), C.c_double(0)
        Ycm = Y.T.contiguous()      # keep the column-major copy alive across the call
        _check(lib().lyap_res_fac_ldlt(self.h, _ptr(A), _ptr(Lt), m, _ptr(S), c, _ptr(Zt),
                                       _ptr(Ycm), eta_r, _ptr(Ld), _ptr(Sd), C.byref(r),
                                       C.byref(resF)), "lyap_res_fac_ldlt")
        k = r.value
        return Ld[:k].T, Sd[:k * k].reshape(k, k).T, resF.value

    def res_fac_chol(self, A, Lt, Zt, eta_r=1e-4):
        import torch
        n, m, c = self.n, Lt.shape[0], Zt.shape[0]
        p = 2 * c + m
        Lp = torch.empty((p, n), dtype=torch.float64, device="cuda")
        Lm = torch.empty((p, n), dtype=torch.float64, device="cuda")
        rp, rm, resF = C.c_int(0), C.c_int(0), C.c_double(0)
        _check(lib().lyap_res_fac_chol(self.h, _ptr(A), _ptr(Lt), m, c, _ptr(Zt), eta_r, _ptr(Lp),
                                       C.byref(rp), _ptr(Lm), C.byref(rm), C.byref(resF)), "lyap_res_fac_chol")
        return Lp[:rp.value].T, Lm[:rm.value].T, resF.value

    def sol_upt_ldlt(self, Zt, Y, Zdt, Yd, eta_s=None):
        import torch
        eta_s = self.opt.eta_s if eta_s is None else eta_s
        n, c, cd = self.n, Zt.shape[0], Zdt.shape[0]
        Zn = torch.empty((c + cd, n), dtype=torch.float64, device="cuda")
        Yn = torch.zeros(((c + cd) ** 2,), dtype=torch.float64, device="cuda")
        r = C.c_int(0)
        Ycm, Ydcm = Y.T.contiguous(), Yd.T.contiguous()
        _check(lib().lyap_sol_upt_ldlt(self.h, c, _ptr(Zt), _ptr(Ycm), cd, _ptr(Zdt),
                                       _ptr(Ydcm), eta_s, _ptr(Zn), _ptr(Yn), C.byref(r)),
               "lyap_sol_upt_ldlt")
        k = r.value
        return Zn[:k].T, Yn.reshape(c + cd, c + cd)[:k, :k].T

    def sol_upt_chol(self, Zt, Zpt, Zmt, eta_s=None):
        import torch
        eta_s = self.opt.eta_s if eta_s is None else eta_s
        n, c, cp, cmm = self.n, Zt.shape[0], Zpt.shape[0], Zmt.shape[0]
        Zn = torch.empty((c + cp + cmm, n), dtype=torch.float64, device="cuda")
        r = C.c_int(0)
        _check(lib().lyap_sol_upt_chol(self.h, c, _ptr(Zt), cp, _ptr(Zpt), cmm,
                                       _ptr(Zmt) if cmm else None, eta_s, _ptr(Zn), C.byref(r)),
               "lyap_sol_upt_chol")
        return Zn[:r.value].T


# ---------------------------------------------------------------- standalone steps
def invert(A, ipiv=None):
    """In-place inversion of a square row-major CUDA tensor (fp64/fp32/fp16/bf16)."""
    import torch
    dt = {torch.float64: FP64, torch.float32: FP32, torch.float16: FP16, torch.bfloat16: BF16}[A.dtype]
    _check(lib().lyap_invert(A.shape[0], dt, _ptr(A), _ptr(ipiv), _stream()), "lyap_invert")
    return A


def tc_gemm(A, B, C, alpha=1.0, beta=0.0):
    """C = alpha A B^T + beta C on the tcgen05 tensor cores (A: M x K, B: N x K, C: M x N,
    contiguous bf16/fp16 CUDA tensors of one dtype)."""
    import torch
    prec = {torch.bfloat16: BF16, torch.float16: FP16}[A.dtype]
    M, K = A.shape
    N = B.shape[0]
    _check(lib().lyap_tc_gemm(prec, M, N, K, alpha, _ptr(A), K, _ptr(B), K, beta, _ptr(C), N, _stream()),
           "lyap_tc_gemm")
    return C


def qr(At):
    """Thin Householder QR of the column-major matrix A = At.T (At: (n, m) fp64 CUDA).
    Returns (Qt, Rt) with Q = Qt.T (m x k), R = Rt.T (k x n)."""
    import torch
    n, m = At.shape
    k = min(m, n)
    Qt = torch.empty((k, m), dtype=torch.float64, device="cuda")
    Rt = torch.empty((n, k), dtype=torch.float64, device="cuda")
    _check(lib().lyap_qr(m, n, _ptr(At), _ptr(Qt), _ptr(Rt), _stream()), "lyap_qr")
    return Qt, Rt


def syev(A):
    """Symmetric eigendecomposition (A symmetric (n,n) fp64 CUDA). Returns (w desc, V) with V[:, j]."""
    import torch
    n = A.shape[0]
    w = torch.empty(n, dtype=torch.float64, device="cuda")
    Vt = torch.empty((n, n), dtype=torch.float64, device="cuda")
    _check(lib().lyap_syev(n, _ptr(A), _ptr(w), _ptr(Vt), _stream()), "lyap_syev")
    return w, Vt.T


def rank_trunc_chol(Zt, tol, prec="fp64"):
    import torch
    c, n = Zt.shape
    out = torch.zeros((c, n), dtype=torch.float64, device="cuda")
    k = C.c_int(0)
    _check(lib().lyap_rank_trunc_chol(n, c, _ptr(Zt), tol, _prec(prec), _ptr(out), C.byref(k), _stream()),
           "lyap_rank_trunc_chol")
    return out[:k.value].T


def rank_trunc_ldlt(Zt, Y, prec="fp64"):
    import torch
    c, n = Zt.shape
    Zo = torch.zeros((c, n), dtype=torch.float64, device="cuda")
    Yo = torch.zeros((c * c,), dtype=torch.float64, device="cuda")
    k = C.c_int(0)
    Ycm = Y.T.contiguous()
    _check(lib().lyap_rank_trunc_ldlt(n, c, _ptr(Zt), _ptr(Ycm), _prec(prec), _ptr(Zo), _ptr(Yo),
                                      C.byref(k), _stream()), "lyap_rank_trunc_ldlt")
    r = k.value
    return Zo[:r].T, Yo[:r * r].reshape(r, r).T
