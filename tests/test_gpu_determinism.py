"""Bitwise reproducibility of the CUDA path (-m gpu).

Every reduction in the library has a fixed order, so a result that changes when the GPU
is shared with other work (or when several solver handles run concurrently on different
streams) means a race inside a kernel.  This caught a double-buffering bug in the
cooperative tridiagonalisation (a fast CTA overwrote the P vector that a slower CTA was
still reading)."""
import threading

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


class _Noise:
    """Keeps the GPU busy with GEMMs on another stream."""

    def __enter__(self):
        self.stop = False
        self.t = threading.Thread(target=self._run)
        self.t.start()
        return self

    def _run(self):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            x = torch.randn(2048, 2048, device="cuda")
            while not self.stop:
                for _ in range(8):
                    x = (x @ x).clamp_(-1, 1)
                st.synchronize()

    def __exit__(self, *exc):
        self.stop = True
        self.t.join()


def _cases(G):
    g = torch.Generator(device="cuda").manual_seed(11)
    B = torch.randn(700, 700, dtype=torch.float64, device="cuda", generator=g)
    B = B + B.T
    Aq = torch.randn(600, 800, dtype=torch.float64, device="cuda", generator=g)
    M = (torch.randn(1024, 1024, device="cuda", generator=g) / 32 - 2 * torch.eye(1024, device="cuda")).to(torch.bfloat16)
    Z = torch.randn(200, 700, dtype=torch.float64, device="cuda", generator=g)

    M2 = (torch.randn(2048, 2048, device="cuda", generator=g) / 45 - 2 * torch.eye(2048, device="cuda")).to(torch.float16)

    def inv():
        X = M.clone()
        G.invert(X)
        return X.float().flatten()

    def inv2():          # n = 2048: implicit pivoting with the look-ahead stream and dependent launches
        X = M2.clone()
        G.invert(X)
        return X.float().flatten()
    return {
        "syev": lambda: torch.cat([t.flatten() for t in G.syev(B)]),
        "qr": lambda: torch.cat([t.flatten() for t in G.qr(Aq)]),
        "invert": inv,
        "invert_lookahead": inv2,
        "rank_trunc_chol": lambda: G.rank_trunc_chol(Z, 2 ** -6, "fp64").flatten(),
    }


def test_primitives_bitwise_reproducible_under_gpu_load(gpu):
    cases = _cases(gpu)
    base = {k: f() for k, f in cases.items()}
    torch.cuda.synchronize()
    with _Noise():
        for _ in range(3):
            for k, f in cases.items():
                out = f()
                torch.cuda.synchronize()
                assert torch.equal(out, base[k]), k


def test_concurrent_handles_match_sequential(gpu):
    p = P.cfg0()
    A = torch.tensor(p.A, dtype=torch.float64, device="cuda")
    Lt = torch.tensor(np.ascontiguousarray(p.L.T), dtype=torch.float64, device="cuda")
    sig = lambda r: (r.report["steps"], r.report["rank"], r.report["final_res"])
    ref = sig(gpu.Solver(p.n, us="fp16", max_cols=128).solve(A, Lt, None, tol=1e-14, maxit=10))
    streams = [torch.cuda.Stream() for _ in range(3)]
    handles = []
    for st in streams:
        with torch.cuda.stream(st):
            handles.append(gpu.Solver(p.n, us="fp16", max_cols=128))
    out = [None] * 3

    def run(k):
        with torch.cuda.stream(streams[k]):
            out[k] = sig(handles[k].solve(A, Lt, None, tol=1e-14, maxit=10))
    th = [threading.Thread(target=run, args=(k,)) for k in range(3)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert all(o == ref for o in out)
