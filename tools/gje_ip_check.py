"""Implicit-pivoting Gauss-Jordan sweep (gje_ip.cu) against the row-swapping sweep (gje.cu):
same pivots and bitwise equal inverses expected; then timings of both."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_02126_b200 as G

def mat(n, dt):
    g = torch.Generator(device="cuda").manual_seed(n)
    return (torch.randn(n, n, device="cuda", generator=g) / n ** 0.5 - 2 * torch.eye(n, device="cuda")).to(dt)

def run(A0, swap):
    if swap: os.environ["LYAP_GJE_SWAP"] = "1"
    else: os.environ.pop("LYAP_GJE_SWAP", None)
    A = A0.clone(); ip = torch.zeros(A.shape[0], dtype=torch.int32, device="cuda")
    G.invert(A, ip); torch.cuda.synchronize()
    return A, ip

def timeit(A0, swap, reps=3):
    if swap: os.environ["LYAP_GJE_SWAP"] = "1"
    else: os.environ.pop("LYAP_GJE_SWAP", None)
    A = A0.clone(); G.invert(A); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        A.copy_(A0); G.invert(A)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

ns = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1024,2048,4096").split(",")]
dts = (sys.argv[2] if len(sys.argv) > 2 else "fp16,bf16,fp32").split(",")
DT = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32}
for n in ns:
    for d in dts:
        A0 = mat(n, DT[d])
        X1, p1 = run(A0, False)
        X2, p2 = run(A0, True)
        same = torch.equal(X1, X2)
        diff = (X1.double() - X2.double()).norm() / X2.double().norm()
        res = (A0.double() @ X1.double() - torch.eye(n, device="cuda", dtype=torch.float64)).norm() / n ** 0.5
        print(f"n={n} {d}: pivots equal {torch.equal(p1, p2)}  bitwise equal {same}  rel diff {diff:.2e}  resid {res:.2e}", flush=True)
        if "time" in sys.argv:
            t1 = timeit(A0, False); t2 = timeit(A0, True)
            print(f"   implicit {t1:8.2f} ms ({2 * n ** 3 / t1 / 1e9:7.1f} TFLOP/s)   swapping {t2:8.2f} ms", flush=True)
            os.environ.pop("LYAP_GJE_SWAP", None)
            for cls in ("gje_panel", "gje_update"):
                G.kernel_timing(cls); A = A0.clone(); G.invert(A); t, c = G.kernel_stats()[:2]
                print(f"   {cls:10s} {t:8.2f} ms {c:6d} launches")
            G.kernel_timing(None)
