"""fp16 sign-Newton A-sequence at order n: total device time and per-class kernel times
(each class timed in its own repetition).  usage: python tools/aseq_breakdown.py 16384[,4096] [us]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_02126_b200 as G
us = sys.argv[2] if len(sys.argv) > 2 else "fp16"
for n in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "4096").split(",")]:
    g = torch.Generator(device="cuda").manual_seed(n)
    Q, _ = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g))
    lam = torch.logspace(0, 2, n, dtype=torch.float64, device="cuda")
    A = -(Q * lam[None, :]) @ Q.T
    del Q
    s = G.Solver(n, us=us, max_cols=64)
    out = s.newton_aseq(A)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(2):
        out = s.newton_aseq(A)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 2
    k = out["steps"]
    print(f"n={n} {us}: A-sequence {ms:8.2f} ms, {k} inversions, {ms / k:7.2f} ms/inversion, "
          f"{k * 2 * n ** 3 / (ms / 1e3) / 1e12:7.2f} TFLOP/s", flush=True)
    for name in ["gje_panel", "gje_update", "tc_gemm", "newton_update"]:
        G.kernel_timing(name)
        s.newton_aseq(A)
        torch.cuda.synchronize()
        t, c, fl, by = G.kernel_stats()
        print(f"  {name:14s} {t:9.2f} ms {c:6d} launches  {fl / max(t, 1e-9) / 1e9:8.1f} TFLOP/s "
              f"{by / max(t, 1e-9) / 1e6:8.1f} GB/s", flush=True)
    G.kernel_timing(None)
    del s, A
    torch.cuda.empty_cache()
