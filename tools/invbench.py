"""Time the u_s inversion (blocked Gauss-Jordan) and the tcgen05 GEMM at large n."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_02126_b200 as G
ns = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1024,4096").split(",")]
dt = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32}[sys.argv[2] if len(sys.argv) > 2 else "bf16"]
for n in ns:
    g = torch.Generator(device="cuda").manual_seed(n)
    A0 = (torch.randn(n, n, device="cuda", generator=g) / n ** 0.5 - 2 * torch.eye(n, device="cuda")).to(dt)
    for _ in range(2):                                   # warm-up (clocks ramp from idle)
        A = A0.clone(); G.invert(A)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        A.copy_(A0); G.invert(A)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    res = (A0.double() @ A.double() - torch.eye(n, device="cuda", dtype=torch.float64)).norm() / n ** 0.5
    print(f"invert n={n} {dt}: {ms:8.2f} ms  {2 * n ** 3 / ms / 1e9:8.2f} TFLOP/s (2n^3)  resid {res:.2e}")
    for cls in ("gje_panel", "gje_update", "tc_gemm", "dgemm"):
        G.kernel_timing(cls); A.copy_(A0); G.invert(A); t, c = G.kernel_stats()[:2]
        print(f"   {cls:10s} {t:8.2f} ms {c:6d} launches")
    G.kernel_timing(None)
    if dt == torch.float32:
        continue
    for K in (32, 256):
        X = torch.randn(n, K, device="cuda").to(dt); B = torch.randn(n, K, device="cuda").to(dt)
        C = torch.zeros(n, n, device="cuda", dtype=dt)
        G.tc_gemm(X, B, C); torch.cuda.synchronize()
        e0.record()
        for _ in range(10):
            G.tc_gemm(X, B, C, 1.0, 1.0)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        ref = (X.float() @ B.float().T)
        print(f"   tc_gemm M=N={n} K={K}: {ms * 1e3:8.1f} us  {2 * n * n * K / ms / 1e9:7.1f} TFLOP/s  "
              f"{(4 * n * n) / ms / 1e6:7.1f} GB/s(C rw)")
