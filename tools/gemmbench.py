import os, sys, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, paper_2510_02126_b200 as G
# exercise the fp64 GEMM through lyap_qr (trailing updates) and syev; direct timing of QR
for (m, n) in [(1024, 256), (1024, 1024), (4096, 512)]:
    A = torch.randn(n, m, dtype=torch.float64, device="cuda")
    G.qr(A); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3): G.qr(A)
    torch.cuda.synchronize(); print("qr", m, n, "ms", (time.perf_counter() - t) / 3 * 1e3)
    Qt, Rt = G.qr(A)
    Q, R = Qt.T, Rt.T
    print("   err", (torch.linalg.norm(Q @ R - A.T) / torch.linalg.norm(A)).item(), (torch.linalg.norm(Q.T @ Q - torch.eye(Q.shape[1], device='cuda', dtype=torch.float64))).item())
