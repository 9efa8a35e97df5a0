"""Time the fp64 Householder QR and the eigensolver alone at IR-sized shapes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_02126_b200 as G
m = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
n = int(sys.argv[2]) if len(sys.argv) > 2 else 900
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
A = torch.randn(n, m, dtype=torch.float64, device="cuda")   # column-major m x n
for _ in range(2):
    G.qr(A)
torch.cuda.synchronize()
for cls in ("qr", "qr_panel", "wy_apply"):
    G.kernel_timing(cls)
    for _ in range(reps):
        G.qr(A)
    ms, c = G.kernel_stats()[:2]
    print(f"qr {m}x{n}: {cls:10s} {ms / reps:8.3f} ms/call  {c // reps} launches/call")
G.kernel_timing(None)
B = torch.randn(n, n, dtype=torch.float64, device="cuda"); B = B + B.T
G.syev(B)
for cls in ("eig", "tridiag", "wy_apply", "dgemm"):
    G.kernel_timing(cls)
    for _ in range(reps):
        G.syev(B)
    ms, c = G.kernel_stats()[:2]
    print(f"syev {n}: {cls:10s} {ms / reps:8.3f} ms/call  {c // reps} launches/call")
G.kernel_timing(None)
