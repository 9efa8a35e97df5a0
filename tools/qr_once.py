"""One thin QR of an m x n fp64 matrix (for ncu captures of the QR kernels)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_02126_b200 as G
m = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1100
At = torch.randn((n, m), dtype=torch.float64, device="cuda")
for _ in range(2):
    G.qr(At)
torch.cuda.synchronize()
