"""One u_s inversion at size n (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_02126_b200 as G
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
A = (torch.randn(n, n, device="cuda") / n ** 0.5 - 2 * torch.eye(n, device="cuda")).to(torch.bfloat16)
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1      # >1: the first inversion warms up
for _ in range(reps):
    X = A.clone()
    G.invert(X)
torch.cuda.synchronize()
