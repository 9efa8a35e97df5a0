"""Warm timing of the eigensolver phases at several orders (LYAP_PROFILE_EIG=1 prints them)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_02126_b200 as G
for p in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "100,200,400,500,900").split(",")]:
    B = torch.randn(p, p, dtype=torch.float64, device="cuda"); B = B + B.T
    for _ in range(3):
        G.syev(B)
    torch.cuda.synchronize()
