"""One fp64 symmetric eigendecomposition of order p (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_02126_b200 as G
p = int(sys.argv[1]) if len(sys.argv) > 1 else 900
B = torch.randn(p, p, dtype=torch.float64, device="cuda"); B = B + B.T
G.syev(B); torch.cuda.synchronize()
