"""Per-repetition times of the u_s inversion at size n (spread / outliers)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_02126_b200 as G
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 12
g = torch.Generator(device="cuda").manual_seed(n)
A0 = (torch.randn(n, n, device="cuda", generator=g) / n ** 0.5 - 2 * torch.eye(n, device="cuda")).to(torch.bfloat16)
ts = []
for r in range(reps):
    A = A0.clone()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(); G.invert(A); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"n={n} per-rep ms: " + " ".join(f"{t:.1f}" for t in ts))
