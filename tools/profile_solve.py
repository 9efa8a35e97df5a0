"""One warm-up solve + one solve of a bench workload (for ncu launch lists / captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_02126_b200 as G  # noqa: E402
import problems as P  # noqa: E402
from bench import WORKLOADS  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
wl = WORKLOADS[cfg]
p = getattr(P, wl["gen"])()
A = torch.tensor(p.A, dtype=torch.float64, device="cuda")
Lt = torch.tensor(np.ascontiguousarray(p.L.T), dtype=torch.float64, device="cuda")
S = torch.tensor(p.S, dtype=torch.float64, device="cuda") if p.S is not None else None
s = G.Solver(p.n, us=wl["us"], max_cols=wl["max_cols"])
n0 = G.launch_count()
r = s.solve(A, Lt, S, tol=wl["tol"], maxit=wl["maxit"])
n1 = G.launch_count()
r = s.solve(A, Lt, S, tol=wl["tol"], maxit=wl["maxit"])
torch.cuda.synchronize()
print("launches per solve:", n1 - n0, G.launch_count() - n1, r.report)
