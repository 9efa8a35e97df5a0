"""Kernel-class time breakdown of one solve (each class timed in a separate solve)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_02126_b200 as G
import problems as P
from bench import WORKLOADS
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
if cfg.startswith("cfg4"):                      # cfg4:<index> -- one member of the batched config
    p = P.cfg4_member(int(cfg.split(":")[1]) if ":" in cfg else 0)
    wl = dict(us="fp16", tol=1e-14, maxit=30, max_cols=1536)
else:
    wl = dict(WORKLOADS[cfg])
    p = getattr(P, wl["gen"])()
if len(sys.argv) > 3:
    wl["us"] = sys.argv[3]                      # solver precision override (e.g. cfg2 fp32)
mc = int(sys.argv[2]) if len(sys.argv) > 2 else wl["max_cols"]
A = torch.tensor(p.A, dtype=torch.float64, device="cuda")
Lt = torch.tensor(np.ascontiguousarray(p.L.T), dtype=torch.float64, device="cuda")
S = torch.tensor(p.S, dtype=torch.float64, device="cuda") if p.S is not None else None
s = G.Solver(p.n, us=wl["us"], max_cols=mc)
t = time.time(); r = s.solve(A, Lt, S, tol=wl["tol"], maxit=wl["maxit"]); torch.cuda.synchronize()
print("solve wall %.3f s" % (time.time() - t), {k: v for k, v in r.report.items() if k not in ("res",)})
for name in G.KERNEL_CLASSES:
    G.kernel_timing(name); s.solve(A, Lt, S, tol=wl["tol"], maxit=wl["maxit"]); ms, c = G.kernel_stats()[:2]
    print(f"{name:14s} {ms:10.2f} ms  {c:6d} launches")
G.kernel_timing(None)
