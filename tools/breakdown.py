"""Kernel-class time breakdown of one solve (each class timed in a separate solve).
usage: python tools/breakdown.py <cfg0..cfg3|cfg4:i> [us] [max_cols] [classes,...]"""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_02126_b200 as G
import problems as P
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
p = P.cfg4_member(int(cfg.split(":")[1])) if cfg.startswith("cfg4") else getattr(P, cfg)()
us = sys.argv[2] if len(sys.argv) > 2 else p.us
mc = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
classes = sys.argv[4].split(",") if len(sys.argv) > 4 else list(G.KERNEL_CLASSES)
A = torch.tensor(p.A, dtype=torch.float64, device="cuda")
Lt = torch.tensor(np.ascontiguousarray(p.L.T), dtype=torch.float64, device="cuda")
S = torch.tensor(p.S, dtype=torch.float64, device="cuda") if p.S is not None else None
s = G.Solver(p.n, us=us, max_cols=mc, newton_cols=int(os.environ.get("NEWTON_COLS", "0")),
             work_cols=int(os.environ.get("WORK_COLS", "0")))
t = time.time(); r = s.solve(A, Lt, S, tol=1e-14, maxit=30); torch.cuda.synchronize()
print(f"{cfg} {us} solve wall %.3f s" % (time.time() - t), json.dumps({k: v for k, v in r.report.items()}), flush=True)
for name in classes:
    G.kernel_timing(name); s.solve(A, Lt, S, tol=1e-14, maxit=30); ms, c, fl, by = G.kernel_stats()
    print(f"{name:14s} {ms:10.2f} ms  {c:6d} launches  {fl/max(ms,1e-9)/1e9:8.2f} TFLOP/s  {by/max(ms,1e-9)/1e6:8.1f} GB/s", flush=True)
G.kernel_timing(None)
