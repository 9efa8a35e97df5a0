"""Solve one equation of a configuration on the GPU and print the report.
usage: python tools/solve_cfg.py cfg2|cfg3|cfg4:<index> [us] [max_cols] [tol]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_02126_b200 as G
import problems as P
name = sys.argv[1] if len(sys.argv) > 1 else "cfg4:0"
t0 = time.time()
if name.startswith("cfg4"):
    p = P.cfg4_member(int(name.split(":")[1]) if ":" in name else 0)
else:
    p = getattr(P, name)()
print(f"generated {name} n={p.n} m={p.m} in {time.time() - t0:.1f} s", flush=True)
us = sys.argv[2] if len(sys.argv) > 2 else p.us
mc = int(sys.argv[3]) if len(sys.argv) > 3 else 512
tol = float(sys.argv[4]) if len(sys.argv) > 4 else 1e-14
A = torch.tensor(p.A, dtype=torch.float64, device="cuda")
Lt = torch.tensor(np.ascontiguousarray(p.L.T), dtype=torch.float64, device="cuda")
S = torch.tensor(p.S, dtype=torch.float64, device="cuda") if p.S is not None else None
s = G.Solver(p.n, us=us, max_cols=mc)
for rep in range(2):
    torch.cuda.synchronize(); t = time.time()
    r = s.solve(A, Lt, S, tol=tol, maxit=30)
    torch.cuda.synchronize()
    print(f"{name} {us}: wall {time.time() - t:.3f} s", {k: v for k, v in r.report.items() if k != "res"}, flush=True)
