"""Solve one configuration on the GPU (verbose library log), report time and residual.
usage: python tools/explore_cfg.py <cfg> <us> <max_cols> [maxit]"""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_02126_b200 as G
import problems as P
name, us, mc = sys.argv[1], sys.argv[2], int(sys.argv[3])
maxit = int(sys.argv[4]) if len(sys.argv) > 4 else 30
t0 = time.time()
p = P.cfg4_member(int(name.split(":")[1])) if name.startswith("cfg4") else getattr(P, name)()
print(f"generated {name} n={p.n} m={p.m} in {time.time() - t0:.1f} s", flush=True)
A = torch.tensor(p.A, dtype=torch.float64, device="cuda")
Lt = torch.tensor(np.ascontiguousarray(p.L.T), dtype=torch.float64, device="cuda")
S = torch.tensor(p.S, dtype=torch.float64, device="cuda") if p.S is not None else None
s = G.Solver(p.n, us=us, max_cols=mc, newton_cols=int(os.environ.get("NEWTON_COLS", "0")),
             work_cols=int(os.environ.get("WORK_COLS", "0")))
for rep in range(int(os.environ.get("REPS", "1"))):
    torch.cuda.synchronize(); t = time.time()
    r = s.solve(A, Lt, S, tol=1e-14, maxit=maxit)
    torch.cuda.synchronize()
    wall = time.time() - t
    print(json.dumps(dict(cfg=name, us=us, wall=wall, **{k: v for k, v in r.report.items()})), flush=True)
    if os.environ.get("CHECK"):
        # explicit fp64 residual of Eq. res-fac-sol on the device (test-side check)
        Z = r.Z
        X = Z @ (r.Y @ Z.T if r.Y is not None else Z.T)
        W = Lt.T @ (S @ Lt if S is not None else Lt)
        R = A @ X + X @ A.T + W
        rel = (torch.linalg.norm(R) / (torch.linalg.norm(W) + 2 * torch.linalg.norm(X) * torch.linalg.norm(A))).item()
        print(f"explicit relative residual {rel:.3e}", flush=True)
        del X, W, R
