"""configs[3]: fp32 solve then fp16 solve in one process (the test_cfg3_full_size order)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_02126_b200 as G
import problems as P
p = P.cfg3()
A = torch.as_tensor(p.A, device="cuda"); Lt = torch.as_tensor(np.ascontiguousarray(p.L.T), device="cuda")
order = sys.argv[1].split(",") if len(sys.argv) > 1 else ["fp32", "fp16"]
caps = {"fp32": dict(max_cols=6144, newton_cols=14336, work_cols=16384),
        "fp16": dict(max_cols=4096, newton_cols=8192, work_cols=10240)}
for us in order:
    s = G.Solver(p.n, us=us, **caps[us])
    r = s.solve(A, Lt, None, tol=1e-14, maxit=10)
    print(us, {k: v for k, v in r.report.items() if k in ("status", "steps", "res", "total_ms")}, flush=True)
    if os.environ.get("RESID"):
        X = r.Z @ r.Z.T
        W = Lt.T @ Lt
        R = A @ X + X @ A.T + W
        print("explicit", (torch.linalg.norm(R) / (torch.linalg.norm(W) + 2 * torch.linalg.norm(X) * torch.linalg.norm(A))).item(), flush=True)
        del X, W, R
    del s, r
