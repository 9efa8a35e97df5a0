"""R-TC table: IR outcomes of the GPU path, the oracle's chop model (every
operation rounded to u_s, the paper's simulation l.1400-1401) and its tc model (u_s
operands/results, fp32 accumulation), and each against a model-independent fp64
solution (scipy Bartels-Stewart).  usage: python tools/rtc_table.py [--no-gpu] [cases]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scipy.linalg as sla
import oracle
import problems as P

CASES = {
    "cfg0_fp16": (lambda: P.cfg0(), "fp16", False, 10),
    "cfg0_bf16": (lambda: P.cfg0(), "bf16", False, 10),
    "ldlt96_fp16": (lambda: P.cfg1(seed=5, n=96, m=3), "fp16", True, 20),
    "ldlt96_bf16": (lambda: P.cfg1(seed=5, n=96, m=3), "bf16", True, 20),
    "cfg1_bf16": (lambda: P.cfg1(), "bf16", True, 30),
}


def X_of(Z, Y):
    return Z @ Z.T if Y is None else Z @ Y @ Z.T


def rel(X, Xr):
    return float(np.linalg.norm(X - Xr) / np.linalg.norm(Xr))


def main():
    gpu = "--no-gpu" not in sys.argv
    names = [a for a in sys.argv[1:] if not a.startswith("--")] or list(CASES)
    oracle.lib()
    if gpu:
        import torch
        import paper_2510_02126_b200 as G
    for name in names:
        gen, us, ldlt, imax = CASES[name]
        p = gen()
        W = p.W()
        Xbs = sla.solve_continuous_lyapunov(p.A, -W)
        row = dict(case=name, n=p.n, us=us)
        outs = {}
        for mdl in ("chop", "tc"):
            t = time.time()
            with oracle.model(mdl):
                r = (oracle.ir_ldlt(p.A, p.L, p.S, us=us, tol=1e-14, imax=imax) if ldlt
                     else oracle.ir_chol(p.A, p.L, us=us, tol=1e-14, imax=imax))
            X = X_of(r.Z, r.Y if ldlt else None)
            outs[mdl] = X
            row[mdl] = dict(steps=r.steps, status=r.status, newton=f"{r.newton_total}({r.newton_max})",
                            final_res=r.final_res, err_vs_bs=rel(X, Xbs), cpu_s=round(time.time() - t, 1))
        row["chop_vs_tc"] = rel(outs["chop"], outs["tc"])
        if gpu:
            s = G.Solver(p.n, us=us, max_cols=640)
            c = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
            res = s.solve(c(p.A), c(p.L.T), c(p.S) if ldlt else None, tol=1e-14, maxit=imax)
            Z = res.Z.cpu().numpy()
            Y = res.Y.cpu().numpy() if ldlt else None
            X = X_of(Z, Y)
            rp = res.report
            row["gpu"] = dict(steps=rp["steps"], status=rp["status"], newton_max=rp["newton_steps"],
                              final_res=rp["final_res"], err_vs_tc=rel(X, outs["tc"]),
                              err_vs_chop=rel(X, outs["chop"]), err_vs_bs=rel(X, Xbs),
                              explicit_res=oracle.rel_residual_explicit(p.A, X, W))
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
