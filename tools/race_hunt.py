"""Bitwise reproducibility of each GPU primitive while another stream keeps the GPU busy
(a timing-dependent result means a race inside a kernel)."""
import os, sys, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_02126_b200 as G
torch.manual_seed(0)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cases = {}
A900 = torch.randn(900, 1024, dtype=torch.float64, device="cuda")          # column-major 1024 x 900
cases["qr 1024x900"] = lambda: torch.cat([t.flatten() for t in G.qr(A900)])
B = torch.randn(900, 900, dtype=torch.float64, device="cuda"); B = B + B.T
cases["syev 900"] = lambda: torch.cat([t.flatten() for t in G.syev(B)])
B2 = torch.randn(300, 300, dtype=torch.float64, device="cuda"); B2 = B2 + B2.T
cases["syev 300"] = lambda: torch.cat([t.flatten() for t in G.syev(B2)])
M0 = (torch.randn(1024, 1024, device="cuda") / 32 - 2 * torch.eye(1024, device="cuda")).to(torch.bfloat16)
def inv():
    X = M0.clone(); G.invert(X); return X.float().flatten()
cases["invert bf16 1024"] = inv
M1 = (torch.randn(300, 300, dtype=torch.float64, device="cuda") + 20 * torch.eye(300, dtype=torch.float64, device="cuda"))
def inv64():
    X = M1.clone(); G.invert(X); return X.flatten()
cases["invert fp64 300"] = inv64
Z = torch.randn(300, 1024, dtype=torch.float64, device="cuda")   # column-major 1024 x 300 (rank-deficient tail below)
Z[200:] = Z[:100] * 0.5 + 1e-9 * torch.randn(100, 1024, dtype=torch.float64, device="cuda")
cases["rank_trunc_chol 1024x300"] = lambda: G.rank_trunc_chol(Z, 2 ** -6, "fp64").flatten()
base = {k: f() for k, f in cases.items()}
torch.cuda.synchronize()
stop = [False]
def noise():
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        x = torch.randn(4096, 4096, device="cuda")
        while not stop[0]:
            for _ in range(10):
                x = (x @ x).clamp_(-1, 1)
            st.synchronize()
t = threading.Thread(target=noise); t.start()
try:
    for k, f in cases.items():
        bad = 0
        for _ in range(reps):
            o = f(); torch.cuda.synchronize()
            if o.shape != base[k].shape or not torch.equal(o, base[k]):
                bad += 1
                d = (o - base[k]).abs().max().item() if o.shape == base[k].shape else float("nan")
        print(f"{k:28s} {'OK' if bad == 0 else f'DIFFERS in {bad}/{reps} (max abs diff {d:.3e})'}", flush=True)
finally:
    stop[0] = True; t.join()
