"""Determinism check: the same equation solved repeatedly (sequentially on one handle,
then concurrently on several handles/streams) must give bitwise identical reports."""
import os, sys, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_02126_b200 as G
import problems as P
name = sys.argv[1] if len(sys.argv) > 1 else "cfg4:128"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
p = P.cfg4_member(int(name.split(":")[1])) if name.startswith("cfg4") else getattr(P, name)()
A = torch.tensor(p.A, dtype=torch.float64, device="cuda")
Lt = torch.tensor(np.ascontiguousarray(p.L.T), dtype=torch.float64, device="cuda")
S = torch.tensor(p.S, dtype=torch.float64, device="cuda") if p.S is not None else None
us = p.us if not name.startswith("cfg1") else "bf16"
mc = 1536 if name.startswith("cfg4") else 640
sig = lambda r: (r.report["steps"], r.report["rank"], tuple(r.report["ranks"]), r.report["final_res"])
s0 = G.Solver(p.n, us=us, max_cols=mc)
seq = [sig(s0.solve(A, Lt, S, tol=1e-14, maxit=30)) for _ in range(reps)]
print("sequential identical:", all(x == seq[0] for x in seq), seq[0][:2], seq[0][3])
for x in seq[1:]:
    if x != seq[0]: print("  differs:", x[:2], x[3])
streams = [torch.cuda.Stream() for _ in range(3)]
handles = []
for st in streams:
    with torch.cuda.stream(st):
        handles.append(G.Solver(p.n, us=us, max_cols=mc))
out = [None] * 3
def run(k):
    with torch.cuda.stream(streams[k]):
        out[k] = sig(handles[k].solve(A, Lt, S, tol=1e-14, maxit=30))
th = [threading.Thread(target=run, args=(k,)) for k in range(3)]
[t.start() for t in th]; [t.join() for t in th]
print("concurrent identical to sequential:", all(x == seq[0] for x in out))
for x in out:
    if x != seq[0]: print("  differs:", x[:2], x[3])
# same handle, sequential solves, while another stream keeps the GPU busy with GEMMs
stop = [False]
def noise():
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        x = torch.randn(4096, 4096, device="cuda")
        while not stop[0]:
            for _ in range(20):
                x = (x @ x).clamp_(-1, 1)
            st.synchronize()
t = threading.Thread(target=noise); t.start()
busy = [sig(s0.solve(A, Lt, S, tol=1e-14, maxit=30)) for _ in range(2)]
stop[0] = True; t.join()
print("sequential under GPU noise identical:", all(x == seq[0] for x in busy))
for x in busy:
    if x != seq[0]: print("  differs:", x[:2], x[3])
