"""GPU busy vs idle during one configs[1] solve (torch profiler, CUPTI activity)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_02126_b200 as G
import problems as P
from bench import WORKLOADS
wl = WORKLOADS["cfg1"]
p = P.cfg1()
A = torch.tensor(p.A, dtype=torch.float64, device="cuda")
Lt = torch.tensor(np.ascontiguousarray(p.L.T), dtype=torch.float64, device="cuda")
S = torch.tensor(p.S, dtype=torch.float64, device="cuda")
s = G.Solver(p.n, us=wl["us"], max_cols=wl["max_cols"])
s.solve(A, Lt, S, tol=wl["tol"], maxit=wl["maxit"]); torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    s.solve(A, Lt, S, tol=wl["tol"], maxit=wl["maxit"]); torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
busy, last_end, gaps = 0.0, None, []
for e in ev:
    st, en = e.time_range.start, e.time_range.end
    if last_end is not None and st > last_end:
        gaps.append(st - last_end)
    busy += max(0.0, en - max(st, last_end if last_end is not None else st))
    last_end = en if last_end is None else max(last_end, en)
span = ev[-1].time_range.end - ev[0].time_range.start
gaps.sort(reverse=True)
print(f"span {span / 1e3:.1f} ms, busy {busy / 1e3:.1f} ms, idle {100 * (1 - busy / span):.1f} %, {len(ev)} device ops")
print(f"gaps > 20 us: {sum(1 for g in gaps if g > 20)} totalling {sum(g for g in gaps if g > 20) / 1e3:.1f} ms; "
      f"gaps <= 20 us total {sum(g for g in gaps if g <= 20) / 1e3:.1f} ms")
