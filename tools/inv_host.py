"""Host-side cost of one inversion: wall time to enqueue vs device time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_02126_b200 as G
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
A0 = (torch.randn(n, n, device="cuda") / n ** 0.5 - 2 * torch.eye(n, device="cuda")).to(torch.bfloat16)
A = A0.clone(); G.invert(A); torch.cuda.synchronize()
s = G.Solver(n, us="bf16", max_cols=64)
for it in range(2):
    A.copy_(A0); torch.cuda.synchronize()
    t0 = time.perf_counter(); G.invert(A); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"lyap_invert n={n}: call {1e3*(t1-t0):.1f} ms, sync {1e3*(t2-t1):.1f} ms")
from torch.profiler import profile, ProfilerActivity
A.copy_(A0); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    G.invert(A); torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
ev.sort(key=lambda e: e.time_range.start)
busy = sum(e.time_range.end - e.time_range.start for e in ev)
span = ev[-1].time_range.end - ev[0].time_range.start
print(f"device span {span/1e3:.1f} ms, busy {busy/1e3:.1f} ms over {len(ev)} device events")
gaps = sorted(((ev[i+1].time_range.start - ev[i].time_range.end), ev[i].name[:40], ev[i+1].name[:40]) for i in range(len(ev)-1))[::-1][:8]
for g in gaps: print(f"  gap {g[0]:.0f} us after {g[1]} before {g[2]}")
