"""Run the fp16 sign-Newton A-sequence once at configs[3]'s n = 16384 (ncu target for the
Newton update kernel: `ncu -k regex:newton_update_row -c 1 --set full python tools/nu_probe.py`)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402
import paper_2510_02126_b200 as G  # noqa: E402
import problems as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
p = P.cfg3() if n == 16384 else P.cfg2()
A = torch.tensor(p.A, dtype=torch.float64, device="cuda")
s = G.Solver(A.shape[0], us="fp16", max_cols=64)
out = s.newton_aseq(A)
torch.cuda.synchronize()
print("steps", out["steps"])
for name in ("newton_update", "gje_panel", "tc_gemm"):
    G.kernel_timing(name)
    s.newton_aseq(A)
    ms, cnt, fl, by = G.kernel_stats()
    G.kernel_timing(None)
    extra = f" {by / (ms / 1e3) / 1e9:.0f} GB/s algorithmic" if by else ""
    print(f"{name}: {cnt} launches {ms:.3f} ms{extra}")
