"""Time RankTruncChol (column-pivoted QR of Z^T) at IR-like sizes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_02126_b200 as G
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
c = int(sys.argv[2]) if len(sys.argv) > 2 else 1400
r = int(sys.argv[3]) if len(sys.argv) > 3 else 400          # numerical rank of the test factor
g = torch.Generator(device="cuda").manual_seed(0)
U = torch.randn(n, r, dtype=torch.float64, device="cuda", generator=g)
Vt = torch.randn(r, c, dtype=torch.float64, device="cuda", generator=g)
sv = torch.logspace(0, -6, r, dtype=torch.float64, device="cuda")
Z = (U * sv) @ Vt                                            # n x c, decaying spectrum
Zt = Z.T.contiguous()                                        # column-major storage of Z
for _ in range(2):
    out = G.rank_trunc_chol(Zt, 2 ** -6, "fp64")
torch.cuda.synchronize()
G.kernel_timing("rrqr")
t = time.time()
out = G.rank_trunc_chol(Zt, 2 ** -6, "fp64")
torch.cuda.synchronize()
ms, cnt = G.kernel_stats()[:2]
G.kernel_timing(None)
print(f"n={n} c={c}: out {tuple(out.shape)}, rrqr kernel {ms:.2f} ms ({ms * 1e3 / max(min(out.shape), 1):.1f} us/step), wall {1e3 * (time.time() - t):.1f} ms")
