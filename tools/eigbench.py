import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, paper_2510_02126_b200 as G
for n in [256, 512, 1024]:
    B = np.random.default_rng(n).standard_normal((n, n)); A = torch.tensor(B + B.T, device="cuda")
    G.syev(A); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3): G.syev(A)
    torch.cuda.synchronize(); print(n, "ms per syev", (time.perf_counter() - t) / 3 * 1e3)
