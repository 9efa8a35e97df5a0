import numpy as np, torch, oracle as orc, problems as P, paper_2510_02126_b200 as G


def cuda(x):
    return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")


def colmajor(x):
    return cuda(np.ascontiguousarray(np.asarray(x).T))


rng = np.random.default_rng(11)
p = P.random_stable(60, 3, 2)
Z = rng.standard_normal((60, 7)); Y = np.diag(rng.uniform(0.1, 1, 7))
s = G.Solver(60, us="fp64", max_cols=64)
_ = s.res_fac_ldlt(cuda(p.A), colmajor(p.L), cuda(np.diag([1.0, 0.5, 2.0])), colmajor(Z), cuda(Y))
_ = s.res_fac_chol(cuda(p.A), colmajor(p.L), colmajor(Z))
Zd = rng.standard_normal((60, 4)); Yd = np.diag([1.0, -0.2, 0.3, -1e-3])
G2 = np.hstack([Z, Zd]); U = np.zeros((11, 11)); U[:7, :7] = Y; U[7:, 7:] = Yd
Q, R = np.linalg.qr(G2); K = R @ U @ R.T
print("numpy eig K", np.sort(np.linalg.eigvalsh(K))[::-1])
w, V = G.syev(cuda(K)); print("gpu syev K", w.cpu().numpy())
Zn, Yn = s.sol_upt_ldlt(colmajor(Z), cuda(Y), colmajor(Zd), cuda(Yd))
print("gpu Yn", np.diag(Yn.cpu().numpy()))
Zno, Yno = orc.sol_upt_ldlt("fp64", Z, Y, Zd, Yd, 10 * 2.0 ** -53)
print("orc Yn", np.diag(Yno))
