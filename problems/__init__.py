"""Seeded synthetic Lyapunov problems (BASELINE.json ``configs``).

This module holds input generation ONLY -- none of the method's arithmetic.
It is the single module shared by the oracle side (tests, cpu baseline) and
the CUDA side (tests, bench, smoke).  Every generator is deterministic in
``seed`` (numpy PCG64).  All matrices are returned as float64 numpy arrays:
``A`` (n x n, C order), ``L`` (n x m), ``S`` (m x m) or None (Cholesky type).

Recipes:

* cfg0  n=64,  m=2,  Cholesky: A = Q diag(-lambda) Q^T, lambda log-spaced in
  [1, 100], Q Haar; L ~ N(0,1).
* cfg1  n=1024, m=4, LDL^T: A = -(Q diag(lambda) Q^T) + K, lambda log-spaced
  in [1, 1e2], K skew-symmetric with N(0, 0.1^2) entries, Q Haar;
  S = diag(Uniform[0.5, 2]); L ~ N(0,1).
* cfg2  n=4096, m=8: A = -(5-point Laplacian, 64x64 grid, h=1/65) minus
  first-order upwind convection (coefficient 10 in x), scaled by 1/||A||_F;
  L columns = indicator functions of random 8x8 grid patches.
* cfg3  n=16384, m=16: same family on a 128x128 grid, convection 50; L ~ N(0,1).
* cfg4  batch: n=2048, m=4, Cholesky: A = V diag(-lambda) V^{-1},
  V = I + 0.1 N(0,1)/sqrt(n), lambda log-spaced in [1, kappa],
  kappa in {1e1, 1e2, 1e3, 1e4} (64 equations each in the full batch).
* paper_synthetic  PAPER.md Section 5.2 (l.1432-1441): A = -V diag(logspace(0,q,n)) V^T
  with the symmetric orthogonal sine matrix V_ij = sqrt(2/(n+1)) sin(ij pi/(n+1)).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Problem:
    name: str
    A: np.ndarray
    L: np.ndarray
    S: np.ndarray | None
    kind: str           # "chol" or "ldlt"
    us: str             # solver precision named by the config
    meta: dict

    @property
    def n(self) -> int:
        return self.A.shape[0]

    @property
    def m(self) -> int:
        return self.L.shape[1]

    def W(self) -> np.ndarray:
        S = np.eye(self.m) if self.S is None else self.S
        return self.L @ S @ self.L.T


def haar_orthogonal(n: int, rng: np.random.Generator) -> np.ndarray:
    """Haar-distributed orthogonal matrix (QR of a Gaussian, sign-fixed)."""
    G = rng.standard_normal((n, n))
    Q, R = np.linalg.qr(G)
    return Q * np.sign(np.diag(R))[None, :]


def sine_orthogonal(n: int) -> np.ndarray:
    """Symmetric orthogonal V_ij = sqrt(2/(n+1)) sin(i j pi/(n+1)), i,j = 1..n."""
    i = np.arange(1, n + 1)
    return np.sqrt(2.0 / (n + 1)) * np.sin(np.outer(i, i) * np.pi / (n + 1))


def paper_synthetic(n: int, m: int, q: float, seed: int, kind: str = "chol", us: str = "bf16") -> Problem:
    """PAPER.md Section 5.2 generator (l.1432-1441)."""
    rng = np.random.default_rng(seed)
    L = rng.standard_normal((n, m))
    V = sine_orthogonal(n)
    lam = np.logspace(0, q, n)
    A = -(V * lam[None, :]) @ V.T
    S = np.eye(m) if kind == "ldlt" else None
    return Problem(f"paper_synthetic_n{n}_q{q}", A, L, S, kind, us, {"q": q, "seed": seed})


def cfg0(seed: int = 0, n: int = 64, m: int = 2) -> Problem:
    rng = np.random.default_rng(seed)
    Q = haar_orthogonal(n, rng)
    lam = np.logspace(0, 2, n)
    A = -(Q * lam[None, :]) @ Q.T
    L = rng.standard_normal((n, m))
    return Problem("cfg0", A, L, None, "chol", "fp16", {"seed": seed, "tol": 1e-14, "imax": 10})


def cfg1(seed: int = 1, n: int = 1024, m: int = 4) -> Problem:
    rng = np.random.default_rng(seed)
    Q = haar_orthogonal(n, rng)
    lam = np.logspace(0, 2, n)
    G = np.triu(rng.normal(0.0, 0.1, (n, n)), 1)
    K = G - G.T
    A = -(Q * lam[None, :]) @ Q.T + K
    S = np.diag(rng.uniform(0.5, 2.0, m))
    L = rng.standard_normal((n, m))
    return Problem("cfg1", A, L, S, "ldlt", "bf16", {"seed": seed})


def convection_diffusion(g: int, conv: float) -> np.ndarray:
    """Dense -(Laplacian) - conv * D_x^- on a g x g grid, h = 1/(g+1), scaled to unit F-norm.

    Both terms are negative (semi)definite in their symmetric part, so A is
    Hurwitz (its field of values lies in the open left half plane)."""
    n = g * g
    h = 1.0 / (g + 1)
    A = np.zeros((n, n))
    idx = np.arange(n).reshape(g, g)          # idx[iy, ix]
    for iy in range(g):
        for ix in range(g):
            r = idx[iy, ix]
            A[r, r] = -4.0 / h**2 - conv / h
            if ix > 0:
                A[r, idx[iy, ix - 1]] += 1.0 / h**2 + conv / h   # upwind (backward) difference
            if ix < g - 1:
                A[r, idx[iy, ix + 1]] += 1.0 / h**2
            if iy > 0:
                A[r, idx[iy - 1, ix]] += 1.0 / h**2
            if iy < g - 1:
                A[r, idx[iy + 1, ix]] += 1.0 / h**2
    return A / np.linalg.norm(A)


def cfg2(seed: int = 2, g: int = 64, m: int = 8) -> Problem:
    rng = np.random.default_rng(seed)
    A = convection_diffusion(g, 10.0)
    n = g * g
    L = np.zeros((n, m))
    for j in range(m):
        iy, ix = rng.integers(0, g - 8 + 1, size=2)
        patch = np.zeros((g, g))
        patch[iy:iy + 8, ix:ix + 8] = 1.0
        L[:, j] = patch.reshape(-1)
    return Problem("cfg2", A, L, None, "chol", "fp16", {"seed": seed, "grid": g})


def cfg3(seed: int = 3, g: int = 128, m: int = 16) -> Problem:
    rng = np.random.default_rng(seed)
    A = convection_diffusion(g, 50.0)
    L = rng.standard_normal((g * g, m))
    return Problem("cfg3", A, L, None, "chol", "fp16", {"seed": seed, "grid": g})


def cfg4_member(index: int, seed: int = 4, n: int = 2048, m: int = 4) -> Problem:
    """Equation `index` (0..255) of the batched config; kappa = 10^(1 + index // 64)."""
    kappa = 10.0 ** (1 + (index // 64) % 4)
    rng = np.random.default_rng([seed, index])
    V = np.eye(n) + 0.1 * rng.standard_normal((n, n)) / np.sqrt(n)
    lam = np.logspace(0, np.log10(kappa), n)
    A = (V * (-lam)[None, :]) @ np.linalg.inv(V)
    L = rng.standard_normal((n, m))
    return Problem(f"cfg4[{index}]", A, L, None, "chol", "fp16", {"seed": seed, "kappa": kappa})


CONFIGS = {"cfg0": cfg0, "cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3}


def diagonal_problem(n: int, m: int, seed: int) -> Problem:
    """Diagonal Hurwitz A: closed form X_ij = -W_ij / (a_i + a_j)."""
    rng = np.random.default_rng(seed)
    a = -rng.uniform(0.5, 5.0, n)
    L = rng.standard_normal((n, m))
    return Problem("diag", np.diag(a), L, None, "chol", "fp64", {"a": a})


def random_stable(n: int, m: int, seed: int, shift: float = 1.0, kind: str = "chol") -> Problem:
    """Small random nonsymmetric Hurwitz A = G/sqrt(n) - (rho(G/sqrt n) + shift) I."""
    rng = np.random.default_rng(seed)
    G = rng.standard_normal((n, n)) / np.sqrt(n)
    A = G - (np.max(np.abs(np.linalg.eigvals(G))) + shift) * np.eye(n)
    L = rng.standard_normal((n, m))
    S = np.eye(m) if kind == "ldlt" else None
    return Problem("random_stable", A, L, S, kind, "fp64", {"seed": seed})
