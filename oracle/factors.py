"""Truncated-SVD compensation factors (oracle; test infrastructure only).

P:142-145 (§4.1): Y = XŴ + XΔW ≈ XŴ + (XA_r)B_r, with A_r, B_r "obtained from
the singular value decomposition of ΔW".  SPEC S:61-65 fixes the split
A = U[:, :r]·diag(σ[:r]) (Σ absorbed into the first-applied factor), B = Vᵀ[:r, :].

This build uses the north_star orientation y = Ŵ·x + U[:, :r]·(V[:r, :]·x) with
W stored N×K (out × in), i.e. the transpose of the paper's d×k.  With
numpy.linalg.svd(ΔW) = P·diag(σ)·Qᵀ (ΔW is N×K):

    U = P[:, :r]                 (N × r, orthonormal columns;  = B_rᵀ)
    V = diag(σ[:r])·Q[:, :r]ᵀ    (r × K, absorbs Σ;            = A_rᵀ)

Sign convention (S:54 transported): first nonzero entry of each U column ≥ 0.
Rank-prefix property: the rank-r factors are the first r columns/rows of the
full factorisation (Eckart–Young), so one stored pool serves every r.
"""
from __future__ import annotations

import numpy as np


def svd_full(delta_w: np.ndarray):
    """Return (P, sigma, Qt) of ΔW with the sign convention applied."""
    dw = np.asarray(delta_w, dtype=np.float64)
    P, sigma, Qt = np.linalg.svd(dw, full_matrices=False)
    for j in range(P.shape[1]):
        col = P[:, j]
        nz = np.flatnonzero(col != 0.0)
        if nz.size and col[nz[0]] < 0:
            P[:, j] = -P[:, j]
            Qt[j, :] = -Qt[j, :]
    return P, sigma, Qt


def svd_factors(delta_w: np.ndarray, r: int):
    """(U [N, r], V [r, K], sigma) for the rank-r compensation of ΔW."""
    P, sigma, Qt = svd_full(delta_w)
    n = sigma.shape[0]
    if r < 0 or r > n:
        raise ValueError(f"rank {r} out of range [0, {n}] (SPEC S:65 range error)")
    U = P[:, :r].copy()
    V = sigma[:r, None] * Qt[:r, :]
    return U, V, sigma


def frobenius_sq(m: np.ndarray) -> float:
    m = np.asarray(m, dtype=np.float64)
    return float(np.sum(m * m))
