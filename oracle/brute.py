"""Optimality oracles for the allocation problem (Appendix B.2; test infrastructure only).

P:764-767: max Σ_i gain_i(r_i)  s.t.  Σ_i r_i <= r_std, r_i >= 0, with the concave
marginal model "∂/∂r ‖(ΔW_i)_r‖_F² ≈ σ_{i,r}²" weighted by 𝒮·𝒢.

  gain_table(sigma, w, levels)  gain_i(L) = w · Σ_{j<=L} σ_j²   (recovered energy)
  brute_force(tables, levels, budget)   exhaustive search, <= 5 matrices
  greedy(tables, levels, budget)        largest marginal gain per unit rank, one level at a time
"""
from __future__ import annotations

import itertools


def gain_table(sigma, weight: float, levels) -> list:
    """gain(L) = weight · Σ_{j < L} σ_j² for each admissible level L (Eckart–Young recovered energy)."""
    out = []
    for L in levels:
        e = 0.0
        for j in range(min(L, len(sigma))):
            e = e + float(sigma[j]) ** 2
        out.append(weight * e)
    return out


def brute_force(tables: list, levels: list, budget: float):
    """Exact maximiser over all level assignments (ties: lexicographically smallest plan)."""
    m = len(tables)
    if m > 5 or len(levels) > 8:
        raise ValueError("instance too large for exhaustive search")
    best_val, best = -1.0, None
    for combo in itertools.product(range(len(levels)), repeat=m):
        if sum(levels[c] for c in combo) > budget:
            continue
        val = 0.0
        for i, c in enumerate(combo):
            val = val + tables[i][c]
        if val > best_val:
            best_val, best = val, [levels[c] for c in combo]
    return best, best_val


def greedy(tables: list, levels: list, budget: float):
    """Repeatedly take the single-level step with the largest gain per unit of rank
    that still fits the budget (the "greedy argument" of P:782)."""
    m = len(tables)
    idx = [0] * m
    used = 0
    while True:
        best_i, best_rate = -1, 0.0
        for i in range(m):
            if idx[i] + 1 >= len(levels):
                continue
            step = levels[idx[i] + 1] - levels[idx[i]]
            if used + step > budget:
                continue
            rate = (tables[i][idx[i] + 1] - tables[i][idx[i]]) / step
            if rate > best_rate:
                best_i, best_rate = i, rate
        if best_i < 0:
            break
        used += levels[idx[best_i] + 1] - levels[idx[best_i]]
        idx[best_i] += 1
    plan = [levels[k] for k in idx]
    val = 0.0
    for i in range(m):
        val = val + tables[i][idx[i]]
    return plan, val
