"""Sensitivity-aware dynamic rank allocation, step by step (oracle; test infrastructure only).

Follows PAPER.md Appendix B.1 in the paper's order and notation, with
the readings listed in DESIGN.md §"Readings" (R10-R17).  All sums run
sequentially over a window's members in input order (Python float adds, no
numpy pairwise summation) so that the C++ host implementation can reproduce the
result bit-for-bit.

  φ_i   singular-value salience            P:579-610   (reading R10: literal S = {1..argmax})
  𝒱_i   = φ_i / Σ_W φ_j
  𝒮_i   = D_i / Σ_W D_j                    P:630-633   (window scope, R11)
  𝒮_ℓ   top-K rule                         P:640-648   (K given; R12)
  𝒢     = k·g_e
  𝒫     = 𝒢·Norm_W(𝒱𝒮)·𝒮_ℓ
  r̃     = 𝒫·r_std
  two-stage                                P:682-694   (mode 0 per-matrix, mode 1 pooled; R13)
  Align  nearest of {0} ∪ {2^k, k>=k0}     P:698-711   (ties up, R14)
  cap    largest level <= cap              (R15, paper silent)
  enforce Σ_W r <= r_std by demotion       (R16; paper silent)
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

HC_ERR_CONFIG = 2
HC_ERR_NUMERIC = 4


class AllocError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def _seqsum(vals) -> float:
    s = 0.0
    for v in vals:
        s = s + float(v)
    return s


# ---------------------------------------------------------------- φ
@dataclass
class Salience:
    phi: float
    cut: int          # |S_i| (0 when S_i = ∅)
    n: int            # number of singular values (|S_i| + |R_i|)


def salience(sigma, tau: float = 0.01) -> Salience:
    """σ̂_j = σ_j/σ_1; k_j = σ̂_{j−1} − 2σ̂_j + σ̂_{j+1} for interior j;
    r_i = argmax_j k_j (smallest index on ties); S_i = {1..r_i} iff max k > τ
    (P:593-598); φ = mean_S σ / mean_R σ, or 1 when S = ∅."""
    sig = [float(v) for v in sigma]
    n = len(sig)
    if n < 3 or sig[0] == 0.0:                 # S:194, S:198 degenerate paths
        return Salience(1.0, 0, n)
    s1 = sig[0]
    hat = [v / s1 for v in sig]
    best_j, best_k = -1, -math.inf
    for j in range(1, n - 1):                  # 0-based interior = 1-based j in [2, n-1]
        kj = hat[j - 1] - 2.0 * hat[j] + hat[j + 1]
        if kj > best_k:                        # strict '>' keeps the smallest index on ties
            best_k, best_j = kj, j
    if not best_k > tau:
        return Salience(1.0, 0, n)
    cut = best_j + 1                           # 1-based argmax = size of S_i
    mean_s = _seqsum(sig[:cut]) / cut
    mean_r = _seqsum(sig[cut:]) / (n - cut)
    return Salience(mean_s / max(mean_r, 1e-300), cut, n)   # reading R10b: mean_R = 0 guarded


# ---------------------------------------------------------------- normalisations
def window_normalise(vals) -> list:
    """x_i / Σ_W x_j, sequential sum; zero sum -> uniform 1/m."""
    tot = _seqsum(vals)
    m = len(vals)
    if tot == 0.0:
        return [1.0 / m] * m
    return [float(v) / tot for v in vals]


def layer_scores(D_layer, K: int) -> list:
    """𝒯 = top-K layers by D_ℓ (ties: smaller index);
    𝒮_ℓ = 1 on 𝒯, else D_ℓ / min_𝒯 D (0 when that minimum is 0, reading R12)."""
    L = len(D_layer)
    if not (1 <= K <= L):
        raise AllocError(HC_ERR_CONFIG, f"top_k_layers {K} out of range [1, {L}]")
    order = sorted(range(L), key=lambda l: (-float(D_layer[l]), l))
    top = set(order[:K])
    dmin = min(float(D_layer[l]) for l in top)
    out = []
    for l in range(L):
        if l in top:
            out.append(1.0)
        elif dmin == 0.0:
            out.append(0.0)
        else:
            out.append(float(D_layer[l]) / dmin)
    return out


def expert_scores(gates, k: int) -> list:
    """𝒢_e = k·g_e with Σ g_e = 1 over the activated set (S:373 error otherwise)."""
    if abs(_seqsum(gates) - 1.0) > 1e-9:
        raise AllocError(HC_ERR_NUMERIC, "gates not normalised")
    return [k * float(g) for g in gates]


# ---------------------------------------------------------------- align / enforce
def align(rt: float, k0: int = 3) -> int:
    """nearest admissible level in {0} ∪ {2^k : k >= k0}; ties round up."""
    lo, hi = 0, 1 << k0
    while rt >= hi:
        lo, hi = hi, hi * 2
    return lo if (rt - lo) < (hi - rt) else hi


def cap_level(r: int, cap: int, k0: int = 3) -> int:
    """Reading R15: the largest admissible level <= cap when the aligned rank exceeds cap."""
    if r <= cap:
        return r
    lvl = 0
    v = 1 << k0
    while v <= cap:
        lvl, v = v, v * 2
    return lvl


def demote(r: int, k0: int = 3) -> int:
    return r // 2 if r // 2 >= (1 << k0) else 0


def enforce_budget(ranks: list, prio: list, r_std: float, k0: int = 3) -> list:
    """S:439-447 (R16): while Σ r > r_std, demote the lowest-𝒫 nonzero member one level;
    equal 𝒫 -> the later member (larger index) first."""
    r = list(ranks)
    while sum(r) > r_std:
        cand = [i for i in range(len(r)) if r[i] > 0]
        if not cand:
            break
        worst = cand[0]
        for i in cand[1:]:
            if prio[i] < prio[worst] or (prio[i] == prio[worst] and i > worst):
                worst = i
        r[worst] = demote(r[worst], k0)
    return r


# ---------------------------------------------------------------- two-stage
def two_stage(rt: list, prio: list, n_sal: list, n_all: list, mode: int) -> list:
    """Mode 0: per matrix min(r̃, |S|) salient + the rest residual -> the count is r̃.
    Mode 1 (literal P:689-693, pooled over the window): water-fill Σr̃ into the salient
    sets ∝ 𝒫 capped at |S_i|; any excess over Σ|S_i| spread ∝ |R_i|."""
    m = len(rt)
    if mode == 0:
        out = []
        for i in range(m):
            sal = min(rt[i], float(n_sal[i]))
            out.append(sal + (rt[i] - sal))
        return out
    total = _seqsum(rt)
    caps = [float(c) for c in n_sal]
    alloc = [0.0] * m
    capsum = _seqsum(caps)
    rem = min(total, capsum)
    active = [i for i in range(m) if caps[i] > 0.0]
    while active and rem > 0.0:
        psum = _seqsum(prio[i] for i in active)
        w = {i: (prio[i] / psum if psum > 0.0 else 1.0 / len(active)) for i in active}
        sat = [i for i in active if alloc[i] + rem * w[i] >= caps[i]]
        if not sat:
            for i in active:
                alloc[i] = alloc[i] + rem * w[i]
            rem = 0.0
            break
        for i in sat:
            rem = rem - (caps[i] - alloc[i])
            alloc[i] = caps[i]
        active = [i for i in active if i not in sat]
    if total > capsum:
        excess = total - capsum
        res = [float(n_all[i] - n_sal[i]) for i in range(m)]
        rsum = _seqsum(res)
        if rsum > 0.0:
            for i in range(m):
                alloc[i] = alloc[i] + excess * res[i] / rsum
    return alloc


# ---------------------------------------------------------------- the whole chain
@dataclass
class Record:
    layer: int
    window: int            # 0 QKV, 1 O, 2 UPGATE, 3 DOWN
    slot: int
    expert: int = -1
    sigma: object = None   # non-increasing singular values, or None -> phi/n_sal/n_all given
    phi: float = 1.0
    n_sal: int = 0
    n_all: int = 0
    D: float = 0.0
    gate: float = 1.0


@dataclass
class Budget:
    D_layer: list
    top_k_layers: int
    r_std: list            # per window kind [4]
    tau: float = 0.01
    k0: int = 3
    two_stage_mode: int = 0
    moe_k: int = 0         # activated experts per window (0 = dense)


@dataclass
class Allocation:
    ranks: list
    priority: list
    rtilde: list
    phi: list = field(default_factory=list)


def allocate_ranks(recs: list, budget: Budget, caps: list) -> Allocation:
    n = len(recs)
    if len(caps) != n:
        raise AllocError(HC_ERR_CONFIG, "caps length")
    L = len(budget.D_layer)
    for r in recs:
        if not (0 <= r.layer < L) or not (0 <= r.window < 4):
            raise AllocError(HC_ERR_CONFIG, "layer/window out of range")
        if not math.isfinite(r.D) or r.D < 0.0 or not math.isfinite(r.gate):
            raise AllocError(HC_ERR_NUMERIC, "non-finite or negative sensitivity")
    for d in budget.D_layer:
        if not math.isfinite(float(d)) or float(d) < 0.0:
            raise AllocError(HC_ERR_NUMERIC, "non-finite or negative layer sensitivity")
    # φ per record
    phi, nsal, nall = [], [], []
    for r in recs:
        if r.sigma is not None:
            s = salience(r.sigma, budget.tau)
            phi.append(s.phi); nsal.append(s.cut); nall.append(s.n)
        else:
            phi.append(float(r.phi)); nsal.append(int(r.n_sal)); nall.append(int(r.n_all))
    S_l = layer_scores(budget.D_layer, budget.top_k_layers)
    # windows keyed by (layer, kind), members in input order
    windows: dict = {}
    for i, r in enumerate(recs):
        windows.setdefault((r.layer, r.window), []).append(i)
    prio = [0.0] * n
    rt = [0.0] * n
    ranks = [0] * n
    for (layer, kind), mem in windows.items():
        V = window_normalise([phi[i] for i in mem])                 # 𝒱_i
        S = window_normalise([recs[i].D for i in mem])              # 𝒮_i
        if budget.moe_k > 0:                                        # 𝒢 = k·g_e
            # gates must be normalised over the activated experts of each slot
            for slot in sorted(set(recs[i].slot for i in mem)):
                gs = [recs[i].gate for i in mem if recs[i].slot == slot]
                expert_scores(gs, budget.moe_k)
            G = [budget.moe_k * float(recs[i].gate) for i in mem]
        else:
            G = [1.0] * len(mem)
        P0 = window_normalise([V[j] * S[j] for j in range(len(mem))])   # Norm_W(𝒱𝒮)
        P = [(G[j] * P0[j]) * S_l[layer] for j in range(len(mem))]      # 𝒫
        rstd = float(budget.r_std[kind])
        RT = [P[j] * rstd for j in range(len(mem))]                     # r̃
        RT2 = two_stage(RT, P, [nsal[i] for i in mem], [nall[i] for i in mem],
                        budget.two_stage_mode)
        al = [cap_level(align(RT2[j], budget.k0), int(caps[i]), budget.k0)
              for j, i in enumerate(mem)]
        al = enforce_budget(al, P, rstd, budget.k0)
        for j, i in enumerate(mem):
            prio[i], rt[i], ranks[i] = P[j], RT2[j], al[j]
    return Allocation(ranks=ranks, priority=prio, rtilde=rt, phi=phi)


def records_from_synth(case: dict) -> list:
    return [Record(layer=r["layer"], window=r["window"], slot=r["slot"], expert=r["expert"],
                   sigma=np.asarray(r["sigma"], dtype=np.float64), D=r["D"], gate=r["gate"])
            for r in case["records"]]


# ---------------------------------------------------------------- r_std on B200 (R17)
def r_std_bytes(Ns, K: int, bits: int, group: int = 128, eps: float = 0.1) -> float:
    """B200 reading of the budget r_std (SURVEY.md §8(c) "Proposed B200 meaning", R17; the paper's
    r_std is a CPU-time budget): the largest rank whose factor bytes 2·r·(N̄ + K) stay within eps
    of the window's base bytes Σ_i N_i·K·b/8 + N_i·(K/g)·(16 + b)/8 (codes, bf16 scale, b-bit zero)."""
    base = sum(N * K * bits // 8 + N * (K // group) * (16 + bits) // 8 for N in Ns)
    nbar = sum(Ns) / len(Ns)
    return float(math.floor(eps * base / (2 * (nbar + K))))
