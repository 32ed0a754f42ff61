"""The compensated quantized linear and its compositions (oracle; test infrastructure only).

Definition (north_star; §4.1 "Y = XŴ + XΔW ≈ XŴ + (XA_r)B_r"
"(X·A)·B, evaluated in that association order"):

    y* = Ŵ·x + U[:, :r] · (V[:r, :] · x)            (float64, associated as (V·x) then U)

with Ŵ = s·(q − z) (oracle.quant.dequant) and every bf16 input upcast exactly.

Windows (App. A.1.3): members sharing one input are evaluated on the
same x and their outputs concatenated in member order (QKV = q,k,v; UPGATE = up,gate).

Stack (reading R9, attention is out of scope and
replaced by the identity on the q-part): per layer
    qkv = QKV(h); a = bf16(q-part); h1 = bf16(h + O(a));
    gu = UPGATE(h1); m = bf16(silu(gate) ⊙ up); h2 = bf16(h1 + DOWN(m)).
MoE ("Y_MoE = Σ_e g_e E_e(X)"): per activated expert e over its
routed tokens: m_e = bf16(silu(gate_e) ⊙ up_e), y[t] += g_{t,e} · DOWN_e(m_e)[t].
bf16 rounding points are part of the definition (the activations a model passes
between linears are bf16); both the oracle and the kernels round there (RNE).
"""
from __future__ import annotations

import numpy as np

from .allocate import align, cap_level
from .packing import unpack_codes, bf16_to_f64, e4m3_to_f64
from .quant import dequant_abi


def deq_weight(codes, scales, zeros, K: int, bits: int, group: int) -> np.ndarray:
    """Ŵ in float64 from the canonical C-ABI formats."""
    q = unpack_codes(codes, K, bits)
    return dequant_abi(q, scales, zeros, group)


def compensated_product(W_hat: np.ndarray, U: np.ndarray, V: np.ndarray, r: int,
                        x: np.ndarray) -> np.ndarray:
    """y*[b, :] = Ŵ·x_b + U[:, :r]·(V[:r, :]·x_b); x is float64 [B, K]; returns [B, N]."""
    x = np.asarray(x, dtype=np.float64)
    y = x @ W_hat.T                                   # Ŵ·x for every row b
    if r > 0:
        t = x @ V[:r, :].T                            # t = V[:r,:]·x   -> [B, r]
        y = y + t @ U[:, :r].T                        # + U[:, :r]·t    -> [B, N]
    return y


def factors_f64(case: dict, rows=None):
    """(U, V) in float64 from the ABI formats: bf16 bits, or (factor_dtype "fp8") e4m3 bytes
    U8 [N, r_stored] / V8 [r_stored, K] with fp32 per-rank scales us / vs:
    U_eff = e4m3(U8)·us[j] (column j), V_eff = e4m3(V8)·vs[j] (row j), exact in float64."""
    if case.get("factor_dtype", "bf16") == "fp8":
        U8 = case["U8"] if rows is None else case["U8"][rows]
        us = np.asarray(case["us"], dtype=np.float32).astype(np.float64)
        vs = np.asarray(case["vs"], dtype=np.float32).astype(np.float64)
        return e4m3_to_f64(U8) * us[None, :], e4m3_to_f64(case["V8"]) * vs[:, None]
    U = case["U"] if rows is None else case["U"][rows]
    return bf16_to_f64(U), bf16_to_f64(case["V"])


def compensated_linear(case: dict, r: int, x_bits=None, rows=None) -> np.ndarray:
    """Oracle for one matrix given a synth.linear_case-style dict (ABI formats).

    ``rows`` (optional index array) restricts the output rows (sampled checks at full size).
    """
    K, bits, group = case["K"], case["bits"], case["group"]
    codes, scales, zeros = case["codes"], case["scales"], case["zeros"]
    if rows is not None:
        codes, scales, zeros = codes[rows], scales[rows], zeros[rows]
    W_hat = deq_weight(codes, scales, zeros, K, bits, group)
    x = bf16_to_f64(case["x"] if x_bits is None else x_bits)
    U, V = factors_f64(case, rows)
    return compensated_product(W_hat, U, V, r, x)


def window_linear(members: list, ranks: list, x_bits) -> np.ndarray:
    """Members sharing x (one compensation window): concatenate outputs in member order."""
    return np.concatenate([compensated_linear(m, r, x_bits=x_bits) for m, r in zip(members, ranks)],
                          axis=1)


def _round_bf16(a: np.ndarray) -> np.ndarray:
    """float64 -> nearest bf16 value (round half to even on the float64 value), as float64.

    v = m·2^e with 0.5 <= |m| < 1; bf16 keeps 8 significant bits, so the value is
    round_half_even(m·256)/256·2^e.  (Normal range only; the activations here are
    far from bf16 under/overflow.)"""
    a = np.asarray(a, dtype=np.float64)
    m, e = np.frexp(a)
    sm = m * 256.0
    fl = np.floor(sm)
    d = sm - fl
    odd = np.mod(fl, 2.0) != 0.0
    up = (d > 0.5) | ((d == 0.5) & odd)
    out = np.ldexp((fl + up) / 256.0, e)
    return np.where((a == 0.0) | ~np.isfinite(a), a, out)


def round_bf16(a: np.ndarray) -> np.ndarray:
    return _round_bf16(a)


def silu(v: np.ndarray) -> np.ndarray:
    """SiLU(v) = v·σ(v) = v / (1 + e^-v) (σ = SiLU as SPEC); e^-v overflowing to inf for very
    negative v gives the correct limit -0."""
    v = np.asarray(v, dtype=np.float64)
    with np.errstate(over="ignore"):
        return v / (1.0 + np.exp(-v))


def stack_forward(layers: list, ranks: list, x_bits) -> np.ndarray:
    """Oracle for the decode stack (C2/C5).

    layers[l] = dict(qkv=[q, k, v], o=[o], upgate=[up, gate], down=[down]) of linear_case dicts;
    ranks[l] = dict with the same keys holding per-member ranks.
    Returns the final hidden state h (float64 [B, d], bf16-valued).
    """
    h = bf16_to_f64(x_bits)
    for L, R in zip(layers, ranks):
        qkv = np.concatenate([_lin(m, r, h) for m, r in zip(L["qkv"], R["qkv"])], axis=1)
        d = L["o"][0]["K"]
        a = round_bf16(qkv[:, :d])
        h1 = round_bf16(h + _lin(L["o"][0], R["o"][0], a))
        up = _lin(L["upgate"][0], R["upgate"][0], h1)
        gate = _lin(L["upgate"][1], R["upgate"][1], h1)
        m = round_bf16(silu(gate) * up)
        h = round_bf16(h1 + _lin(L["down"][0], R["down"][0], m))
    return h


def _lin(case: dict, r: int, x_f64: np.ndarray) -> np.ndarray:
    W_hat = deq_weight(case["codes"], case["scales"], case["zeros"], case["K"], case["bits"], case["group"])
    U, V = factors_f64(case)
    return compensated_product(W_hat, U, V, r, x_f64)


def moe_forward(experts: list, ranks: list, x_bits, topk_idx, topk_gate) -> np.ndarray:
    """Oracle for the grouped MoE expert path (C3).

    experts[e] = dict(up=case, gate=case, down=case); ranks[e] = dict(up=r, gate=r, down=r).
    x_bits [T, d] bf16; topk_idx int [T, k]; topk_gate float32 [T, k] (used as given, as fp32 values).
    y[t] = Σ_{j} g[t, j] · DOWN_e(bf16(silu(GATE_e(x_t)) ⊙ UP_e(x_t))),  e = topk_idx[t, j].
    """
    x = bf16_to_f64(x_bits)
    T = x.shape[0]
    d = next(ex for ex in experts if ex is not None)["down"]["N"]   # inactive experts may be None
    y = np.zeros((T, d), dtype=np.float64)
    for e in sorted(set(int(v) for v in np.asarray(topk_idx).reshape(-1))):
        toks, slots = np.nonzero(np.asarray(topk_idx) == e)
        xe = x[toks]
        up = _lin(experts[e]["up"], ranks[e]["up"], xe)
        gate = _lin(experts[e]["gate"], ranks[e]["gate"], xe)
        m = round_bf16(silu(gate) * up)
        de = _lin(experts[e]["down"], ranks[e]["down"], m)
        g = np.asarray(topk_gate, dtype=np.float32)[toks, slots].astype(np.float64)
        y[toks] += g[:, None] * de
    return y


def dynamic_rank(k: int, g, rtilde, cap: int, k0: int = 3) -> int:
    """Per-(token, expert) rank of one matrix ("G_{i,e} = k·g_e"):
    r̃_{i,e} = G_{i,e}·r̃_i with G = k·g_e, then Align (ties up R14) and the cap rule (R15).

    g (the routing weight) and r̃ arrive as fp32 values (the C-ABI's types) and are upcast exactly; the
    product (k·g)·r̃ is then taken in float64, where it is EXACT (k <= 16 has <= 5 significant bits, g and
    r̃ 24 each: <= 53 bits), so the integer decision is the exact-arithmetic one (R21)."""
    rt = (float(k) * float(np.float32(g))) * float(np.float32(rtilde))
    return cap_level(align(rt, k0), int(cap), k0)


def moe_forward_dynamic(experts: list, caps: list, x_bits, topk_idx, topk_gate, rtilde: list, k0: int = 3):
    """Grouped MoE with per-(token, expert) dynamic ranks: for token t and slot j (expert e, gate g),
    the up / gate / down products use r = dynamic_rank(k, g, rtilde[e][s], caps[e][s]), s = up, gate,
    down; y[t] = Σ_j g · DOWN_e(bf16(silu(GATE_e(x_t)) ⊙ UP_e(x_t))).  caps[e] / rtilde[e] are dicts
    with keys up, gate, down.  One token row at a time (plain, slow, test-sized)."""
    x = bf16_to_f64(x_bits)
    idx = np.asarray(topk_idx)
    gates = np.asarray(topk_gate, dtype=np.float32)
    T, k = idx.shape
    d = experts[int(idx[0, 0])]["down"]["N"]
    y = np.zeros((T, d), dtype=np.float64)
    for t in range(T):
        for j in range(k):
            e, g = int(idx[t, j]), gates[t, j]
            r = {s: dynamic_rank(k, g, rtilde[e][s], caps[e][s], k0) for s in ("up", "gate", "down")}
            xt = x[t:t + 1]
            up = _lin(experts[e]["up"], r["up"], xt)
            gt = _lin(experts[e]["gate"], r["gate"], xt)
            m = round_bf16(silu(gt) * up)
            y[t] += float(g) * _lin(experts[e]["down"], r["down"], m)[0]
    return y
