"""Seeded synthetic input generators shared by the oracle tests, the GPU parity
tests and ``bench.py``.

This module holds NONE of the method's arithmetic (no unpacking, no dequant, no
products, no allocation rule).  It only draws random numbers (numpy PCG64) and
rounds them to the storage formats the C-ABI takes (bf16 bit patterns, uint32
code words, uint8 zeros).  Uniform random uint32 words are uniformly random
b-bit codes under any bit layout, so no packing code is needed here.

Recipe (DESIGN.md §"Input recipe"):
  * codes   uniform over [0, 2^b) (random words)
  * zeros   2^(b-1) ("sym", the symmetric RTN case) or uniform [0, 2^b) ("asym")
  * scales  bf16(0.002 + 0.01 * U(0,1))      (~ max|w|/7 for w ~ N(0, 0.02))
  * x       bf16(N(0, 1))
  * U       bf16(N(0, 1/N))                   (orthonormal-ish columns)
  * V       bf16(N(0, 0.02^2))                (absorbs Sigma; compensation ~5% of |y|)
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "rng", "f32_to_bf16_bits", "bf16_bits_to_f32", "linear_case", "sensitivity_case",
    "routing_case", "SHAPES",
]

# Layer shapes (N x K = out x in), SURVEY.md §8 table.
SHAPES = {
    "llama2_7b": dict(hidden=4096, q=4096, kv=4096, ffn=11008, layers=32),
    "llama3_8b": dict(hidden=4096, q=4096, kv=1024, ffn=14336, layers=32),
    "llama3_70b": dict(hidden=8192, q=8192, kv=1024, ffn=28672, layers=80),
    "qwen3_30b_a3b_expert": dict(hidden=2048, ffn=768, experts=128, topk=8, layers=48),
}


# decode-stack gains per slot (q, k, v, o, up, gate, down)
STACK_GAINS = (1.0, 1.0, 1.0, 0.25, 0.25, 0.25, 0.05)


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def f32_to_bf16_bits(a) -> np.ndarray:
    """Round float32 values to bf16 (round-to-nearest-even) and return uint16 bits."""
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float32))
    u = a.view(np.uint32).astype(np.uint64)
    rounding = ((u >> 16) & 1) + 0x7FFF
    return ((u + rounding) >> 16).astype(np.uint16)


def bf16_bits_to_f32(b) -> np.ndarray:
    b = np.ascontiguousarray(np.asarray(b, dtype=np.uint16))
    return (b.astype(np.uint32) << 16).view(np.float32)


def linear_case(seed: int, N: int, K: int, bits: int = 4, group: int = 128,
                r_stored: int = 64, B: int = 1, zeros: str = "sym", unit_gain=False) -> dict:
    """One compensated linear's inputs in the C-ABI storage formats.

    codes  uint32 [N, K*bits/32]   (canonical little-endian bitstream per row)
    scales uint16 [N, K/group]     (bf16 bits)
    zeros  uint8  [N, K/group]
    U      uint16 [N, r_stored]    (bf16 bits)
    V      uint16 [r_stored, K]    (bf16 bits)
    x      uint16 [B, K]           (bf16 bits)
    """
    assert (K * bits) % 32 == 0 and K % group == 0
    g = rng(seed)
    words = K * bits // 32
    codes = g.integers(0, 2**32, size=(N, words), dtype=np.uint64).astype(np.uint32)
    ng = K // group
    if unit_gain:
        # stack recipe: |W x| ~ |x| so activations stay O(1) through many layers.
        # E[(q - z)^2] = (4^b - 1)/12 + 1/4 for uniform codes and z = 2^(b-1)
        # unit_gain may be a float gain (True = 1.0); see STACK_GAINS
        e2 = ((4 ** bits) - 1) / 12.0 + 0.25
        gain = np.float32(1.0 if unit_gain is True else float(unit_gain))
        scales = f32_to_bf16_bits(gain * (0.5 + g.random((N, ng), dtype=np.float32)) / np.float32(np.sqrt(e2 * K)))
    else:
        scales = f32_to_bf16_bits(0.002 + 0.01 * g.random((N, ng), dtype=np.float32))
    if zeros == "sym":
        z = np.full((N, ng), 1 << (bits - 1), dtype=np.uint8)
    elif zeros == "asym":
        z = g.integers(0, 1 << bits, size=(N, ng), dtype=np.uint8)
    else:
        raise ValueError(zeros)
    U = f32_to_bf16_bits(g.standard_normal((N, r_stored), dtype=np.float32) / np.float32(np.sqrt(N)))
    # compensation ~5% of |y|: unit gain -> sigma_V = 0.05 sqrt(N / (r K)); C1 recipe -> 0.02
    sv = 0.05 * np.sqrt(N / (max(r_stored, 1) * K)) if unit_gain else 0.02
    V = f32_to_bf16_bits(np.float32(sv) * g.standard_normal((r_stored, K), dtype=np.float32))
    x = f32_to_bf16_bits(g.standard_normal((B, K), dtype=np.float32))
    return dict(codes=codes, scales=scales, zeros=z, U=U, V=V, x=x,
                N=N, K=K, bits=bits, group=group, r_stored=r_stored, B=B)


def fp8_factors(case: dict, seed: int, all_codes: bool = False) -> dict:
    """Replace a linear_case's factors by e4m3 bytes + fp32 per-rank scales (SURVEY.md §8(f)4 inputs).
    Random BYTES, no arithmetic: sign uniform, exponent field uniform in [4, 10] (|v| in [2^-3, 15]) with
    1/16 of the bytes drawn from the subnormal / zero codes; all_codes cycles through every non-NaN code.
    Scales fp32: us ~ U(0.5, 1.5)/(4·sqrt(N)), vs ~ U(0.5, 1.5)·σ_V/4 (σ_V of linear_case's bf16 V)."""
    g = rng(seed)
    N, K, rs = case["N"], case["K"], case["r_stored"]

    def draw(shape):
        if all_codes:
            valid = np.array([c for c in range(256) if (c & 0x7F) != 0x7F], dtype=np.uint8)
            return valid[np.arange(int(np.prod(shape))) % valid.size].reshape(shape)
        sign = g.integers(0, 2, size=shape, dtype=np.uint8) << 7
        e = g.integers(4, 11, size=shape, dtype=np.uint8)
        sub = g.random(shape) < 1.0 / 16.0
        e = np.where(sub, 0, e).astype(np.uint8)
        m = g.integers(0, 8, size=shape, dtype=np.uint8)
        return (sign | (e << 3) | m).astype(np.uint8)
    out = dict(case)
    out["factor_dtype"] = "fp8"
    out["U8"] = draw((N, rs))
    out["V8"] = draw((rs, K))
    sv = 0.05 * np.sqrt(N / (max(rs, 1) * K)) if K else 0.02
    out["us"] = ((0.5 + g.random(rs, dtype=np.float32)) / np.float32(4.0 * np.sqrt(N))).astype(np.float32)
    out["vs"] = ((0.5 + g.random(rs, dtype=np.float32)) * np.float32(sv / 4.0)).astype(np.float32)
    return out


def activations(seed: int, B: int, K: int) -> np.ndarray:
    """bf16 bits of x ~ N(0, 1), shape [B, K]."""
    return f32_to_bf16_bits(rng(seed).standard_normal((B, K), dtype=np.float32))


def sensitivity_case(seed: int, n_layers: int, members_per_window=(3, 1, 2, 1),
                     n_sigma: int = 256) -> dict:
    """Synthetic allocator inputs (SURVEY.md §8(d) C2 recipe).

    Planted spectra sigma_j = exp(-j/c) + 0.05 with c ~ U[2, 16]; D_i ~ LogNormal(0, 1);
    D_layer ~ LogNormal(0, 0.5).  Returns per-record dicts in window order
    (layer-major; windows QKV=0, O=1, UPGATE=2, DOWN=3; slots in member order).
    """
    g = rng(seed)
    recs = []
    for layer in range(n_layers):
        for kind, m in enumerate(members_per_window):
            for slot in range(m):
                c = g.uniform(2.0, 16.0)
                j = np.arange(n_sigma, dtype=np.float64)
                sigma = np.exp(-j / c) + 0.05
                recs.append(dict(layer=layer, window=kind, slot=slot, expert=-1,
                                 sigma=sigma, D=float(g.lognormal(0.0, 1.0)), gate=1.0))
    D_layer = g.lognormal(0.0, 0.5, size=n_layers)
    return dict(records=recs, D_layer=D_layer)


def routing_case(seed: int, T: int, E: int, topk: int):
    """Synthetic routing: logits ~ N(0,1) per token,
    softmax -> top-k (ties by lower expert index) -> renormalised gates.
    Returns (topk_idx int32 [T, topk], topk_gate float32 [T, topk])."""
    g = rng(seed)
    logits = g.standard_normal((T, E))
    p = np.exp(logits - logits.max(axis=1, keepdims=True))
    p /= p.sum(axis=1, keepdims=True)
    idx = np.argsort(-p, axis=1, kind="stable")[:, :topk]
    gate = np.take_along_axis(p, idx, axis=1)
    gate /= gate.sum(axis=1, keepdims=True)
    return idx.astype(np.int32), gate.astype(np.float32)
