"""Group-wise dequantisation and the RTN quantiser (oracle; test infrastructure only).

Dequant ("the weight matrix becomes Ŵ"; SPEC S:131-135 with the
north_star's per-group zeros; readings R2/R3):

    Ŵ[n, k] = s[n, ⌊k/g⌋] · (q[n, k] − z[n, ⌊k/g⌋])

groups of g consecutive input (K) elements per output row.

RTN (the GPTQ stand-in the SPEC prescribes): per group
scale = max|w| / (2^(b-1) − 1); code = clamp(round_half_away(w / scale));
an all-zero group gets scale 1 and codes 0.
"""
from __future__ import annotations

import numpy as np

from .packing import bf16_to_f64


def dequant(q: np.ndarray, scales: np.ndarray, zeros: np.ndarray, group: int) -> np.ndarray:
    """Ŵ = s·(q − z), float64 [N, K].  ``scales`` are float64 values (already decoded)."""
    q = np.asarray(q, dtype=np.float64)
    N, K = q.shape
    s = np.repeat(np.asarray(scales, dtype=np.float64), group, axis=1)[:, :K]
    z = np.repeat(np.asarray(zeros, dtype=np.float64), group, axis=1)[:, :K]
    return s * (q - z)


def dequant_abi(q: np.ndarray, scales_bf16: np.ndarray, zeros_u8: np.ndarray, group: int) -> np.ndarray:
    """Dequant from the C-ABI storage formats (bf16 scale bits, uint8 zeros)."""
    return dequant(q, bf16_to_f64(scales_bf16), zeros_u8.astype(np.float64), group)


def round_half_away(v: np.ndarray) -> np.ndarray:
    """SPEC S:124 / S:156: ties round away from zero (numpy's round is half-even)."""
    v = np.asarray(v, dtype=np.float64)
    return np.sign(v) * np.floor(np.abs(v) + 0.5)


def rtn_quantize(w: np.ndarray, bits: int, group: int):
    """Symmetric RTN quantiser.

    Returns (codes_signed int64 [N, K] in [-(2^(b-1)-1), 2^(b-1)-1], scales float64 [N, K/g]).
    Stored unsigned for the kernel as q = code + 2^(b-1), z = 2^(b-1).
    """
    w = np.asarray(w, dtype=np.float64)
    N, K = w.shape
    assert K % group == 0
    qmax = (1 << (bits - 1)) - 1
    codes = np.zeros((N, K), dtype=np.int64)
    scales = np.ones((N, K // group), dtype=np.float64)
    for gi in range(K // group):
        blk = w[:, gi * group:(gi + 1) * group]
        amax = np.max(np.abs(blk), axis=1)
        for n in range(N):
            if amax[n] == 0.0:
                scales[n, gi] = 1.0
                codes[n, gi * group:(gi + 1) * group] = 0
                continue
            s = amax[n] / qmax
            scales[n, gi] = s
            c = round_half_away(blk[n] / s)
            codes[n, gi * group:(gi + 1) * group] = np.clip(c, -qmax - 1, qmax).astype(np.int64)
    return codes, scales


def rtn_dequantize(codes: np.ndarray, scales: np.ndarray, group: int) -> np.ndarray:
    """entry = code × group scale."""
    s = np.repeat(np.asarray(scales, dtype=np.float64), group, axis=1)
    return np.asarray(codes, dtype=np.float64) * s
