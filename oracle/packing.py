"""Storage-format decoding for the oracle (test infrastructure only).

Canonical code format (reading R1; the paper never fixes sub-byte
packing — SPEC S:162 lists packed storage as a non-goal): row n of a b-bit
matrix is a little-endian bitstream of uint32 words; element k occupies bits
[b*k, b*k + b) of that stream, i.e.

    q[n, k] = (stream_n >> (b*k)) & (2^b - 1)

For b = 3 an element may straddle two words.
"""
from __future__ import annotations

import numpy as np


def unpack_codes(words: np.ndarray, K: int, bits: int) -> np.ndarray:
    """Canonical bitstream -> unsigned codes q[n, k] in [0, 2^bits), int64 [N, K]."""
    words = np.asarray(words, dtype=np.uint32)
    N = words.shape[0]
    w64 = words.astype(np.uint64)
    # a zero word appended so that the "next word" of the last element exists
    w64 = np.concatenate([w64, np.zeros((N, 1), dtype=np.uint64)], axis=1)
    k = np.arange(K, dtype=np.int64)
    pos = bits * k                      # bit offset of element k in the stream
    wi = pos // 32                      # word holding the element's first bit
    off = (pos % 32).astype(np.uint64)  # bit offset inside that word
    lo = w64[:, wi] >> off
    hi = w64[:, wi + 1] << (np.uint64(32) - off)   # bits spilling into the next word
    both = (lo | hi) & np.uint64(0xFFFFFFFF)
    return (both & np.uint64((1 << bits) - 1)).astype(np.int64)


def bf16_to_f64(bits: np.ndarray) -> np.ndarray:
    """bf16 bit patterns (uint16) -> float64, exactly (bf16 is the top half of fp32)."""
    b = np.ascontiguousarray(np.asarray(bits, dtype=np.uint16))
    return (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def f64_to_bf16_bits_rne(a: np.ndarray) -> np.ndarray:
    """Round float values to bf16, round-to-nearest-even, via float32 (exact
    double->float rounding first is NOT what the kernel does, so only call this
    on float32-representable inputs, e.g. kernel fp32 outputs)."""
    f = np.ascontiguousarray(np.asarray(a, dtype=np.float32))
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + (((u >> 16) & 1) + 0x7FFF)) >> 16
    return u.astype(np.uint16)


def e4m3_to_f64(b: np.ndarray) -> np.ndarray:
    """OCP FP8 E4M3 (e4m3fn) bytes -> float64 by the format's definition: sign bit 7,
    exponent bits 6-3 (bias 7), mantissa bits 2-0; e > 0: (-1)^s·2^(e-7)·(1 + m/8); e = 0: (-1)^s·2^-6·m/8;
    0x7F / 0xFF (e = 15, m = 7) are NaN (no infinities)."""
    b = np.asarray(b, dtype=np.uint8).astype(np.int64)
    s = np.where(b & 0x80, -1.0, 1.0)
    e = (b >> 3) & 0xF
    m = (b & 0x7).astype(np.float64)
    v = np.where(e > 0, np.ldexp(1.0 + m / 8.0, (e - 7).astype(np.int64)), np.ldexp(m / 8.0, -6))
    v = s * v
    return np.where((e == 15) & ((b & 0x7) == 7), np.nan, v)
