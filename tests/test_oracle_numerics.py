"""Pins for oracle.packing / oracle.quant / oracle.factors / oracle.linear.

Each test pins the oracle to something other than itself: hand-packed words, the
SPEC's printed worked examples (tests/golden), closed forms (Eckart–Young), exact
identities (rank 0, full rank), or an independent brute-force construction.
"""
import numpy as np
import pytest

import synth
from oracle import packing, quant, factors, linear


# ------------------------------------------------------------------ unpack (c1)
def _pack_bigint(q, bits):
    """Independent construction of the canonical stream: Python big int Σ q_k << (b·k)."""
    N, K = q.shape
    words = K * bits // 32
    out = np.zeros((N, words), dtype=np.uint32)
    for n in range(N):
        v = 0
        for k in range(K):
            v |= int(q[n, k]) << (bits * k)
        for w in range(words):
            out[n, w] = (v >> (32 * w)) & 0xFFFFFFFF
    return out


def test_unpack_hand_words_4bit():
    w = np.array([[0x76543210, 0xFEDCBA98]], dtype=np.uint32)
    assert packing.unpack_codes(w, 16, 4).tolist() == [list(range(16))]


def test_unpack_hand_words_2bit():
    # 0xE4 = 0b11_10_01_00 -> 0,1,2,3 then zeros
    w = np.array([[0x000000E4]], dtype=np.uint32)
    assert packing.unpack_codes(w, 16, 2).tolist() == [[0, 1, 2, 3] + [0] * 12]


def test_unpack_hand_words_3bit_straddle():
    # q[0] = 1 (bits 0-2); q[10] = 5 = 0b101 occupies bits 30,31,32: bit30=1, bit31=0, bit32=1
    w = np.array([[0x40000001, 0x00000001, 0x00000000]], dtype=np.uint32)
    q = packing.unpack_codes(w, 32, 3)[0]
    exp = [0] * 32
    exp[0], exp[10] = 1, 5
    assert q.tolist() == exp


@pytest.mark.parametrize("bits", [2, 3, 4, 8])
def test_unpack_inverts_bigint_pack(bits):
    g = synth.rng(bits)
    q = g.integers(0, 1 << bits, size=(5, 256))
    assert np.array_equal(packing.unpack_codes(_pack_bigint(q, bits), 256, bits), q)


def test_bf16_decode_exact():
    assert packing.bf16_to_f64(np.array([0x3F80, 0xC000, 0x3DCD], dtype=np.uint16)).tolist() == \
        [1.0, -2.0, float(np.float32(np.uint32(0x3DCD0000).view(np.float32)))]


# ------------------------------------------------------------------ quantiser / dequant (c2, c3)
def test_rtn_spec_examples(golden):
    e4 = golden["rtn_4bit"]
    c, s = quant.rtn_quantize(np.array([e4["w"]]), 4, 2)
    assert c.tolist() == [e4["codes"]] and abs(s[0, 0] - e4["scale"]) < 1e-15
    assert np.allclose(quant.rtn_dequantize(c, s, 2), [e4["deq"]], atol=1e-15)
    e3 = golden["rtn_3bit"]
    c, s = quant.rtn_quantize(np.array([e3["w"]]), 3, 2)
    assert c.tolist() == [e3["codes"]] and abs(s[0, 0] - e3["scale"]) < 1e-15
    res = np.array([e3["w"]]) - quant.rtn_dequantize(c, s, 2)
    assert np.allclose(res, [e3["residual"]], atol=e3["residual_tol"])


def test_rtn_zero_group_and_rounding():
    c, s = quant.rtn_quantize(np.zeros((2, 4)), 4, 4)
    assert (c == 0).all() and (s == 1.0).all()
    assert quant.round_half_away(np.array([2.5, -2.5, 0.5, 1.49])).tolist() == [3.0, -3.0, 1.0, 1.0]


@pytest.mark.parametrize("bits", [2, 3, 4])
def test_half_step_bound_tight(bits):
    # |W - Ŵ| <= scale/2 elementwise; tight (ratio -> 1) on random weights
    w = synth.rng(10 + bits).standard_normal((64, 256)) * 0.02
    c, s = quant.rtn_quantize(w, bits, 128)
    res = np.abs(w - quant.rtn_dequantize(c, s, 128))
    half = np.repeat(s, 128, axis=1) / 2
    ratio = (res / half).max()
    assert ratio <= 1.0 + 1e-12 and ratio > 0.98
    # S:149 idempotence of quantize∘dequantize on codes
    c2, _ = quant.rtn_quantize(quant.rtn_dequantize(c, s, 128), bits, 128)
    assert np.array_equal(c, c2)


def test_dequant_hand_group():
    q = np.arange(16)[None, :]
    W = quant.dequant(q, np.array([[0.5, 2.0]]), np.array([[8, 3]]), 8)
    exp = [0.5 * (k - 8) for k in range(8)] + [2.0 * (k - 3) for k in range(8, 16)]
    assert W[0].tolist() == exp


# ------------------------------------------------------------------ factors (c4)
def test_eckart_young_diag(golden):
    for key in ("eckart_young_r1", "eckart_young_r2"):
        e = golden[key]
        M = np.diag(np.array(e["diag"], dtype=np.float64))
        U, V, _ = factors.svd_factors(M, e["r"])
        assert abs(factors.frobenius_sq(M - U @ V) - e["err_sq"]) < 1e-12


def test_eckart_young_random_and_monotone():
    # SPEC acceptance 1: ||ΔW - U_r V_r||² = Σ_{j>r} σ_j², and monotone in r
    for seed in range(10):
        M = synth.rng(100 + seed).standard_normal((64, 64))
        prev = np.inf
        for r in (0, 8, 16, 32, 64):
            U, V, sig = factors.svd_factors(M, r)
            err = factors.frobenius_sq(M - U @ V)
            tail = float(np.sum(sig[r:] ** 2))
            assert abs(err - tail) <= 1e-9 * max(1.0, factors.frobenius_sq(M))
            assert err <= prev + 1e-12
            prev = err


@pytest.mark.parametrize("bits", [2, 3, 4])
def test_full_rank_reconstructs_W(bits):
    # north_star: "exact reconstruction of W when the error SVD is kept at full rank"
    W = synth.rng(7).standard_normal((96, 128)) * 0.02
    c, s = quant.rtn_quantize(W, bits, 128)
    W_hat = quant.rtn_dequantize(c, s, 128)
    U, V, _ = factors.svd_factors(W - W_hat, 96)
    assert np.abs(W_hat + U @ V - W).max() <= 1e-14 * 96


def test_rank_prefix_and_sign_convention():
    M = synth.rng(3).standard_normal((40, 30))
    U30, V30, _ = factors.svd_factors(M, 30)
    U8, V8, _ = factors.svd_factors(M, 8)
    assert np.array_equal(U30[:, :8], U8) and np.array_equal(V30[:8], V8)
    for j in range(8):
        nz = np.flatnonzero(U8[:, j])
        assert U8[nz[0], j] > 0
    with pytest.raises(ValueError):
        factors.svd_factors(M, 31)


# ------------------------------------------------------------------ compensated product (c5)
def _brute_linear(case, r):
    """Element-by-element construction from the definition, independent of the
    vectorised oracle: per (b, n) a Python loop over k, extracting each code from a
    Python big-int stream."""
    N, K, bits, g = case["N"], case["K"], case["bits"], case["group"]
    f = lambda u16: float(np.uint32(int(u16) << 16).view(np.float32))
    out = np.zeros((case["B"], N))
    for n in range(N):
        stream = 0
        for w in range(K * bits // 32):
            stream |= int(case["codes"][n, w]) << (32 * w)
        for b in range(case["B"]):
            acc = 0.0
            for k in range(K):
                q = (stream >> (bits * k)) & ((1 << bits) - 1)
                acc += f(case["scales"][n, k // g]) * (q - int(case["zeros"][n, k // g])) * f(case["x"][b, k])
            t = [sum(f(case["V"][j, k]) * f(case["x"][b, k]) for k in range(K)) for j in range(r)]
            acc += sum(f(case["U"][n, j]) * t[j] for j in range(r))
            out[b, n] = acc
    return out


@pytest.mark.parametrize("bits,zeros", [(4, "sym"), (3, "asym"), (2, "asym")])
def test_compensated_linear_matches_brute_force(bits, zeros):
    case = synth.linear_case(5, N=6, K=256, bits=bits, group=128, r_stored=16, B=2, zeros=zeros)
    for r in (0, 8, 16):
        y = linear.compensated_linear(case, r)
        yb = _brute_linear(case, r)
        assert np.abs(y - yb).max() <= 1e-12 * max(1.0, np.abs(yb).max())


def test_rank0_equals_plain_quantized_product():
    # S:226 / S:730: rank 0 equals the plain quantised product exactly
    case = synth.linear_case(1, N=64, K=256, bits=4, r_stored=16, B=3)
    W_hat = linear.deq_weight(case["codes"], case["scales"], case["zeros"], 256, 4, 128)
    x = packing.bf16_to_f64(case["x"])
    assert np.array_equal(linear.compensated_linear(case, 0), x @ W_hat.T)


def test_full_rank_factors_give_W_x_and_association():
    # full-rank factors -> X·ΔW;  S:231: (Vx)U == x(UV) (association equivalence)
    W = synth.rng(11).standard_normal((48, 128)) * 0.02
    c, s = quant.rtn_quantize(W, 3, 128)
    W_hat = quant.rtn_dequantize(c, s, 128)
    U, V, _ = factors.svd_factors(W - W_hat, 48)
    x = synth.rng(12).standard_normal((4, 128))
    y = linear.compensated_product(W_hat, U, V, 48, x)
    assert np.abs(y - x @ W.T).max() <= 1e-12
    assert np.abs(linear.compensated_product(W_hat, U, V, 16, x) - x @ (W_hat + U[:, :16] @ V[:16]).T).max() <= 1e-12


def test_round_bf16_matches_fp32_route():
    # bf16 RNE of float64 values that are exactly float32-representable equals the
    # classic fp32 bit trick (independent construction)
    a = synth.rng(2).standard_normal(10000).astype(np.float32).astype(np.float64)
    r = linear.round_bf16(a)
    bits = packing.f64_to_bf16_bits_rne(a)
    assert np.array_equal(r, packing.bf16_to_f64(bits))
    assert linear.round_bf16(np.array([1.0 + 2.0 ** -8]))[0] == 1.0          # tie -> even
    assert linear.round_bf16(np.array([1.0 + 3 * 2.0 ** -8]))[0] == 1.0 + 2.0 ** -6


def _silu_ref(v):
    # independent SiLU: v·σ(v) with the library logistic (scipy.special.expit), not oracle.linear.silu
    from scipy.special import expit
    return np.asarray(v, np.float64) * expit(np.asarray(v, np.float64))


def test_silu_closed_forms():
    # SiLU(v) = v·σ(v) ("σ(W_gate X)", SPEC's σ = SiLU): closed forms that catch a dropped term,
    # a sign flip or a wrong exponent.  σ(ln 3) = 3/4, σ(-ln 3) = 1/4; silu(v) - silu(-v) = v (σ(v) +
    # σ(-v) = 1); silu(0) = 0, silu(h) = h/2 + h²/4 + O(h⁴); silu(v) -> v for large v and -> 0 for very negative v.
    L3 = np.log(3.0)
    assert linear.silu(np.array([0.0]))[0] == 0.0
    assert abs(linear.silu(np.array([L3]))[0] - 0.75 * L3) <= 1e-15
    assert abs(linear.silu(np.array([-L3]))[0] + 0.25 * L3) <= 1e-15
    v = synth.rng(77).standard_normal(1000) * 6
    assert np.abs(linear.silu(v) - linear.silu(-v) - v).max() <= 1e-13
    assert abs(linear.silu(np.array([1e-8]))[0] - (0.5e-8 + 0.25e-16)) <= 1e-23     # h/2 + h²/4 + O(h⁴)
    assert abs(linear.silu(np.array([40.0]))[0] - 40.0) <= 1e-14 * 40 and abs(linear.silu(np.array([-40.0]))[0]) < 1e-15
    assert np.abs(linear.silu(v) - _silu_ref(v)).max() <= 1e-14


def test_window_linear_member_order_and_widths():
    # App. A.1.3: members sharing x run as one window; the output is the concatenation of the
    # members' compensated products in member order, each at its own rank and width.  Checked column block
    # by column block against the element-by-element brute force (_brute_linear, independent of oracle code).
    cases = [synth.linear_case(60 + i, N=n, K=256, bits=b, r_stored=16, B=2, zeros="asym")
             for i, (n, b) in enumerate(((6, 4), (2, 4), (4, 4)))]
    x = cases[0]["x"]
    for c in cases:
        c["x"] = x
    ranks = [8, 0, 16]
    y = linear.window_linear(cases, ranks, x)
    assert y.shape == (2, 12)
    off = 0
    for c, r in zip(cases, ranks):
        yb = _brute_linear(c, r)
        assert np.abs(y[:, off:off + c["N"]] - yb).max() <= 1e-12 * max(1.0, np.abs(yb).max())
        off += c["N"]


def test_moe_single_expert_equals_dense():
    # SPEC toymodel example: MoE with one expert, g = 1 == dense FFN (SiLU from the library logistic)
    d, f = 128, 128
    up = synth.linear_case(20, f, d, 3, 128, 16, 1, "asym")
    gate = synth.linear_case(21, f, d, 3, 128, 16, 1, "asym")
    down = synth.linear_case(22, d, f, 3, 128, 16, 1, "asym")
    x = synth.activations(23, 5, d)
    y = linear.moe_forward([dict(up=up, gate=gate, down=down)], [dict(up=8, gate=0, down=16)],
                           x, np.zeros((5, 1), np.int32), np.ones((5, 1), np.float32))
    xf = packing.bf16_to_f64(x)
    m = linear.round_bf16(_silu_ref(linear._lin(gate, 0, xf)) * linear._lin(up, 8, xf))
    assert np.allclose(y, linear._lin(down, 16, m), rtol=0, atol=1e-12 * np.abs(y).max())


def test_moe_gate_linearity_two_identical_experts():
    # P:852 Y = Σ_e g_e E_e(X): two copies of one expert routed with gates (g, 1 - g) equal the dense FFN,
    # and a single expert with gate g scales its output by exactly g (float64 weighting)
    d, f = 128, 128
    up = synth.linear_case(30, f, d, 4, 128, 16, 1, "asym")
    gate = synth.linear_case(31, f, d, 4, 128, 16, 1, "asym")
    down = synth.linear_case(32, d, f, 4, 128, 16, 1, "asym")
    ex = dict(up=up, gate=gate, down=down)
    r = dict(up=16, gate=8, down=0)
    x = synth.activations(33, 4, d)
    one = linear.moe_forward([ex], [r], x, np.zeros((4, 1), np.int32), np.ones((4, 1), np.float32))
    g = np.float32(0.375)                                             # exact in binary: no rounding in g, 1-g
    two = linear.moe_forward([ex, ex], [r, r], x, np.array([[0, 1]] * 4, np.int32),
                             np.array([[g, 1 - g]] * 4, np.float32))
    assert np.allclose(two, one, rtol=1e-14, atol=0)
    half = linear.moe_forward([ex], [r], x, np.zeros((4, 1), np.int32), np.full((4, 1), g, np.float32))
    assert np.array_equal(half, one * float(g))


def test_dynamic_rank_rule_worked_examples():
    # G = k·g, r̃ = G·r̃_i, Align ties up (R14), cap to the largest level <= cap (R15)
    assert linear.dynamic_rank(2, 0.75, 16.0, 64) == 32          # 24 is the 16/32 midpoint: ties up
    assert linear.dynamic_rank(2, 0.75, 16.0, 16) == 16          # capped
    assert linear.dynamic_rank(8, 0.125, 40.0, 64) == 32         # k·g = 1 leaves r̃ = 40 -> 32
    assert linear.dynamic_rank(8, 0.01, 40.0, 64) == 0           # 3.2 < 4 -> 0
    assert linear.dynamic_rank(4, 0.5, 3.0, 64) == 8             # 6 -> nearest of {0, 8}: 8
    assert linear.dynamic_rank(1, 1.0, 300.0, 48) == 32          # 256 aligned, cap 48 -> 32


# (k, g, r̃, exact rank, what an fp32 product would give): the exact product sits just below an Align
# midpoint (48, 96, 12) while its fp32 rounding lands ON the midpoint and ties up (found by search)
DYN_EXACT_CASES = [(9, 0.7322015762329102, 7.283968448638916, 32, 64),
                   (5, 0.012711115181446075, 1510.489013671875, 64, 128),
                   (2, 0.42846035957336426, 14.003628730773926, 8, 16)]


def _align_exact(rt, k0=3):
    from fractions import Fraction
    lo, hi = Fraction(0), Fraction(1 << k0)
    while rt >= hi:
        lo, hi = hi, hi * 2
    return int(lo) if (rt - lo) < (hi - rt) else int(hi)


def test_dynamic_rank_is_exact_arithmetic():
    # R21: (k·g)·r̃ is exact in float64 for fp32 g, r̃ and k <= 16, so the decision equals the one taken
    # in exact rational arithmetic (fractions.Fraction); an fp32 product would flip these ties
    from fractions import Fraction
    for k, g, rt, exact, f32 in DYN_EXACT_CASES:
        assert np.float32(g) == g and np.float32(rt) == rt
        assert linear.dynamic_rank(k, np.float32(g), np.float32(rt), 256) == exact
        assert _align_exact(Fraction(float(np.float32(np.float32(k) * np.float32(g)) * np.float32(rt)))) == f32
    r = synth.rng(78)
    for _ in range(3000):
        k = int(r.integers(1, 17))
        g = np.float32(r.uniform(0, 1))
        rt = np.float32(r.uniform(0, 300))
        ex = Fraction(k) * Fraction(float(g)) * Fraction(float(rt))
        assert float(k) * float(g) * float(rt) == ex                       # no rounding in float64
        cap = int(r.choice([0, 8, 16, 48, 64, 256]))
        lv = _align_exact(ex)
        want = lv if lv <= cap else max([0] + [v for v in (8, 16, 32, 64, 128, 256) if v <= cap])
        assert linear.dynamic_rank(k, g, rt, cap) == want


def test_moe_dynamic_reduces_to_static_and_zero():
    d, f = 128, 128
    mk = lambda s: synth.linear_case(40 + s, 128, 128, 3, 128, 16, 1, "asym")
    ex = [dict(up=mk(0), gate=mk(1), down=mk(2)), dict(up=mk(3), gate=mk(4), down=mk(5))]
    caps = [dict(up=16, gate=8, down=16), dict(up=8, gate=16, down=0)]
    x = synth.activations(46, 3, d)
    idx = np.array([[0, 1], [1, 0], [0, 1]], np.int32)
    gate = np.array([[0.5, 0.5], [0.75, 0.25], [0.625, 0.375]], np.float32)
    big = [dict(up=1e6, gate=1e6, down=1e6)] * 2                 # every rank saturates at its cap
    dyn = linear.moe_forward_dynamic(ex, caps, x, idx, gate, big)
    stat = linear.moe_forward(ex, caps, x, idx, gate)
    assert np.allclose(dyn, stat, rtol=1e-13, atol=1e-13)
    zero = linear.moe_forward_dynamic(ex, caps, x, idx, gate, [dict(up=0.0, gate=0.0, down=0.0)] * 2)
    z_stat = linear.moe_forward(ex, [dict(up=0, gate=0, down=0)] * 2, x, idx, gate)
    assert np.allclose(zero, z_stat, rtol=1e-13, atol=1e-13)


def test_e4m3_decode_pins():
    """OCP E4M3 by hand: zero, the smallest subnormal 2^-9, the largest subnormal 7·2^-9,
    the smallest normal 2^-6, 1.0, 1.875, 2.0, the largest finite 448, signed zero, -1, NaN; the codes
    0x00..0x7E increase strictly and within a binade step by 2^(e-10)."""
    from oracle.packing import e4m3_to_f64
    vals = e4m3_to_f64(np.array([0x00, 0x01, 0x07, 0x08, 0x38, 0x3F, 0x40, 0x7E, 0x80, 0xB8], dtype=np.uint8))
    assert list(vals) == [0.0, 2.0 ** -9, 7 * 2.0 ** -9, 2.0 ** -6, 1.0, 1.875, 2.0, 448.0, 0.0, -1.0]
    assert np.signbit(vals[8])
    assert np.isnan(e4m3_to_f64(np.array([0x7F, 0xFF], dtype=np.uint8))).all()
    pos = e4m3_to_f64(np.arange(0x7F, dtype=np.uint8))
    assert np.all(np.diff(pos) > 0)
    for c in range(8, 0x7E):
        e = c >> 3
        if (c & 7) != 7:
            assert pos[c + 1] - pos[c] == 2.0 ** (e - 10)
    assert np.array_equal(e4m3_to_f64(np.arange(0x80, 0xFF, dtype=np.uint8)), -pos)


def test_fp8_factor_product_definition():
    """The fp8 compensated product is the bf16 one with U_eff = e4m3(U8)·us, V_eff = e4m3(V8)·vs: when every
    byte is a power-of-two code and the scales are 1, U_eff / V_eff equal bf16 factors holding the same values,
    so both oracle paths agree exactly."""
    from oracle import linear
    from oracle.packing import e4m3_to_f64, f64_to_bf16_bits_rne
    case = synth.linear_case(5, N=32, K=128, bits=4, r_stored=16)
    g = np.random.default_rng(1)
    U8 = (g.integers(0, 2, (32, 16)) << 7 | g.integers(3, 12, (32, 16)) << 3).astype(np.uint8)
    V8 = (g.integers(0, 2, (16, 128)) << 7 | g.integers(3, 12, (16, 128)) << 3).astype(np.uint8)
    f8 = dict(case, factor_dtype="fp8", U8=U8, V8=V8, us=np.ones(16, np.float32), vs=np.ones(16, np.float32))
    bf = dict(case, U=f64_to_bf16_bits_rne(e4m3_to_f64(U8)), V=f64_to_bf16_bits_rne(e4m3_to_f64(V8)))
    for r in (0, 8, 16):
        assert np.array_equal(linear.compensated_linear(f8, r), linear.compensated_linear(bf, r))
