"""fp8 (e4m3) compensation factors on the GPU against the float64 oracle fed the same
e4m3 bytes and fp32 per-rank scales (oracle.linear.factors_f64): decode windows (int8 and fp16 paths,
multi-member, fused SiLU, stack), every non-NaN code, prefill (fp16 copies of U_eff / V_eff) and the load
errors."""
import numpy as np
import pytest

import synth
from oracle import linear
from oracle.packing import bf16_to_f64

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hc():
    import paper_2605_05819_b200 as m
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return m


@pytest.fixture(scope="module")
def ctx(hc):
    return hc.Context(0)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


_L = [3000]


def next_layer():
    _L[0] += 1
    return _L[0]


def desc8(hc, case, layer, window, slot, r, glue=0, host=False):
    t = (lambda a: np.ascontiguousarray(a)) if host else dev
    return dict(layer=layer, window=window, slot=slot, N=case["N"], K=case["K"], bits=case["bits"],
                codes=t(case["codes"]), scales=t(case["scales"]), zeros=t(case["zeros"]),
                U=t(case["U8"]), V=t(case["V8"]), u_scale=t(case["us"]), v_scale=t(case["vs"]),
                factor_dtype=hc.FACTORS_FP8, r_stored=case["r_stored"], r_alloc=r, glue=glue)


def rel(y, ref):
    return np.abs(y - ref).max() / np.abs(ref).max()


@pytest.mark.parametrize("bits,B,K", [(4, 1, 1024), (2, 2, 1280), (4, 4, 640), (3, 1, 1024), (3, 16, 640),
                                      (4, 1, 11008)])
@pytest.mark.parametrize("r", [16, 64, 128])
def test_fp8_window_parity(hc, ctx, bits, B, K, r):
    """One 3-member window (q/k/v-like) with e4m3 factors: every path (int8 at B <= 2 for 2/4-bit, fp16 else,
    x staged or x-prep at K = 11008) within 1e-5 of the float64 oracle at the window's scale; r = 0 equals
    the uncompensated product exactly."""
    cases = [synth.fp8_factors(synth.linear_case(600 + bits * 10 + B + i, N=n, K=K, bits=bits, r_stored=128, B=B,
                                                 zeros="asym"), 700 + i) for i, n in enumerate((256, 128, 128))]
    L = next_layer()
    ranks = (r, r // 2, 0)
    ctx.load_layer([desc8(hc, c, L, 0, s, rr) for s, (c, rr) in enumerate(zip(cases, ranks))])
    y = torch.empty((B, 512), dtype=torch.float32, device="cuda")
    ctx.compensated_linear(L, 0, dev(cases[0]["x"]), y)
    torch.cuda.synchronize()
    ref = linear.window_linear(cases, list(ranks), cases[0]["x"])
    assert rel(y.cpu().numpy(), ref) <= 1e-5, rel(y.cpu().numpy(), ref)
    # the compensation is really applied (r matters)
    ref0 = linear.window_linear(cases, [0, 0, 0], cases[0]["x"])
    assert rel(ref0, ref) > 100 * rel(y.cpu().numpy(), ref)


def test_fp8_every_code(hc, ctx):
    """U8 / V8 cycling through all 254 non-NaN codes (normals, subnormals, ±0): the in-register e4m3 -> bf16
    conversion is exact for each (the product matches the oracle to fp32 accumulation)."""
    case = synth.fp8_factors(synth.linear_case(650, N=256, K=512, bits=4, r_stored=64, B=2, zeros="asym"), 651,
                             all_codes=True)
    L = next_layer()
    ctx.load_layer([desc8(hc, case, L, 0, 0, 64)])
    y = torch.empty((2, 256), dtype=torch.float32, device="cuda")
    ctx.compensated_linear(L, 0, dev(case["x"]), y)
    torch.cuda.synchronize()
    ref = linear.compensated_linear(case, 64)
    assert rel(y.cpu().numpy(), ref) <= 1e-5


@pytest.mark.parametrize("bits,B", [(4, 1), (3, 5)])
def test_fp8_fused_silu(hc, ctx, bits, B):
    up = synth.fp8_factors(synth.linear_case(660 + bits, N=384, K=640, bits=bits, r_stored=32, B=B, zeros="asym",
                                             unit_gain=True), 661)
    gate = synth.fp8_factors(synth.linear_case(670 + bits, N=384, K=640, bits=bits, r_stored=32, B=B, zeros="asym",
                                               unit_gain=True), 671)
    L = next_layer()
    ctx.load_layer([desc8(hc, up, L, hc.UPGATE, 0, 32, hc.GLUE_SILU_MUL), desc8(hc, gate, L, hc.UPGATE, 1, 16, hc.GLUE_SILU_MUL)])
    y = torch.empty((B, 384), dtype=torch.float32, device="cuda")
    ctx.compensated_linear(L, hc.UPGATE, dev(up["x"]), y)
    torch.cuda.synchronize()
    u = linear.compensated_linear(up, 32)
    g = linear.compensated_linear(gate, 16, x_bits=up["x"])
    ref = linear.silu(g) * u
    assert rel(y.cpu().numpy(), ref) <= 1e-5


def test_fp8_stack(hc):
    """A 2-layer decode stack with e4m3 factors in every window, per element within the stack bound."""
    STACK_GAINS = (1.0, 1.0, 1.0, 0.25, 0.25, 0.25, 0.05)
    d, kv, f, L = 256, 128, 512, 2
    layers, ranks = [], []
    for l in range(L):
        c = lambda n, k, s: synth.fp8_factors(synth.linear_case(680 + l * 10 + s, N=n, K=k, bits=4, r_stored=32,
                                                                zeros="asym", unit_gain=STACK_GAINS[s]), 690 + l * 10 + s)
        layers.append(dict(qkv=[c(d, d, 0), c(kv, d, 1), c(kv, d, 2)], o=[c(d, d, 3)], upgate=[c(f, d, 4), c(f, d, 5)],
                           down=[c(d, f, 6)]))
        ranks.append(dict(qkv=[32, 16, 0], o=[16], upgate=[32, 8], down=[16]))
    ctx = hc.Context(0)
    for l, (L_, R_) in enumerate(zip(layers, ranks)):
        mats = [desc8(hc, L_["qkv"][i], l, hc.QKV, i, R_["qkv"][i]) for i in range(3)]
        mats += [desc8(hc, L_["o"][0], l, hc.O, 0, R_["o"][0])]
        mats += [desc8(hc, L_["upgate"][i], l, hc.UPGATE, i, R_["upgate"][i], hc.GLUE_SILU_MUL) for i in range(2)]
        mats += [desc8(hc, L_["down"][0], l, hc.DOWN, 0, R_["down"][0])]
        ctx.load_layer(mats)
    x = synth.activations(9, 2, d)
    y = torch.empty((2, d), dtype=torch.int16, device="cuda")
    ctx.stack_forward(dev(x), y)
    torch.cuda.synchronize()
    ref = linear.stack_forward(layers, ranks, x)
    yv = bf16_to_f64(y.cpu().numpy().view(np.uint16))
    assert np.all(np.abs(yv - ref) <= 2e-3 * np.abs(ref).max() + np.abs(ref) * 2.0 ** -6 * L)
    ctx.close()


def test_fp8_prefill(hc, ctx):
    """B = 96 runs the tcgen05 prefill on fp16 copies of U_eff / V_eff (one fp16 rounding each): 2e-3."""
    case = synth.fp8_factors(synth.linear_case(700, N=512, K=1024, bits=4, r_stored=64, B=96, zeros="asym"), 701)
    L = next_layer()
    ctx.load_layer([desc8(hc, case, L, 0, 0, 64)])
    y = torch.empty((96, 512), dtype=torch.float32, device="cuda")
    ctx.compensated_linear(L, 0, dev(case["x"]), y)
    torch.cuda.synchronize()
    ref = linear.compensated_linear(case, 64)
    assert rel(y.cpu().numpy(), ref) <= 2e-3


def test_fp8_load_errors(hc, ctx):
    case = synth.fp8_factors(synth.linear_case(710, N=128, K=256, bits=4, r_stored=16), 711)
    bad = dict(case, U8=case["U8"].copy())
    bad["U8"][3, 5] = 0x7F                                   # NaN encoding
    with pytest.raises(hc.HCError) as e:
        ctx.load_layer([desc8(hc, bad, next_layer(), 0, 0, 16, host=True)])
    assert e.value.code == hc.HC_ERR_NUMERIC
    m = desc8(hc, case, next_layer(), hc.UPGATE, 0, 16, host=True)
    m["expert"] = 0                                          # MoE experts take bf16 factors
    with pytest.raises(hc.HCError) as e:
        ctx.load_layer([m])
    assert e.value.code == hc.HC_ERR_CONFIG
    m = desc8(hc, case, next_layer(), 0, 0, 16, host=True)
    m["u_scale"] = None
    with pytest.raises(hc.HCError):
        ctx.load_layer([m])
