"""GPU parity of the fused decode kernel (through the C-ABI) against the float64 oracle.

Bar (BASELINE.json north_star): max|y − y*| / max|y*| <= 2e-3 on fp32 output; bf16 output
bit-equal to RNE(fp32 output); r = 0 bit-identical to the uncompensated product; results
deterministic and identical across repeated launches (self-resetting counters)."""
import numpy as np
import pytest

import synth
from oracle import linear
from oracle.packing import bf16_to_f64, f64_to_bf16_bits_rne

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 2e-3


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


def load(ctx, case, layer, window=0, slot=0, r=0, expert=-1):
    ctx.load_layer([dict(layer=layer, window=window, slot=slot, expert=expert, N=case["N"], K=case["K"],
                         bits=case["bits"], codes=dev(case["codes"]), scales=dev(case["scales"]),
                         zeros=dev(case["zeros"]), U=dev(case["U"]) if case["r_stored"] else None,
                         V=dev(case["V"]) if case["r_stored"] else None, r_stored=case["r_stored"], r_alloc=r)])


def run(hc, ctx, layer, x_bits, rows, window=0, out=0):
    B = x_bits.shape[0]
    y = torch.empty((B, rows), dtype=torch.float32 if out == 0 else torch.int16, device="cuda")
    ctx.compensated_linear(layer, window, dev(x_bits), y, out_dtype=out)
    torch.cuda.synchronize()
    return y.cpu().numpy()


def rel_err(y, ref):
    return np.abs(y - ref).max() / np.abs(ref).max()


_layer = [100]


def next_layer():
    _layer[0] += 1
    return _layer[0]


@pytest.mark.parametrize("bits,zeros", [(4, "sym"), (4, "asym"), (3, "asym"), (3, "sym"), (2, "asym")])
@pytest.mark.parametrize("B", [1, 3, 8, 9, 16])
def test_single_matrix_parity(hc, ctx, bits, zeros, B):
    # 17 row blocks, 11 groups (uneven split over 8 warps), several V slices
    case = synth.linear_case(bits * 31 + B, N=272, K=1408, bits=bits, r_stored=64, B=B, zeros=zeros)
    L = next_layer()
    for r in (0, 8, 32, 64):
        load(ctx, case, L, r=r)
        y = run(hc, ctx, L, case["x"], 272)
        ref = linear.compensated_linear(case, r)
        assert rel_err(y, ref) <= TOL, (r, rel_err(y, ref))
        assert rel_err(y, ref) <= 1e-5      # exact products, fp32 accumulation (DESIGN R20)


def test_rank0_bit_identical_to_zero_compensation(hc, ctx):
    # r = 0 launch (no U/V reads) == r = 64 launch with U = 0 (compensation exactly 0)
    case = synth.linear_case(5, N=512, K=1024, bits=4, r_stored=64, B=4, zeros="asym")
    L = next_layer()
    load(ctx, case, L, r=0)
    y0 = run(hc, ctx, L, case["x"], 512)
    case0 = dict(case, U=np.zeros_like(case["U"]))
    load(ctx, case0, L, r=64)
    y64 = run(hc, ctx, L, case["x"], 512)
    assert np.array_equal(y0, y64)
    ref = linear.compensated_linear(case, 0)
    assert rel_err(y0, ref) <= 1e-5


def test_bf16_output_is_rne_of_fp32(hc, ctx):
    case = synth.linear_case(6, N=256, K=2048, bits=4, r_stored=32, B=5)
    L = next_layer()
    load(ctx, case, L, r=32)
    y32 = run(hc, ctx, L, case["x"], 256, out=0)
    y16 = run(hc, ctx, L, case["x"], 256, out=1).view(np.uint16)
    assert np.array_equal(y16, f64_to_bf16_bits_rne(y32))


def test_window_three_members_and_determinism(hc, ctx):
    L = next_layer()
    K = 1024
    cases = [synth.linear_case(40 + i, N=n, K=K, bits=4, r_stored=64, B=2, zeros="asym")
             for i, n in enumerate((512, 128, 128))]
    ranks = (64, 0, 16)
    for slot, (c, r) in enumerate(zip(cases, ranks)):
        load(ctx, c, L, window=0, slot=slot, r=r)
    assert ctx.window_rows(L, 0) == 768
    x = cases[0]["x"]
    y1 = run(hc, ctx, L, x, 768)
    y2 = run(hc, ctx, L, x, 768)
    y3 = run(hc, ctx, L, x, 768)
    assert np.array_equal(y1, y2) and np.array_equal(y2, y3)      # deterministic, counters reset
    ref = linear.window_linear(cases, list(ranks), x)
    assert rel_err(y1, ref) <= 1e-5


def test_host_buffers_path_equals_device_path(hc, ctx):
    case = synth.linear_case(8, N=256, K=1024, bits=3, r_stored=32, B=3, zeros="asym")
    L = next_layer()
    load(ctx, case, L, r=32)
    yd = run(hc, ctx, L, case["x"], 256)
    yh = np.zeros((3, 256), np.float32)
    ctx.compensated_linear(L, 0, np.ascontiguousarray(case["x"]), yh)     # host numpy in/out
    assert np.array_equal(yd, yh)


def test_c1_full_size_parity(hc, ctx):
    # BASELINE C1: 4096 x 4096, 4-bit g128, rank 64, batch 1 — the bench launch configuration
    for zeros in ("sym", "asym"):
        case = synth.linear_case(0, N=4096, K=4096, bits=4, r_stored=64, B=1, zeros=zeros)
        L = next_layer()
        load(ctx, case, L, r=64)
        y = run(hc, ctx, L, case["x"], 4096)
        ref = linear.compensated_linear(case, 64)
        assert rel_err(y, ref) <= 1e-5


def test_errors(hc, ctx):
    case = synth.linear_case(9, N=128, K=256, bits=4, r_stored=16, B=1)
    with pytest.raises(hc.HCError) as ei:
        ctx.load_layer([dict(layer=0, window=0, slot=0, N=120, K=256, bits=4, codes=dev(case["codes"]),
                             scales=dev(case["scales"]), zeros=dev(case["zeros"]))])
    assert ei.value.code == hc.HC_ERR_CONFIG
    with pytest.raises(hc.HCError) as ei:
        load(ctx, case, 999, r=24)                       # not admissible
    assert ei.value.code == hc.HC_ERR_CONFIG
    with pytest.raises(hc.HCError) as ei:
        ctx.compensated_linear(12345, 0, dev(case["x"]), torch.empty(1, 128, device="cuda"))
    assert ei.value.code == hc.HC_ERR_STATE


def _wide_range_x(seed, B, K):
    """bf16 x spanning ~12 decades within each group, one all-zero group, one group of values near
    the bf16 normal minimum, one group with a single large outlier (int8 path edge cases)."""
    g = np.random.default_rng(seed)
    x = g.standard_normal((B, K)) * 10.0 ** g.uniform(-9, 3, (B, K))
    x[:, 128:256] = 0.0                                    # all-zero group
    if K >= 512:
        x[:, 256:384] = g.standard_normal((B, 128)) * 1e-37   # tiny group (exponent clamp)
        x[:, 384:512] = g.standard_normal((B, 128)) * 1e-3
        x[:, 400] = 3.0e4                                  # outlier: the rest sits 2^24 below it
    return f64_to_bf16_bits_rne(x)


@pytest.mark.parametrize("bits,zeros", [(4, "asym"), (4, "sym"), (2, "asym")])
@pytest.mark.parametrize("B", [1, 2])
@pytest.mark.parametrize("K", [640, 1408])
def test_int8_path_edge_cases(hc, ctx, bits, zeros, B, K):
    """The int8 mma path (4-/2-bit, B <= 2, x staged): x in per-group block fixed
    point.  Wide-range, zero, tiny and outlier groups; K = 640 leaves three of the eight warps without
    groups; every result within 1e-5 of the float64 oracle (relative to max|y*|) and deterministic."""
    case = synth.linear_case(700 + 10 * bits + B, N=272, K=K, bits=bits, r_stored=32, B=B, zeros=zeros)
    case["x"] = _wide_range_x(K + B, B, K)
    L = next_layer()
    for r in (0, 16):
        load(ctx, case, L, r=r)
        y = run(hc, ctx, L, case["x"], 272)
        ref = linear.compensated_linear(case, r)
        assert np.all(np.isfinite(y))
        assert rel_err(y, ref) <= 1e-5, (r, rel_err(y, ref))
        assert np.array_equal(y, run(hc, ctx, L, case["x"], 272))


def _range_x(seed, B, K, kind):
    """bf16 x outside fp16's exact band (R20): all-zero rows, tiny rows (~1e-12, far below
    fp16's 2^-14), rows with outliers >= 65504 (up to 1e6), and a wide mix (each 128-group at its own
    scale 1e-12 .. 1e7, elements spread a further 1e±3 inside the group)."""
    g = np.random.default_rng(seed)
    if kind == "zero":
        x = np.zeros((B, K))
    elif kind == "tiny":
        x = g.standard_normal((B, K)) * 1e-12
    elif kind == "outlier":
        x = g.standard_normal((B, K))
        x[:, 5] = 7.0e4
        x[:, K // 3] = -2.5e5
        x[:, K - 3] = 1.0e6
    else:
        gs = 10.0 ** g.uniform(-12, 7, (B, K // 128, 1))
        x = (g.standard_normal((B, K // 128, 128)) * gs * 10.0 ** g.uniform(-3, 3, (B, K // 128, 128))).reshape(B, K)
    return f64_to_bf16_bits_rne(x)


def row_rel(y, ref):
    """max over batch rows of max|y_b - y*_b| / max|y*_b| (each row judged at its own scale)."""
    return max(np.abs(y[b] - ref[b]).max() / np.abs(ref[b]).max() for b in range(ref.shape[0]))


@pytest.mark.parametrize("bits,B,K", [(3, 4, 1408), (3, 16, 1408), (4, 4, 11008), (4, 16, 11008), (2, 8, 1408),
                                      (3, 1, 2560), (4, 1, 11008)])
@pytest.mark.parametrize("kind", ["zero", "tiny", "outlier", "wide"])
def test_fp16_path_full_bf16_range(hc, ctx, bits, B, K, kind):
    """The fp16 mma path (3-bit; B > 2; K = 11008 DOWN-shaped at B = 1, 4, 16; both the shared-memory
    staged x' and the x-prep kernel) accepts any bf16 x: per-(group, row) power-of-two prescale of x'
    (R20) and the two-word t accumulators (R22).  Each batch row within 1e-5 of the float64 oracle at its
    own scale; an all-zero x gives exactly zero."""
    case = synth.linear_case(900 + 7 * bits + B, N=272, K=K, bits=bits, r_stored=32, B=B, zeros="asym")
    case["x"] = _range_x(K + B + len(kind), B, K, kind)
    L = next_layer()
    for r in (0, 32):
        load(ctx, case, L, r=r)
        y = run(hc, ctx, L, case["x"], 272)
        assert np.all(np.isfinite(y))
        if kind == "zero":
            assert np.all(y == 0.0)
            continue
        ref = linear.compensated_linear(case, r)
        assert row_rel(y, ref) <= 1e-5, (r, row_rel(y, ref))
        assert np.array_equal(y, run(hc, ctx, L, case["x"], 272))


@pytest.mark.parametrize("bits,B", [(4, 1), (4, 2), (3, 4), (4, 16)])
def test_nonfinite_x_propagates(hc, ctx, bits, B):
    """A non-finite activation makes its batch row non-finite (as in float64, where inf·0 is NaN) on the
    int8 path (B <= 2) and the fp16 path; the other rows are unaffected."""
    case = synth.linear_case(950 + bits + B, N=144, K=1024, bits=bits, r_stored=16, B=B, zeros="asym")
    xb = case["x"].copy()
    xb[0, 300] = 0x7F80                      # +inf
    if B > 1:
        xb[B - 1, 17] = 0x7FC0               # NaN
    L = next_layer()
    load(ctx, case, L, r=16)
    y = run(hc, ctx, L, xb, 144)
    ref = linear.compensated_linear(case, 16, x_bits=xb)
    assert np.all(~np.isfinite(y[0])) and np.all(~np.isfinite(ref[0]))
    if B > 1:
        assert np.all(~np.isfinite(y[B - 1]))
    for b in range(1, B - 1):
        assert np.abs(y[b] - ref[b]).max() <= 1e-5 * np.abs(ref[b]).max()


@pytest.mark.parametrize("bits,B", [(4, 1), (2, 2), (4, 4), (3, 9)])
@pytest.mark.parametrize("r", [128, 256])
def test_high_rank_parity(hc, ctx, bits, B, r):
    """Ranks 128 and 256 (the largest admissible level): U chunks beyond the shared-memory prefetch are
    read from global memory; 16 rank chunks in the t accumulators."""
    case = synth.linear_case(970 + bits * 3 + B, N=288, K=1280, bits=bits, r_stored=256, B=B, zeros="asym")
    L = next_layer()
    load(ctx, case, L, r=r)
    y = run(hc, ctx, L, case["x"], 288)
    ref = linear.compensated_linear(case, r)
    assert rel_err(y, ref) <= 1e-5, rel_err(y, ref)
    ref_low = linear.compensated_linear(case, r // 2)
    assert rel_err(y, ref_low) > 10 * rel_err(y, ref)      # the top half of the ranks is really used


@pytest.mark.parametrize("scale", [1.0, 1e-9, 1e9])
@pytest.mark.parametrize("B", [1, 2])
def test_int8_two_epilogue_warps_multi_item(hc, ctx, scale, B):
    """Int8 path with several row-block items per CTA (decode grid capped at one CTA per SM): consecutive items
    alternate between the two epilogue warps (own reduction slot, U buffer and t fragments).
    Tiny / huge activations move the V·x partials out of tier 0 (below 2^-24 / above 2^12), so the lane-distributed
    extra-tier t pass runs (R22; tier 1 holds partials up to 2^50).  Within the oracle bound, and bit-identical to the full-grid launch (items on other CTAs / warps)."""
    case = synth.linear_case(70 + B, N=4096, K=512, bits=4, r_stored=32, B=B, zeros="asym")
    xf = bf16_to_f64(case["x"]) * scale
    case["x"] = f64_to_bf16_bits_rne(xf)
    L = next_layer()
    load(ctx, case, L, r=32)
    ref = linear.compensated_linear(case, 32)
    y_full = run(hc, ctx, L, case["x"], 4096)
    hc.set_option("decode_ctas_per_sm", 1)
    try:
        y_one = run(hc, ctx, L, case["x"], 4096)
    finally:
        hc.set_option("decode_ctas_per_sm", 0)
    assert row_rel(y_one, ref) <= 1e-5, row_rel(y_one, ref)
    assert np.array_equal(y_one, y_full)
