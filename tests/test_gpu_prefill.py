"""GPU parity of the tcgen05 prefill path (hc_compensated_linear with B > 16) against the float64
oracle.  fp16 operands: X bf16 -> fp16 (exact in range), fp16(s·(q − z)) weights, T = X·Vᵀ rounded to
fp16, U in fp16; fp32 accumulation in TMEM.  Expected max|err|/max|ref| ~2e-4,
bar 2e-3 (north_star)."""
import numpy as np
import pytest

import synth
from oracle import linear
from oracle.packing import f64_to_bf16_bits_rne

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]

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


def desc(case, layer, window, slot, r):
    return dict(layer=layer, window=window, slot=slot, N=case["N"], K=case["K"], bits=case["bits"],
                codes=dev(case["codes"]), scales=dev(case["scales"]), zeros=dev(case["zeros"]),
                U=dev(case["U"]), V=dev(case["V"]), r_stored=case["r_stored"], r_alloc=r)


def rel(y, ref):
    return np.abs(y - ref).max() / np.abs(ref).max()


_layer = [500]


def nl():
    _layer[0] += 1
    return _layer[0]


@pytest.mark.parametrize("M", [17, 128, 200, 300])
@pytest.mark.parametrize("zeros", ["sym", "asym"])
def test_prefill_single_matrix(hc, ctx, M, zeros):
    case = synth.linear_case(600 + M, N=512, K=1024, bits=4, r_stored=128, B=M, zeros=zeros)
    L = nl()
    for r in (0, 8, 64, 128):
        ctx.load_layer([desc(case, L, 0, 0, r)])
        y = torch.empty((M, 512), dtype=torch.float32, device="cuda")
        ctx.compensated_linear(L, 0, dev(case["x"]), y)
        torch.cuda.synchronize()
        y = y.cpu().numpy()
        ref = linear.compensated_linear(case, r)
        assert rel(y, ref) <= TOL, (r, rel(y, ref))


def test_prefill_window_bf16_and_rank_effect(hc, ctx):
    M, K = 256, 2048
    cases = [synth.linear_case(700 + i, N=n, K=K, bits=4, r_stored=64, B=M, zeros="asym")
             for i, n in enumerate((512, 256, 256))]
    ranks = (64, 0, 16)
    L = nl()
    for s, (c, r) in enumerate(zip(cases, ranks)):
        ctx.load_layer([desc(c, L, 0, s, r)])
    x = dev(cases[0]["x"])
    y = torch.empty((M, 1024), dtype=torch.float32, device="cuda")
    yb = torch.empty((M, 1024), dtype=torch.int16, device="cuda")
    ctx.compensated_linear(L, 0, x, y)
    ctx.compensated_linear(L, 0, x, yb, out_dtype=hc.OUT_BF16)
    torch.cuda.synchronize()
    y = y.cpu().numpy()
    ref = linear.window_linear(cases, list(ranks), cases[0]["x"])
    assert rel(y, ref) <= TOL
    assert np.array_equal(yb.cpu().numpy().view(np.uint16), f64_to_bf16_bits_rne(y))
    # the compensation is visible: the r = 0 oracle is clearly worse than the kernel
    ref0 = linear.window_linear(cases, [0, 0, 0], cases[0]["x"])
    assert rel(y, ref0) > 10 * rel(y, ref)


def test_prefill_c4_shape_sampled(hc, ctx):
    # BASELINE C4: 2048 tokens through a Llama-3-8B-shaped o_proj (4096 x 4096), 4-bit, r = 64;
    # the full output is computed on the GPU, the oracle checks 64 sampled token rows
    M, N, K = 2048, 4096, 4096
    case = synth.linear_case(800, N=N, K=K, bits=4, r_stored=64, B=M, zeros="asym")
    L = nl()
    ctx.load_layer([desc(case, L, 0, 0, 64)])
    y = torch.empty((M, N), dtype=torch.float32, device="cuda")
    ctx.compensated_linear(L, 0, dev(case["x"]), y)
    torch.cuda.synchronize()
    rows = synth.rng(1).choice(M, size=64, replace=False)
    ref = linear.compensated_linear(case, 64, x_bits=case["x"][rows])
    assert rel(y.cpu().numpy()[rows], ref) <= TOL


def test_prefill_merged_window_matches_per_member(hc, ctx):
    """A multi-member window runs as ONE GEMM (rows concatenated, rank slices stacked, block-diagonal U);
    it must agree with the oracle, with the per-member launches (option prefill_merge = 0), and follow rank
    changes (the merged copies are rebuilt)."""
    M, K = 384, 1024
    cases = [synth.linear_case(800 + i, N=n, K=K, bits=4, r_stored=32, B=M, zeros="asym")
             for i, n in enumerate((512, 256, 256))]
    L = nl()
    for ranks in ((32, 8, 0), (0, 16, 32)):
        for s, (c, r) in enumerate(zip(cases, ranks)):
            ctx.load_layer([desc(c, L, 0, s, r)])
        x = dev(cases[0]["x"])
        y = torch.empty((M, 1024), dtype=torch.float32, device="cuda")
        ctx.compensated_linear(L, 0, x, y)
        hc.set_option("prefill_merge", 0)
        try:
            y2 = torch.empty_like(y)
            ctx.compensated_linear(L, 0, x, y2)
        finally:
            hc.set_option("prefill_merge", 1)
        torch.cuda.synchronize()
        ref = linear.window_linear(cases, list(ranks), cases[0]["x"])
        assert rel(y.cpu().numpy(), ref) <= TOL
        assert rel(y.cpu().numpy(), y2.cpu().numpy()) <= 1e-6
    # rank change through hc_set_rank rebuilds the merged rank slice
    ctx.set_rank(L, 0, 0, 8)
    y = torch.empty((M, 1024), dtype=torch.float32, device="cuda")
    ctx.compensated_linear(L, 0, dev(cases[0]["x"]), y)
    torch.cuda.synchronize()
    assert rel(y.cpu().numpy(), linear.window_linear(cases, [8, 16, 32], cases[0]["x"])) <= TOL


@pytest.mark.parametrize("kind", ["zero", "tiny", "outlier", "wide"])
def test_prefill_full_bf16_range(hc, ctx, kind):
    """Prefill (tcgen05) with activations outside fp16's exact band: the per-token power-of-two prescale
    of X (R20) keeps every row within the bar at its own scale; an all-zero X gives exactly zero."""
    M, N, K = 200, 512, 1024
    case = synth.linear_case(1200 + len(kind), N=N, K=K, bits=4, r_stored=64, B=M, zeros="asym")
    g = np.random.default_rng(len(kind))
    if kind == "zero":
        x = np.zeros((M, K))
    elif kind == "tiny":
        x = g.standard_normal((M, K)) * 1e-12
    elif kind == "outlier":
        x = g.standard_normal((M, K))
        x[:, 7] = 7.0e4
        x[::3, 500] = -3.0e5
        x[::5, 900] = 2.0e6
    else:
        x = g.standard_normal((M, K)) * 10.0 ** g.uniform(-12, 7, (M, 1)) * 10.0 ** g.uniform(-2, 2, (M, K))
    case["x"] = f64_to_bf16_bits_rne(x)
    L = nl()
    for r in (0, 64):
        ctx.load_layer([desc(case, L, 0, 0, r)])
        y = torch.empty((M, N), dtype=torch.float32, device="cuda")
        ctx.compensated_linear(L, 0, dev(case["x"]), y)
        torch.cuda.synchronize()
        y = y.cpu().numpy()
        assert np.all(np.isfinite(y))
        if kind == "zero":
            assert np.all(y == 0.0)
            continue
        ref = linear.compensated_linear(case, r)
        worst = max(np.abs(y[m] - ref[m]).max() / np.abs(ref[m]).max() for m in range(M))
        assert worst <= TOL, (r, worst)


@pytest.mark.parametrize("r", [128, 256])
def test_prefill_high_rank(hc, ctx, r):
    """Rank 128 and 256 (C4's rank sweep reaches 256): the rank slice is a 256-wide K extension."""
    M, N, K = 160, 512, 1024
    case = synth.linear_case(1300 + r, N=N, K=K, bits=4, r_stored=256, B=M, zeros="asym")
    L = nl()
    ctx.load_layer([desc(case, L, 0, 0, r)])
    y = torch.empty((M, N), dtype=torch.float32, device="cuda")
    ctx.compensated_linear(L, 0, dev(case["x"]), y)
    torch.cuda.synchronize()
    ref = linear.compensated_linear(case, r)
    assert rel(y.cpu().numpy(), ref) <= TOL
    assert rel(y.cpu().numpy(), linear.compensated_linear(case, r // 2)) > 3 * rel(y.cpu().numpy(), ref)
