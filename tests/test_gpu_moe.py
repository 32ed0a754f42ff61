"""GPU parity of the grouped MoE expert path (hc_moe_forward, C3) against the float64 oracle
(oracle.linear.moe_forward): routed token batches over several experts, 3-bit weights with per-expert
compensation ranks, entries of > 16 rows per expert, host and device inputs, determinism."""
import numpy as np
import pytest

import synth
from oracle import linear

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hc():
    import paper_2605_05819_b200 as m
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def desc(case, layer, window, slot, expert, r, glue=0):
    return dict(layer=layer, window=window, slot=slot, expert=expert, N=case["N"], K=case["K"], bits=case["bits"],
                codes=dev(case["codes"]), scales=dev(case["scales"]), zeros=dev(case["zeros"]),
                U=dev(case["U"]), V=dev(case["V"]), r_stored=case["r_stored"], r_alloc=r, glue=glue)


def make_experts(E, d, f, bits, seed, r_stored=16):
    g = synth.rng(seed)
    experts, ranks = [], []
    for e in range(E):
        c = lambda n, k, s: synth.linear_case(seed * 100 + 3 * e + s, N=n, K=k, bits=bits, r_stored=r_stored,
                                              zeros="asym", unit_gain=synth.STACK_GAINS[4 + s])
        experts.append(dict(up=c(f, d, 0), gate=c(f, d, 1), down=c(d, f, 2)))
        lv = [0, 8, 16]
        ranks.append(dict(up=lv[int(g.integers(0, 3))], gate=lv[int(g.integers(0, 3))], down=lv[int(g.integers(0, 3))]))
    return experts, ranks


def load(hc, ctx, layer, experts, ranks):
    for e, (ex, r) in enumerate(zip(experts, ranks)):
        ctx.load_layer([desc(ex["up"], layer, hc.UPGATE, 0, e, r["up"], hc.GLUE_SILU_MUL),
                        desc(ex["gate"], layer, hc.UPGATE, 1, e, r["gate"], hc.GLUE_SILU_MUL),
                        desc(ex["down"], layer, hc.DOWN, 0, e, r["down"])])


@pytest.mark.parametrize("bits", [3, 4])
@pytest.mark.parametrize("T,topk", [(1, 2), (5, 3), (40, 2)])
def test_moe_forward_parity(hc, bits, T, topk):
    E, d, f = 6, 256, 384
    experts, ranks = make_experts(E, d, f, bits, seed=bits * 10 + T)
    ctx = hc.Context(0)
    load(hc, ctx, 0, experts, ranks)
    x = synth.activations(T + 3, T, d)
    idx, gate = synth.routing_case(T + 7, T, E, topk)
    y = torch.empty((T, d), dtype=torch.float32, device="cuda")
    ctx.moe_forward(0, dev(x), dev(idx), dev(gate), y)
    y2 = torch.empty_like(y)
    ctx.moe_forward(0, dev(x), dev(idx), dev(gate), y2)
    torch.cuda.synchronize()
    yc = y.cpu().numpy()
    assert np.array_equal(yc, y2.cpu().numpy())                     # deterministic
    ref = linear.moe_forward(experts, ranks, x, idx, gate)
    # m = bf16(silu(gate)·up) is a rounding point (R8): an fp32-vs-float64 flip of one m element
    # moves y by one bf16 ulp of m times a DOWN weight, far inside 2e-3·max|y|
    err = np.abs(yc - ref).max() / np.abs(ref).max()
    assert err <= 2e-3, err
    # host inputs / output through the same entry point
    yh = np.zeros((T, d), dtype=np.float32)
    ctx.moe_forward(0, np.ascontiguousarray(x), idx, gate, yh)
    assert np.array_equal(yh, yc)
    ctx.close()


def test_moe_rank_change_and_skipped_ids(hc):
    E, d, f = 4, 128, 256
    experts, ranks = make_experts(E, d, f, 3, seed=99)
    ctx = hc.Context(0)
    load(hc, ctx, 2, experts, ranks)
    T = 9
    x = synth.activations(5, T, d)
    idx, gate = synth.routing_case(6, T, E, 2)
    idx[0, 1] = E + 3                                               # outside [0, E): skipped
    y = torch.empty((T, d), dtype=torch.float32, device="cuda")
    for e in range(E):                                              # all ranks to 16 / 0 via hc_set_rank
        ctx.set_rank(2, hc.UPGATE, 0, 16, expert=e)
        ctx.set_rank(2, hc.DOWN, 0, 0, expert=e)
        ranks[e]["up"], ranks[e]["down"] = 16, 0
    ctx.moe_forward(2, dev(x), dev(idx), dev(gate), y)
    torch.cuda.synchronize()
    keep = idx < E
    ref = linear.moe_forward(experts, ranks, x, np.where(keep, idx, 0), np.where(keep, gate, 0.0).astype(np.float32))
    err = np.abs(y.cpu().numpy() - ref).max() / np.abs(ref).max()
    assert err <= 2e-3, err
    with pytest.raises(hc.HCError):
        ctx.moe_forward(7, dev(x), dev(idx), dev(gate), y)           # no experts on layer 7
    ctx.close()


@pytest.mark.parametrize("T,topk", [(6, 2), (40, 4)])
def test_moe_dynamic_ranks(hc, T, topk):
    """Per-(token, expert) ranks r = Cap(Align((k·g)·r̃)) (hc_moe_set_dynamic_ranks) against the oracle
    (oracle.linear.moe_forward_dynamic); huge r̃ reproduces the static path bit for bit; NULL restores it."""
    E, d, f = 5, 256, 256
    experts, _ = make_experts(E, d, f, 3, seed=123 + T)
    caps = [dict(up=16, gate=16, down=16) for _ in range(E)]
    ctx = hc.Context(0)
    load(hc, ctx, 1, experts, caps)
    x = synth.activations(T + 30, T, d)
    idx, gate = synth.routing_case(T + 31, T, E, topk)
    g = synth.rng(T)
    rtilde = (g.random((E, 3)) * 24.0).astype(np.float32)          # mixes ranks 0 / 8 / 16 per token
    ctx.moe_set_dynamic_ranks(1, rtilde)
    y = torch.empty((T, d), dtype=torch.float32, device="cuda")
    ctx.moe_forward(1, dev(x), dev(idx), dev(gate), y)
    torch.cuda.synchronize()
    rt = [dict(up=float(r[0]), gate=float(r[1]), down=float(r[2])) for r in rtilde]
    ref = linear.moe_forward_dynamic(experts, caps, x, idx, gate, rt)
    err = np.abs(y.cpu().numpy() - ref).max() / np.abs(ref).max()
    assert err <= 2e-3, err
    # the integer ranks the device decided, bit-exact against the oracle's rule (R21)
    got = ctx.moe_last_ranks(T, topk)
    want = np.array([[[linear.dynamic_rank(topk, gate[t, j], rtilde[idx[t, j]][s], 16) for s in range(3)]
                      for j in range(topk)] for t in range(T)], dtype=np.int32)
    assert np.array_equal(got, want)
    assert len(np.unique(want)) >= 2
    # the ranks really vary: the static-rank oracle differs from the dynamic one
    assert np.abs(linear.moe_forward(experts, caps, x, idx, gate) - ref).max() > 1e-6
    ctx.moe_set_dynamic_ranks(1, np.full((E, 3), 1e6, np.float32))  # saturate at the caps
    ctx.moe_forward(1, dev(x), dev(idx), dev(gate), y)
    ctx.moe_set_dynamic_ranks(1, None)
    y_stat = torch.empty_like(y)
    ctx.moe_forward(1, dev(x), dev(idx), dev(gate), y_stat)
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), y_stat.cpu().numpy())
    with pytest.raises(hc.HCError):
        ctx.moe_set_dynamic_ranks(1, np.full((E, 3), -1.0, np.float32))
    ctx.close()


def test_moe_dynamic_rank_exact_ties_and_range(hc):
    """Device ranks at the cases where an fp32 product would round onto an Align midpoint (the float64
    product is exact, R21), r_stored = r_alloc = 256 (a rank of 256 must not be truncated), and a huge
    r̃ (1e9: saturates at the cap, no overflow)."""
    from test_oracle_numerics import DYN_EXACT_CASES
    E, d, f = 16, 256, 256
    for i, (k, g, rt, exact, _f32) in enumerate(DYN_EXACT_CASES):
        cap = 256
        experts, _ = make_experts(E, d, f, 4, seed=300 + i, r_stored=256)
        caps = [dict(up=cap, gate=cap, down=cap) for _ in range(E)]
        ctx = hc.Context(0)
        load(hc, ctx, 0, experts, caps)
        T = 2
        idx = np.array([list(range(k)), list(range(k))], np.int32)
        gate = np.full((T, k), np.float32(g), np.float32)
        rtilde = np.full((E, 3), np.float32(rt), np.float32)
        ctx.moe_set_dynamic_ranks(0, rtilde)
        x = synth.activations(400 + i, T, d)
        y = torch.empty((T, d), dtype=torch.float32, device="cuda")
        ctx.moe_forward(0, dev(x), dev(idx), dev(gate), y)
        torch.cuda.synchronize()
        assert np.all(ctx.moe_last_ranks(T, k) == exact)
        rtd = [dict(up=float(rt), gate=float(rt), down=float(rt))] * E
        ref = linear.moe_forward_dynamic(experts, caps, x, idx, gate, rtd)
        assert np.abs(y.cpu().numpy() - ref).max() <= 2e-3 * np.abs(ref).max()
        # r = 256 everywhere (r̃ huge) must use all 256 ranks: equal to the static path at r_alloc = 256
        ctx.moe_set_dynamic_ranks(0, np.full((E, 3), 1e9, np.float32))
        ctx.moe_forward(0, dev(x), dev(idx), dev(gate), y)
        torch.cuda.synchronize()
        assert np.all(ctx.moe_last_ranks(T, k) == 256)
        ref256 = linear.moe_forward(experts, caps, x, idx, gate)
        assert np.abs(y.cpu().numpy() - ref256).max() <= 2e-3 * np.abs(ref256).max()
        ctx.close()


@pytest.mark.parametrize("scale", [1e-12, 3e5])
def test_moe_full_bf16_range(hc, scale):
    """MoE expert GEMVs (fp16 mma path) with activations far outside fp16's exact band: the per-(row,
    group) prescale of x' (R20) keeps every token row within the bar at its own scale."""
    E, d, f, T, topk = 6, 256, 256, 5, 3
    experts, ranks = make_experts(E, d, f, 3, seed=77)
    ctx = hc.Context(0)
    load(hc, ctx, 2, experts, ranks)
    g = np.random.default_rng(5)
    xf = g.standard_normal((T, d)) * scale
    xf[1, 3] *= 40.0
    from oracle.packing import f64_to_bf16_bits_rne
    x = f64_to_bf16_bits_rne(xf)
    idx, gate = synth.routing_case(78, T, E, topk)
    y = torch.empty((T, d), dtype=torch.float32, device="cuda")
    ctx.moe_forward(2, dev(x), dev(idx), dev(gate), y)
    torch.cuda.synchronize()
    y = y.cpu().numpy()
    ref = linear.moe_forward(experts, ranks, x, idx, gate)
    assert np.all(np.isfinite(y))
    worst = max(np.abs(y[t] - ref[t]).max() / np.abs(ref[t]).max() for t in range(T))
    assert worst <= 2e-3, worst
    ctx.close()
