"""Peer mode: the column-sharded decode stack with the gather fused into the decode
epilogue over peer memory and the next window's t exchanged as per-slice partials.  The GPU pool has one
GPU per box, so G ranks run here as G contexts in ONE process on ONE device (hc_peer_set with the
regions' device pointers; the kernels of the ranks run concurrently on their own streams: the decode grid
is capped at one CTA per SM and programmatic dependent launch is off, so every rank's window fits beside
the others').  Checked against the float64 oracle (per element, DESIGN.md stack bound) and bit for bit
against the single-GPU stack with t forwarding (the same per-block t partials, the same integer sums)."""
import numpy as np
import pytest

import synth
from oracle import linear
from oracle.packing import bf16_to_f64, f64_to_bf16_bits_rne

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

STACK_GAINS = (1.0, 1.0, 1.0, 0.25, 0.25, 0.25, 0.05)


@pytest.fixture(scope="module")
def hc():
    import paper_2605_05819_b200 as m
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def make_stack(L, d, kv, f, bits, r_stored, seed):
    layers, ranks = [], []
    g = synth.rng(seed)
    levels = [0, 8, 16, 32]
    for l in range(L):
        c = lambda n, k, s: synth.linear_case(seed * 1000 + l * 10 + s, N=n, K=k, bits=bits, r_stored=r_stored,
                                              zeros="asym", unit_gain=STACK_GAINS[s])
        L_ = dict(qkv=[c(d, d, 0), c(kv, d, 1), c(kv, d, 2)], o=[c(d, d, 3)], upgate=[c(f, d, 4), c(f, d, 5)],
                  down=[c(d, f, 6)])
        R_ = {k: [int(levels[int(v)]) for v in g.integers(0, 4, size=len(L_[k]))] for k in L_}
        R_["o"] = [16]                        # every window compensated somewhere in the stack
        layers.append(L_)
        ranks.append(R_)
    return layers, ranks


def load_stack(hc, ctx, layers, ranks, shard=None):
    """shard = (rank, G): rows [rank·N/G, (rank+1)·N/G) of every member (the full matrices are passed)."""
    def desc(case, layer, window, slot, r, glue=0):
        lo, hi = (0, case["N"]) if shard is None else hc.shard_rows(case["N"], shard[1], shard[0])
        return dict(layer=layer, window=window, slot=slot, N=case["N"], K=case["K"], bits=case["bits"],
                    codes=dev(case["codes"]), scales=dev(case["scales"]), zeros=dev(case["zeros"]),
                    U=dev(case["U"]), V=dev(case["V"]), r_stored=case["r_stored"], r_alloc=r, glue=glue,
                    row_begin=lo, row_end=hi)
    for l, (L_, R_) in enumerate(zip(layers, ranks)):
        mats = [desc(L_["qkv"][i], l, hc.QKV, i, R_["qkv"][i]) for i in range(3)]
        mats += [desc(L_["o"][0], l, hc.O, 0, R_["o"][0])]
        mats += [desc(L_["upgate"][i], l, hc.UPGATE, i, R_["upgate"][i], hc.GLUE_SILU_MUL) for i in range(2)]
        mats += [desc(L_["down"][0], l, hc.DOWN, 0, R_["down"][0])]
        ctx.load_layer(mats)


@pytest.fixture
def emulation(hc):
    """G ranks on one GPU: one CTA per SM per window, no programmatic dependent launch (restored after)."""
    hc.set_option("decode_ctas_per_sm", 1)
    hc.set_option("pdl", 0)
    yield
    hc.set_option("decode_ctas_per_sm", 0)
    hc.set_option("pdl", 1)


def run_peers(hc, layers, ranks, G, x, steps=2):
    ctxs = [hc.Context(0) for _ in range(G)]
    for p, c in enumerate(ctxs):
        load_stack(hc, c, layers, ranks, shard=(p, G))
    bases = [c.peer_region(G)[0] for c in ctxs]
    for p, c in enumerate(ctxs):
        c.peer_set(p, G, bases)
    B, d = x.shape
    xs = dev(x)
    streams = [torch.cuda.Stream() for _ in range(G)]
    outs = []
    for _ in range(steps):                     # first call captures the graph, the second replays it
        ys = [torch.empty((B, d), dtype=torch.int16, device="cuda") for _ in range(G)]
        for c, y, s in zip(ctxs, ys, streams):
            c.stack_forward(xs, y, stream=s)
        torch.cuda.synchronize()
        outs.append([y.cpu().numpy().view(np.uint16).copy() for y in ys])
    for c in ctxs:
        c.close()
    return outs


@pytest.mark.parametrize("bits,B", [(4, 1), (2, 2), (4, 4), (3, 3)])
def test_peer_stack_matches_oracle_and_single_gpu(hc, emulation, bits, B):
    L, d, kv, f, G = 2, 256, 128, 512, 2
    layers, ranks = make_stack(L, d, kv, f, bits, 32, seed=50 + bits * 7 + B)
    x = synth.activations(11 + B, B, d)
    outs = run_peers(hc, layers, ranks, G, x)
    for step in outs:
        for y in step:
            assert np.array_equal(y, outs[0][0])                  # every rank, every replay: the same h
    y = outs[0][0]
    # the single-GPU stack with t forwarding computes the same t partials (one per 16-row output block)
    hc.set_option("t_forward", 1)
    try:
        c1 = hc.Context(0)
        load_stack(hc, c1, layers, ranks)
        y1 = torch.empty((B, d), dtype=torch.int16, device="cuda")
        c1.stack_forward(dev(x), y1)
        torch.cuda.synchronize()
        y1 = y1.cpu().numpy().view(np.uint16)
        c1.close()
    finally:
        hc.set_option("t_forward", 0)
    assert np.array_equal(y, y1)
    ref = linear.stack_forward(layers, ranks, x)
    yv = bf16_to_f64(y)
    bound = 2e-3 * np.abs(ref).max() + np.abs(ref) * 2.0 ** -6 * L
    assert np.all(np.abs(yv - ref) <= bound), np.abs(yv - ref).max() / np.abs(ref).max()
    assert np.mean(y == f64_to_bf16_bits_rne(ref)) >= 0.97


def test_peer_stack_four_ranks(hc, emulation):
    """G = 4 (k / v members of 128 rows -> 32-row shards, two row blocks per rank)."""
    L, d, kv, f, G = 1, 256, 128, 384, 4
    layers, ranks = make_stack(L, d, kv, f, 4, 32, seed=91)
    x = synth.activations(5, 1, d)
    outs = run_peers(hc, layers, ranks, G, x, steps=1)
    ref = linear.stack_forward(layers, ranks, x)
    for y in outs[0]:
        assert np.array_equal(y, outs[0][0])
        yv = bf16_to_f64(y)
        assert np.all(np.abs(yv - ref) <= 2e-3 * np.abs(ref).max() + np.abs(ref) * 2.0 ** -6 * L)


def test_peer_api_errors(hc):
    ctx = hc.Context(0)
    with pytest.raises(hc.HCError):
        ctx.peer_region(2)                         # nothing loaded
    layers, ranks = make_stack(1, 256, 128, 384, 4, 32, seed=3)
    load_stack(hc, ctx, layers, ranks, shard=(0, 2))
    with pytest.raises(hc.HCError):
        ctx.peer_region(9)                         # world > 8
    base, nbytes = ctx.peer_region(2)
    assert base != 0 and nbytes > 0
    with pytest.raises(hc.HCError):
        ctx.peer_set(0, 2, [base + 256, base])     # bases[rank] must be this context's region
    ctx.close()
