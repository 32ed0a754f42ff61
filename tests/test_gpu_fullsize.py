"""Parity at BASELINE.json's full sizes, in the launch configurations bench.py times:
  C2  one Llama-2-7B-shaped layer (d 4096, ffn 11008, 4-bit g128) through hc_stack_forward at B = 1 with
      allocator ranks (t forwarding + dataflow waits, as in the 32-layer bench graph), checked whole;
  C3  a Qwen3-30B-A3B-shaped MoE layer (128 experts, top-8, 16 routed tokens, 3-bit) through
      hc_moe_forward, checked whole;
  C5  Llama-3-70B-shaped 2-bit windows (QKV 10240x8192, DOWN 8192x28672) through hc_compensated_linear,
      checked on sampled output rows (the oracle computes each sampled row on its own).
The oracle is oracle/ (float64); inputs are synth/ (seeded)."""
import numpy as np
import pytest

import synth
from oracle import allocate as A
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


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def desc(case, layer, window, slot, r, glue=0, expert=-1):
    return dict(layer=layer, window=window, slot=slot, expert=expert, N=case["N"], K=case["K"], bits=case["bits"],
                codes=dev(case["codes"]), scales=dev(case["scales"]), zeros=dev(case["zeros"]),
                U=dev(case["U"]), V=dev(case["V"]), r_stored=case["r_stored"], r_alloc=r, glue=glue)


def test_c2_full_layer_stack(hc):
    d, kv, f, rs = 4096, 4096, 11008, 128
    gains = synth.STACK_GAINS
    c = lambda n, k, s: synth.linear_case(7000 + s, N=n, K=k, bits=4, r_stored=rs, zeros="asym", unit_gain=gains[s])
    L = dict(qkv=[c(d, d, 0), c(kv, d, 1), c(kv, d, 2)], o=[c(d, d, 3)], upgate=[c(f, d, 4), c(f, d, 5)], down=[c(d, f, 6)])
    # ranks from the oracle allocator on the bench's synthetic sensitivities (one layer, 7 matrices)
    sc = synth.sensitivity_case(3, n_layers=1, members_per_window=(3, 1, 2, 1), n_sigma=256)
    recs = [A.Record(r["layer"], r["window"], r["slot"], sigma=r["sigma"], D=r["D"]) for r in sc["records"]]
    Ns = {(0, 0): d, (0, 1): kv, (0, 2): kv, (1, 0): d, (2, 0): f, (2, 1): f, (3, 0): d}
    caps = [min(rs, Ns[(r.window, r.slot)], f if r.window == 3 else d) for r in recs]
    out = A.allocate_ranks(recs, A.Budget(sc["D_layer"], 1, [159.0, 102.0, 138.0, 163.0]), caps)
    R = {k: [] for k in ("qkv", "o", "upgate", "down")}
    for r, rk in zip(recs, out.ranks):
        R[("qkv", "o", "upgate", "down")[r.window]].append(int(rk))
    assert sum(sum(v) for v in R.values()) > 0
    ctx = hc.Context(0)
    mats = [desc(L["qkv"][i], 0, hc.QKV, i, R["qkv"][i]) for i in range(3)] + [desc(L["o"][0], 0, hc.O, 0, R["o"][0])]
    mats += [desc(L["upgate"][i], 0, hc.UPGATE, i, R["upgate"][i], hc.GLUE_SILU_MUL) for i in range(2)]
    mats += [desc(L["down"][0], 0, hc.DOWN, 0, R["down"][0])]
    ctx.load_layer(mats)
    x = synth.activations(71, 1, d)
    y = torch.empty((1, d), dtype=torch.int16, device="cuda")
    for _ in range(3):
        ctx.stack_forward(dev(x), y)                                   # graph replays: counters / t reset
    torch.cuda.synchronize()
    yb = y.cpu().numpy().view(np.uint16)
    ref = linear.stack_forward([L], [R], x)
    yv = bf16_to_f64(yb)
    bound = 2e-3 * np.abs(ref).max() + np.abs(ref) * 2.0 ** -6         # 2e-3 bar + bf16 rounding flips (R7/R8)
    assert np.all(np.abs(yv - ref) <= bound), np.abs(yv - ref).max() / np.abs(ref).max()
    ctx.close()


def test_c3_full_moe_layer(hc):
    E, d, f, k, T = 128, 2048, 768, 8, 16
    g = synth.rng(17)
    idx, gate = synth.routing_case(18, T, E, k)
    act = sorted(set(int(v) for v in idx.reshape(-1)))
    ctx = hc.Context(0)
    experts, ranks = [], []
    for e in range(E):
        mk = lambda n, kk, s: synth.linear_case(9000 + 3 * e + s, N=n, K=kk, bits=3, r_stored=16, zeros="asym",
                                               unit_gain=synth.STACK_GAINS[4 + s])
        ex = dict(up=mk(f, d, 0), gate=mk(f, d, 1), down=mk(d, f, 2))
        rr = dict(up=int((0, 8, 16)[g.integers(0, 3)]), gate=int((0, 8, 16)[g.integers(0, 3)]),
                  down=int((0, 8, 16)[g.integers(0, 3)]))
        ctx.load_layer([desc(ex["up"], 0, hc.UPGATE, 0, rr["up"], hc.GLUE_SILU_MUL, e),
                        desc(ex["gate"], 0, hc.UPGATE, 1, rr["gate"], hc.GLUE_SILU_MUL, e),
                        desc(ex["down"], 0, hc.DOWN, 0, rr["down"], 0, e)])
        experts.append(ex if e in act else None)
        ranks.append(rr)
    x = synth.activations(19, T, d)
    y = torch.empty((T, d), dtype=torch.float32, device="cuda")
    ctx.moe_forward(0, dev(x), dev(idx), dev(gate), y)
    torch.cuda.synchronize()
    ref = linear.moe_forward(experts, ranks, x, idx, gate)
    err = np.abs(y.cpu().numpy() - ref).max() / np.abs(ref).max()
    assert err <= 2e-3, err
    ctx.close()


@pytest.mark.parametrize("shape", [("qkv", 10240, 8192), ("down", 8192, 28672)])
def test_c5_window_sampled_rows(hc, shape):
    name, N, K = shape
    case = synth.linear_case(5100 + N, N=N, K=K, bits=2, r_stored=64, B=1, zeros="asym")
    ctx = hc.Context(0)
    ctx.load_layer([desc(case, 0, hc.QKV, 0, 64)])
    y = torch.empty((1, N), dtype=torch.float32, device="cuda")
    ctx.compensated_linear(0, hc.QKV, dev(case["x"]), y)
    torch.cuda.synchronize()
    rows = np.sort(synth.rng(N).choice(N, size=96, replace=False))
    ref = linear.compensated_linear(case, 64, rows=rows)
    got = y.cpu().numpy()[:, rows]
    # the 2e-3 bar is relative to max|y| over the full output; the sampled rows' max stands in for it
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert err <= 1e-5, err                                              # exact products, fp32 accumulation
    ctx.close()
