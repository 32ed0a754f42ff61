"""Pins for oracle.allocate and oracle.brute (App. B.1-B.2; SPEC worked examples)."""
import math

import numpy as np
import pytest

import synth
from oracle import allocate as A
from oracle import brute


def test_salience_examples(golden):
    e = golden["salience_flat"]
    s = A.salience(e["sigma"])
    assert (s.phi, s.cut) == (1.0, 0)
    e = golden["salience_chain"]
    s = A.salience(e["sigma"], 0.01)
    assert s.cut == e["cut"] and abs(s.phi - e["phi"]) < e["phi_tol"]
    # the chain's exact value from the formula: mean(1,0.9,0.1)/mean(0.05,0.04)
    assert abs(s.phi - (2.0 / 3.0) / 0.045) < 1e-12
    # interior second differences as printed
    sig = e["sigma"]
    k = [sig[j - 1] - 2 * sig[j] + sig[j + 1] for j in range(1, 4)]
    assert np.allclose(k, e["k"], atol=1e-12)
    assert A.salience([0, 0, 0, 0]).phi == 1.0
    assert A.salience([3.0, 1.0]).phi == 1.0           # n < 3


def test_salience_threshold_and_ties():
    # max k below tau -> not salient
    assert A.salience([1.0, 1.0, 0.99, 0.98], tau=0.01).cut == 0
    # k = (-0.5, 0.5, -0.5, 0.5) at j = 2..5: tie between j = 3 and j = 5, smallest wins
    s = A.salience([1.0, 1.0, 0.5, 0.5, 0.0, 0.0], tau=0.01)
    assert s.cut == 3 and abs(s.phi - (2.5 / 3) / (0.5 / 3)) < 1e-12


def test_salience_phi_at_least_one_and_planted_recovery():
    # φ >= 1.  Planted c salient values followed by a drop: the second difference
    # peaks at the first value AFTER the drop (k_j = σ̂_{j-1} − 2σ̂_j + σ̂_{j+1} is largest where
    # the curve turns), so the literal S = {1..argmax k} (reading R10) holds c + 1 values —
    # exactly as in the paper's own example (where S includes the knee value 0.1).
    g = synth.rng(5)
    hits = 0
    for trial in range(200):
        c = int(g.integers(2, 5))
        sig = np.concatenate([np.linspace(1.0, 0.8, c), 0.05 * np.exp(-np.arange(60) / 30.0)])
        sig = np.sort(sig)[::-1]
        s = A.salience(sig)
        assert s.phi >= 1.0
        hits += (s.cut == c + 1)
    assert hits >= 180


def test_normalisations(golden):
    e = golden["salience_scores"]
    assert np.allclose(A.window_normalise(e["phi"]), e["V"], atol=e["tol"])
    e = golden["matrix_scores"]
    assert A.window_normalise(e["D"]) == e["S"]
    assert A.window_normalise([0.0, 0.0, 0.0]) == [1 / 3] * 3
    assert A.window_normalise([2.5]) == [1.0]
    for key in ("layer_scores_K1", "layer_scores_K2"):
        e = golden[key]
        assert np.allclose(A.layer_scores(e["D"], e["K"]), e["S"], atol=1e-15)
    assert A.layer_scores([5, 3, 1], 3) == [1.0, 1.0, 1.0]
    assert A.layer_scores([2.0, 5.0, 5.0, 1.0], 1) == [0.4, 1.0, 1.0, 0.2]   # tie -> smaller index in 𝒯
    with pytest.raises(A.AllocError):
        A.layer_scores([1.0], 0)
    e = golden["expert_scores"]
    assert np.allclose(A.expert_scores(e["g"], e["k"]), e["G"], atol=1e-15)
    assert A.expert_scores([0.5, 0.5], 2) == [1.0, 1.0]
    with pytest.raises(A.AllocError):
        A.expert_scores([0.5, 0.4], 2)


def _chain_records():
    # S:197/S:207/S:386: member 0 has the B.1 example spectrum, members 1-2 flat spectra (φ = 1)
    return [A.Record(0, 0, 0, sigma=np.array([1, 0.9, 0.1, 0.05, 0.04]), D=0.75),
            A.Record(0, 0, 1, sigma=np.array([1.0, 1.0, 1.0, 1.0]), D=0.15),
            A.Record(0, 0, 2, sigma=np.array([1.0, 1.0, 1.0, 1.0]), D=0.10)]


def test_priority_and_continuous_rank_chain(golden):
    al = A.allocate_ranks(_chain_records(), A.Budget([1.0], 1, [64, 64, 64, 64]), [256] * 3)
    e = golden["priority_chain"]
    assert np.allclose(al.priority, e["P"], rtol=e["rel_tol"])
    e = golden["continuous_rank"]
    assert np.allclose(al.rtilde, e["rtilde"], rtol=e["rel_tol"])
    assert al.ranks == [64, 0, 0]                       # aligned plan within budget 64
    # the cap reading (R15): a matrix with only 5 singular values cannot take rank 64
    al = A.allocate_ranks(_chain_records(), A.Budget([1.0], 1, [64] * 4), [5, 4, 4])
    assert al.ranks == [0, 0, 0]
    al = A.allocate_ranks(_chain_records(), A.Budget([1.0], 1, [64] * 4), [40, 256, 256])
    assert al.ranks == [32, 0, 0]


def test_align_cap_demote(golden):
    e = golden["align"]
    for rt, r in e["cases"]:
        assert A.align(rt, e["k0"]) == r
    assert [A.align(v) for v in (3.99, 11.99, 12.0, 23.9, 24.0, 95.9, 96.0, 1000.0)] == \
        [0, 8, 16, 16, 32, 64, 128, 1024]
    assert A.cap_level(64, 40) == 32 and A.cap_level(8, 7) == 0 and A.cap_level(16, 16) == 16
    assert A.demote(8) == 0 and A.demote(64) == 32


def test_enforce_budget(golden):
    e = golden["enforce_budget"]
    assert A.enforce_budget(e["ranks"], e["priorities"], e["r_std"]) == e["out"]
    assert A.enforce_budget([32, 8], [0.5, 0.5], 48) == [32, 8]          # feasible: unchanged
    assert A.enforce_budget([32, 8, 8], [0.2, 0.5, 0.3], 0) == [0, 0, 0]  # r_std = 0
    assert A.enforce_budget([16, 16], [0.5, 0.5], 24) == [16, 8]          # equal 𝒫: later member first


def test_two_stage(golden):
    e = golden["two_stage_mode0"]
    assert A.two_stage([float(e["rtilde"])], [1.0], [e["n_sal"]], [e["n_sal"] + e["n_res"]], 0) == [e["out"]]
    # mode 1 hand trace (P:689-693 pooled reading): 𝒫 = (0.75, 0.25), r̃ = (12, 4), |S| = (4, 8), |R| = (60, 56)
    out = A.two_stage([12.0, 4.0], [0.75, 0.25], [4, 8], [64, 64], 1)
    assert np.allclose(out, [4 + 4 * 60 / 116, 8 + 4 * 56 / 116], atol=1e-12)
    # stage 2 inert when Σr̃ <= Σ|S|: r̃ = (6, 2) into caps (8, 8) -> proportional to 𝒫 = (6, 2)
    assert np.allclose(A.two_stage([6.0, 2.0], [0.75, 0.25], [8, 8], [64, 64], 1), [6.0, 2.0], atol=1e-12)
    # conservation: the pooled total is preserved
    out = A.two_stage([30.0, 10.0, 5.0], [0.6, 0.3, 0.1], [3, 0, 20], [100, 50, 60], 1)
    assert abs(sum(out) - 45.0) < 1e-9


def _random_window_case(seed):
    c = synth.sensitivity_case(seed, n_layers=4, n_sigma=64)
    recs = A.records_from_synth(c)
    rstd = [float(v) for v in synth.rng(seed + 1).integers(0, 200, size=4)]
    return recs, A.Budget(list(c["D_layer"]), 1, rstd)


def test_budget_invariant_admissible_and_capped():
    for seed in range(300):
        recs, bud = _random_window_case(seed)
        caps = [int(v) for v in synth.rng(seed + 2).integers(0, 300, size=len(recs))]
        for mode in (0, 1):
            bud.two_stage_mode = mode
            al = A.allocate_ranks(recs, bud, caps)
            sums = {}
            for rec, r, cap in zip(recs, al.ranks, caps):
                assert r == 0 or (r >= 8 and r & (r - 1) == 0)
                assert r <= cap
                sums[(rec.layer, rec.window)] = sums.get((rec.layer, rec.window), 0) + r
            for (layer, kind), s in sums.items():
                assert s <= bud.r_std[kind]


def test_priority_scale_invariance_and_determinism():
    # scaling every D (hence every 𝒱·𝒮) by a positive constant leaves 𝒫 and the plan unchanged
    recs, bud = _random_window_case(42)
    caps = [256] * len(recs)
    base = A.allocate_ranks(recs, bud, caps)
    for rec in recs:
        rec.D *= 4.0                       # power of two: exact scaling
    again = A.allocate_ranks(recs, bud, caps)
    assert again.ranks == base.ranks and again.priority == base.priority


def test_moe_gate_conservation_and_error():
    recs = [A.Record(0, 2, s, expert=e, phi=1.0, n_all=64, D=1.0, gate=g)
            for e, g in ((3, 0.7), (9, 0.3)) for s in (0, 1)]
    al = A.allocate_ranks(recs, A.Budget([1.0], 1, [0, 0, 64, 0], moe_k=2), [256] * 4)
    # 𝒢 = (1.4, 0.6) per slot; Norm_W over the 4 members gives 0.25 each -> 𝒫 = (0.35, 0.35, 0.15, 0.15)
    assert np.allclose(al.priority, [0.35, 0.35, 0.15, 0.15], atol=1e-15)
    bad = [A.Record(0, 2, 0, expert=e, phi=1.0, D=1.0, gate=g) for e, g in ((1, 0.7), (2, 0.2))]
    with pytest.raises(A.AllocError) as ei:
        A.allocate_ranks(bad, A.Budget([1.0], 1, [64] * 4, moe_k=2), [256] * 2)
    assert ei.value.code == A.HC_ERR_NUMERIC


def test_errors():
    with pytest.raises(A.AllocError) as ei:
        A.allocate_ranks([A.Record(0, 0, 0, D=-1.0)], A.Budget([1.0], 1, [64] * 4), [64])
    assert ei.value.code == A.HC_ERR_NUMERIC
    with pytest.raises(A.AllocError) as ei:
        A.allocate_ranks([A.Record(2, 0, 0, D=1.0)], A.Budget([1.0], 1, [64] * 4), [64])
    assert ei.value.code == A.HC_ERR_CONFIG


# ------------------------------------------------------------------ optimality (App. B.2)
def test_greedy_counterexample_on_power_of_two_levels(golden):
    e = golden["greedy_counterexample"]
    lv = e["levels"]
    tables = []
    for rates in e["per_unit_gains"]:
        t = [0.0]
        for i in range(1, len(lv)):
            t.append(t[-1] + rates[i - 1] * (lv[i] - lv[i - 1]))
        tables.append(t)
    gp, gv = brute.greedy(tables, lv, e["budget"])
    bp, bv = brute.brute_force(tables, lv, e["budget"])
    assert gp == e["greedy_plan"] and abs(gv - e["greedy_value"]) < 1e-9
    assert bp == e["brute_plan"] and abs(bv - e["brute_value"]) < 1e-9


def test_greedy_equals_brute_force_on_uniform_levels():
    # SPEC acceptance 4 under reading R17 (uniform steps, where the concave greedy argument holds)
    g = synth.rng(77)
    levels = [0, 8, 16, 24, 32]
    for _ in range(200):
        tables = []
        for i in range(3):
            sig = np.sort(g.random(40))[::-1]
            tables.append(brute.gain_table(sig, float(g.random()), levels))
        budget = int(g.integers(0, 49))
        _, gv = brute.greedy(tables, levels, budget)
        _, bv = brute.brute_force(tables, levels, budget)
        assert abs(gv - bv) <= 1e-12 * max(1.0, bv)


def test_brute_force_examples():
    # S:455-457
    t = [brute.gain_table([3.0, 2.0, 1.0] * 10, 1.0, [0, 8, 16])]
    assert brute.brute_force(t, [0, 8, 16], 16)[0] == [16]
    t2 = [brute.gain_table([5.0] * 20, 1.0, [0, 8, 16]), brute.gain_table([1.0] * 20, 1.0, [0, 8, 16])]
    assert brute.brute_force(t2, [0, 8, 16], 16)[0] == [16, 0]
    assert brute.brute_force(t2, [0, 8, 16], 0) == ([0, 0], 0.0)


def test_r_std_bytes_hand_values():
    """R17 pinned by hand: Llama-2-7B QKV (3 x 4096x4096, 4-bit g128) has base bytes 3·(8388608 + 327680) =
    26148864, N̄ + K = 8192, so r_std = floor(0.1·26148864 / 16384) = floor(159.6) = 159 (SURVEY.md §8(c)
    quotes ≈ 159); a single 4096² 2-bit matrix: 4194304 + 4096·32·18/8 = 4489216 -> floor(448921.6/16384) = 27."""
    from oracle.allocate import r_std_bytes
    assert r_std_bytes([4096, 4096, 4096], 4096, 4) == 159.0
    assert r_std_bytes([4096], 4096, 2) == 27.0
    # scale invariance of the rule: doubling every N and K doubles the bytes per unit rank and the base
    # bytes by 4 -> r_std doubles (up to the floor)
    assert abs(r_std_bytes([8192], 8192, 4) - 2 * r_std_bytes([4096], 4096, 4)) <= 1


def test_r_std_library_bit_exact():
    """hc_calib_r_std (host C++) equals the oracle's rule bit for bit on the bench windows and random ones."""
    import paper_2605_05819_b200 as hc
    from oracle.allocate import r_std_bytes
    g = np.random.default_rng(5)
    cases = [([4096, 4096, 4096], 4096, 4), ([4096], 4096, 4), ([11008, 11008], 4096, 4), ([4096], 11008, 4),
             ([8192, 1024, 1024], 8192, 2), ([28672, 28672], 8192, 2), ([768, 768], 2048, 3), ([2048], 768, 3)]
    for _ in range(50):
        cases.append(([int(v) * 16 for v in g.integers(1, 800, size=int(g.integers(1, 5)))], int(g.integers(1, 100)) * 128,
                      int(g.choice([2, 3, 4, 8]))))
    for Ns, K, b in cases:
        for eps in (0.1, 0.05, 0.25):
            assert hc.calib_r_std(Ns, K, b, 128, eps) == r_std_bytes(Ns, K, b, 128, eps), (Ns, K, b, eps)
