"""CPU-only tests of the C-ABI library: it loads, exports every declared symbol, the host
allocator is bit-exact with the oracle, and the load-time repack round-trips bit-exactly
through the kernel's own fragment/slot mapping.  No compute call needs a GPU here."""
import os
import re

import numpy as np
import pytest

import synth
from oracle import allocate as A
from oracle import packing

import paper_2605_05819_b200 as hc
from paper_2605_05819_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "hcinfer.h")).read()
    declared = set(re.findall(r"\b(hc_[a-z_]+)\s*\(", hdr))
    L = hc.lib()
    for name in declared:
        assert hasattr(L, name), f"{name} declared in hcinfer.h but not exported"
    bound = {n for n, _, _ in _lib.SIGNATURES}
    assert declared == bound, f"binding/header mismatch: {declared ^ bound}"
    assert b"sm_100a" in L.hc_version()


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(hc.HCError) as ei:
        hc.Context(0)
    assert ei.value.code == hc.HC_ERR_RUNTIME


def _to_dicts(recs):
    return [dict(layer=r.layer, window=r.window, slot=r.slot, expert=r.expert, sigma=r.sigma, phi=r.phi,
                 n_sal=r.n_sal, n_all=r.n_all, D=r.D, gate=r.gate) for r in recs]


def _both(recs, bud, caps):
    o = A.allocate_ranks(recs, bud, caps)
    r, p = hc.allocate_ranks(_to_dicts(recs), bud.D_layer, bud.top_k_layers, bud.r_std, caps, bud.tau, bud.k0,
                             bud.two_stage_mode, bud.moe_k)
    return o, r, p


def test_allocator_spec_chain_bit_exact():
    recs = [A.Record(0, 0, 0, sigma=np.array([1, 0.9, 0.1, 0.05, 0.04]), D=0.75),
            A.Record(0, 0, 1, sigma=np.array([1.0, 1.0, 1.0, 1.0]), D=0.15),
            A.Record(0, 0, 2, sigma=np.array([1.0, 1.0, 1.0, 1.0]), D=0.10)]
    o, r, p = _both(recs, A.Budget([1.0], 1, [64.0] * 4), [256] * 3)
    assert r.tolist() == o.ranks == [64, 0, 0]
    assert p.tolist() == o.priority            # bit-identical doubles


@pytest.mark.parametrize("mode", [0, 1])
def test_allocator_random_instances_bit_exact(mode):
    for seed in range(400):
        c = synth.sensitivity_case(seed, n_layers=int(synth.rng(seed).integers(1, 6)), n_sigma=48)
        recs = A.records_from_synth(c)
        g = synth.rng(seed + 9)
        rstd = [float(v) for v in g.uniform(0, 300, size=4)]
        K = int(g.integers(1, len(c["D_layer"]) + 1))
        caps = [int(v) for v in g.integers(0, 300, size=len(recs))]
        o, r, p = _both(recs, A.Budget(list(c["D_layer"]), K, rstd, two_stage_mode=mode), caps)
        assert r.tolist() == o.ranks, seed
        assert p.tolist() == o.priority, seed


def test_allocator_moe_and_errors_match_oracle():
    recs = [A.Record(0, 2, s, expert=e, phi=1.0 + e, n_sal=2, n_all=64, D=1.0 + s, gate=g)
            for e, g in ((3, 0.7), (9, 0.3)) for s in (0, 1)]
    o, r, p = _both(recs, A.Budget([1.0], 1, [0, 0, 64.0, 0], moe_k=2), [256] * 4)
    assert r.tolist() == o.ranks and p.tolist() == o.priority
    bad = [A.Record(0, 2, 0, expert=e, phi=1.0, D=1.0, gate=g) for e, g in ((1, 0.7), (2, 0.2))]
    with pytest.raises(A.AllocError):
        A.allocate_ranks(bad, A.Budget([1.0], 1, [64.0] * 4, moe_k=2), [256] * 2)
    with pytest.raises(hc.HCError) as ei:
        hc.allocate_ranks(_to_dicts(bad), [1.0], 1, [64.0] * 4, [256] * 2, moe_k=2)
    assert ei.value.code == hc.HC_ERR_NUMERIC
    with pytest.raises(hc.HCError) as ei:
        hc.allocate_ranks([dict(layer=0, window=0, slot=0, D=-1.0)], [1.0], 1, [64] * 4, [64])
    assert ei.value.code == hc.HC_ERR_NUMERIC
    with pytest.raises(hc.HCError) as ei:
        hc.allocate_ranks([dict(layer=3, window=0, slot=0, D=1.0)], [1.0], 1, [64] * 4, [64])
    assert ei.value.code == hc.HC_ERR_CONFIG


@pytest.mark.parametrize("bits", [2, 3, 4])
@pytest.mark.parametrize("zeros", ["sym", "asym"])
def test_repack_round_trip_bit_exact(bits, zeros):
    case = synth.linear_case(bits * 7, N=48, K=384, bits=bits, r_stored=0, zeros=zeros)
    packed = hc.repack_host(case["codes"], case["scales"], case["zeros"], 48, 384, bits)
    assert packed.size == 3 * 3 * (256 * bits + 48)
    q, s, z = hc.unpack_repacked_host(packed, 48, 384, bits)
    assert np.array_equal(q, packing.unpack_codes(case["codes"], 384, bits))   # oracle's unpack
    assert np.array_equal(s, case["scales"]) and np.array_equal(z, case["zeros"])


def test_repack_rejects_bad_shapes():
    c = np.zeros((17, 16), np.uint32)
    with pytest.raises(hc.HCError) as ei:
        hc.repack_host(c, np.zeros((17, 1), np.uint16), np.zeros((17, 1), np.uint8), 17, 128, 4)
    assert ei.value.code == hc.HC_ERR_CONFIG


def test_options_roundtrip_and_errors():
    """hc_set_option / hc_get_option (host only): every documented switch round-trips, unknown names and
    negative values are HC_ERR_CONFIG, and the defaults are the measured-best plan."""
    import paper_2605_05819_b200 as hc
    defaults = {"t_forward": 0, "x_handoff": 1, "dep_wait": 1, "int8_path": 1, "prefill_merge": 1,
                "decode_ctas_per_sm": 0, "pdl": 1, "l2_prefetch": 0, "l2_prefetch_at_start": 0}
    for name, d in defaults.items():
        assert hc.get_option(name) == d
        hc.set_option(name, 3)
        assert hc.get_option(name) == 3
        hc.set_option(name, d)
    with pytest.raises(hc.HCError) as e:
        hc.set_option("no_such_switch", 1)
    assert e.value.code == hc.HC_ERR_CONFIG
    with pytest.raises(hc.HCError):
        hc.set_option("x_handoff", -1)
    with pytest.raises(hc.HCError):
        hc.get_option("no_such_switch")
