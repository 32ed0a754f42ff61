#!/usr/bin/env python
"""Benchmark of the HCInfer compensated quantized linear on B200 (driver contract: one JSON line).

Workloads (BASELINE.json configs):
  c1  single 4096x4096 linear, 4-bit g128, rank-64 compensation, batch-1 decode.
      One step = one compensated linear over one batch; L2 is defeated by rotating through
      128 distinct weight copies (1.25 GB > 126 MB L2) — config["l2"] says so.

`python bench.py [--gpus N --steps K --warmup W --impl {ours,reference} --workload c1]`
Under torchrun each rank runs an independent replica of the workload (the path partitions into
independent problems: weak scaling, no data-path collective); value = all ranks' bytes / max time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "compensated quant-linear HBM GB/s vs peak; decode tokens/s at 1/2/4/8 GPUs"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.summary = {"sm_mhz": None, "sm_max_mhz": None, "reasons": []}
        if not self.proc:
            return
        time.sleep(0.15)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            return
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [v.strip() for v in line.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0])); mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if sm:
            self.summary = {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                            "samples": len(sm)}


# ------------------------------------------------------------------ workload C1
C1 = dict(N=4096, K=4096, bits=4, group=128, r=64, r_stored=64, B=1)


FACTOR_BYTES = {"bf16": 2, "fp8": 1}   # bytes per factor element (fp8: e4m3 + 2 fp32 scales per rank)


def factor_bytes(r, N, K, kind="bf16"):
    return FACTOR_BYTES[kind] * r * (N + K) + (8 * r if kind == "fp8" else 0)


def c1_bytes(c=C1, r=None, kind="bf16"):
    """Algorithmic bytes of one C1 call: codes b/8 per element, a bf16
    scale + a b-bit zero per group, the rank-r slices of U and V (bf16, or e4m3 + per-rank scales), x (bf16)
    and y (fp32)."""
    N, K, b, g, B = c["N"], c["K"], c["bits"], c["group"], c["B"]
    r = c["r"] if r is None else r
    base = N * K * b // 8 + N * (K // g) * (16 + b) // 8
    fac = factor_bytes(r, N, K, kind)
    io = B * (2 * K + 4 * N)
    return base + fac + io


def dtype_of(args, config):
    """The arithmetic the timed path computes in: int8 mma for 2/4-bit decode at
    B <= 2 (codes x s8 digits of x, exact int32), else fp16 mma on exact dequantised integers."""
    import paper_2605_05819_b200 as hc
    bits = config.get("bits", 4)
    if args.workload == "c4":
        return f"fp16 tcgen05 (s·(q−z) of int{bits}, bf16 X as fp16), fp32 accumulate"
    if bits in (2, 4) and args.batch <= 2 and hc.get_option("int8_path") != 0 and args.workload != "c3":
        return f"int8 mma (u{bits} codes x s8 digits of bf16 x, exact int32), fp32 per-group accumulate"
    return f"fp16 mma (exact int{bits} dequant x fp16 x), fp32 accumulate"


def e4m3_random(shape, g):
    """Random e4m3 bytes on the device (random BYTES: sign, exponent field in [4, 10], mantissa; 1/16 of them
    subnormal / zero codes) -- the synth.fp8_factors recipe."""
    import torch
    sign = torch.randint(0, 2, shape, generator=g, device="cuda", dtype=torch.int32) << 7
    e = torch.randint(4, 11, shape, generator=g, device="cuda", dtype=torch.int32)
    e = torch.where(torch.rand(shape, generator=g, device="cuda") < 1.0 / 16.0, torch.zeros_like(e), e)
    m = torch.randint(0, 8, shape, generator=g, device="cuda", dtype=torch.int32)
    return (sign | (e << 3) | m).to(torch.uint8)


def factor_fields(U, V, N, K, rs, g, kind):
    """Matrix-descriptor fields of the factors: bf16 U / V as given, or e4m3 bytes + per-rank scales with the
    same RMS as the bf16 factors (|e4m3| RMS of the recipe ~ 4.9)."""
    import torch
    import paper_2605_05819_b200 as hc
    if kind != "fp8":
        return dict(U=U, V=V)
    su = float(U.float().pow(2).mean().sqrt()) / 4.9
    sv = float(V.float().pow(2).mean().sqrt()) / 4.9
    return dict(U=e4m3_random((N, rs), g), V=e4m3_random((rs, K), g), factor_dtype=hc.FACTORS_FP8,
                u_scale=(su * (0.5 + torch.rand(rs, generator=g, device="cuda"))).contiguous(),
                v_scale=(sv * (0.5 + torch.rand(rs, generator=g, device="cuda"))).contiguous())


def run_c1_ours(args, rank, world, device):
    import torch
    import paper_2605_05819_b200 as hc
    c = C1
    ncopy = 128
    ctx = hc.Context(device)
    g = torch.Generator(device="cuda").manual_seed(1234 + rank)
    N, K, b, G = c["N"], c["K"], c["bits"], c["K"] // c["group"]
    mats = []
    for i in range(ncopy):
        codes = torch.randint(-2**31, 2**31, (N, K * b // 32), generator=g, device="cuda", dtype=torch.int32)
        scales = (0.002 + 0.01 * torch.rand((N, G), generator=g, device="cuda")).to(torch.bfloat16)
        zeros = torch.full((N, G), 1 << (b - 1), dtype=torch.uint8, device="cuda")
        U = (torch.randn((N, c["r_stored"]), generator=g, device="cuda") / N ** 0.5).to(torch.bfloat16)
        V = (0.02 * torch.randn((c["r_stored"], K), generator=g, device="cuda")).to(torch.bfloat16)
        ctx.load_layer([dict(layer=i, window=0, slot=0, N=N, K=K, bits=b, codes=codes, scales=scales, zeros=zeros,
                             r_stored=c["r_stored"], r_alloc=c["r"],
                             **factor_fields(U, V, N, K, c["r_stored"], g, getattr(args, "factors", "bf16")))])
        del codes, scales, zeros, U, V
    x = torch.randn((c["B"], K), generator=g, device="cuda").to(torch.bfloat16)
    y = torch.empty((c["B"], N), dtype=torch.float32, device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for i in range(ncopy):                           # first call allocates workspaces
            ctx.compensated_linear(i, 0, x, y)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=st):
            for i in range(ncopy):
                ctx.compensated_linear(i, 0, x, y, stream=st)
    torch.cuda.synchronize()
    reps = max(1, (args.steps + ncopy - 1) // ncopy)
    warm = max(1, (args.warmup + ncopy - 1) // ncopy)
    with torch.cuda.stream(st):
        for _ in range(warm):
            graph.replay()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(device) as clk, torch.cuda.stream(st):
        e0.record(st)
        for _ in range(reps):
            graph.replay()                               # replays on the current stream = st
        e1.record(st)
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    steps = reps * ncopy
    # the same copies at r = 0 (no U / V reads, the uncompensated body): the compensation overhead
    for i in range(ncopy):
        ctx.set_rank(i, 0, 0, 0)
    with torch.cuda.stream(st):
        for i in range(ncopy):
            ctx.compensated_linear(i, 0, x, y)
        torch.cuda.synchronize()
        graph0 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph0, stream=st):
            for i in range(ncopy):
                ctx.compensated_linear(i, 0, x, y, stream=st)
        for _ in range(warm):
            graph0.replay()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(st)
        for _ in range(reps):
            graph0.replay()
        f1.record(st)
        torch.cuda.synchronize()
    ms_r0 = f0.elapsed_time(f1)
    for i in range(ncopy):
        ctx.set_rank(i, 0, 0, c["r"])
    # end-to-end through the public API with HOST buffers (pinned x in, y out every step)
    xh = x.cpu().pin_memory()
    yh = torch.empty((c["B"], N), dtype=torch.float32).pin_memory()
    n_e2e = min(steps, 512)
    for i in range(8):
        ctx.compensated_linear(i, 0, xh, yh, stream=st)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(n_e2e):
        ctx.compensated_linear(i % ncopy, 0, xh, yh, stream=st)   # syncs per call (host result)
    e2e_s = time.perf_counter() - t0
    ctx.close()
    return dict(ms=ms, steps=steps, clocks=clk.summary, e2e_s=e2e_s, n_e2e=n_e2e, ms_r0=ms_r0,
                launches=steps, h2d=c["B"] * K * 2, d2h=c["B"] * N * 4)


def oracle_c1_sample(seconds: float = 12.0):
    """The float64 oracle on a bounded sample of the C1 workload (whole calls)."""
    import synth
    from oracle import linear
    case = synth.linear_case(0, N=C1["N"], K=C1["K"], bits=4, r_stored=64, B=1)
    t0 = time.perf_counter()
    n = 0
    while True:
        linear.compensated_linear(case, C1["r"])
        n += 1
        el = time.perf_counter() - t0
        if el >= seconds or n >= 200:
            break
    return n, el


# ------------------------------------------------------------------ stacks: C2 (headline), C5 (multi-GPU)
C2 = dict(name="c2", model="llama2_7b", hidden=4096, kv=4096, ffn=11008, layers=32, bits=4, group=128,
          r_stored=128, fixed_rank=None)
C5 = dict(name="c5", model="llama3_70b", hidden=8192, kv=1024, ffn=28672, layers=80, bits=2, group=128,
          r_stored=64, fixed_rank=64)
STACKS = {"c2": C2, "c5": C5}


def window_bytes_base(Ns, K, bits, g=128):
    return sum(N * K * bits // 8 + N * (K // g) * (16 + bits) // 8 for N in Ns)


def c2_windows(c=C2):
    d, kv, f = c["hidden"], c["kv"], c["ffn"]
    # (kind, member N list, K)
    return [(0, [d, kv, kv], d), (1, [d], d), (2, [f, f], d), (3, [d], f)]


def c2_r_std(c=C2):
    """B200 reading of r_std (R17): the largest rank whose extra bytes stay
    within 10% of the window's base bytes: floor(0.1·bytes_base / (2·(mean N + K)))."""
    out = []
    for kind, Ns, K in c2_windows(c):
        nbar = sum(Ns) / len(Ns)
        out.append(float(int(0.1 * window_bytes_base(Ns, K, c["bits"]) / (2 * (nbar + K)))))
    return out


def c2_ranks(c=C2, seed=0):
    """Ranks from the library's allocator on synthetic sensitivity inputs (planted spectra); C5 uses the
    fixed rank of its BASELINE config (r = 64)."""
    if c.get("fixed_rank") is not None:
        return {(l, kind, s): c["fixed_rank"] for l in range(c["layers"]) for kind, Ns, K in c2_windows(c)
                for s in range(len(Ns))}
    import synth
    import paper_2605_05819_b200 as hc
    case = synth.sensitivity_case(seed, n_layers=c["layers"], members_per_window=(3, 1, 2, 1), n_sigma=256)
    caps = []
    for rec in case["records"]:
        kind, Ns, K = c2_windows(c)[rec["window"]]
        caps.append(min(c["r_stored"], Ns[rec["slot"]], K))
    ranks, prio = hc.allocate_ranks(case["records"], case["D_layer"], (c["layers"] + 3) // 4, c2_r_std(c), caps)
    out = {}
    for rec, r in zip(case["records"], ranks):
        out[(rec["layer"], rec["window"], rec["slot"])] = int(r)
    return out


def c2_ranks_oracle(c=C2, seed=0):
    """The same plan as c2_ranks, computed by the float64 oracle allocator (oracle/allocate.py, bit-exact
    with hc_allocate_ranks): the reference arm does not call the library."""
    import synth
    from oracle import allocate as oa
    case = synth.sensitivity_case(seed, n_layers=c["layers"], members_per_window=(3, 1, 2, 1), n_sigma=256)
    caps = []
    for rec in case["records"]:
        kind, Ns, K = c2_windows(c)[rec["window"]]
        caps.append(min(c["r_stored"], Ns[rec["slot"]], K))
    bud = oa.Budget(D_layer=list(case["D_layer"]), top_k_layers=(c["layers"] + 3) // 4, r_std=c2_r_std(c))
    al = oa.allocate_ranks(oa.records_from_synth(case), bud, caps)
    return {(rec["layer"], rec["window"], rec["slot"]): int(r) for rec, r in zip(case["records"], al.ranks)}


def c2_bytes(ranks, B, c=C2, G=1, kind="bf16"):
    """Algorithmic bytes one GPU moves per decode step: its rows of every base weight (codes, bf16 scale,
    b-bit zero), its rows of the allocated U slices and ALL of the allocated V slices (V·x is replicated
    under column sharding), and the activations in/out of each window."""
    tot = 0
    for l in range(c["layers"]):
        for wk, Ns, K in c2_windows(c):
            tot += window_bytes_base([N // G for N in Ns], K, c["bits"])
            for s, N in enumerate(Ns):
                tot += factor_bytes(ranks[(l, wk, s)], N // G, K, kind)
            tot += B * 2 * K + B * 2 * ((sum(Ns) if wk != 2 else Ns[0]) // G)
    return tot


def build_c2(ctx, ranks, c=C2, shard=None, factors="bf16"):
    """Random-init weights of the named shapes, generated on the device; every matrix has its own seed so
    all ranks of a column-sharded run see the same model and load rows [rank·N/G, (rank+1)·N/G)."""
    import torch
    import paper_2605_05819_b200 as hc
    gains = (1.0, 1.0, 1.0, 0.25, 0.25, 0.25, 0.05)   # synth.STACK_GAINS (finite over 32 layers)
    if c["layers"] > 32:
        gains = (1.0, 1.0, 1.0, 0.2, 0.2, 0.2, 0.02)  # 80 layers: stronger damping keeps the output finite
    b = c["bits"]
    e2 = ((4 ** b) - 1) / 12.0 + 0.25
    slot_gain = {(0, 0): 0, (0, 1): 1, (0, 2): 2, (1, 0): 3, (2, 0): 4, (2, 1): 5, (3, 0): 6}
    for l in range(c["layers"]):
        mats = []
        for kind, Ns, K in c2_windows(c):
            G = K // c["group"]
            for s, N in enumerate(Ns):
                g = torch.Generator(device="cuda").manual_seed(4242 + 100 * l + 10 * kind + s)
                gain = gains[slot_gain[(kind, s)]]
                rs = c["r_stored"]
                lo, hi = (0, N) if shard is None else hc.shard_rows(N, shard[1], shard[0])
                mats.append(dict(
                    layer=l, window=kind, slot=s, N=N, K=K, bits=b, row_begin=lo, row_end=hi,
                    codes=torch.randint(-2**31, 2**31, (N, K * b // 32), generator=g, device="cuda", dtype=torch.int32),
                    scales=(gain * (0.5 + torch.rand((N, G), generator=g, device="cuda")) / (e2 * K) ** 0.5).to(torch.bfloat16),
                    zeros=torch.randint(0, 1 << b, (N, G), generator=g, device="cuda", dtype=torch.uint8),
                    r_stored=rs, r_alloc=ranks[(l, kind, s)], glue=1 if kind == 2 else 0,
                    **factor_fields((torch.randn((N, rs), generator=g, device="cuda") / N ** 0.5).to(torch.bfloat16),
                                    (0.05 * (N / (rs * K)) ** 0.5 * torch.randn((rs, K), generator=g, device="cuda")).to(torch.bfloat16),
                                    N, K, rs, g, factors)))
        ctx.load_layer(mats)
        del mats
    torch.cuda.synchronize()


def run_c2_ours(args, rank, world, device, B, c=C2, tp=False, sweep=()):
    """Build the stack once; time B (the bench line), the same stack at r = 0 (compensation overhead,
    SURVEY.md §8(d)), and the batch sweep `sweep`, all with device events on the launching stream."""
    import torch
    import paper_2605_05819_b200 as hc
    ranks = c2_ranks(c)
    if getattr(args, "rank_override", None) is not None:
        ranks = {k: args.rank_override for k in ranks}
    ctx = hc.Context(device)
    G = world if tp else 1
    peer = tp and getattr(args, "tp_path", "peer") == "peer"
    if tp and not peer:
        ctx.init_comm(rank, world)
    fk = getattr(args, "factors", "bf16")
    build_c2(ctx, ranks, c, shard=(rank, world) if tp else None, factors=fk)
    if peer:
        ctx.init_peers(rank, world)      # gather fused into the decode epilogue over peer memory
    st = torch.cuda.Stream()

    def timed(Bt, clocks=False):
        gx = torch.Generator(device="cuda").manual_seed(7 + (0 if tp else rank))
        x = torch.randn((Bt, c["hidden"]), generator=gx, device="cuda").to(torch.bfloat16)
        y = torch.empty((Bt, c["hidden"]), dtype=torch.bfloat16, device="cuda")
        for _ in range(max(args.warmup, 3)):
            ctx.stack_forward(x, y, stream=st)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        clk = Clocks(device) if clocks else None
        if clk:
            clk.__enter__()
        e0.record(st)
        for _ in range(args.steps):
            ctx.stack_forward(x, y, stream=st)
        e1.record(st)
        torch.cuda.synchronize()
        if clk:
            clk.__exit__(None, None, None)
        if world > 1:
            torch.distributed.barrier()
        return e0.elapsed_time(e1), x, y, (clk.summary if clk else None)

    ms, x, y, clocks = timed(B, clocks=True)
    finite = bool(torch.isfinite(y.float()).all().item())
    # end to end through the public API with pinned HOST buffers (H2D of x, D2H of y every step)
    xh = x.cpu().pin_memory()
    yh = torch.empty((B, c["hidden"]), dtype=torch.bfloat16).pin_memory()
    ctx.stack_forward(xh, yh, stream=st)
    n_e2e = max(3, min(args.steps, 50))
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for _ in range(n_e2e):
        ctx.stack_forward(xh, yh, stream=st)      # synchronises (host result)
    e2e_s = time.perf_counter() - t0
    # the same weights at r = 0 everywhere (uncompensated body: no U / V bytes, no rank projection)
    for (l, kind, sl) in ranks:
        ctx.set_rank(l, kind, sl, 0)
    ms_r0 = timed(B)[0]
    for (l, kind, sl), r in ranks.items():
        ctx.set_rank(l, kind, sl, r)
    sw = {}
    for Bs in sweep:
        mss = timed(Bs)[0]
        sw[str(Bs)] = {"tokens_per_s": round((1 if tp else world) * Bs * args.steps / (mss * 1e-3), 1),
                       "ms_per_step": round(mss / args.steps, 4),
                       "GBps": round(c2_bytes(ranks, Bs, c, G, fk) / (mss / args.steps * 1e-3) / 1e9, 1)}
    ctx.close()
    mean_rank = sum(ranks.values()) / len(ranks)
    # decode kernels (+ the NCCL path's unshard permute per window; + the peer path's final gather wait)
    launches = args.steps * (4 * c["layers"] * (2 if (tp and not peer) else 1) + (1 if peer else 0))
    return dict(ms=ms, steps=args.steps, clocks=clocks, e2e_s=e2e_s, n_e2e=n_e2e, finite=finite,
                launches=launches, h2d=B * c["hidden"] * 2, d2h=B * c["hidden"] * 2,
                bytes=c2_bytes(ranks, B, c, G, fk), bytes_r0=c2_bytes({k: 0 for k in ranks}, B, c, G), ms_r0=ms_r0,
                mean_rank=mean_rank, ranks=ranks, sweep=sw)


def oracle_c2_sample(seconds: float = 15.0, c=C2):
    """The float64 oracle on a bounded sample of the C2 workload: whole layers (all 4 windows, glue
    included) of the Llama-2-7B-shaped stack at B = 1, at the ranks hc_allocate_ranks gives layer 0 of the
    bench's own plan (c2_ranks).  A sampled step is one layer; tokens/s = 1 / (32 x the time per layer)."""
    import synth
    from oracle import linear
    d, kv, f = c["hidden"], c["kv"], c["ffn"]
    ranks = c2_ranks_oracle(c)
    rr = {w: [ranks[(0, k, sl)] for sl in range(n)] for w, k, n in (("qkv", 0, 3), ("o", 1, 1), ("upgate", 2, 2), ("down", 3, 1))}
    rs = max(16, -(-max(max(v) for v in rr.values()) // 16) * 16)
    mk = lambda N, K, s: synth.linear_case(100 + s, N=N, K=K, bits=c["bits"], r_stored=rs, zeros="asym",
                                           unit_gain=synth.STACK_GAINS[s])
    L = dict(qkv=[mk(d, d, 0), mk(kv, d, 1), mk(kv, d, 2)], o=[mk(d, d, 3)], upgate=[mk(f, d, 4), mk(f, d, 5)],
             down=[mk(d, f, 6)])
    h = synth.activations(1, 1, d)
    t0 = time.perf_counter()
    n = 0
    while True:
        linear.stack_forward([L], [rr], h)
        n += 1
        el = time.perf_counter() - t0
        if el >= seconds or n >= 8:
            break
    per_layer = el / n
    return 1.0 / (per_layer * c["layers"]), n, el


# ------------------------------------------------------------------ workload C3 (grouped MoE experts)
C3 = dict(name="c3", model="qwen3_30b_a3b", hidden=2048, ffn=768, experts=128, topk=8, layers=48, bits=3, group=128,
          r_stored=16)


def c3_matrix_bytes(N, K, bits, r):
    return N * K * bits // 8 + N * (K // 128) * (16 + bits) // 8 + 2 * r * (N + K)


def run_c3_ours(args, rank, world, device, T, c=C3):
    """48 MoE layers of 128 experts (3-bit, per-expert ranks in {0, 8, 16}); one step = hc_moe_forward on every
    layer for the same T routed tokens (routing drawn per layer as in SURVEY.md §8(d) C3)."""
    import torch
    import synth
    import paper_2605_05819_b200 as hc
    d, f, E, k, b, rs = c["hidden"], c["ffn"], c["experts"], c["topk"], c["bits"], c["r_stored"]
    ctx = hc.Context(device)
    levels = (0, 8, 16)
    rng = np.random.default_rng(123)
    ranks = {}
    e2 = ((4 ** b) - 1) / 12.0 + 0.25
    for l in range(c["layers"]):
        for e in range(E):
            rr = [levels[int(v)] for v in rng.integers(0, 3, size=3)]
            ranks[(l, e)] = rr
            mats = []
            for (win, slot, N, K, gl, r) in ((2, 0, f, d, 1, rr[0]), (2, 1, f, d, 1, rr[1]), (3, 0, d, f, 0, rr[2])):
                g = torch.Generator(device="cuda").manual_seed(10007 * l + 31 * e + 7 * win + slot)
                G = K // 128
                gain = 0.25 if win == 2 else 0.05
                mats.append(dict(layer=l, window=win, slot=slot, expert=e, N=N, K=K, bits=b, glue=gl,
                                 codes=torch.randint(-2**31, 2**31, (N, K * b // 32), generator=g, device="cuda", dtype=torch.int32),
                                 scales=(gain * (0.5 + torch.rand((N, G), generator=g, device="cuda")) / (e2 * K) ** 0.5).to(torch.bfloat16),
                                 zeros=torch.randint(0, 1 << b, (N, G), generator=g, device="cuda", dtype=torch.uint8),
                                 U=(torch.randn((N, rs), generator=g, device="cuda") / N ** 0.5).to(torch.bfloat16),
                                 V=(0.05 * (N / (rs * K)) ** 0.5 * torch.randn((rs, K), generator=g, device="cuda")).to(torch.bfloat16),
                                 r_stored=rs, r_alloc=r))
            ctx.load_layer(mats)
    torch.cuda.synchronize()
    x = torch.randn((T, d), generator=torch.Generator(device="cuda").manual_seed(5), device="cuda").to(torch.bfloat16)
    routes = [synth.routing_case(900 + l, T, E, k) for l in range(c["layers"])]
    idx = [torch.from_numpy(r[0]).cuda() for r in routes]
    gate = [torch.from_numpy(r[1]).cuda() for r in routes]
    ys = [torch.empty((T, d), dtype=torch.float32, device="cuda") for _ in range(c["layers"])]
    if getattr(args, "moe_dynamic", False):
        # per-(token, expert) ranks r = Cap(Align((k·g)·r̃)) (hc_moe_set_dynamic_ranks), r̃ ~ U[0, 24)
        for l in range(c["layers"]):
            ctx.moe_set_dynamic_ranks(l, (rng.random((E, 3)) * 24.0).astype(np.float32))
    nbytes = 0
    for l, (ri, _) in enumerate(routes):
        for e in sorted(set(int(v) for v in ri.reshape(-1))):
            ru, rg, rd = ranks[(l, e)]
            nbytes += c3_matrix_bytes(f, d, b, ru) + c3_matrix_bytes(f, d, b, rg) + c3_matrix_bytes(d, f, b, rd)
        nbytes += T * (2 * d + 4 * d) + T * k * 8
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for l in range(c["layers"]):
            ctx.moe_forward(l, x, idx[l], gate[l], ys[l], stream=st)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=st):
            for l in range(c["layers"]):
                ctx.moe_forward(l, x, idx[l], gate[l], ys[l], stream=st)
        for _ in range(max(args.warmup, 3)):
            graph.replay()
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(device) as clk, torch.cuda.stream(st):
        e0.record(st)
        for _ in range(args.steps):
            graph.replay()
        e1.record(st)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    finite = bool(all(torch.isfinite(yy).all().item() for yy in ys))
    # end to end with host buffers: x, routing in; y of the last layer out, every layer through the API
    xh = x.cpu()
    yh = np.zeros((T, d), dtype=np.float32)
    ih = [r[0] for r in routes]
    gh = [r[1] for r in routes]
    n_e2e = max(2, min(args.steps, 5))
    t0 = time.perf_counter()
    for _ in range(n_e2e):
        for l in range(c["layers"]):
            ctx.moe_forward(l, xh, ih[l], gh[l], yh)
    e2e_s = time.perf_counter() - t0
    ctx.close()
    return dict(ms=ms, steps=args.steps, clocks=clk.summary, e2e_s=e2e_s, n_e2e=n_e2e, finite=finite,
                launches=args.steps * c["layers"] * 8, bytes=nbytes,
                h2d=c["layers"] * (T * d * 2 + T * k * 8), d2h=c["layers"] * T * d * 4)


def oracle_c3_sample(seconds: float = 15.0, c=C3, T=16):
    """The float64 oracle on a bounded sample of C3: whole MoE layers (T routed tokens, top-8 of 128
    experts) of Qwen3-30B-A3B expert shapes; tokens/s extrapolated x48 layers."""
    import synth
    from oracle import linear
    d, f, E, k = c["hidden"], c["ffn"], c["experts"], c["topk"]
    idx, gate = synth.routing_case(901, T, E, k)
    act = sorted(set(int(v) for v in idx.reshape(-1)))
    mk = lambda N, K, s: synth.linear_case(200 + s, N=N, K=K, bits=c["bits"], r_stored=16, zeros="asym")
    experts = [dict(up=mk(f, d, 3 * i), gate=mk(f, d, 3 * i + 1), down=mk(d, f, 3 * i + 2)) if i in act else None
               for i in range(E)]
    ranks = [dict(up=8, gate=8, down=8) for _ in range(E)]
    x = synth.activations(3, T, d)
    t0 = time.perf_counter()
    n = 0
    while True:
        linear.moe_forward(experts, ranks, x, idx, gate)
        n += 1
        el = time.perf_counter() - t0
        if el >= seconds or n >= 4:
            break
    return T / (el / n * c["layers"]), n, el


# ------------------------------------------------------------------ workload C4 (prefill, tcgen05)
C4 = dict(name="c4", model="llama3_8b", hidden=4096, kv=1024, ffn=14336, layers=32, bits=4, group=128, M=2048,
          r_stored=256)


def c4_windows(c=C4):
    d, kv, f = c["hidden"], c["kv"], c["ffn"]
    return [(0, [d, kv, kv], d), (1, [d], d), (2, [f, f], d), (3, [d], f)]


def run_c4_ours(args, rank, world, device, r_all, c=C4):
    """Prefill of M = 2048 tokens through 32 Llama-3-8B-shaped layers (4 windows each; UPGATE runs as a
    plain 2-member window: the SiLU glue is a decode-path fusion), every matrix at rank r_all.  One
    step = the 128 window GEMMs on the same X (attention and the inter-window activations are out of
    scope); TFLOPS = algorithmic 2MNK + 2Mr(N+K) over the step."""
    import torch
    import paper_2605_05819_b200 as hc
    M, b, rs = c["M"], c["bits"], c["r_stored"]
    ctx = hc.Context(device)
    flops = 0
    outs = {}
    for l in range(c["layers"]):
        mats = []
        for kind, Ns, K in c4_windows(c):
            G = K // 128
            for sl, N in enumerate(Ns):
                g = torch.Generator(device="cuda").manual_seed(7919 * l + 13 * kind + sl)
                mats.append(dict(layer=l, window=kind, slot=sl, N=N, K=K, bits=b,
                                 codes=torch.randint(-2**31, 2**31, (N, K * b // 32), generator=g, device="cuda", dtype=torch.int32),
                                 scales=((0.5 + torch.rand((N, G), generator=g, device="cuda")) / (21.5 * K) ** 0.5).to(torch.bfloat16),
                                 zeros=torch.randint(0, 16, (N, G), generator=g, device="cuda", dtype=torch.uint8),
                                 U=(torch.randn((N, rs), generator=g, device="cuda") / N ** 0.5).to(torch.bfloat16),
                                 V=(0.05 * torch.randn((rs, K), generator=g, device="cuda") / K ** 0.5).to(torch.bfloat16),
                                 r_stored=rs, r_alloc=r_all))
                flops += 2 * M * N * K + 2 * M * r_all * (N + K)
        ctx.load_layer(mats)
        del mats
    torch.cuda.synchronize()
    xs = {K: torch.randn((M, K), generator=torch.Generator(device="cuda").manual_seed(K), device="cuda").to(torch.bfloat16)
          for K in (c["hidden"], c["ffn"])}
    for kind, Ns, K in c4_windows(c):
        outs[kind] = torch.empty((M, sum(Ns)), dtype=torch.bfloat16, device="cuda")
    st = torch.cuda.Stream()

    def step():
        for l in range(c["layers"]):
            for kind, Ns, K in c4_windows(c):
                ctx.compensated_linear(l, kind, xs[K], outs[kind], out_dtype=hc.OUT_BF16, stream=st)
    with torch.cuda.stream(st):
        step()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=st):
            step()
        for _ in range(max(args.warmup, 3)):
            graph.replay()
        torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(device) as clk, torch.cuda.stream(st):
        e0.record(st)
        for _ in range(args.steps):
            graph.replay()
        e1.record(st)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    finite = bool(all(torch.isfinite(o.float()).all().item() for o in outs.values()))
    # the rank sweep of C4 on the same weights: r = 0 (the uncompensated GEMM) and r = 256 (the largest level)
    rank_ms = {}
    for rr in (0, 256):
        if rr == r_all:
            continue
        for l in range(c["layers"]):
            for kind, Ns, K in c4_windows(c):
                for sl in range(len(Ns)):
                    ctx.set_rank(l, kind, sl, rr)
        with torch.cuda.stream(st):
            step()
            torch.cuda.synchronize()
            g2 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g2, stream=st):
                step()
            g2.replay()
            torch.cuda.synchronize()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record(st)
            for _ in range(args.steps):
                g2.replay()
            f1.record(st)
            torch.cuda.synchronize()
        fl = sum(2 * M * N * K + 2 * M * rr * (N + K) for _, Ns, K in c4_windows(c) for N in Ns) * c["layers"]
        rank_ms[rr] = (f0.elapsed_time(f1), fl)
        del g2
    for l in range(c["layers"]):
        for kind, Ns, K in c4_windows(c):
            for sl in range(len(Ns)):
                ctx.set_rank(l, kind, sl, r_all)
    # end to end: host X in, the last window's output back to the host, every window through the API
    xh = {K: v.cpu() for K, v in xs.items()}
    yh = np.zeros((M, c["hidden"]), dtype=np.uint16)
    t0 = time.perf_counter()
    n_e2e = 1
    for l in range(c["layers"]):
        for kind, Ns, K in c4_windows(c):
            ctx.compensated_linear(l, kind, xh[K], yh if kind in (1, 3) else outs[kind], out_dtype=hc.OUT_BF16)
    e2e_s = time.perf_counter() - t0
    ctx.close()
    return dict(ms=ms, steps=args.steps, clocks=clk.summary, e2e_s=e2e_s, n_e2e=n_e2e, finite=finite, flops=flops,
                rank_ms=rank_ms, launches=args.steps * c["layers"] * 4 * 3, h2d=c["layers"] * 4 * M * 4096 * 2, d2h=c["layers"] * 2 * M * 4096 * 2)


def oracle_c4_sample(seconds: float = 15.0, c=C4, r=64):
    """The float64 oracle on a bounded sample of C4: the O window (4096x4096, rank r) on 256 of the 2048
    tokens, repeated; converted to tokens/s of the whole 32-layer prefill step by the flop ratio."""
    import synth
    from oracle import linear
    case = synth.linear_case(41, N=4096, K=4096, bits=4, r_stored=max(r, 16), B=256)
    t0 = time.perf_counter()
    n = 0
    while True:
        linear.compensated_linear(case, r)
        n += 1
        el = time.perf_counter() - t0
        if el >= seconds or n >= 20:
            break
    fl_sample = 2 * 256 * 4096 * 4096 + 2 * 256 * r * (8192)
    fl_token = sum(2 * N * K + 2 * r * (N + K) for _, Ns, K in c4_windows(c) for N in Ns) * c["layers"]
    return fl_sample * n / el / fl_token, n, el


def traffic_of(args):
    """DRAM bytes per step of the timed kernels from one ncu capture of this code version
    (profiles/r02/traffic.json: dram__bytes_read.sum + dram__bytes_write.sum over the decode launches of one
    step, summed, written by tools/ncu_traffic.py); the algorithmic bytes of the same step are
    roofline.bytes_per_step.  Null where no capture exists for the workload / batch."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "traffic.json")) as f:
            t = json.load(f)
        return t.get(f"{args.workload}_B{args.batch}")
    except Exception:
        return None


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--mode", default="auto", choices=["auto", "tp", "replicas"],
                    help="N>1: tp = column-sharded stack with NCCL all-gather (strong scaling, default); "
                         "replicas = independent full-model replicas (weak scaling)")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--sweep", action="store_true", help="c2: also time B = 2, 4, 8, 16")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--rank-override", type=int, default=None, help="dev: use this rank for every matrix")
    ap.add_argument("--moe-dynamic", action="store_true", help="c3: per-(token, expert) dynamic ranks (P:652-665)")
    ap.add_argument("--no-sweep", action="store_true", help="c2: skip the default B = 2/4/8/16 sweep")
    ap.add_argument("--set-option", action="append", default=[], metavar="NAME=VALUE",
                    help="dev A/B: hc_set_option before the run (e.g. t_forward=1)")
    ap.add_argument("--factors", default="bf16", choices=["bf16", "fp8"],
                    help="compensation factor storage (fp8: e4m3 + per-rank fp32 scales, SURVEY 8(f)4)")
    ap.add_argument("--tp-path", default="peer", choices=["peer", "nccl"],
                    help="N>1 column sharding: peer = gather fused into the decode epilogue over NVLink peer "
                         "memory with partial-t exchange (default); nccl = ncclAllGather + unshard per window")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        # one process per GPU: re-launch this command under torch.distributed.run (the driver's own launch
        # sets WORLD_SIZE and skips this)
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        if os.environ.get("HC_BENCH_DRYRUN") == "1":     # test hook: show the launch instead of running it
            print(json.dumps({"spawn": cmd}))
            sys.exit(0)
        sys.exit(subprocess.call(cmd))

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    hbm, tflops, peak_src = peaks()
    tp = world > 1 and args.mode in ("auto", "tp")
    if args.workload == "c4":
        r4 = args.rank_override if args.rank_override is not None else 64
        config = {"workload": f"c4: prefill of 2048 tokens through 32 Llama-3-8B-shaped layers (QKV 6144, O 4096, "
                              f"UPGATE 2x14336, DOWN 4096x14336), 4-bit g128, rank {r4} on every matrix, tcgen05 GEMM",
                  "hidden": 4096, "kv": 1024, "ffn": 14336, "layers": 32, "bits": 4, "group": 128, "tokens": 2048,
                  "rank": r4, "parallelism": f"dp{world}",
                  "l2": "per-window weights (<= 60 MB) may be L2-resident across replays; prefill is tensor-bound"}
    elif args.workload == "c3":
        config = {"workload": f"c3: Qwen3-30B-A3B-shaped MoE expert linears (128 experts, top-8, 48 layers), 3-bit g128 + "
                              f"per-expert ranks in {{0, 8, 16}}, {args.batch} routed tokens per step, grouped launches",
                  "hidden": 2048, "expert_ffn": 768, "experts": 128, "topk": 8, "layers": 48, "bits": 3, "group": 128,
                  "tokens": args.batch, "parallelism": f"dp{world}",
                  "l2": "inputs larger than L2 (11.4 GB of expert weights; each step touches every layer)",
                  "routing": "softmax(N(0,1) logits) top-8, renormalised gates (synth.routing_case)",
                  "dynamic_ranks": bool(args.moe_dynamic)}
    elif args.workload == "c1":
        config = {"workload": "c1: single 4096x4096 linear, 4-bit g128, rank-64 compensation, batch-1 decode",
                  "N": 4096, "K": 4096, "bits": 4, "group": 128, "rank": 64, "batch": 1, "factors": args.factors,
                  "l2": "defeated: 128 distinct weight copies (1.25 GB) rotated per step"}
    else:
        c = STACKS[args.workload]
        desc = ("c2: Llama-2-7B-shaped 32-layer decode stack, 4-bit g128 + dynamic ranks (hc_allocate_ranks, "
                "r_std = 10%-bytes rule)" if args.workload == "c2" else
                "c5: Llama-3-70B-shaped 80-layer decode stack, 2-bit g128 + rank-64 compensation")
        config = {"workload": desc + ((f", column-sharded over {world} GPUs (" + ("gather fused into the decode epilogue over "
                                       "peer memory, partial-t exchange" if args.tp_path == "peer" else "NCCL all-gather per window")
                                       + ")") if tp else
                                      (f", {world} independent replicas" if world > 1 else ", 1 GPU")),
                  "layers": c["layers"], "hidden": c["hidden"], "kv": c["kv"], "ffn": c["ffn"], "bits": c["bits"],
                  "group": 128, "r_stored": c["r_stored"], "batch": args.batch, "factors": args.factors,
                  "parallelism": f"tp{world}" if tp else f"dp{world}",
                  "l2": "inputs larger than L2 (all weights streamed per step)",
                  "attention": "identity stand-in on the q-part (out of scope, DESIGN.md R9)"}

    if args.impl == "reference":
        if rank != 0:
            return
        # a sampled step is one unit of the workload the oracle ran in full (C1: one call; C2: one layer;
        # C3: one MoE layer; C4: one O-window product on 256 tokens); ms_per_step is its measured time, so
        # steps x ms_per_step is the wall time of the sample, and value converts it to the workload's metric
        if args.workload == "c1":
            n, el = oracle_c1_sample(seconds=max(5.0, min(60.0, 0.05 * (args.steps + args.warmup))))
            val, unit = c1_bytes() * n / el / 1e9, "GB/s"
            sample = f"{n} whole C1 calls (numpy float64, unpack+dequant+matvec); step = one call"
        elif args.workload == "c4":
            val, n, el = oracle_c4_sample(seconds=20.0, r=config["rank"])
            unit = "tokens/s"
            sample = (f"{n} O-window products (256 tokens, 4096x4096, rank {config['rank']}, float64), flop-scaled "
                      f"to the 32-layer step; step = one product")
        elif args.workload == "c3":
            val, n, el = oracle_c3_sample(seconds=20.0, T=args.batch)
            unit = "tokens/s"
            sample = f"{n} whole MoE layers ({args.batch} tokens, top-8 of 128 experts, float64), x48 layers; step = one layer"
        else:
            val, n, el = oracle_c2_sample(seconds=20.0)
            unit = "tokens/s"
            sample = (f"{n} whole Llama-2-7B layers at B=1 (float64, all 4 windows + glue, allocator ranks of layer 0), "
                      f"x32 layers; step = one layer")
        ms = 1e3 * el / n
        line = {"impl": "reference", "metric": METRIC, "value": round(val, 6), "unit": unit, "n_gpus": args.gpus,
                "steps": n, "warmup": 0, "ms_per_step": round(ms, 3), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config,
                "cpu_baseline": {"value": round(val, 6), "unit": unit, "cores": cores(), "kind": "oracle",
                                 "sample": sample},
                "e2e": {"value": round(val, 6), "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import paper_2605_05819_b200 as hc
    for kv in args.set_option:
        k, v = kv.split("=")
        hc.set_option(k, int(v))
    if args.set_option:
        config["options"] = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in args.set_option}
    if world > 1:
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    if args.workload == "c4":
        r = run_c4_ours(args, rank, world, local, config["rank"])
        nbytes = 0
        unit, kernel = "tokens/s", "hc::prefill_kernel (tcgen05, 128x256 tiles)"
    elif args.workload == "c3":
        r = run_c3_ours(args, rank, world, local, args.batch)
        nbytes = r["bytes"]
        unit, kernel = "tokens/s", "hc::moe_gemv_kernel<3> (grouped UPGATE + DOWN per layer)"
    elif args.workload == "c1":
        r = run_c1_ours(args, rank, world, local)
        nbytes = c1_bytes(kind=args.factors)
        unit, kernel = "GB/s", "hc::decode_kernel<4,1,true,true> (int8 mma path)"
    else:
        sweep = () if (args.workload != "c2" or args.no_sweep) else tuple(b for b in (1, 2, 4, 8, 16) if b != args.batch)
        if args.sweep and args.workload == "c5":
            sweep = (2, 4, 8, 16)
        r = run_c2_ours(args, rank, world, local, args.batch, STACKS[args.workload], tp, sweep=sweep)
        nbytes = r["bytes"]
        unit, kernel = "tokens/s", "hc::decode_kernel (4 fused windows per layer; int8 mma path where x8 fits)"
    per_rank = torch.tensor([r["ms"]], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(per_rank, op=torch.distributed.ReduceOp.MAX)
    ms_max = float(per_rank.item())
    achieved = nbytes / (r["ms"] / r["steps"] * 1e-3) / 1e9
    if args.workload == "c4":
        value = world * 2048 * r["steps"] / (ms_max * 1e-3)
        tfl = r["flops"] / (r["ms"] / r["steps"] * 1e-3) / 1e12
        e2e = {"value": round(2048 * r["n_e2e"] / r["e2e_s"], 2), "unit": "tokens/s",
               "h2d_bytes_per_step": r["h2d"], "d2h_bytes_per_step": r["d2h"]}
        config["flops_per_step"] = r["flops"]
        config["output_finite"] = r["finite"]
    elif args.workload == "c1":
        value = world * nbytes * r["steps"] / (ms_max * 1e-3) / 1e9
        e2e = {"value": round(nbytes * r["n_e2e"] / r["e2e_s"] / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": r["h2d"], "d2h_bytes_per_step": r["d2h"]}
    else:
        streams = 1 if tp else world           # column sharding serves one stream; replicas serve `world`
        value = streams * args.batch * r["steps"] / (ms_max * 1e-3)
        e2e = {"value": round(streams * args.batch * r["n_e2e"] / r["e2e_s"], 2), "unit": "tokens/s",
               "h2d_bytes_per_step": r["h2d"], "d2h_bytes_per_step": r["d2h"]}
        if "mean_rank" in r:
            config["mean_rank"] = round(r["mean_rank"], 2)
        config["bytes_per_step"] = nbytes
        config["output_finite"] = r["finite"]
    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 2), "unit": unit, "n_gpus": world, "steps": r["steps"],
                "warmup": args.warmup, "ms_per_step": round(ms_max / r["steps"], 6), "higher_is_better": True,
                "scaling": "strong" if tp else "weak", "vs_baseline": None, "dtype": dtype_of(args, config),
                "data": "synthetic (seeded on device, random weights of the named shapes)", "config": config,
                "roofline": ({"bound": "hbm", "achieved": round(achieved, 2), "peak": hbm, "unit": "GB/s",
                              "frac": round(achieved / hbm, 4), "traffic": traffic_of(args), "peak_source": peak_src,
                              "kernel": kernel, "bytes_per_step": nbytes} if args.workload != "c4" else
                             {"bound": "tensor", "achieved": round(tfl, 1), "peak": tflops, "unit": "TFLOP/s",
                              "frac": round(tfl / tflops, 4), "traffic": None, "peak_source": peak_src,
                              "kernel": kernel, "flops_per_step": r["flops"]}),
                "clocks": r["clocks"], "gpu_launches": r["launches"], "e2e": e2e}
        if args.workload == "c3" and args.sweep:
            sweep = {}
            for Ts in (1, 16, 64, 256):
                rs = run_c3_ours(args, rank, world, local, Ts)
                sweep[str(Ts)] = {"tokens_per_s": round(Ts * rs["steps"] / (rs["ms"] * 1e-3), 1),
                                  "ms_per_step": round(rs["ms"] / rs["steps"], 4),
                                  "GBps": round(rs["bytes"] / (rs["ms"] / rs["steps"] * 1e-3) / 1e9, 1)}
            line["token_sweep"] = sweep
        elif r.get("sweep"):
            line["batch_sweep"] = r["sweep"]
        # compensation overhead against the same weights at r = 0 (the paper's analogue is
        # "≥85% of throughput"): time ratio - 1 beside the algorithmic byte / flop floor of the factors
        if args.workload == "c1":
            b0 = c1_bytes(r=0)
            line["overhead_vs_r0"] = {"rank": C1["r"], "time": round(r["ms"] / r["ms_r0"] - 1, 4),
                                      "bytes_floor": round(nbytes / b0 - 1, 4),
                                      "r0_GBps_of_r0_bytes": round(b0 * r["steps"] / (r["ms_r0"] * 1e-3) / 1e9, 1)}
        elif args.workload in ("c2", "c5"):
            line["overhead_vs_r0"] = {"rank": "allocated" if args.workload == "c2" else STACKS[args.workload]["fixed_rank"],
                                      "time": round(r["ms"] / r["ms_r0"] - 1, 4),
                                      "bytes_floor": round(r["bytes"] / r["bytes_r0"] - 1, 4),
                                      "r0_tokens_per_s": round(args.batch * r["steps"] / (r["ms_r0"] * 1e-3), 2)}
        elif args.workload == "c4":
            rs_ = {str(config["rank"]): {"TFLOPS": round(tfl, 1), "ms_per_step": round(r["ms"] / r["steps"], 4)}}
            for rr, (mss, fl) in r["rank_ms"].items():
                rs_[str(rr)] = {"TFLOPS": round(fl / (mss / r["steps"] * 1e-3) / 1e12, 1),
                                "ms_per_step": round(mss / r["steps"], 4)}
            line["rank_sweep"] = rs_
            if 0 in r["rank_ms"]:
                ms0, fl0 = r["rank_ms"][0]
                ov = {str(config["rank"]): {"time": round(r["ms"] / ms0 - 1, 4), "flops_floor": round(r["flops"] / fl0 - 1, 4)}}
                if 256 in r["rank_ms"]:
                    ms2, fl2 = r["rank_ms"][256]
                    ov["256"] = {"time": round(ms2 / ms0 - 1, 4), "flops_floor": round(fl2 / fl0 - 1, 4)}
                line["overhead_vs_r0"] = ov
        if not args.no_cpu_baseline:
            if args.workload == "c1":
                n, el = oracle_c1_sample(12.0)
                line["cpu_baseline"] = {"value": round(nbytes * n / el / 1e9, 4), "unit": "GB/s", "cores": cores(),
                                        "kind": "oracle", "sample": f"{n} whole C1 calls, numpy float64"}
            elif args.workload == "c4":
                tps, n, el = oracle_c4_sample(15.0, r=config["rank"])
                line["cpu_baseline"] = {"value": round(tps, 6), "unit": "tokens/s", "cores": cores(), "kind": "oracle",
                                        "sample": f"{n} O-window products (256 tokens, float64), flop-scaled"}
            elif args.workload == "c3":
                tps, n, el = oracle_c3_sample(15.0, T=args.batch)
                line["cpu_baseline"] = {"value": round(tps, 6), "unit": "tokens/s", "cores": cores(), "kind": "oracle",
                                        "sample": f"{n} whole MoE layers ({args.batch} tokens, float64), extrapolated x48"}
            elif args.workload == "c2":
                tps, n, el = oracle_c2_sample(15.0)
                line["cpu_baseline"] = {"value": round(tps, 6), "unit": "tokens/s", "cores": cores(), "kind": "oracle",
                                        "sample": f"{n} whole Llama-2-7B layers at B=1 (float64), extrapolated x32"}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
