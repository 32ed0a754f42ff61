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


def c1_bytes(c=C1):
    """Algorithmic bytes of one C1 call: codes b/8 per element, a bf16
    scale + a b-bit zero per group, the rank-r slices of U and V (bf16), x (bf16) and y (fp32)."""
    N, K, b, g, r, B = c["N"], c["K"], c["bits"], c["group"], c["r"], c["B"]
    base = N * K * b // 8 + N * (K // g) * (16 + b) // 8
    fac = 2 * r * (N + K)
    io = B * (2 * K + 4 * N)
    return base + fac + io


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
                             U=U, V=V, r_stored=c["r_stored"], r_alloc=c["r"])])
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
    return dict(ms=ms, steps=steps, clocks=clk.summary, e2e_s=e2e_s, n_e2e=n_e2e,
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


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1024)
    ap.add_argument("--warmup", type=int, default=256)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c1", choices=["c1"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    hbm, tflops, peak_src = peaks()
    config = {"workload": "c1: single 4096x4096 linear, 4-bit g128, rank-64 compensation, batch-1 decode",
              "N": 4096, "K": 4096, "bits": 4, "group": 128, "rank": 64, "batch": 1,
              "l2": "defeated: 128 distinct weight copies (1.25 GB) rotated per step"}

    if args.impl == "reference":
        if rank != 0:
            return
        n, el = oracle_c1_sample(seconds=max(5.0, min(60.0, 0.05 * (args.steps + args.warmup))))
        gbs = c1_bytes() * n / el / 1e9
        line = {"impl": "reference", "metric": METRIC, "value": round(gbs, 4), "unit": "GB/s", "n_gpus": args.gpus,
                "steps": n, "warmup": 0, "ms_per_step": round(1e3 * el / n, 3), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config,
                "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": cores(), "kind": "oracle",
                                 "sample": f"{n} whole C1 calls (numpy float64, unpack+dequant+matvec)"},
                "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    if world > 1:
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    r = run_c1_ours(args, rank, world, local)
    ms_step = r["ms"] / r["steps"]
    nbytes = c1_bytes()
    per_rank = torch.tensor([r["ms"]], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(per_rank, op=torch.distributed.ReduceOp.MAX)
    ms_max = float(per_rank.item())
    value = world * nbytes * r["steps"] / (ms_max * 1e-3) / 1e9
    achieved = nbytes / (r["ms"] / r["steps"] * 1e-3) / 1e9
    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": r["steps"],
                "warmup": args.warmup, "ms_per_step": round(ms_max / r["steps"], 6), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "bf16x int4 (fp32 accumulate)",
                "data": "synthetic (seeded on device)", "config": config,
                "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": hbm, "unit": "GB/s",
                             "frac": round(achieved / hbm, 4), "traffic": None, "peak_source": peak_src,
                             "kernel": "hc::decode_kernel<4,1>", "bytes_per_launch": nbytes},
                "clocks": r["clocks"], "gpu_launches": r["launches"],
                "e2e": {"value": round(nbytes * r["n_e2e"] / r["e2e_s"] / 1e9, 3), "unit": "GB/s",
                        "h2d_bytes_per_step": r["h2d"], "d2h_bytes_per_step": r["d2h"]}}
        if not args.no_cpu_baseline:
            n, el = oracle_c1_sample(12.0)
            line["cpu_baseline"] = {"value": round(nbytes * n / el / 1e9, 4), "unit": "GB/s", "cores": cores(),
                                    "kind": "oracle", "sample": f"{n} whole C1 calls, numpy float64"}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
