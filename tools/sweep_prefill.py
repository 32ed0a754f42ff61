"""Prefill (tcgen05) timing sweep (development tool): C4 = 2048 tokens through Llama-3-8B-shaped
windows, 4-bit g128, rank sweep.  TFLOPS = algorithmic flops (2MNK + 2Mr(N+K)) / time."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_05819_b200 as hc

SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "upgate": (28672, 4096), "down": (4096, 14336)}


def load(ctx, layer, N, K, r, rs=256):
    g = torch.Generator(device="cuda").manual_seed(layer)
    G = K // 128
    ctx.load_layer([dict(layer=layer, window=0, slot=0, N=N, K=K, bits=4,
                         codes=torch.randint(-2**31, 2**31, (N, K // 8), generator=g, device="cuda", dtype=torch.int32),
                         scales=(0.002 + 0.01 * torch.rand((N, G), generator=g, device="cuda")).to(torch.bfloat16),
                         zeros=torch.randint(0, 16, (N, G), generator=g, device="cuda", dtype=torch.uint8),
                         U=(torch.randn((N, rs), generator=g, device="cuda") / N ** 0.5).to(torch.bfloat16),
                         V=(0.02 * torch.randn((rs, K), generator=g, device="cuda")).to(torch.bfloat16),
                         r_stored=rs, r_alloc=r)])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=2048)
    ap.add_argument("--ranks", default="0,8,16,32,64,128,256")
    ap.add_argument("--shapes", default="qkv,o,upgate,down")
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    ctx = hc.Context(0)
    M = args.M
    layer = 0
    for name in args.shapes.split(","):
        N, K = SHAPES[name]
        x = torch.randn((M, K), device="cuda").to(torch.bfloat16)
        y = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
        for r in [int(v) for v in args.ranks.split(",")]:
            layer += 1
            load(ctx, layer, N, K, r)
            st = torch.cuda.current_stream()
            for _ in range(3):
                ctx.compensated_linear(layer, 0, x, y, out_dtype=hc.OUT_BF16)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.reps):
                ctx.compensated_linear(layer, 0, x, y, out_dtype=hc.OUT_BF16)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / args.reps
            flops = 2 * M * N * K + 2 * M * r * (N + K)
            print(json.dumps(dict(shape=name, M=M, N=N, K=K, r=r, us=round(us, 1),
                                  tflops=round(flops / us / 1e6, 1))), flush=True)


if __name__ == "__main__":
    main()
