"""Decode-kernel timing sweep (development tool, not the driver bench): one window of the given
shape, rotating through enough distinct copies to defeat L2, CUDA-graph replayed."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_05819_b200 as hc


def bytes_of(N, K, bits, r, B):
    return N * K * bits // 8 + N * (K // 128) * (16 + bits) // 8 + 2 * r * (N + K) + B * (2 * K + 4 * N)


def run(ctx, N, K, bits, r, B, layer0, copies=None, reps=20):
    per = bytes_of(N, K, bits, 0, 0)
    copies = copies or max(4, min(256, int(1.5e9 // per)))
    g = torch.Generator(device="cuda").manual_seed(N + K + r)
    G = K // 128
    for i in range(copies):
        ctx.load_layer([dict(layer=layer0 + i, window=0, slot=0, N=N, K=K, bits=bits,
                             codes=torch.randint(-2**31, 2**31, (N, K * bits // 32), generator=g, device="cuda", dtype=torch.int32),
                             scales=(0.002 + 0.01 * torch.rand((N, G), generator=g, device="cuda")).to(torch.bfloat16),
                             zeros=torch.randint(0, 1 << bits, (N, G), generator=g, device="cuda", dtype=torch.uint8),
                             U=(torch.randn((N, 64), generator=g, device="cuda") / N ** 0.5).to(torch.bfloat16),
                             V=(0.02 * torch.randn((64, K), generator=g, device="cuda")).to(torch.bfloat16),
                             r_stored=64, r_alloc=r)])
    x = torch.randn((B, K), generator=g, device="cuda").to(torch.bfloat16)
    y = torch.empty((B, N), dtype=torch.float32, device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for i in range(copies):
            ctx.compensated_linear(layer0 + i, 0, x, y, stream=st)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=st):
            for i in range(copies):
                ctx.compensated_linear(layer0 + i, 0, x, y, stream=st)
        gr.replay(); gr.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            gr.replay()
        e1.record(st)
        torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (reps * copies)
    nb = bytes_of(N, K, bits, r, B)
    return dict(N=N, K=K, bits=bits, r=r, B=B, us=round(us, 3), gbs=round(nb / us / 1e3, 1), copies=copies)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="2368,128,4,0,1;4096,4096,4,0,1;4096,4096,4,64,1;16384,4096,4,0,1;16384,4096,4,64,1;4096,16384,4,64,1;22016,4096,4,64,1;4096,4096,4,64,8;4096,4096,4,64,16;4096,4096,3,64,1;4096,4096,2,64,1")
    args = ap.parse_args()
    ctx = hc.Context(0)
    layer = 0
    for c in args.cases.split(";"):
        N, K, bits, r, B = map(int, c.split(","))
        res = run(ctx, N, K, bits, r, B, layer)
        layer += 1000
        print(json.dumps(res), flush=True)
