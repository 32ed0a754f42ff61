"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck):
decode windows (int8 path, fp16 staged and x-prep paths, fused SiLU, fp8 factors), a 2-layer stack graph,
the grouped MoE layer, the tcgen05 prefill, the calibration SVD.  Each result is checked against the oracle
so a sanitizer run also shows the outputs stayed correct.
    compute-sanitizer --tool memcheck python tools/sanitize_cases.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_05819_b200 as hc  # noqa: E402
import synth  # noqa: E402
from oracle import linear  # noqa: E402

dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()


def desc(c, layer, window, slot, r, glue=0):
    return dict(layer=layer, window=window, slot=slot, N=c["N"], K=c["K"], bits=c["bits"], codes=dev(c["codes"]),
                scales=dev(c["scales"]), zeros=dev(c["zeros"]), U=dev(c["U"]), V=dev(c["V"]), r_stored=c["r_stored"],
                r_alloc=r, glue=glue)


def check(y, ref, tol, what):
    e = float(np.abs(y - ref).max() / np.abs(ref).max())
    assert e <= tol, (what, e)
    print(f"{what}: ok ({e:.2e})", flush=True)


ctx = hc.Context(0)
L = 0
for bits, B, K in ((4, 1, 512), (3, 4, 512), (4, 16, 384), (2, 2, 1280)):
    c = synth.linear_case(10 + bits + B, N=128, K=K, bits=bits, r_stored=32, B=B, zeros="asym")
    ctx.load_layer([desc(c, L, 0, 0, 32)])
    y = torch.empty((B, 128), dtype=torch.float32, device="cuda")
    ctx.compensated_linear(L, 0, dev(c["x"]), y)
    torch.cuda.synchronize()
    check(y.cpu().numpy(), linear.compensated_linear(c, 32), 1e-5, f"decode bits {bits} B {B} K {K}")
    L += 1
# int8 path with several items per CTA (both epilogue warps: items alternate between them) and the extra-tier t
# pass (tiny activations put the V·x partials below 2^-24): decode grid capped at one CTA per SM
hc.set_option("decode_ctas_per_sm", 1)
for scale, tag in ((1.0, "int8 multi-item"), (1e-9, "int8 multi-item, extra-tier t")):
    c = synth.linear_case(30, N=4096, K=512, bits=4, r_stored=32, B=1, zeros="asym")
    xb = (c["x"].astype(np.uint32) << 16).view(np.float32) * np.float32(scale)
    c["x"] = (xb.view(np.uint32) >> 16).astype(np.uint16)          # exact: a power-of-ten scale of bf16 values, truncated
    ctx.load_layer([desc(c, L, 0, 0, 32)])
    y = torch.empty((1, 4096), dtype=torch.float32, device="cuda")
    ctx.compensated_linear(L, 0, dev(c["x"]), y)
    torch.cuda.synchronize()
    check(y.cpu().numpy(), linear.compensated_linear(c, 32), 1e-5, tag)
    L += 1
hc.set_option("decode_ctas_per_sm", 0)
# fused SiLU + fp8 factors
up = synth.linear_case(40, N=128, K=256, bits=4, r_stored=16, B=2, zeros="asym", unit_gain=True)
gate = synth.linear_case(41, N=128, K=256, bits=4, r_stored=16, B=2, zeros="asym", unit_gain=True)
ctx.load_layer([desc(up, L, hc.UPGATE, 0, 16, hc.GLUE_SILU_MUL), desc(gate, L, hc.UPGATE, 1, 8, hc.GLUE_SILU_MUL)])
y = torch.empty((2, 128), dtype=torch.float32, device="cuda")
ctx.compensated_linear(L, hc.UPGATE, dev(up["x"]), y)
torch.cuda.synchronize()
check(y.cpu().numpy(), linear.silu(linear.compensated_linear(gate, 8, x_bits=up["x"])) * linear.compensated_linear(up, 16),
      1e-5, "fused SiLU")
L += 1
f8 = synth.fp8_factors(synth.linear_case(42, N=128, K=512, bits=4, r_stored=32, B=1, zeros="asym"), 43)
ctx.load_layer([dict(desc(f8, L, 0, 0, 32), U=dev(f8["U8"]), V=dev(f8["V8"]), u_scale=dev(f8["us"]),
                     v_scale=dev(f8["vs"]), factor_dtype=hc.FACTORS_FP8)])
y = torch.empty((1, 128), dtype=torch.float32, device="cuda")
ctx.compensated_linear(L, 0, dev(f8["x"]), y)
torch.cuda.synchronize()
check(y.cpu().numpy(), linear.compensated_linear(f8, 32), 1e-5, "fp8 factors")
# prefill (tcgen05)
c = synth.linear_case(50, N=256, K=512, bits=4, r_stored=32, B=64, zeros="asym")
ctx.load_layer([desc(c, 100, 0, 0, 32)])
y = torch.empty((64, 256), dtype=torch.float32, device="cuda")
ctx.compensated_linear(100, 0, dev(c["x"]), y)
torch.cuda.synchronize()
check(y.cpu().numpy(), linear.compensated_linear(c, 32), 2e-3, "prefill")
ctx.close()
# stack (2 layers)
STACK_GAINS = (1.0, 1.0, 1.0, 0.25, 0.25, 0.25, 0.05)
cs = hc.Context(0)
layers, ranks = [], []
for l in range(2):
    mk = lambda n, k, s: synth.linear_case(60 + 10 * l + s, N=n, K=k, bits=4, r_stored=16, zeros="asym", unit_gain=STACK_GAINS[s])
    Ly = dict(qkv=[mk(128, 128, 0), mk(128, 128, 1), mk(128, 128, 2)], o=[mk(128, 128, 3)],
              upgate=[mk(256, 128, 4), mk(256, 128, 5)], down=[mk(128, 256, 6)])
    Ry = dict(qkv=[16, 8, 0], o=[16], upgate=[8, 16], down=[16])
    mats = [desc(Ly["qkv"][i], l, hc.QKV, i, Ry["qkv"][i]) for i in range(3)] + [desc(Ly["o"][0], l, hc.O, 0, 16)]
    mats += [desc(Ly["upgate"][i], l, hc.UPGATE, i, Ry["upgate"][i], hc.GLUE_SILU_MUL) for i in range(2)]
    mats += [desc(Ly["down"][0], l, hc.DOWN, 0, 16)]
    cs.load_layer(mats)
    layers.append(Ly)
    ranks.append(Ry)
x = synth.activations(3, 1, 128)
y = torch.empty((1, 128), dtype=torch.int16, device="cuda")
cs.stack_forward(dev(x), y)
torch.cuda.synchronize()
from oracle.packing import bf16_to_f64  # noqa: E402
check(bf16_to_f64(y.cpu().numpy().view(np.uint16)), linear.stack_forward(layers, ranks, x), 2e-2, "stack")
cs.close()
# MoE (8 experts, top-2, 3 tokens)
cm = hc.Context(0)
E, d, f = 8, 256, 128
experts, eranks = [], []
for e in range(E):
    ex = dict(up=synth.linear_case(80 + 3 * e, N=f, K=d, bits=3, r_stored=16, zeros="asym"),
              gate=synth.linear_case(81 + 3 * e, N=f, K=d, bits=3, r_stored=16, zeros="asym"),
              down=synth.linear_case(82 + 3 * e, N=d, K=f, bits=3, r_stored=16, zeros="asym"))
    experts.append(ex)
    eranks.append(dict(up=8, gate=16, down=8))
    cm.load_layer([dict(desc(ex["up"], 0, hc.UPGATE, 0, 8, hc.GLUE_SILU_MUL), expert=e),
                   dict(desc(ex["gate"], 0, hc.UPGATE, 1, 16, hc.GLUE_SILU_MUL), expert=e),
                   dict(desc(ex["down"], 0, hc.DOWN, 0, 8), expert=e)])
idx, gw = synth.routing_case(5, 3, E, 2)
xm = synth.activations(4, 3, d)
ym = torch.empty((3, d), dtype=torch.float32, device="cuda")
cm.moe_forward(0, dev(xm), dev(idx.astype(np.int32)), dev(gw.astype(np.float32)), ym)
torch.cuda.synchronize()
check(ym.cpu().numpy(), linear.moe_forward(experts, eranks, xm, idx, gw), 1e-4, "moe")
# calibration SVD
W = 0.02 * torch.randn((1, 64, 128), device="cuda")
codes = torch.randint(-2**31, 2**31, (1, 64, 128 * 4 // 32), device="cuda", dtype=torch.int32)
scales = torch.full((1, 64, 1), 0.003, device="cuda").to(torch.bfloat16)
zeros = torch.full((1, 64, 1), 8, dtype=torch.uint8, device="cuda")
U = torch.empty((1, 64, 16), dtype=torch.float64, device="cuda")
V = torch.empty((1, 16, 128), dtype=torch.float64, device="cuda")
S = torch.empty((1, 64), dtype=torch.float64, device="cuda")
sw = cm.calib_svd(W, codes, scales, zeros, 4, 128, 16, U, V, S)
torch.cuda.synchronize()
print(f"calib svd: {sw} sweeps, sigma1 {S[0, 0].item():.4g}", flush=True)
cm.close()
print("all cases done")
