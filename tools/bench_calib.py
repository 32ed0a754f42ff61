"""Time the GPU calibration (hc_calib_svd + hc_calib_salience) on model-sized matrices (dev tool).
    python tools/bench_calib.py [N K bits r n_mats]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_05819_b200 as hc  # noqa: E402

N, K, bits, r, M = (int(v) for v in (sys.argv[1:] + ["4096", "4096", "4", "256", "1"][len(sys.argv) - 1:])[:5])
g = torch.Generator(device="cuda").manual_seed(0)
W = 0.02 * torch.randn((M, N, K), generator=g, device="cuda")
codes = torch.randint(-2**31, 2**31, (M, N, K * bits // 32), generator=g, device="cuda", dtype=torch.int32)
scales = (W.abs().amax(dim=2, keepdim=True).expand(M, N, K // 128) / ((1 << (bits - 1)) - 1)).to(torch.bfloat16).contiguous()
zeros = torch.full((M, N, K // 128), 1 << (bits - 1), dtype=torch.uint8, device="cuda")
U = torch.empty((M, N, r), dtype=torch.float64, device="cuda")
V = torch.empty((M, r, K), dtype=torch.float64, device="cuda")
S = torch.empty((M, min(N, K)), dtype=torch.float64, device="cuda")
ctx = hc.Context(0)
torch.cuda.synchronize()
t0 = time.perf_counter()
sweeps = ctx.calib_svd(W, codes, scales, zeros, bits, 128, r, U, V, S)
torch.cuda.synchronize()
t1 = time.perf_counter()
phi = torch.empty(M, dtype=torch.float64, device="cuda")
cut = torch.empty(M, dtype=torch.int32, device="cuda")
ctx.calib_salience(S, phi, cut)
torch.cuda.synchronize()
print(f"calib_svd {M}x{N}x{K} bits {bits} r {r}: {t1 - t0:.2f} s, {sweeps} sweeps, sigma1 {S[0, 0].item():.4g}, "
      f"phi {phi[0].item():.4g} cut {int(cut[0].item())}")
