"""Per-window timeline of the per-window decode graph (dev tool; needs an HC_DEC_TRACE=1 build via
HC_LIB_PATH).  For each window kind: when its CTAs start (relative to the previous window's last
epilogue), when the PDL wait releases, first / last FULL (tile work), epilogue end."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_05819_b200 as hc  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
c = bench.C2
ranks = bench.c2_ranks(c)
if os.environ.get("HC_TRACE_R0"):
    ranks = {key: 0 for key in ranks}
for kv in os.environ.get("HC_TRACE_OPTS", "").split():   # e.g. t_forward=1
    hc.set_option(kv.split("=")[0], int(kv.split("=")[1]))
ctx = hc.Context(0)
bench.build_c2(ctx, ranks, c)
n_win, grid = 4 * c["layers"], 512
buf = torch.zeros((n_win, grid, 16), dtype=torch.int64, device="cuda")
L = hc.lib()
L.hc_dev_decode_trace.argtypes = [ctypes.c_void_p]
assert L.hc_dev_decode_trace(buf.data_ptr()) == 0
x = torch.randn((B, c["hidden"]), device="cuda").to(torch.bfloat16)
y = torch.empty((B, c["hidden"]), dtype=torch.bfloat16, device="cuda")
for _ in range(5):
    ctx.stack_forward(x, y)
torch.cuda.synchronize()
buf.zero_()
ctx.stack_forward(x, y)
torch.cuda.synchronize()
t = buf.cpu().numpy().astype(np.float64)
t0 = t[t > 0].min()
t = np.where(t > 0, (t - t0) / 1e3, np.nan)
end = np.nanmax(t[:, :, 4], axis=1)
print("step µs", np.nanmax(end))
prev = np.concatenate([[0.0], end[:-1]])
names = ["qkv", "o", "upgate", "down"]
for k in range(4):
    idx = np.arange(k, n_win, 4)
    rel = t[idx] - prev[idx, None, None]
    q = lambda ev, f: np.nanmean(f(rel[:, :, ev], axis=1))
    print(f"{names[k]:7s} win {np.mean(end[idx] - prev[idx]):6.2f} | start min {q(0, np.nanmin):6.2f} max {q(0, np.nanmax):6.2f}"
          f" | pdl {q(1, np.nanmin):6.2f}/{q(1, np.nanmax):6.2f} | 1stFULL {q(2, np.nanmin):6.2f}/{q(2, np.nanmedian):6.2f}/{q(2, np.nanmax):6.2f}"
          f" | t {q(5, np.nanmin):6.2f}/{q(5, np.nanmax):6.2f} | stg {q(6, np.nanmedian):6.2f}->{q(8, np.nanmedian):6.2f}->{q(7, np.nanmedian):6.2f} | Vx {q(9, np.nanmedian):6.2f}/{q(9, np.nanmax):6.2f} Vflush {q(10, np.nanmedian):6.2f}/{q(10, np.nanmax):6.2f} rel {q(12, np.nanmax):6.2f} vdone {q(11, np.nanmin):6.2f}/{q(11, np.nanmedian):6.2f} t0 {q(13, np.nanmedian):6.2f} tdeep {q(14, np.nanmedian):6.2f} | lastFULL {q(3, np.nanmedian):6.2f}/{q(3, np.nanmax):6.2f} | epi {q(4, np.nanmedian):6.2f}/{q(4, np.nanmax):6.2f}")
ctx.close()
