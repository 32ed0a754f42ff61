"""Per-window timeline of the persistent stack kernel (dev tool; needs an HC_STK_TRACE=1 build via
HC_LIB_PATH).  Prints, per window kind, the mean time from the previous window's completion to
x-ready / staged / tiles-done / epilogue-done, min and max over CTAs."""
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
ctx = hc.Context(0)
bench.build_c2(ctx, ranks, c)
n_win, grid = 4 * c["layers"], 148
buf = torch.zeros((n_win, grid, 4), dtype=torch.int64, device="cuda")
L = hc.lib()
L.hc_dev_stack_trace.argtypes = [ctypes.c_void_p]
assert L.hc_dev_stack_trace(buf.data_ptr()) == 0
acct = torch.zeros((grid, 17, 8), dtype=torch.int64, device="cuda")
L.hc_dev_stack_acct.argtypes = [ctypes.c_void_p]
assert L.hc_dev_stack_acct(acct.data_ptr()) == 0
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
t = np.where(t > 0, (t - t0) / 1e3, np.nan)          # µs from the first stamp
done = np.nanmax(t[:, :, 3], axis=1)                  # window complete (last epilogue)
print("total µs", np.nanmax(done))
names = ["qkv", "o", "upgate", "down"]
prev = np.concatenate([[0.0], done[:-1]])
for k in range(4):
    idx = np.arange(k, n_win, 4)
    rows = []
    for ev in range(4):
        d = t[idx, :, ev] - prev[idx, None]
        rows.append((np.nanmean(np.nanmin(d, axis=1)), np.nanmean(np.nanmedian(d, axis=1)), np.nanmean(np.nanmax(d, axis=1))))
    dur = np.mean(done[idx] - prev[idx])
    print(f"{names[k]:7s} window {dur:7.2f} µs | " + " | ".join(f"ev{e} min {a:6.2f} med {b:6.2f} max {m:6.2f}" for e, (a, b, m) in enumerate(rows)))
a = acct.cpu().numpy().astype(np.float64)
tile = a[:, :16, :]
tot = tile[:, :, 3].mean()
print("tile warps: data wait %.1f%%  EMPTY wait %.1f%%  x wait %.1f%%  V %.1f%%  bar1 %.1f%%  staging(incl x wait) %.1f%% (of %.0f cycles)" % (
    100 * tile[:, :, 0].mean() / tot, 100 * tile[:, :, 1].mean() / tot, 100 * tile[:, :, 2].mean() / tot,
    100 * tile[:, :, 4].mean() / tot, 100 * tile[:, :, 5].mean() / tot, 100 * tile[:, :, 6].mean() / tot, tot))
e = a[:, 16, :]
print("epilogue: FULL wait %.1f%%  t wait %.1f%%  U wait %.1f%%" % (100 * e[:, 0].mean() / e[:, 3].mean(),
      100 * e[:, 1].mean() / e[:, 3].mean(), 100 * e[:, 2].mean() / e[:, 3].mean()))
ctx.close()
