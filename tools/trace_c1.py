"""Timeline of the C1 decode launch (dev tool; needs an HC_DEC_TRACE=1 build via HC_LIB_PATH):
per launch, when CTAs start, the PDL wait, first / last FULL and the epilogue end, relative to the
previous launch's last epilogue."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_05819_b200 as hc  # noqa: E402

c = bench.C1
ncopy = 16
ctx = hc.Context(0)
g = torch.Generator(device="cuda").manual_seed(1)
N, K, b, G = c["N"], c["K"], c["bits"], c["K"] // c["group"]
r = int(sys.argv[1]) if len(sys.argv) > 1 else c["r"]
for i in range(ncopy):
    ctx.load_layer([dict(layer=i, window=0, slot=0, N=N, K=K, bits=b,
                         codes=torch.randint(-2**31, 2**31, (N, K * b // 32), generator=g, device="cuda", dtype=torch.int32),
                         scales=(0.002 + 0.01 * torch.rand((N, G), generator=g, device="cuda")).to(torch.bfloat16),
                         zeros=torch.full((N, G), 8, dtype=torch.uint8, device="cuda"),
                         U=(torch.randn((N, c["r_stored"]), generator=g, device="cuda") / N ** 0.5).to(torch.bfloat16),
                         V=(0.02 * torch.randn((c["r_stored"], K), generator=g, device="cuda")).to(torch.bfloat16),
                         r_stored=c["r_stored"], r_alloc=r)])
n_slot, grid = 64, 512
buf = torch.zeros((n_slot, grid, int(os.environ.get("HC_TRACE_W", "16"))), dtype=torch.int64, device="cuda")
L = hc.lib()
L.hc_dev_decode_trace.argtypes = [ctypes.c_void_p]
assert L.hc_dev_decode_trace(buf.data_ptr()) == 0
x = torch.randn((1, K), device="cuda").to(torch.bfloat16)
y = torch.empty((1, N), dtype=torch.float32, device="cuda")
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for i in range(ncopy):
        ctx.compensated_linear(i, 0, x, y)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=st):
        for i in range(ncopy):
            ctx.compensated_linear(i, 0, x, y, stream=st)
torch.cuda.synchronize()
for _ in range(3):
    with torch.cuda.stream(st):
        graph.replay()
torch.cuda.synchronize()
buf.zero_()
with torch.cuda.stream(st):
    graph.replay()
torch.cuda.synchronize()
t = buf.cpu().numpy().astype(np.float64)
used = [s for s in range(n_slot) if (t[s] > 0).any()]
t = t[used]
t0 = t[t > 0].min()
t = np.where(t > 0, (t - t0) / 1e3, np.nan)
end = np.nanmax(t[:, :, 4], axis=1)
print(f"rank {r}: {len(used)} launches, total µs {np.nanmax(end):.2f}, per launch {np.nanmax(end) / len(used):.2f}")
prev = np.concatenate([[np.nan], end[:-1]])
for i in range(1, len(used)):
    rel = t[i] - prev[i]
    f = lambda ev, fn: fn(rel[:, ev])
    print(f"launch {i:2d} dur {end[i] - prev[i]:6.2f} | start {f(0, np.nanmin):6.2f}/{f(0, np.nanmax):6.2f}"
          f" | pdl {f(1, np.nanmin):6.2f}/{f(1, np.nanmax):6.2f} | 1stFULL {f(2, np.nanmin):6.2f}/{f(2, np.nanmedian):6.2f}/{f(2, np.nanmax):6.2f}"
          f" | Vx {f(9, np.nanmax):6.2f} Vflush {f(10, np.nanmax):6.2f} rel {f(12, np.nanmax):6.2f} vdone {f(11, np.nanmin):6.2f}/{f(11, np.nanmax):6.2f} t0 {f(13, np.nanmin):6.2f}/{f(13, np.nanmax):6.2f} tb {f(14, np.nanmin):6.2f}/{f(14, np.nanmax):6.2f}"
          f" | t {f(5, np.nanmin):6.2f}/{f(5, np.nanmax):6.2f} | lastFULL {f(3, np.nanmedian):6.2f}/{f(3, np.nanmax):6.2f} | epi {f(4, np.nanmedian):6.2f}/{f(4, np.nanmax):6.2f}")
ctx.close()
