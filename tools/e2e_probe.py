"""Where does the host-buffer e2e time go? (dev tool)"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2303_14335_b200 as mp  # noqa: E402
import synth  # noqa: E402

graphs = []
for r in range(16):
    gs, k, alpha = synth.config_graphs(1, seed=10 * r)
    graphs += gs
b = synth.concat(graphs)
L = b.n_layouts
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
h = [pin(x) for x in (b.layout_offsets, b.ce_rowptr, b.ce_col, b.se_rowptr, b.se_col)]


def out():
    return {"colors": torch.empty(b.n, dtype=torch.int32).pin_memory(),
            "n_conflicts": torch.zeros(L, dtype=torch.int64).pin_memory(),
            "n_stitches": torch.zeros(L, dtype=torch.int64).pin_memory(),
            "cost": torch.zeros(L, dtype=torch.float64).pin_memory(),
            "stats": torch.zeros(len(mp.STAT_NAMES), dtype=torch.int64).pin_memory()}


outs = [out(), out(), out()]
ctx = mp.Context(0, b.n, L)
se = b.se_edges()
pairs = pin(np.ascontiguousarray(se[se[:, 0] < se[:, 1]], dtype=np.int32))
sub = lambda i: ctx.submit_pairs(h[0], b.n, h[1], h[2], pairs, k, alpha, 0, 1, out=outs[i % 3])  # noqa: E731
for i in range(3):
    ctx.wait(sub(i))
N = 10
t0 = time.perf_counter()
for i in range(N):
    ctx.wait(sub(i))
print("serial submit+wait ms/step", (time.perf_counter() - t0) * 1e3 / N)
# the upper-triangle upload (uint8 row lengths + upper columns; CSR built on the device)
ud, uc = synth.upper_csr(b)
ud, uc = pin(ud), pin(uc)
subu = lambda i: ctx.submit_upper(h[0], b.n, ud, uc, pairs, k, alpha, 0, 1, out=outs[i % 3])  # noqa: E731
for i in range(3):
    ctx.wait(subu(i))
t0 = time.perf_counter()
for i in range(N):
    ctx.wait(subu(i))
print("upper: serial submit+wait ms/step", (time.perf_counter() - t0) * 1e3 / N)
t0 = time.perf_counter()
for i in range(N):
    t = subu(i)
    if i >= 2:
        ctx.wait(t - 2)
ctx.wait(t - 1)
ctx.wait(t)
print("upper: pipelined ms/step", (time.perf_counter() - t0) * 1e3 / N)
ctx.reset_timing()
ctx.set_timing(True)
for i in range(N):
    ctx.wait(subu(i))
ctx.set_timing(False)
kt = ctx.kernel_times()
print("upper: device us per submit", {k: round(v[0] / v[1] * 1e3, 1) for k, v in kt.items() if v[1]})
t0 = time.perf_counter()
ts = []
for i in range(N):
    a = time.perf_counter()
    t = sub(i)
    ts.append(time.perf_counter() - a)
    if i >= 2:
        ctx.wait(t - 2)
ctx.wait(t - 1)
ctx.wait(t)
print("pipelined ms/step", (time.perf_counter() - t0) * 1e3 / N, "submit call ms", [round(x * 1e3, 3) for x in ts])
# H2D alone (the pairs entry point's inputs), D2H alone (its outputs)
hin = h[:3] + [pairs]
d = [torch.empty_like(x, device="cuda") for x in hin]
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(N):
    for dd, x in zip(d, hin):
        dd.copy_(x, non_blocking=True)
torch.cuda.synchronize()
print("H2D only ms/step", (time.perf_counter() - t0) * 1e3 / N, "bytes", sum(x.numel() * 4 for x in hin))
dc = torch.empty(b.n, dtype=torch.int32, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(N):
    outs[0]["colors"].copy_(dc, non_blocking=True)
torch.cuda.synchronize()
print("D2H colours only ms/step", (time.perf_counter() - t0) * 1e3 / N)
# blocking host call
t0 = time.perf_counter()
for i in range(N):
    mp.mpld_decompose_batch(h[0], b.n, h[1], h[2], h[3], h[4], k, alpha, 0, 1, out_colors=outs[0]["colors"])
print("blocking host call ms/step", (time.perf_counter() - t0) * 1e3 / N)
