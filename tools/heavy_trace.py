"""Heavy-search trace of configs[2] (dev tool; needs a MPLD_DIAG_HEAVY build via MPLD_LIB):
per unit (component or spilled item) its size, nodes, start / end time; summary of the
critical path.

MPLD_LIB=.../libmpld_diag.so python tools/heavy_trace.py [CONFIG]
"""
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2303_14335_b200 as mp  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
dev = torch.device("cuda:0")
torch.cuda.set_device(0)
s = torch.cuda.current_stream()
it = bench.workload_items(cfg, 0, bench.default_replicas(cfg))[0]
d = bench.DeviceItem(it, dev)
ctx = mp.Context(0, it.g.n, it.g.n_layouts)
for _ in range(3):
    d.run(ctx, s, mp.MPLD_FLAG_VALIDATE)
torch.cuda.synchronize()
dbg = ctx.debug(4 * 200000)
nrec = int(dbg[96 + 0 * 0 - 96 + 0]) if False else None
tr = dbg[96:].reshape(-1, 4)
tr = tr[tr[:, 2] > 0]
t0 = tr[:, 2].min()
ci = tr[:, 0] & 0xffffffff
n = (tr[:, 0] >> 32) & 0xffff
item = tr[:, 0] >> 48
dur = (tr[:, 3] - tr[:, 2]) / 1e3
end = (tr[:, 3] - t0) / 1e3
start = (tr[:, 2] - t0) / 1e3
nodes_u = tr[:, 1] & 0xffffffff
iters_u = tr[:, 1] >> 32
tr[:, 1] = nodes_u
print("units", len(tr), "components", int((item == 0).sum()), "items", int((item > 0).sum()),
      "span_us", round(float(end.max()), 1), "nodes", int(nodes_u.sum()), "iters", int(iters_u.sum()))
for i in np.argsort(-dur)[:10]:
    print(f"  unit ci {int(ci[i])} n {int(n[i])} item {int(item[i])} nodes {int(nodes_u[i])} iters {int(iters_u[i])} "
          f"lanes/iter {nodes_u[i] / max(iters_u[i], 1):.1f} dur {dur[i]:.1f} us ns/iter {1e3 * dur[i] / max(iters_u[i], 1):.0f}")
by = collections.defaultdict(lambda: [0, 0, 0.0, 0.0, 1e18, 0])
for c, nn, it_, nd, st, en in zip(ci, n, item, tr[:, 1], start, end):
    b = by[int(c)]
    b[0] = int(nn); b[1] += 1; b[2] += float(nd); b[4] = min(b[4], st); b[5] = max(b[5], en)
top = sorted(by.items(), key=lambda kv: -kv[1][5])[:12]
for c, (nn, units, nodes, _, st, en) in top:
    print(f"ci {c:6d} n {nn:3d} units {units:6d} nodes {int(nodes):8d} start {st:7.1f} end {en:7.1f} us")
hist = np.histogram(dur[item == 0], bins=[0, 5, 10, 20, 50, 100, 200, 500, 1e9])[0]
print("component unit durations (us) <5,<10,<20,<50,<100,<200,<500,>=500:", hist.tolist())
busy = np.zeros(200)
for st, en in zip(start, end):
    a, b = int(st // 10), int(en // 10)
    busy[a:min(b + 1, 200)] += 1
print("units running per 10us:", busy[: int(end.max() // 10) + 1].astype(int).tolist())
