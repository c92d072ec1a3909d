"""Step and per-kernel device times of one configuration under different flags (dev tool).

python tools/flags_probe.py CONFIG FLAGS...
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2303_14335_b200 as mp  # noqa: E402

cfg = int(sys.argv[1])
dev = torch.device("cuda:0")
torch.cuda.set_device(0)
s = torch.cuda.current_stream()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)
it = bench.workload_items(cfg, 0, bench.default_replicas(cfg))[0]
d = bench.DeviceItem(it, dev)
ctx = mp.Context(0, it.g.n, it.g.n_layouts)
for fl in [int(x) for x in sys.argv[2:]]:
    for _ in range(3):
        d.run(ctx, s, fl)
    ms = []
    for _ in range(15):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        d.run(ctx, s, fl)
        b.record(s)
        b.synchronize()
        ms.append(a.elapsed_time(b))
    ctx.reset_timing()
    ctx.set_timing(True)
    for _ in range(5):
        flush.fill_(1)
        d.run(ctx, s, fl)
    torch.cuda.synchronize()
    ctx.set_timing(False)
    kt = {k: round(v[0] / v[1] * 1e3, 1) for k, v in ctx.kernel_times().items() if v[1]}
    print(json.dumps({"config": cfg, "flags": fl, "step_ms_median": round(sorted(ms)[7], 4), "kernels_us": kt}))
