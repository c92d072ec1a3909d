"""configs[4] per-(size, k) device times (dev tool): python tools/c4_probe.py LABEL..."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2303_14335_b200 as mp  # noqa: E402

dev = torch.device("cuda:0")
torch.cuda.set_device(0)
s = torch.cuda.current_stream()
want = sys.argv[1:] or ["n8_k3", "n16_k3", "n16_k4"]
items = [it for it in bench.workload_items(4, 0, 1) if it.label in want]
ctx = mp.Context(0, max(it.g.n for it in items), 1)
for it in items:
    d = bench.DeviceItem(it, dev)
    for _ in range(2):
        d.run(ctx, s, mp.MPLD_FLAG_VALIDATE)
    ms = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        d.run(ctx, s, mp.MPLD_FLAG_VALIDATE)
        b.record(s)
        b.synchronize()
        ms.append(a.elapsed_time(b))
    print(json.dumps({"item": it.label, "ms_median": round(sorted(ms)[2], 3)}))
