"""Recovery level trace of the configs[1] bench batch (dev tool): per level the
ready count and the globaltimer gap to the next level (CTA 0's stamps, ns),
plus the step time (CUDA events, L2 flushed).

MPLD_LIB=... python tools/level_trace.py [config]
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2303_14335_b200 as mp  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    dev = torch.device("cuda:0")
    torch.cuda.set_device(0)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)
    items = bench.workload_items(cfg, 0, bench.default_replicas(cfg))
    ctx = mp.Context(0, max(it.g.n for it in items), max(it.g.n_layouts for it in items))
    d = bench.DeviceItem(items[0], dev)
    for _ in range(5):
        d.run(ctx, stream, mp.MPLD_FLAG_VALIDATE)
    ms = []
    for _ in range(20):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        d.run(ctx, stream, mp.MPLD_FLAG_VALIDATE)
        b.record(stream)
        b.synchronize()
        ms.append(a.elapsed_time(b))
    dbg = ctx.debug()
    nl = int(dbg[16])
    tr = [int(x) for x in dbg[20:52]]
    nr = [int(x) for x in dbg[52:84]]
    levels = [(nr[16 + i], (tr[17 + i] - tr[16 + i]) if 16 + i + 1 < 32 and tr[17 + i] > tr[16 + i] else None)
              for i in range(min(nl, 16))]
    ctx.reset_timing()
    ctx.set_timing(True)
    for _ in range(10):
        d.run(ctx, stream, mp.MPLD_FLAG_VALIDATE)
    torch.cuda.synchronize()
    ctx.set_timing(False)
    kt = {k: round(v[0] / v[1] * 1e3, 1) for k, v in ctx.kernel_times().items() if v[1]}
    print(json.dumps({"lib": os.environ.get("MPLD_LIB", "default").rsplit("/", 1)[-1], "config": cfg,
                      "step_ms_median": round(sorted(ms)[len(ms) // 2], 4), "n_levels": nl,
                      "levels_cnt_gap_ns": levels, "kernels_us": kt}), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
