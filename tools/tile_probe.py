"""Tile pipeline against the whole-graph pipeline (dev tool): for each config,
both flags on the same device inputs — outputs compared element by element,
the tile gate, step times (CUDA events, L2 flushed) and per-kernel times.

python tools/tile_probe.py [configs ...]
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
    cfgs = [int(x) for x in sys.argv[1:]] or [1, 2, 3, 4]
    dev = torch.device("cuda:0")
    torch.cuda.set_device(0)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)
    for cfg in cfgs:
        items = bench.workload_items(cfg, 0, bench.default_replicas(cfg))
        if cfg == 4:
            items = [it for it in items if it.label in ("n8_k3", "n16_k4", "n32_k3", "n64_k4")]
        ctx = mp.Context(0, max(it.g.n for it in items), max(it.g.n_layouts for it in items))
        for it in items:
            d = bench.DeviceItem(it, dev)
            res = {}
            for name, fl in (("whole", mp.MPLD_FLAG_VALIDATE),
                             ("tile", mp.MPLD_FLAG_VALIDATE | mp.MPLD_FLAG_TILES)):
                for _ in range(3):
                    d.run(ctx, stream, fl)
                torch.cuda.synchronize()
                out = (d.colors.clone(), d.counts.clone(), d.cost.clone(), d.stats.clone())
                gate = int(ctx.debug()[88])
                ms = []
                for _ in range(10):
                    flush.fill_(1)
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    d.run(ctx, stream, fl)
                    b.record(stream)
                    b.synchronize()
                    ms.append(a.elapsed_time(b))
                ctx.reset_timing()
                ctx.set_timing(True)
                for _ in range(5):
                    d.run(ctx, stream, fl)
                torch.cuda.synchronize()
                ctx.set_timing(False)
                kt = {k: round(v[0] / v[1] * 1e3, 1) for k, v in ctx.kernel_times().items() if v[1]}
                res[name] = (out, gate, sorted(ms)[len(ms) // 2], kt)
            (w, _, wms, wkt), (t, gate, tms, tkt) = res["whole"], res["tile"]
            same = [bool(torch.equal(x, y)) for x, y in zip(w, t)]
            st_w = dict(zip(mp.STAT_NAMES, w[3].tolist()))
            st_t = dict(zip(mp.STAT_NAMES, t[3].tolist()))
            print(json.dumps({"config": cfg, "item": it.label, "n": it.g.n, "gate": gate,
                              "same_colors_counts_cost_stats": same, "whole_ms": round(wms, 4),
                              "tile_ms": round(tms, 4), "whole_kernels_us": wkt, "tile_kernels_us": tkt,
                              "stats_whole": st_w, "stats_tile": st_t}), flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
