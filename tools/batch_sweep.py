"""Batch-size sweep of configs[1] (dev tool): step time and per-kernel times for
x1 / x4 / x16 / x64 copies of the ISCAS-85 suite, to split the per-level
latency of the level-synchronous kernels from their per-vertex cost.

python tools/batch_sweep.py [OUT.json]
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
    out = {"source": "tools/batch_sweep.py: configs[1] (ten ISCAS-85-shaped layouts per replica), exact mode, "
                     "validation on, L2 flushed before every step, CUDA events; per-kernel times from a second "
                     "pass with events around every launch", "rows": []}
    dev = torch.device("cuda:0")
    torch.cuda.set_device(0)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)
    kb_names = ("mpld_simplify_components", "mpld_recover")
    for reps in (1, 4, 16, 64):
        items = bench.workload_items(1, 0, reps)
        d = bench.DeviceItem(items[0], dev)
        ctx = mp.Context(0, items[0].g.n, items[0].g.n_layouts)
        for _ in range(3):
            d.run(ctx, stream, mp.MPLD_FLAG_VALIDATE)
        torch.cuda.synchronize()
        step_ms, _ = bench.time_steps(ctx, [d], 10, flush, stream, mp.MPLD_FLAG_VALIDATE)
        ctx.reset_timing()
        ctx.set_timing(True)
        bench.time_steps(ctx, [d], 10, flush, stream, mp.MPLD_FLAG_VALIDATE)
        ctx.set_timing(False)
        kt = {k: v[0] / v[1] * 1e3 for k, v in ctx.kernel_times().items() if v[1]}
        st = d.stats_dict()
        kb = bench.kernel_bytes(items, st)
        g = items[0].g
        row = {"replicas": reps, "vertices": int(g.n), "ce_entries": int(g.ce_col.size),
               "components": int(st["components"]), "step_ms": sum(step_ms) / len(step_ms),
               "components_per_s": st["components"] / (sum(step_ms) / len(step_ms) / 1e3),
               "kernel_us": {k: round(v, 1) for k, v in kt.items()},
               "gbs": {k: round(kb[k] / (kt[k] / 1e6) / 1e9, 1) for k in kb_names if k in kt}}
        out["rows"].append(row)
        print(json.dumps(row), flush=True)
        ctx.close()
        del d
        torch.cuda.empty_cache()
    # per-level latency vs per-vertex cost: least-squares fit t = a + b * n over the sweep
    for k in kb_names + ("step",):
        xs = [r["vertices"] for r in out["rows"]]
        ys = [r["step_ms"] * 1e3 if k == "step" else r["kernel_us"].get(k, 0.0) for r in out["rows"]]
        n = len(xs)
        mx, my = sum(xs) / n, sum(ys) / n
        b = sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sum((x - mx) ** 2 for x in xs)
        a = my - b * mx
        out.setdefault("fit_us", {})[k] = {"fixed_us": round(a, 2), "ns_per_vertex": round(b * 1e3, 4)}
    print(json.dumps(out["fit_us"]))
    if len(sys.argv) > 1:
        json.dump(out, open(sys.argv[1], "w"), indent=1)


if __name__ == "__main__":
    main()
