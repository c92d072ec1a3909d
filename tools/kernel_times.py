"""Per-kernel device times of the hot path on a few workload variants (dev tool).

python tools/kernel_times.py [--replicas R ...]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2303_14335_b200 as mp  # noqa: E402
import synth  # noqa: E402


def run(b, k, alpha, iters=10, flush=None, max_steps=1 << 20, flags=1):
    dev = torch.device("cuda:0")
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    args = [T(b.layout_offsets), b.n, T(b.ce_rowptr), T(b.ce_col), T(b.se_rowptr), T(b.se_col)]
    L = b.n_layouts
    colors = torch.empty(b.n, dtype=torch.int32, device=dev)
    counts = torch.empty(2 * L, dtype=torch.int64, device=dev)
    cost = torch.empty(L, dtype=torch.float64, device=dev)
    stats = torch.empty(len(mp.STAT_NAMES), dtype=torch.int64, device=dev)
    ctx = mp.Context(0, b.n, L)
    for _ in range(3):
        ctx.decompose_device(*args, k, alpha, max_steps, colors, counts, cost, stats, flags=flags)
    torch.cuda.synchronize()
    ctx.reset_timing()
    ctx.set_timing(True)
    for _ in range(iters):
        if flush is not None:
            flush.zero_()
        ctx.decompose_device(*args, k, alpha, max_steps, colors, counts, cost, stats, flags=flags)
    torch.cuda.synchronize()
    t = ctx.kernel_times()
    ctx.set_timing(False)
    ctx.decompose_device(*args, k, alpha, max_steps, colors, counts, cost, stats, flags=flags)
    torch.cuda.synchronize()
    d = ctx.debug()
    t0 = d[12]
    rel = lambda i: round((int(d[i]) - int(t0)) / 1e3, 1) if d[i] else None  # noqa: E731
    print("  phases(us from simplify start): simplify r01/rounds-end/hook:", [rel(i) for i in (0, 1, 3)],
          "search start", rel(14), "recover start", rel(13), "recover level0/levels-end", [rel(i) for i in (8, 9)],
          "evaluate start", rel(15), "levels", int(d[16]), "rounds", int(d[18]))
    rr = [(i, rel(20 + i), int(d[52 + i])) for i in range(32) if d[20 + i]]
    print("  rounds/levels (index, us, frontier):", rr)
    dd, ds = int(d[84]), int(d[86])
    print("  slowest discovery: cycles, n(|groups<<8|chunks<<16 in diag builds):", dd >> 16, dd & 0xffff,
          "| slowest light search: cycles, steps, n:", ds >> 24, (ds >> 8) & 0xffff, ds & 0xff)
    h = int(d[91])
    print("  heavy search: slowest component cycles, its n, iterations, steal rounds; slowest warp cycles:", int(d[89]),
          h & 0xff, (h >> 8) & 0xffffffff, h >> 40, int(d[90]))
    print("  seeds, heavy components, components:", int(d[92]), int(d[93]), int(d[94]))
    st = dict(zip(mp.STAT_NAMES, stats.cpu().tolist()))
    ctx.close()
    return {name: round(1e3 * ms / max(n, 1), 1) for name, (ms, n) in t.items()}, st


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--replicas", type=int, nargs="+", default=[1, 4, 16])
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--max-steps", type=int, default=0)
    ap.add_argument("--flags", type=int, default=1, help="1 = validate the CSR (bench default)")
    ap.add_argument("--single", action="store_true", help="skip the one-layout variant")
    a = ap.parse_args()
    flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda:0")
    for R in a.replicas:
        graphs = []
        for r in range(R):
            gs, k, alpha = synth.config_graphs(a.config, seed=10 * r)
            graphs += gs
        b = synth.concat(graphs)
        us, st = run(b, k, alpha, flush=flush, max_steps=a.max_steps, flags=a.flags)
        print(json.dumps({"replicas": R, "layouts": b.n_layouts, "n": b.n, "us_per_launch": us, "stats": st}))
        if a.single:
            continue
        one = synth.concat(graphs)
        one.layout_offsets = np.array([0, one.n], dtype=np.int32)
        us, st = run(one, k, alpha, flush=flush, max_steps=a.max_steps, flags=a.flags)
        print(json.dumps({"replicas": R, "layouts": 1, "n": one.n, "us_per_launch": us}))


if __name__ == "__main__":
    main()
