#!/usr/bin/env python
"""Benchmark of the MPLD hot path (BASELINE.json metric: components/s and ms per
layout; cost bit-exact vs the CPU oracle).

One step = one pass of the whole hot path (validate -> simplify -> components ->
exact-cover search -> recover -> evaluate) over one batch of synthetic layouts:
the ten ISCAS-85-shaped layouts of BASELINE.json configs[1] (Table 1
|V|/|E| for c432..c7552, k = 3, alpha = 0.1, stitch candidates), replicated
with `--replicas` seeds, resident in HBM.  Under torchrun every rank decomposes
its own batch (different seeds, no collective on the data path: components and
layouts are independent) and `value` is all components of all
ranks over the max-over-ranks device time (weak scaling).

`--impl reference` times the CPU oracle (oracle/, the "reference arm" of this
tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "components/s"
MAX_STEPS = 0  # exact mode (R7): no budget, heavy components on the warp-parallel search


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mpld", choices=["mpld", "reference"])
    ap.add_argument("--replicas", type=int, default=None,
                    help="seeds of the configuration per step per rank (default 16 for configs[1], else 1)")
    ap.add_argument("--config", type=int, default=1, choices=[1, 2, 3], help="BASELINE.json configs[] index")
    ap.add_argument("--max-steps", type=int, default=MAX_STEPS)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--profile-launches", action="store_true", help="short run for ncu (no clocks / baselines)")
    ap.add_argument("--mode", default="layouts", choices=["layouts", "shard"],
                    help="layouts: every rank decomposes its own batch (weak scaling, default); "
                         "shard: one batch, its components sharded over the ranks, colours combined "
                         "by an NCCL all-reduce MAX (strong scaling)")
    return ap.parse_args()


CONFIG = 1  # BASELINE.json configs[] index of the workload (set by --config)
WORKLOADS = {
    1: "configs[1]: ISCAS-85-shaped TPLD suite c432..c7552 (Table 1 |V|,|E|) x%d seeds per rank, k=3, "
       "alpha=0.1, stitch candidates",
    2: "configs[2]: QPLD k=4 on the s38584-scale (Table 1 |V|,|E|) ISCAS-89-shaped layout, components up to "
       "~40 vertices, alpha=0.1, x%d seeds per rank",
    3: "configs[3]: TPLD k=3 on a 10^6-polygon industrial-scale layout, alpha=0.1, x%d seeds per rank",
}


def workload(rank: int, replicas: int):
    graphs = []
    for r in range(replicas):
        gs, k, alpha = synth.config_graphs(CONFIG, seed=1000 * rank + 10 * r)
        graphs += gs
    return synth.concat(graphs, name="cfg%d_x%d" % (CONFIG, replicas)), k, alpha


def config_dict(b, replicas, n_gpus, extra=None):
    d = {"workload": WORKLOADS[CONFIG] % replicas,
         "layouts_per_step": int(b.n_layouts), "vertices_per_step": int(b.n),
         "ce_edges_per_step": int(b.n_ce), "se_edges_per_step": int(b.n_se),
         "max_steps": MAX_STEPS, "l2": "flushed between timed steps (256 MiB write)",
         "parallelism": "dp%d (independent layouts per rank)" % n_gpus}
    if os.environ.get("MPLD_BENCH_MODE") == "shard":
        d["parallelism"] = "component shards over %d ranks, NCCL all-reduce MAX of colours" % n_gpus
    if extra:
        d.update(extra)
    return d


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + q,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def kernel_bytes(b, st):
    """Algorithmic bytes per launch of each HBM-side kernel: the
    CSR rows it must read once plus the per-vertex words it must write once."""
    n, m_ce, m_se = b.n, b.ce_col.size, b.se_col.size
    csr = 8 * (n + 1) + 4 * m_ce + 4 * m_se
    return {
        "mpld_validate": csr,
        "mpld_simplify_components": csr + 4 * n,  # CSR + the round of every vertex
        "mpld_recover": 8 * (n + 1) + 4 * m_ce + 4 * int(st["hidden"]),  # CE rows + colours of hidden vertices
        "mpld_evaluate": csr + 4 * n,  # CSR + colours
    }


def aggregate(values, ops, world, device):
    """Whole-job figures: per-rank values reduced with 'sum' (work) or 'max'
    (device time, the slowest rank) over the process group."""
    import torch
    vals = torch.tensor(values, dtype=torch.float64, device=device)
    if world > 1:
        import torch.distributed as dist
        tot, mx = vals.clone(), vals.clone()
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        return [(tot if op == "sum" else mx)[i].item() for i, op in enumerate(ops)]
    return vals.tolist()


def cpu_layouts(b):
    return synth.split(b)


def run_cpu_baseline(layouts, k, alpha, seconds):
    """The oracle as it stands, single-threaded, on the first layouts of the batch
    until `seconds` of CPU work (bounded sample)."""
    import oracle
    if layouts and layouts[0].n > 300_000:  # a single layout alone exceeds the bounded CPU sample
        return {"value": None, "unit": METRIC, "cores": 1, "kind": "oracle",
                "sample": "skipped: one layout of %d vertices exceeds the bounded CPU sample" % layouts[0].n}
    comps = done = 0
    t0 = time.perf_counter()
    for g in layouts:
        r = oracle.decompose(g, k, alpha, max_steps=MAX_STEPS, check=False)
        comps += len(r["components"])
        done += 1
        if time.perf_counter() - t0 > seconds:
            break
    dt = time.perf_counter() - t0
    return {"value": comps / dt, "unit": METRIC, "cores": 1, "kind": "oracle",
            "sample": f"first {done} layouts of the rank-0 batch ({comps} components, {dt:.1f} s, "
                      f"single-threaded CPython oracle/ incl. simplification and recovery)",
            "ms_per_layout": 1e3 * dt / done}


def main_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    b, k, alpha = workload(0, args.replicas)
    import oracle
    # each step: a bounded sample of the workload (one ISCAS-85 suite = 10 layouts, ~1 s of CPU work)
    per_step = cpu_layouts(b)[:10]
    for _ in range(args.warmup):
        for g in per_step[:2]:
            oracle.decompose(g, k, alpha, max_steps=MAX_STEPS, check=False)
    comps = 0
    t0 = time.perf_counter()
    for s in range(args.steps):
        for g in per_step:
            comps += len(oracle.decompose(g, k, alpha, max_steps=MAX_STEPS, check=False)["components"])
    dt = time.perf_counter() - t0
    val = comps / dt
    out = {"metric": METRIC, "value": val, "unit": METRIC, "impl": "reference", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
           "ms_per_layout": 1e3 * dt / (args.steps * len(per_step)), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
           "config": config_dict(b, args.replicas, args.gpus,
                                 {"reference_sample": "one ISCAS-85 suite (10 layouts) per step"}),
           "cpu_baseline": {"value": val, "unit": METRIC, "cores": 1, "kind": "oracle",
                            "sample": "10 layouts (c432..c7552, first suite of the batch) per step, CPython oracle"},
           "e2e": {"value": val, "unit": METRIC, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def main():
    global CONFIG
    args = parse()
    CONFIG = args.config
    if args.replicas is None:
        args.replicas = 16 if CONFIG == 1 else 1
    if args.impl == "reference":
        return main_reference(args)
    if CONFIG == 3:  # the 10^6-polygon layout: a large per-vertex CPU sample is out of reach, use 5 s
        args.cpu_seconds = min(args.cpu_seconds, 5.0)
    import torch
    import torch.distributed as dist

    import paper_2303_14335_b200 as mp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    mp.lib()
    shard = args.mode == "shard"
    os.environ["MPLD_BENCH_MODE"] = args.mode
    b, k, alpha = workload(0 if shard else rank, args.replicas)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    d_lo, d_cr, d_cc, d_sr, d_sc = (T(b.layout_offsets), T(b.ce_rowptr), T(b.ce_col), T(b.se_rowptr),
                                    T(b.se_col))
    L = b.n_layouts
    colors = torch.empty(b.n, dtype=torch.int32, device=dev)
    counts = torch.empty(2 * L, dtype=torch.int64, device=dev)
    cost = torch.empty(L, dtype=torch.float64, device=dev)
    stats = torch.empty(len(mp.STAT_NAMES), dtype=torch.int64, device=dev)
    ctx = mp.Context(local, b.n, L)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    flags = mp.MPLD_FLAG_VALIDATE

    def step():
        if not shard:
            ctx.decompose_device(d_lo, b.n, d_cr, d_cc, d_sr, d_sc, k, alpha, args.max_steps, colors, counts, cost,
                                 stats, flags=flags, stream=stream)
            return
        ctx.prepare_device(d_lo, b.n, d_cr, d_cc, d_sr, d_sc, k, colors, counts, flags=flags, stream=stream)
        ctx.search_device(alpha, args.max_steps, rank, world, colors, stream=stream)
        if world > 1:  # the only exchange: per-component colourings, element-wise max over NVLink
            dist.all_reduce(colors, op=dist.ReduceOp.MAX)
        ctx.finish_device(alpha, colors, counts, cost, stats, stream=stream)

    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize()
    st = dict(zip(mp.STAT_NAMES, stats.cpu().tolist()))
    assert st["error"] == 0, st
    comps_per_step = st["components"]

    if args.profile_launches:
        for _ in range(args.steps):
            step()
        torch.cuda.synchronize()
        print(json.dumps({"profile_run": True, "stats": st}))
        return

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            starts[i].record(stream)
            step()
            ends[i].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = sum(step_ms)
    # per-kernel durations: the same steps again with CUDA events around every
    # launch (on the launch stream); events between kernels serialise them, so
    # this pass is kept out of the timed steps above (programmatic dependent
    # launch overlaps each kernel's launch with its predecessor's drain there)
    ctx.reset_timing()
    ctx.set_timing(True)
    for i in range(args.steps):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    ctx.set_timing(False)
    ktimes = ctx.kernel_times()
    kernel_pass_ms = sum(v[0] for v in ktimes.values())
    st = dict(zip(mp.STAT_NAMES, stats.cpu().tolist()))
    assert st["error"] == 0, st
    # kernels launched in the timed steps: the library's own count per call
    # (simplify, discover, light search, heavy x2 word classes, recovery prep,
    # recovery + its cluster tail)
    launches = int(st["launches"]) * args.steps

    # e2e: the host C-ABI call on pinned host buffers (H2D + kernels + D2H inside)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    h = [pin(x) for x in (b.layout_offsets, b.ce_rowptr, b.ce_col, b.se_rowptr, b.se_col)]
    h_colors = torch.empty(b.n, dtype=torch.int32).pin_memory()
    e2e_steps = max(3, min(3 * args.steps, 30))  # enough submits that pipeline fill and drain amortise

    def e2e_step():
        if not shard:  # the host C-ABI call: H2D, all kernels, D2H inside
            mp.mpld_decompose_batch(h[0], b.n, h[1], h[2], h[3], h[4], k, alpha, args.max_steps, flags,
                                    out_colors=h_colors)
            return
        for dst, src in zip((d_lo, d_cr, d_cc, d_sr, d_sc), h):  # H2D from pinned memory
            dst.copy_(src, non_blocking=True)
        step()
        h_colors.copy_(colors, non_blocking=True)  # D2H of the result
        torch.cuda.synchronize()

    e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    e2e_s = time.perf_counter() - t0
    assert np.array_equal(h_colors.numpy(), colors.cpu().numpy())
    blocking_ms = e2e_s * 1e3 / e2e_steps
    e2e_how = "wall clock around the blocking host C-ABI call mpld_decompose_batch (pinned buffers)"
    if not shard:
        # pipelined: the asynchronous host C-ABI call mpld_decompose_batch_async, two
        # staging slots: step i+1's upload overlaps step i's compute; every step uploads
        # its inputs and the host waits for (reads) every step's result
        def pinned_out():
            return {"colors": torch.empty(b.n, dtype=torch.int32).pin_memory(),
                    "n_conflicts": torch.zeros(L, dtype=torch.int64).pin_memory(),
                    "n_stitches": torch.zeros(L, dtype=torch.int64).pin_memory(),
                    "cost": torch.zeros(L, dtype=torch.float64).pin_memory(),
                    "stats": torch.zeros(len(mp.STAT_NAMES), dtype=torch.int64).pin_memory()}
        outs = [pinned_out(), pinned_out(), pinned_out()]  # one per staging slot of the context
        actx = mp.Context(local, b.n, L)
        # the stitch candidates as (u, v) pairs, the input of the pairs entry point
        # (prepared once, outside the timed region, like every other input array)
        se = b.se_edges()
        se = se[se[:, 0] < se[:, 1]] if se.size else np.zeros((0, 2), np.int32)
        h_pairs = pin(np.ascontiguousarray(se, dtype=np.int32))

        def submit(i):
            return actx.submit_pairs(h[0], b.n, h[1], h[2], h_pairs, k, alpha, args.max_steps, flags,
                                     out=outs[i % 3])

        for i in range(3):  # warm-up allocates the three staging slots outside the timed region
            actx.wait(submit(i))
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        pend = []
        for i in range(e2e_steps):  # up to three submits in flight; every result is waited for
            pend.append(submit(i))
            if len(pend) > 2:
                r = actx.wait(pend.pop(0))
        for t in pend:
            r = actx.wait(t)
        e2e_s = time.perf_counter() - t0
        assert np.array_equal(r["colors"].numpy(), colors.cpu().numpy()) and r["stats"]["error"] == 0
        actx.close()
        e2e_how = ("wall clock around %d pipelined submits of the asynchronous host C-ABI call "
                   "mpld_decompose_batch_pairs_async + mpld_wait (CE as CSR, stitch candidates as pairs; pinned "
                   "buffers, three staging slots: step i+1's upload overlaps step i's compute); blocking "
                   "mpld_decompose_batch: %.3f ms/step" % (e2e_steps, blocking_ms))
    h2d = (sum(x.numel() * 4 for x in h[:3]) + h_pairs.numel() * 4) if not shard else sum(x.numel() * 4 for x in h)
    d2h = b.n * 4 + L * 8 * 3 + 8 * len(mp.STAT_NAMES)

    # aggregate over ranks
    # components: every rank counts the ones it searched (shard mode: disjoint
    # shards of one batch) -> sum; layouts: shard mode holds the same batch on
    # every rank -> max
    comps_all, ms_max, e2e_comps_all, e2e_ms_max, layouts_all = aggregate(
        [comps_per_step * args.steps, total_ms, comps_per_step * e2e_steps, e2e_s * 1e3, L],
        ["sum", "max", "sum", "max", "max" if shard else "sum"], world, dev)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    value = comps_all / (ms_max / 1e3)
    ms_per_step = ms_max / args.steps
    # roofline of the dominant kernel
    kb = kernel_bytes(b, st)
    dom_name, (dom_ms, dom_n) = max(ktimes.items(), key=lambda kv: kv[1][0])
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        hbm_peak, peak_src = float(peaks["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured)"
    except Exception:
        hbm_peak, peak_src = 6650.0, "B200_PROFILING.md fallback 6.65 TB/s"
    traffic = None  # DRAM bytes per launch of the dominant kernel from the committed ncu --set full capture
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "r1_kernels.json")))["kernels"]
        traffic = prof.get(dom_name, {}).get("dram_bytes")
    except Exception:
        pass
    if kb.get(dom_name):
        achieved = kb[dom_name] / (dom_ms / dom_n / 1e3) / 1e9
        roof = {"kernel": dom_name, "bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": traffic, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": kb[dom_name],
                "note": "dependency-latency bound in practice (one grid barrier per level), DESIGN.md §5"}
    else:
        # ALU roofline: 148 SMs x 4 SMSPs x 32 lanes x 1 instr/clk at sm_max, 60 instr per node
        achieved = st["steps"] / (dom_ms / dom_n / 1e3) / 1e9
        peak_nodes = 148 * 4 * 32 * 1965e6 / 60.0 / 1e9
        roof = {"kernel": dom_name, "bound": "alu", "achieved": achieved, "peak": peak_nodes,
                "unit": "Gnodes/s", "frac": achieved / peak_nodes, "traffic": None,
                "peak_source": "148 SM x 4 SMSP x 32 lanes x 1.965 GHz / 60 instr per node (DESIGN.md §5)"}
    share = {name: (v[0] / kernel_pass_ms if kernel_pass_ms else None) for name, v in ktimes.items() if v[1]}
    out = {"metric": METRIC, "value": value, "unit": METRIC, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms_per_step,
           "ms_per_layout": ms_max / args.steps / (layouts_all if shard else layouts_all / world),
           "higher_is_better": True, "scaling": "strong" if shard else "weak", "vs_baseline": None, "dtype": "int32",
           "data": "synthetic (seeded, synth/layouts.py)",
           "config": config_dict(b, args.replicas, world, {"components_per_step_per_rank": comps_per_step}),
           "e2e": {"value": e2e_comps_all / (e2e_ms_max / 1e3), "unit": METRIC, "h2d_bytes_per_step": int(h2d),
                   "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_ms_max / e2e_steps,
                   "blocking_ms_per_step": blocking_ms, "timing": e2e_how},
           "gpu_launches": int(launches),
           "kernel_share": share,
           "kernel_timing": "per-kernel CUDA events on the launch stream, a second pass of the same %d steps "
                            "(shares of the summed kernel time)" % args.steps,
           "roofline": roof,
           "clocks": clk.summary(),
           "stats": st}
    if not args.no_cpu_baseline:
        out["cpu_baseline"] = run_cpu_baseline(cpu_layouts(b), k, alpha, args.cpu_seconds)
    print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
