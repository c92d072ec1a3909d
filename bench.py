#!/usr/bin/env python
"""Benchmark of the MPLD hot path (BASELINE.json metric: components/s and ms per
layout; cost bit-exact vs the CPU oracle).

One step = one pass of the whole hot path (validate -> simplify -> components ->
exact-cover search -> recover -> Eq. 1) over one batch of synthetic input,
resident in HBM.  The headline line (no flags) is BASELINE.json configs[1]: the
ten ISCAS-85-shaped layouts (Table 1 |V|/|E| for c432..c7552, k = 3,
alpha = 0.1, stitch candidates), x16 seeds per step.  The same JSON line carries
`secondary` measurements of configs[2] (QPLD k = 4, s38584 scale), configs[3]
(10^6 polygons) and configs[4] (the stress sweep), single-layout latencies and
the paper's own numbers as context.  `--config N` makes configs[N] the headline.

Under torchrun every rank decomposes its own batch (different seeds, no
collective on the data path: components and layouts are independent, DESIGN.md
§6) and `value` is all components of all ranks over the max-over-ranks device
time (weak scaling).  `--mode shard` decomposes ONE batch with its components
sharded over the ranks.

`--impl reference` times the CPU oracle (oracle/, the "reference arm" of this
tier) on a bounded sample of the same workload, over all host cores.
"""
from __future__ import annotations

import argparse
import json
import multiprocessing
import os
import statistics
import subprocess
import sys
import threading
import time
from dataclasses import dataclass

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "components/s"
MAX_STEPS = 0  # exact mode (R7): no budget, heavy components on the warp-parallel search

# configs[4], the stress sweep (R13): 10^5 components per (size, k),
# 500 distinct seeded components repeated in 200 layouts; exact search up to
# STRESS_EXACT_MAX vertices, a budget of STRESS_BUDGET nodes per component above
# (the exact search of random min-degree-k components is exponential in n).
STRESS_SIZES = [4, 8, 16, 24, 32, 48, 64]
STRESS_KS = [3, 4]
STRESS_TEMPLATES = 500
STRESS_COPIES = 200
STRESS_EXACT_MAX = 16
STRESS_BUDGET = 20000

# PAPER.md §3 / Table 1 (context only: another machine, another implementation)
PAPER_CONTEXT = {
    "source": "PAPER.md §3 and Table 1",
    "hardware": "Intel Core 2.9 GHz + NVIDIA GeForce RTX 2080, nvcc 11.0, 32 threads per block, one block per sub-graph",
    "speedup_vs_original_EC": 17.6,
    "speedup_vs_OpenMPL_EC": 20.0,
    "table1_time_s": {"c432": 0.000367, "c499": 0.000044, "c880": 0.000368, "c1355": 0.000767, "c1908": 0.001019,
                      "c2670": 0.00085, "c3540": 0.006474, "c5315": 0.000511, "c6288": 0.007601,
                      "c7552": 0.003175, "s38584": 0.009688},
    "note": "per-circuit simplification + decomposition time of real ISCAS layouts; ours are synthetic layouts of "
            "the same |V|/|E|, so these are context, not a baseline (vs_baseline stays null)",
}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mpld", choices=["mpld", "reference"])
    ap.add_argument("--replicas", type=int, default=None,
                    help="seeds of the configuration per step per rank (default 16 for configs[1], else 1)")
    ap.add_argument("--config", type=int, default=1, choices=[0, 1, 2, 3, 4], help="BASELINE.json configs[] index")
    ap.add_argument("--max-steps", type=int, default=None, help="search budget (default: exact; configs[4]: R13)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--profile-launches", action="store_true", help="short run for ncu (no clocks / baselines)")
    ap.add_argument("--mode", default="layouts", choices=["layouts", "shard"],
                    help="layouts: every rank decomposes its own batch (weak scaling, default); "
                         "shard: one batch, its components sharded over the ranks, compact colour lists "
                         "all-gathered over NCCL (strong scaling)")
    return ap.parse_args(argv)


WORKLOADS = {
    0: "configs[0]: TPLD k=3, 1,000 polygons in components of <= 8 vertices, no stitches, x%d seeds per rank",
    1: "configs[1]: ISCAS-85-shaped TPLD suite c432..c7552 (Table 1 |V|,|E|) x%d seeds per rank, k=3, "
       "alpha=0.1, stitch candidates",
    2: "configs[2]: QPLD k=4 on the s38584-scale (Table 1 |V|,|E|) ISCAS-89-shaped layout, components up to "
       "~40 vertices, alpha=0.1, x%d seeds per rank",
    3: "configs[3]: TPLD k=3 on a 10^6-polygon industrial-scale layout, alpha=0.1, x%d seeds per rank",
    4: "configs[4]: stress sweep, component sizes 4..64 x k=3,4, 10^5 components each (x%d), exact search up to "
       "16 vertices, budget 20000 nodes per component above (DESIGN.md R13)",
}


@dataclass
class Item:
    """One decomposition call of a step: a batch of layouts and its parameters."""
    label: str
    g: object  # synth.DecompGraph (possibly a batch of layouts)
    k: int
    alpha: float
    max_steps: int


def stress_budget(size: int) -> int:
    return 0 if size <= STRESS_EXACT_MAX else STRESS_BUDGET


def stress_template(size: int, k: int, rank: int = 0):
    """The STRESS_TEMPLATES distinct components of one (size, k) of configs[4] (rank 0: the seeds the
    parity tests use)."""
    return synth.stress_components(size, STRESS_TEMPLATES, k, seed=7000 + 10 * size + k + 100003 * rank)


def workload_items(config: int, rank: int, replicas: int, max_steps=None):
    """The calls of one step of configs[config] on `rank` (seeded, synthetic)."""
    if config == 4:
        items = []
        for size in STRESS_SIZES:
            for k in STRESS_KS:
                tmpl = stress_template(size, k, rank)
                g = synth.concat([tmpl] * STRESS_COPIES, name=f"stress_n{size}_k{k}")
                items.append(Item(f"n{size}_k{k}", g, k, 0.1, stress_budget(size) if max_steps is None else max_steps))
        return items
    graphs = []
    k = alpha = None
    for r in range(replicas):
        gs, k, alpha = synth.config_graphs(config, seed=1000 * rank + 10 * r)
        graphs += gs
    b = synth.concat(graphs, name="cfg%d_x%d" % (config, replicas))
    return [Item("cfg%d" % config, b, k, alpha, MAX_STEPS if max_steps is None else max_steps)]


def workload(rank: int, replicas: int, config: int = 1):
    """(batch, k, alpha) of a one-call configuration (configs[0..3])."""
    it = workload_items(config, rank, replicas)[0]
    return it.g, it.k, it.alpha


def default_replicas(config: int) -> int:
    return 16 if config == 1 else 1


def config_dict(config, items, replicas, n_gpus, shard=False, extra=None):
    gs = [it.g for it in items]
    d = {"workload": WORKLOADS[config] % replicas,
         "layouts_per_step": int(sum(g.n_layouts for g in gs)), "vertices_per_step": int(sum(g.n for g in gs)),
         "ce_edges_per_step": int(sum(g.n_ce for g in gs)), "se_edges_per_step": int(sum(g.n_se for g in gs)),
         "max_steps": sorted({it.max_steps for it in items}), "l2": "flushed between timed steps (256 MiB write)",
         "parallelism": "dp%d (independent layouts per rank)" % n_gpus}
    if shard:
        d["parallelism"] = ("component shards over %d ranks (cost-balanced partition), compact (vertex, colour) "
                            "lists all-gathered over NCCL" % n_gpus)
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


def kernel_bytes(items, st):
    """Algorithmic bytes per launch of each HBM-side kernel: the
    CSR rows it must read once plus the per-vertex words it must write once
    (averaged over the calls of a step)."""
    n = sum(it.g.n for it in items) / len(items)
    m_ce = sum(it.g.ce_col.size for it in items) / len(items)
    m_se = sum(it.g.se_col.size for it in items) / len(items)
    csr = 8 * (n + 1) + 4 * m_ce + 4 * m_se
    return {
        "mpld_simplify_components": csr + 4 * n,  # CSR + the round of every vertex
        "mpld_recover": 8 * (n + 1) + 4 * m_ce + 4 * int(st["hidden"]) / len(items),  # CE rows + hidden colours
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


def exchange_compact(pairs, count, world):
    """The exchange of a sharded run: every rank's compact list
    of (vertex, colour) pairs (flat int32, `count` [1] int64 pairs) goes to every
    rank.  The counts are all-gathered first, each list is padded to the longest
    with vertex -1 (skipped by mpld_shard_import), then the lists are
    all-gathered.  Returns the concatenated flat int32 pairs of all ranks."""
    import torch
    import torch.distributed as dist
    counts = [torch.zeros_like(count) for _ in range(world)]
    dist.all_gather(counts, count)
    mine = int(count.item())
    longest = max(1, max(int(c.item()) for c in counts))
    send = pairs[: 2 * longest]
    if longest > mine:
        send[2 * mine:].fill_(-1)
    recv = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(recv, send)
    return torch.cat(recv)


# ---------------------------------------------------------------- CPU oracle (baseline / reference arm)
def cpu_units(config, items):
    """The oracle's work units of a workload: (graph, k, alpha, max_steps) per
    layout (configs[4]: per component of the templates, all (size, k) interleaved)."""
    if config != 4:
        out = []
        for it in items:
            out += [(g, it.k, it.alpha, it.max_steps) for g in synth.split(it.g)]
        return out
    per = []
    for it in items:
        tmpl_n = it.g.n // STRESS_COPIES
        size = int(it.label.split("_")[0][1:])
        first = synth.split(it.g)[0] if it.g.n_layouts > 1 else it.g
        assert first.n == tmpl_n
        first.layout_offsets = np.arange(0, tmpl_n + 1, size, dtype=np.int32)  # one layout per component
        per.append([(c, it.k, it.alpha, it.max_steps) for c in synth.split(first)])
    out = []
    for i in range(max(len(p) for p in per)):  # interleave the sizes: a bounded sample covers all of them
        out += [p[i] for p in per if i < len(p)]
    return out


def _oracle_unit(u):
    import oracle
    g, k, alpha, ms = u
    return len(oracle.decompose(g, k, alpha, max_steps=ms, check=False)["components"])


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_oracle_pool(units, seconds, cores):
    """The oracle as it stands over `units`, one process per host core, until
    `seconds` of wall time (bounded sample).  Returns (components, units done, s)."""
    comps = done = 0
    t0 = time.perf_counter()
    ctx = multiprocessing.get_context("fork")
    with ctx.Pool(cores) as pool:
        for c in pool.imap_unordered(_oracle_unit, units, chunksize=1):
            comps += c
            done += 1
            if time.perf_counter() - t0 > seconds:
                pool.terminate()
                break
    return comps, done, time.perf_counter() - t0


def run_cpu_baseline(config, items, seconds):
    units = cpu_units(config, items)
    if config == 3:
        units = units[:1]  # one 10^6-polygon layout (~20 s of oracle): one core
    cores = min(host_cores(), len(units))
    comps, done, dt = run_oracle_pool(units, seconds, cores)
    return {"value": comps / dt, "unit": METRIC, "cores": cores, "kind": "oracle",
            "sample": f"{done} of {len(units)} oracle units of the rank-0 workload ({comps} components, {dt:.1f} s "
                      f"wall, CPython oracle/ incl. simplification and recovery, one process per host core)",
            "ms_per_unit": 1e3 * dt * cores / max(done, 1)}


def main_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    items = workload_items(args.config, 0, args.replicas, args.max_steps)
    units = cpu_units(args.config, items)
    cores = min(host_cores(), len(units))
    per_step = units[: max(cores, 10)] if args.config != 3 else units[:1]
    import oracle  # noqa: F401  (imported before the pool forks)
    if args.warmup:
        run_oracle_pool(per_step[: min(len(per_step), cores)], 1e9, cores)
    comps = 0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        c, _, _ = run_oracle_pool(per_step, 1e9, min(cores, len(per_step)))
        comps += c
    dt = time.perf_counter() - t0
    val = comps / dt
    sample = (f"{len(per_step)} oracle units of the workload per step (layouts; configs[4]: components), "
              f"one process per host core")
    out = {"metric": METRIC, "value": val, "unit": METRIC, "impl": "reference", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
           "ms_per_layout": 1e3 * dt / (args.steps * len(per_step)), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
           "config": config_dict(args.config, items, args.replicas, args.gpus, extra={"reference_sample": sample}),
           "cpu_baseline": {"value": val, "unit": METRIC, "cores": min(cores, len(per_step)), "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": val, "unit": METRIC, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


# ---------------------------------------------------------------- device runs
class DeviceItem:
    """An Item resident in HBM with its output buffers."""

    def __init__(self, it: Item, dev):
        import torch
        import paper_2303_14335_b200 as mp
        self.it = it
        g = it.g
        T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
        self.lo, self.cr, self.cc, self.sr, self.sc = (T(g.layout_offsets), T(g.ce_rowptr), T(g.ce_col),
                                                       T(g.se_rowptr), T(g.se_col))
        L = g.n_layouts
        self.colors = torch.empty(g.n, dtype=torch.int32, device=dev)
        self.counts = torch.empty(2 * L, dtype=torch.int64, device=dev)
        self.cost = torch.empty(L, dtype=torch.float64, device=dev)
        self.stats = torch.empty(len(mp.STAT_NAMES), dtype=torch.int64, device=dev)

    def run(self, ctx, stream, flags):
        it = self.it
        ctx.decompose_device(self.lo, it.g.n, self.cr, self.cc, self.sr, self.sc, it.k, it.alpha, it.max_steps,
                             self.colors, self.counts, self.cost, self.stats, flags=flags, stream=stream)

    def stats_dict(self):
        import paper_2303_14335_b200 as mp
        return dict(zip(mp.STAT_NAMES, self.stats.cpu().tolist()))


def merge_stats(sts):
    out = {}
    for s in sts:
        for a, v in s.items():
            out[a] = max(out.get(a, v), v) if a in ("max_component", "max_steps", "rounds") else out.get(a, 0) + v
    return out


def time_steps(ctx, ditems, steps, flush, stream, flags, per_item=False):
    """Device time of `steps` steps (CUDA events on the launch stream around each
    step; the L2 is flushed before each).  Returns (step ms list, per-item ms)."""
    import torch
    marks = [[torch.cuda.Event(enable_timing=True) for _ in range(len(ditems) + 1 if per_item else 2)]
             for _ in range(steps)]
    for i in range(steps):
        flush.zero_()
        marks[i][0].record(stream)
        for j, d in enumerate(ditems):
            d.run(ctx, stream, flags)
            if per_item:
                marks[i][j + 1].record(stream)
        if not per_item:
            marks[i][1].record(stream)
    torch.cuda.synchronize()
    step_ms = [m[0].elapsed_time(m[-1]) for m in marks]
    item_ms = [sum(m[j].elapsed_time(m[j + 1]) for m in marks) for j in range(len(ditems))] if per_item else None
    return step_ms, item_ms


def secondary(config, rank, world, dev, stream, flush, local, steps=5, warmup=2):
    """A shorter device-timed measurement of another configuration (no e2e /
    CPU baseline): value, ms per step, largest component, truncated searches."""
    import torch
    import paper_2303_14335_b200 as mp
    t0 = time.perf_counter()
    items = workload_items(config, rank, default_replicas(config))
    gen_s = time.perf_counter() - t0
    ditems = [DeviceItem(it, dev) for it in items]
    ctx = mp.Context(local, max(it.g.n for it in items), max(it.g.n_layouts for it in items))
    flags = mp.MPLD_FLAG_VALIDATE
    for _ in range(warmup):
        for d in ditems:
            d.run(ctx, stream, flags)
    torch.cuda.synchronize()
    sts = [d.stats_dict() for d in ditems]
    for s in sts:
        assert s["error"] == 0, s
    st = merge_stats(sts)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    with Clocks(local) as clk:
        step_ms, item_ms = time_steps(ctx, ditems, steps, flush, stream, flags, per_item=config == 4)
    comps_all, ms_max, lay_all = aggregate([st["components"] * steps, sum(step_ms), sum(it.g.n_layouts for it in items)],
                                           ["sum", "max", "sum"], world, dev)
    out = {"config": "configs[%d]" % config, "workload": WORKLOADS[config] % default_replicas(config),
           "value": comps_all / (ms_max / 1e3), "unit": METRIC, "ms_per_step": ms_max / steps,
           "ms_per_layout": ms_max / steps / (lay_all / world), "steps": steps, "warmup": warmup,
           "components_per_step_per_rank": st["components"], "max_component": st["max_component"],
           "truncated": st["truncated"], "max_steps": sorted({it.max_steps for it in items}),
           "vertices_per_step": int(sum(it.g.n for it in items)), "clocks": clk.summary(),
           "generation_s": round(gen_s, 1)}
    if config == 4:
        out["per_size"] = {}
        for it, d, s, ms in zip(items, ditems, sts, item_ms):
            out["per_size"][it.label] = {"components": s["components"], "ms": ms / steps,
                                         "components_per_s": s["components"] / (ms / steps / 1e3) if ms else None,
                                         "max_steps": it.max_steps, "truncated": s["truncated"],
                                         "nodes": s["steps"]}
    if config in (2, 3):  # one layout per step: the single-layout latency of this circuit size
        out["single_layout_ms"] = ms_max / steps
    ctx.close()
    del ditems
    torch.cuda.empty_cache()
    return out


def single_layout_latency(dev, stream, flush, local, circuit="c7552", reps=20):
    """One ISCAS-85-shaped layout alone: device-resident call (CUDA events, L2
    flushed before each) and the blocking host C-ABI call mpld_decompose
    (wall clock, H2D + D2H inside), medians."""
    import torch
    import paper_2303_14335_b200 as mp
    g = synth.iscas_layout(circuit, seed=0)
    it = Item(circuit, g, 3, 0.1, MAX_STEPS)
    d = DeviceItem(it, dev)
    ctx = mp.Context(local, g.n, 1)
    for _ in range(3):
        d.run(ctx, stream, mp.MPLD_FLAG_VALIDATE)
    dev_ms = []
    for _ in range(reps):
        ms, _ = time_steps(ctx, [d], 1, flush, stream, mp.MPLD_FLAG_VALIDATE)
        dev_ms += ms
    host_ms = []
    for _ in range(reps):
        t0 = time.perf_counter()
        mp.mpld_decompose(g.n, g.ce_rowptr, g.ce_col, g.se_rowptr, g.se_col, 3, 0.1, MAX_STEPS)
        host_ms.append(1e3 * (time.perf_counter() - t0))
    ctx.close()
    return {"layout": circuit + " (synthetic, Table 1 |V|,|E|)", "device_ms": statistics.median(dev_ms),
            "host_call_ms": statistics.median(host_ms),
            "paper_table1_s": PAPER_CONTEXT["table1_time_s"].get(circuit)}


def roofline(ktimes, items, st):
    """Roofline of the dominant kernel."""
    kb = kernel_bytes(items, st)
    dom_name, (dom_ms, dom_n) = max(ktimes.items(), key=lambda kv: kv[1][0])
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        hbm_peak, peak_src = float(peaks["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured)"
    except Exception:
        hbm_peak, peak_src = 6650.0, "B200_PROFILING.md fallback 6.65 TB/s"
    prof = {}
    for name in ("r2_kernels.json", "r1_kernels.json"):
        try:
            prof = json.load(open(os.path.join(ROOT, "profiles", name)))["kernels"]
            prof_src = name
            break
        except Exception:
            continue
    traffic = prof.get(dom_name, {}).get("dram_bytes") if prof else None
    if kb.get(dom_name):
        achieved = kb[dom_name] / (dom_ms / dom_n / 1e3) / 1e9
        return {"kernel": dom_name, "bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": traffic, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": kb[dom_name],
                "note": "dependency-latency bound in practice (one grid barrier per level), DESIGN.md §5"}
    # the search: ALU bound.  Peak nodes/s = issue slots (148 SMs x 4 schedulers x 1 warp-instr/clk at the
    # max SM clock) / warp instructions per node, the latter measured by ncu (inst_executed / nodes) when a
    # profile holds it
    ipn = prof.get(dom_name, {}).get("inst_per_node") if prof else None
    ipn_src = f"profiles/{prof_src} inst_executed / nodes" if ipn else "assumed 60 warp instructions per node"
    ipn = ipn or 60.0
    achieved = st["steps"] / (dom_ms / 1e3) / 1e9 if dom_ms else 0.0
    peak_nodes = 148 * 4 * 1965e6 / ipn / 1e9
    return {"kernel": dom_name, "bound": "alu", "achieved": achieved, "peak": peak_nodes, "unit": "Gnodes/s",
            "frac": achieved / peak_nodes, "traffic": traffic,
            "peak_source": f"148 SM x 4 schedulers x 1 warp-instruction/clk x 1.965 GHz / {ipn:.0f} ({ipn_src})"}


def main():
    args = parse()
    if args.replicas is None:
        args.replicas = default_replicas(args.config)
    if args.impl == "reference":
        return main_reference(args)
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
    if shard and args.config == 4:
        raise SystemExit("--mode shard needs a one-call configuration (configs[0..3])")
    items = workload_items(args.config, 0 if shard else rank, args.replicas, args.max_steps)
    ditems = [DeviceItem(it, dev) for it in items]
    ctx = mp.Context(local, max(it.g.n for it in items), max(it.g.n_layouts for it in items))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    flags = mp.MPLD_FLAG_VALIDATE
    if shard:
        d0 = ditems[0]
        it0 = items[0]
        cap = max(1, it0.g.n)
        exp_pairs = torch.empty(2 * cap, dtype=torch.int32, device=dev)
        exp_count = torch.zeros(1, dtype=torch.int64, device=dev)

        def shard_step():
            ctx.prepare_device(d0.lo, it0.g.n, d0.cr, d0.cc, d0.sr, d0.sc, it0.k, d0.colors, d0.counts,
                               flags=flags, stream=stream)
            ctx.search_device(it0.alpha, it0.max_steps, rank, world, d0.colors, stream=stream)
            if world > 1:  # the only exchange: the compact (vertex, colour) lists of the searched components
                ctx.shard_export(d0.colors, exp_pairs, exp_count, stream=stream)
                ctx.shard_import(exchange_compact(exp_pairs, exp_count, world), d0.colors, stream=stream)
            ctx.finish_device(it0.alpha, d0.colors, d0.counts, d0.cost, d0.stats, stream=stream)

    def step():
        if shard:
            shard_step()
        else:
            for d in ditems:
                d.run(ctx, stream, flags)

    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize()
    sts = [d.stats_dict() for d in ditems]
    for s in sts:
        assert s["error"] == 0, s
    st = merge_stats(sts)
    comps_per_step = st["components"]

    if args.profile_launches:
        for _ in range(args.steps):
            step()
        torch.cuda.synchronize()
        dbg = ctx.debug()  # search nodes of the last call: total, heavy (for ncu's instructions per node)
        print(json.dumps({"profile_run": True, "stats": st, "last_call_nodes": int(dbg[87]),
                          "last_call_heavy_nodes": int(dbg[85])}))
        return

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        if shard:
            import torch as _t
            starts = [_t.cuda.Event(enable_timing=True) for _ in range(args.steps)]
            ends = [_t.cuda.Event(enable_timing=True) for _ in range(args.steps)]
            for i in range(args.steps):
                flush.zero_()
                starts[i].record(stream)
                step()
                ends[i].record(stream)
            torch.cuda.synchronize()
            step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
            item_ms = None
        else:
            step_ms, item_ms = time_steps(ctx, ditems, args.steps, flush, stream, flags,
                                          per_item=args.config == 4)
    if world > 1:
        dist.barrier()
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
    sts = [d.stats_dict() for d in ditems]
    for s in sts:
        assert s["error"] == 0, s
    st = merge_stats(sts)
    # kernels launched in the timed steps: the library's own count per call
    launches = int(sum(s["launches"] for s in sts)) * args.steps

    # e2e: the host C-ABI on pinned host buffers (H2D + kernels + D2H inside)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    e2e_steps = max(3, min(3 * args.steps, 30))  # enough submits that pipeline fill and drain amortise
    if not shard:
        # pipelined: the asynchronous host C-ABI call mpld_decompose_batch_upper_async (the
        # conflict edges as the upper triangle of their CSR with uint8 row lengths, the stitch
        # candidates as pairs; the symmetric CSR is built on the device), three staging slots:
        # step i+1's upload overlaps step i's compute; every call uploads its inputs and the
        # host waits for (reads) every result.  The upload format is prepared once, outside
        # the timed region, like every other input array
        hosts = []
        for it in items:
            g = it.g
            se = synth.stitch_pairs(g)
            up_deg, up_col = synth.upper_csr(g)
            L = g.n_layouts
            outs = [{"colors": torch.empty(g.n, dtype=torch.int32).pin_memory(),
                     "n_conflicts": torch.zeros(L, dtype=torch.int64).pin_memory(),
                     "n_stitches": torch.zeros(L, dtype=torch.int64).pin_memory(),
                     "cost": torch.zeros(L, dtype=torch.float64).pin_memory(),
                     "stats": torch.zeros(len(mp.STAT_NAMES), dtype=torch.int64).pin_memory()} for _ in range(3)]
            hosts.append({"lo": pin(g.layout_offsets), "ud": pin(up_deg), "uc": pin(up_col),
                          "pairs": pin(np.ascontiguousarray(se, dtype=np.int32)), "outs": outs})
        actx = mp.Context(local, max(it.g.n for it in items), max(it.g.n_layouts for it in items))
        seq = [(j, i) for i in range(e2e_steps) for j in range(len(items))]

        def submit(pos):
            j, i = seq[pos]
            it, h = items[j], hosts[j]
            return actx.submit_upper(h["lo"], it.g.n, h["ud"], h["uc"], h["pairs"], it.k, it.alpha, it.max_steps,
                                     flags, out=h["outs"][pos % 3])

        for pos in range(min(3, len(seq))):  # warm-up allocates the staging slots outside the timed region
            actx.wait(submit(pos))
        if world > 1:
            dist.barrier()
        reps = []
        for _rep in range(3):  # three timed runs, the median kept (host wall clock: one preempted
            t0 = time.perf_counter()  # host thread would otherwise decide the number)
            pend = []
            last = {}
            for pos in range(len(seq)):  # up to three submits in flight; every result is waited for
                pend.append((pos, submit(pos)))
                if len(pend) > 2:
                    p, t = pend.pop(0)
                    last[seq[p][0]] = actx.wait(t)
            for p, t in pend:
                last[seq[p][0]] = actx.wait(t)
            reps.append(time.perf_counter() - t0)
        e2e_s = sorted(reps)[1]
        for j, d in enumerate(ditems):
            assert np.array_equal(last[j]["colors"].numpy(), d.colors.cpu().numpy()) and last[j]["stats"]["error"] == 0
        actx.close()
        e2e_how = ("wall clock around %d steps of pipelined submits of the asynchronous host C-ABI call "
                   "mpld_decompose_batch_upper_async + mpld_wait (CE as the upper triangle of its CSR with uint8 "
                   "row lengths, stitch candidates as pairs, symmetric CSR built on the device; pinned buffers, "
                   "three staging slots: step i+1's upload overlaps step i's compute); median of 3 timed runs "
                   "(%s ms)" % (e2e_steps, ", ".join("%.2f" % (1e3 * r) for r in reps)))
        h2d = sum(h["lo"].numel() * 4 + h["ud"].numel() + h["uc"].numel() * 4 + h["pairs"].numel() * 4
                  for h in hosts)
    else:
        g = items[0].g
        h = [pin(x) for x in (g.layout_offsets, g.ce_rowptr, g.ce_col, g.se_rowptr, g.se_col)]
        h_colors = torch.empty(g.n, dtype=torch.int32).pin_memory()
        d0 = ditems[0]

        def e2e_step():
            for dst, src in zip((d0.lo, d0.cr, d0.cc, d0.sr, d0.sc), h):  # H2D from pinned memory
                dst.copy_(src, non_blocking=True)
            step()
            h_colors.copy_(d0.colors, non_blocking=True)  # D2H of the result
            torch.cuda.synchronize()

        e2e_step()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        e2e_s = time.perf_counter() - t0
        e2e_how = "wall clock around the sharded phases with pinned H2D / D2H copies (torch copies)"
        h2d = sum(x.numel() * 4 for x in h)
    d2h = sum(it.g.n * 4 + it.g.n_layouts * 8 * 3 + 8 * len(mp.STAT_NAMES) for it in items)

    # aggregate over ranks
    # components: every rank counts the ones it searched (shard mode: disjoint
    # shards of one batch) -> sum; layouts: shard mode holds the same batch on
    # every rank -> max
    L = sum(it.g.n_layouts for it in items)
    comps_all, ms_max, e2e_comps_all, e2e_ms_max, layouts_all = aggregate(
        [comps_per_step * args.steps, total_ms, comps_per_step * e2e_steps, e2e_s * 1e3, L],
        ["sum", "max", "sum", "max", "max" if shard else "sum"], world, dev)

    sec = {}
    lat = None
    if not args.no_secondary and not shard and args.config == 1:
        for c in (2, 3, 4):
            sec["configs[%d]" % c] = secondary(c, rank, world, dev, stream, flush, local)
        lat = single_layout_latency(dev, stream, flush, local)
        if "configs[2]" in sec:
            lat = {"c7552": lat, "s38584": {"layout": "s38584 (synthetic, Table 1 |V|,|E|, QPLD k=4)",
                                            "device_ms": sec["configs[2]"]["single_layout_ms"],
                                            "paper_table1_s": PAPER_CONTEXT["table1_time_s"]["s38584"]}}
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    value = comps_all / (ms_max / 1e3)
    ms_per_step = ms_max / args.steps
    roof = roofline(ktimes, items, st)
    share = {name: (v[0] / kernel_pass_ms if kernel_pass_ms else None) for name, v in ktimes.items() if v[1]}
    out = {"metric": METRIC, "value": value, "unit": METRIC, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms_per_step,
           "ms_per_layout": ms_max / args.steps / (layouts_all if shard else layouts_all / world),
           "higher_is_better": True, "scaling": "strong" if shard else "weak", "vs_baseline": None, "dtype": "int32",
           "data": "synthetic (seeded, synth/layouts.py)",
           "config": config_dict(args.config, items, args.replicas, world, shard,
                                 {"components_per_step_per_rank": comps_per_step}),
           "e2e": {"value": e2e_comps_all / (e2e_ms_max / 1e3), "unit": METRIC, "h2d_bytes_per_step": int(h2d),
                   "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_ms_max / e2e_steps, "timing": e2e_how},
           "gpu_launches": int(launches),
           "kernel_share": share,
           "kernel_timing": "per-kernel CUDA events on the launch stream, a second pass of the same %d steps "
                            "(shares of the summed kernel time)" % args.steps,
           "roofline": roof,
           "clocks": clk.summary(),
           "stats": st}
    if item_ms and args.config == 4:
        out["per_size"] = {it.label: {"components": s["components"], "ms": ms / args.steps,
                                      "max_steps": it.max_steps, "truncated": s["truncated"]}
                           for it, s, ms in zip(items, sts, item_ms)}
    if sec:
        out["secondary"] = sec
    if lat:
        out["latency"] = lat
    out["paper_context"] = PAPER_CONTEXT
    if not args.no_cpu_baseline:
        out["cpu_baseline"] = run_cpu_baseline(args.config, items, args.cpu_seconds)
    print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
