"""Parity of the CUDA path (through the C ABI) with the CPU oracle, element by
element: colours, conflict and stitch counts and cost are compared bit-exactly
(integer / index results; the cost is the same IEEE expression on both sides)."""
from __future__ import annotations

import functools
import random

import numpy as np
import pytest

import oracle
import synth
from synth import from_edges
from tests._pins import BAD_GRAPHS, GOOD_CE, GOOD_SE, raw_graph

mp = pytest.importorskip("paper_2303_14335_b200")
torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

BUDGET = 1 << 20


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    mp.lib()


def _assert_same(g, k, alpha, max_steps=BUDGET, flags=mp.MPLD_FLAG_VALIDATE, ref=None):
    got = mp.decompose_graph(g, k, alpha, max_steps=max_steps, flags=flags)
    ref = ref or oracle.decompose(g, k, alpha, max_steps=max_steps)
    assert np.array_equal(got["colors"], ref["colors"]), np.nonzero(got["colors"] != ref["colors"])[0][:10]
    for li, (c, s, cost) in enumerate(ref["per_layout"]):
        assert int(got["n_conflicts"][li]) == c
        assert int(got["n_stitches"][li]) == s
        assert float(got["cost"][li]) == cost
    st = got["stats"]
    assert st["components"] == len(ref["components"])
    assert st["rounds"] == ref["n_rounds"]
    assert st["hidden"] == int((ref["hround"] >= 0).sum())
    if max_steps > 0:  # exact mode explores heavy components in parallel: other node counts
        assert st["steps"] == sum(c["steps"] for c in ref["components"])
    assert st["truncated"] == sum(c["truncated"] for c in ref["components"])
    assert st["error"] == 0
    return got, ref


def test_config0_full():
    graphs, k, alpha = synth.config_graphs(0)
    _assert_same(graphs[0], k, alpha)


def test_config1_iscas85_suite_batched():
    graphs, k, alpha = synth.config_graphs(1)
    b = synth.concat(graphs)
    _assert_same(b, k, alpha)


@pytest.mark.parametrize("k", [2, 3, 4])
def test_random_small_graphs(k):
    rng = random.Random(2024 + k)
    for trial in range(40):
        n = rng.randint(1, 24)
        p = rng.choice([0.15, 0.3, 0.5])
        ce, se = [], []
        for u in range(n):
            for v in range(u + 1, n):
                r = rng.random()
                if r < 0.05:
                    se.append((u, v))
                elif r < 0.05 + p:
                    ce.append((u, v))
        g = from_edges(n, ce, se)
        _assert_same(g, k, 0.1, max_steps=20000)


@pytest.mark.parametrize("alpha", [0.0, 0.1, 0.5, 1.0, 2.5])
def test_alpha_values(alpha):
    g = synth.make_layout(3000, 3400, k=3, stitch_prob=0.6, comp_max=12, density=0.9, seed=7)
    _assert_same(g, 3, alpha)


@pytest.mark.parametrize("budget", [1, 5, 37, 200])
def test_truncated_search_parity(budget):
    """With a tiny max_steps the GPU stops at exactly the oracle's node."""
    g = synth.stress_components(16, 30, 3, seed=3)
    _assert_same(g, 3, 0.1, max_steps=budget)


@pytest.mark.parametrize("size", [4, 8, 16, 24, 32, 48, 64])
def test_stress_component_sizes(size):
    g = synth.stress_components(size, 12, 3, seed=size)
    _assert_same(g, 3, 0.1, max_steps=20000)


@pytest.mark.parametrize("case", ["cfg1", "stress12", "stress20", "k4", "k2"])
def test_exact_mode_warp_parallel_search(case):
    """max_steps = 0 (exact mode): heavy components go to the warp-parallel
    search; the result must still be the oracle's first optimal leaf (R7)."""
    if case == "cfg1":
        graphs, k, alpha = synth.config_graphs(1)
        g = synth.concat(graphs[:6])
    elif case.startswith("stress"):
        k, alpha = 3, 0.1
        g = synth.stress_components(int(case[6:]), 40, 3, seed=11)
    elif case == "k4":
        graphs, k, alpha = synth.config_graphs(2, scale=0.05)
        g = graphs[0]
    else:
        k, alpha = 2, 0.1
        g = synth.stress_components(14, 30, 2, seed=5)
    got, ref = _assert_same(g, k, alpha, max_steps=0)
    assert got["stats"]["truncated"] == 0


def test_single_layout_entry_point():
    """The north_star signature mpld_decompose(csr, stitches, k, alpha, max_steps)."""
    g = synth.iscas_layout("c1908", seed=3)
    colors, nc, ns, cost = mp.mpld_decompose(g.n, g.ce_rowptr, g.ce_col, g.se_rowptr, g.se_col, 3, 0.1, 0)
    ref = oracle.decompose(g, 3, 0.1, max_steps=0)
    assert np.array_equal(colors, ref["colors"])
    assert (nc, ns, cost) == (ref["n_conflicts"], ref["n_stitches"], ref["cost"])


def test_industrial_config3_scaled():
    """configs[3] shape (10^6 polygons) scaled to 5 %: full element-by-element parity."""
    graphs, k, alpha = synth.config_graphs(3, scale=0.05)
    _assert_same(graphs[0], k, alpha, max_steps=0)


@pytest.mark.parametrize("k", [3, 4])
def test_stress_sweep_exact_mode(k):
    """configs[4] stress sweep (component sizes 4 -> 64) in exact mode, sampled sizes."""
    for size in (4, 16, 24, 32, 48, 64):
        g = synth.stress_components(size, 6, k, seed=100 + size)
        budget = 0 if size <= 24 else 50000  # exact mode where the oracle can follow
        got = mp.decompose_graph(g, k, 0.1, max_steps=budget)
        if size <= 24:
            ref = oracle.decompose(g, k, 0.1, max_steps=0)
            assert np.array_equal(got["colors"], ref["colors"])
            assert got["stats"]["truncated"] == 0
        # invariants at any size: colours in range, counts recomputed from colours
        c = got["colors"]
        assert ((c >= 0) & (c < k)).all()
        ce = g.ce_edges()
        assert int((c[ce[:, 0]] == c[ce[:, 1]]).sum()) == int(got["n_conflicts"][0])
        assert got["stats"]["components"] == (6 if size > k else 0)  # K_size with size <= k peels away


def test_qpld_k4_scaled():
    graphs, k, alpha = synth.config_graphs(2, scale=0.1)
    _assert_same(graphs[0], k, alpha, max_steps=200000)


def test_edge_cases():
    fx = synth.fixtures()
    for name in ["empty", "single", "K4", "K5", "K7", "W5", "C5", "stitch_pair", "triangle"]:
        for k in (2, 3, 4):
            _assert_same(fx[name], k, 0.1)
    # everything hidden (a long path)
    n = 1000
    _assert_same(from_edges(n, [(i, i + 1) for i in range(n - 1)]), 3, 0.1)
    # a 64-vertex clique fits; 65 is rejected
    K64 = from_edges(64, [(i, j) for i in range(64) for j in range(i + 1, 64)])
    got = mp.decompose_graph(K64, 4, 0.1, max_steps=1000)
    ref = oracle.decompose(K64, 4, 0.1, max_steps=1000)
    assert np.array_equal(got["colors"], ref["colors"])
    K65 = from_edges(65, [(i, j) for i in range(65) for j in range(i + 1, 65)])
    with pytest.raises(mp.MPLDError) as ei:
        mp.decompose_graph(K65, 4, 0.1, max_steps=1000)
    assert ei.value.code == 3


def test_validation_rejects_bad_graphs():
    g = from_edges(4, [(0, 1), (1, 2)])
    bad = from_edges(4, [(0, 1), (1, 2)])
    bad.ce_col = bad.ce_col.copy()
    bad.ce_col[0] = 3  # 0 -> 3 without 3 -> 0
    with pytest.raises(mp.MPLDError) as ei:
        mp.decompose_graph(bad, 3, 0.1, flags=mp.MPLD_FLAG_VALIDATE)
    assert ei.value.code == 2
    _assert_same(g, 3, 0.1)  # the context recovers after an error


_raw = raw_graph
_GOOD_CE, _GOOD_SE, _BAD_GRAPHS = GOOD_CE, GOOD_SE, BAD_GRAPHS


def test_validation_accepts_valid_graphs():
    good = _raw(5, _GOOD_CE, _GOOD_SE)
    r = mp.decompose_graph(good, 2, 0.1, flags=mp.MPLD_FLAG_VALIDATE)
    assert r["stats"]["error"] == 0
    graphs, k, alpha = synth.config_graphs(1)
    b = synth.concat(graphs)
    rv = mp.decompose_graph(b, k, alpha, flags=mp.MPLD_FLAG_VALIDATE)
    rn = mp.decompose_graph(b, k, alpha, flags=0)
    assert np.array_equal(rv["colors"], rn["colors"]) and np.array_equal(rv["cost"], rn["cost"])


@pytest.mark.parametrize("case", sorted(_BAD_GRAPHS))
def test_validation_rejects_each_invariant(case):
    ce, se, lo = _BAD_GRAPHS[case]
    with pytest.raises(mp.MPLDError) as ei:
        mp.decompose_graph(_raw(5, ce, se, lo), 2, 0.1, flags=mp.MPLD_FLAG_VALIDATE)
    assert ei.value.code == (1 if case == "layout_offsets_short" else 2), case
    _assert_same(from_edges(4, [(0, 1), (1, 2)]), 3, 0.1)  # the context recovers


def test_batch_equals_individual_calls():
    graphs = [synth.make_layout(2000, 2300, k=3, stitch_prob=0.5, comp_max=10, density=0.9, seed=s) for s in range(4)]
    b = synth.concat(graphs)
    gb = mp.decompose_graph(b, 3, 0.1)
    for li, g in enumerate(graphs):
        gi = mp.decompose_graph(g, 3, 0.1)
        a, e = b.layout_offsets[li], b.layout_offsets[li + 1]
        assert np.array_equal(gb["colors"][a:e], gi["colors"])
        assert gb["n_conflicts"][li] == gi["n_conflicts"][0] and gb["cost"][li] == gi["cost"][0]


def test_device_entry_point_matches_host_entry_point():
    graphs, k, alpha = synth.config_graphs(1)
    b = synth.concat(graphs[:4])
    host = mp.decompose_graph(b, k, alpha, max_steps=BUDGET)
    dev = torch.device("cuda:0")
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    ctx = mp.Context(0, b.n, b.n_layouts)
    colors = torch.empty(b.n, dtype=torch.int32, device=dev)
    counts = torch.empty(2 * b.n_layouts, dtype=torch.int64, device=dev)
    cost = torch.empty(b.n_layouts, dtype=torch.float64, device=dev)
    stats = torch.empty(len(mp.STAT_NAMES), dtype=torch.int64, device=dev)
    ctx.set_timing(True)
    for _ in range(2):
        ctx.decompose_device(T(b.layout_offsets), b.n, T(b.ce_rowptr), T(b.ce_col), T(b.se_rowptr), T(b.se_col),
                             k, alpha, BUDGET, colors, counts, cost, stats)
    torch.cuda.synchronize()
    assert np.array_equal(colors.cpu().numpy(), host["colors"])
    c = counts.cpu().numpy().reshape(-1, 2)
    assert np.array_equal(c[:, 0], host["n_conflicts"]) and np.array_equal(c[:, 1], host["n_stitches"])
    assert np.array_equal(cost.cpu().numpy(), host["cost"])
    times = ctx.kernel_times()
    assert times["mpld_exact_cover_search"][1] == 2 and times["mpld_exact_cover_search"][0] > 0
    ctx.close()


@pytest.mark.parametrize("shards", [1, 2, 3])
def test_sharded_phases_equal_oracle(shards):
    """The phase-split path of one batch sharded over `shards` processes, simulated
    on one GPU: every shard searches its components into its own colour buffer,
    the buffers are combined by an element-wise maximum (the NCCL all-reduce MAX
    of the multi-GPU run), then recovery + Eq. (1) — equal to the oracle."""
    graphs, k, alpha = synth.config_graphs(1)
    b = synth.concat(graphs[:5])
    dev = torch.device("cuda:0")
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    ctx = mp.Context(0, b.n, b.n_layouts)
    colors = torch.empty(b.n, dtype=torch.int32, device=dev)
    counts = torch.empty(2 * b.n_layouts, dtype=torch.int64, device=dev)
    cost = torch.empty(b.n_layouts, dtype=torch.float64, device=dev)
    stats = torch.empty(len(mp.STAT_NAMES), dtype=torch.int64, device=dev)
    graph = [T(b.layout_offsets), T(b.ce_rowptr), T(b.ce_col), T(b.se_rowptr), T(b.se_col)]  # alive until finish
    ctx.prepare_device(graph[0], b.n, *graph[1:], k, colors, counts, flags=mp.MPLD_FLAG_VALIDATE)
    torch.cuda.synchronize()
    assert int(colors.max()) == -1
    parts = []
    for s in range(shards):
        c = colors.clone()
        ctx.search_device(alpha, 0, s, shards, c)
        parts.append(c)
    torch.cuda.synchronize()
    owned = [(p >= 0) for p in parts]
    assert int(sum(o.int() for o in owned).max()) <= 1  # every kept vertex searched by exactly one shard
    # the cost-balanced partition (include/mpld.h phase 2), recomputed from the
    # oracle's components: estimate n * k^n capped at 2^32, inclusive prefix in
    # root order, shard of the interval's start
    ref_comps = sorted(oracle.decompose(b, k, alpha, max_steps=0)["components"], key=lambda c: c["root"])

    def estimate(n):
        e = n
        for _ in range(n):
            if e >= 1 << 32:
                break
            e *= k
        return min(e, 1 << 32)

    ests = [estimate(c["size"]) for c in ref_comps]
    total, acc = float(sum(ests)), 0
    host_owned = [o.cpu().numpy() for o in owned]
    for c, e in zip(ref_comps, ests):
        acc += e
        want = min(max(int(float(acc - e) / total * float(shards)), 0), shards - 1)
        got = [s for s in range(shards) if host_owned[s][c["root"]]]
        assert got == [want], (c, got, want)
    combined = torch.stack(parts).amax(0).contiguous()
    # the compact exchange (mpld_shard_export / mpld_shard_import): each shard's
    # (vertex, colour) list, concatenated with padding, scattered into the
    # all -1 colours of phase 1 gives the same combined colouring
    lists = []
    for p in parts:
        pr = torch.empty(2 * b.n, dtype=torch.int32, device=dev)
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        ctx.shard_export(p, pr, cnt)
        torch.cuda.synchronize()
        m = int(cnt.item())
        assert m == int((p >= 0).sum())
        exp = pr[: 2 * m].view(-1, 2).cpu().numpy()
        assert sorted(exp[:, 0].tolist()) == torch.nonzero(p >= 0).flatten().cpu().tolist()
        assert (p.cpu().numpy()[exp[:, 0]] == exp[:, 1]).all()
        lists += [pr[: 2 * m], torch.full((6,), -1, dtype=torch.int32, device=dev)]
    imported = colors.clone()
    ctx.shard_import(torch.cat(lists), imported)
    torch.cuda.synchronize()
    assert torch.equal(imported, combined)
    ctx.finish_device(alpha, combined, counts, cost, stats)
    torch.cuda.synchronize()
    ref = oracle.decompose(b, k, alpha, max_steps=0)
    assert np.array_equal(combined.cpu().numpy(), ref["colors"])
    c2 = counts.cpu().numpy().reshape(-1, 2)
    for li, (c, s_, cst) in enumerate(ref["per_layout"]):
        assert (int(c2[li, 0]), int(c2[li, 1]), float(cost[li])) == (c, s_, cst)
    ctx.close()


def test_full_size_config2_exact_element_by_element():
    """configs[2] at full s38584 size exactly as bench.py times it
    (bench.workload_items(2, 0, 1): one QPLD layout, k = 4, components up to
    ~40 vertices, exact mode, validation on): full element-by-element parity
    with the oracle (~15 s of oracle): light lanes, the 32- and 64-bit heavy
    searches and their work-queue spill all take part."""
    import bench
    it = bench.workload_items(2, 0, 1)[0]
    assert it.max_steps == 0 and it.k == 4
    got, ref = _assert_same(it.g, it.k, it.alpha, max_steps=it.max_steps)
    sizes = [c["size"] for c in ref["components"]]
    assert 36 <= max(sizes) <= 48 and sum(1 for n in sizes if n > 32) >= 5  # the shape configs[2] names
    assert got["stats"]["max_component"] == max(sizes)
    assert got["stats"]["truncated"] == 0


def test_async_pipeline_matches_sync_calls():
    """mpld_decompose_batch_async / mpld_wait: three back-to-back submits (the
    third reuses the first's staging slot), pinned and pageable host buffers,
    results identical to the blocking host call."""
    import torch
    batches = []
    for s in range(3):
        gs, k, alpha = synth.config_graphs(1, seed=100 + s)
        batches.append((synth.concat(gs[: 3 + 2 * s]), k, alpha))
    ctx = mp.Context(0, 1 << 10, 2)
    tickets = []
    for i, (b, k, alpha) in enumerate(batches):
        arrs = [b.layout_offsets, b.ce_rowptr, b.ce_col, b.se_rowptr, b.se_col]
        if i == 1:  # pinned host memory: truly asynchronous copies
            arrs = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in arrs]
        lo, crp, ccol, srp, scol = arrs
        tickets.append(ctx.submit(lo, b.n, crp, ccol, srp, scol, k, alpha, max_steps=0, flags=mp.MPLD_FLAG_VALIDATE))
    for (b, k, alpha), t in zip(batches, tickets):
        got = ctx.wait(t)
        ref = mp.decompose_graph(b, k, alpha, max_steps=0)
        assert np.array_equal(got["colors"], ref["colors"])
        assert np.array_equal(got["n_conflicts"], ref["n_conflicts"])
        assert np.array_equal(got["n_stitches"], ref["n_stitches"])
        assert np.array_equal(got["cost"], ref["cost"])
        # exact mode: the CTA-parallel search's node count depends on when lanes
        # publish the shared incumbent, so steps are not compared (the result is)
        nondet = ("steps", "max_steps", "spill_refused")
        assert {a: v for a, v in got["stats"].items() if a not in nondet} == \
               {a: v for a, v in ref["stats"].items() if a not in nondet}
    # a device-side error surfaces from wait(); the context keeps working
    ce, se, lo = _BAD_GRAPHS["asymmetric_ce"]
    bad = _raw(5, ce, se, lo)
    t = ctx.submit(bad.layout_offsets, bad.n, bad.ce_rowptr, bad.ce_col, bad.se_rowptr, bad.se_col, 2, 0.1,
                   flags=mp.MPLD_FLAG_VALIDATE)
    with pytest.raises(mp.MPLDError) as ei:
        ctx.wait(t)
    assert ei.value.code == 2
    b, k, alpha = batches[0]
    t = ctx.submit(b.layout_offsets, b.n, b.ce_rowptr, b.ce_col, b.se_rowptr, b.se_col, k, alpha)
    assert np.array_equal(ctx.wait(t)["colors"], mp.decompose_graph(b, k, alpha)["colors"])
    ctx.close()


@pytest.mark.parametrize("case", ["stress20", "k4", "cfg1"])
def test_heavy_search_spill(monkeypatch, case):
    """Exact mode with the heavy-search spill threshold at its minimum (64 warp
    iterations): long searches hand their open work to the work queue, other
    warps take it, slots merge the best keys — the result must still be the
    oracle's first optimal leaf (R7) for every component."""
    monkeypatch.setenv("MPLD_HEAVY_SPILL", "64")
    if case == "stress20":
        k, alpha = 3, 0.1
        g = synth.stress_components(20, 40, 3, seed=11)
    elif case == "k4":
        graphs, k, alpha = synth.config_graphs(2, scale=0.05)
        g = graphs[0]
    else:
        graphs, k, alpha = synth.config_graphs(1)
        g = synth.concat(graphs[:6])
    dev = torch.device("cuda:0")
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    L = int(g.layout_offsets.size - 1)
    lo = g.layout_offsets
    ctx = mp.Context(0, g.n, L)  # reads MPLD_HEAVY_SPILL
    colors = torch.empty(g.n, dtype=torch.int32, device=dev)
    counts = torch.empty(2 * L, dtype=torch.int64, device=dev)
    cost = torch.empty(L, dtype=torch.float64, device=dev)
    stats = torch.empty(len(mp.STAT_NAMES), dtype=torch.int64, device=dev)
    ctx.decompose_device(T(lo), g.n, T(g.ce_rowptr), T(g.ce_col), T(g.se_rowptr), T(g.se_col),
                         k, alpha, 0, colors, counts, cost, stats, flags=mp.MPLD_FLAG_VALIDATE)
    torch.cuda.synchronize()
    ref = oracle.decompose(g, k, alpha, max_steps=0)
    assert np.array_equal(colors.cpu().numpy(), ref["colors"])
    c2 = counts.cpu().numpy().reshape(-1, 2)
    for li, (c, s_, cst) in enumerate(ref["per_layout"]):
        assert (int(c2[li, 0]), int(c2[li, 1]), float(cost[li])) == (c, s_, cst)
    assert int(stats.cpu().numpy()[mp.STAT_NAMES.index("truncated")]) == 0
    ctx.close()


def _se_pairs(g):
    """Each stitch edge once, (u, v) with u < v, int32 [m, 2]."""
    e = g.se_edges()
    return np.ascontiguousarray(e[e[:, 0] < e[:, 1]], dtype=np.int32) if e.size else np.zeros((0, 2), np.int32)


def test_stitch_pairs_entry_point():
    """mpld_decompose_batch_pairs_async (stitch edges as pairs, SE CSR built on
    the device) gives the oracle's colours and per-layout counts, pair order
    and direction notwithstanding; bad pairs are rejected."""
    graphs, k, alpha = synth.config_graphs(1)
    b = synth.concat(graphs[:6])
    pairs = _se_pairs(b)
    assert pairs.shape[0] > 0
    rng = np.random.default_rng(0)
    shuffled = pairs[rng.permutation(pairs.shape[0])].copy()
    flip = rng.random(shuffled.shape[0]) < 0.5
    shuffled[flip] = shuffled[flip][:, ::-1]
    ref = oracle.decompose(b, k, alpha, max_steps=0)
    ctx = mp.Context(0, b.n, b.n_layouts)
    for pp in (pairs, shuffled):
        t = ctx.submit_pairs(b.layout_offsets, b.n, b.ce_rowptr, b.ce_col, pp, k, alpha, 0, mp.MPLD_FLAG_VALIDATE)
        r = ctx.wait(t)
        assert np.array_equal(r["colors"], ref["colors"])
        for li, (c, s_, cst) in enumerate(ref["per_layout"]):
            assert (int(r["n_conflicts"][li]), int(r["n_stitches"][li]), float(r["cost"][li])) == (c, s_, cst)
    bad = pairs.copy()
    bad[0, 1] = b.n  # out of range
    with pytest.raises(mp.MPLDError):
        ctx.submit_pairs(b.layout_offsets, b.n, b.ce_rowptr, b.ce_col, bad, k, alpha, 0, mp.MPLD_FLAG_VALIDATE)
    dup = np.concatenate([pairs, pairs[:1]])  # a duplicate stitch edge: caught by the device validation
    with pytest.raises(mp.MPLDError):
        ctx.wait(ctx.submit_pairs(b.layout_offsets, b.n, b.ce_rowptr, b.ce_col, dup, k, alpha, 0,
                                  mp.MPLD_FLAG_VALIDATE))
    ctx.close()


@pytest.mark.parametrize("slots", ["0", "4", "64"])
def test_recovery_cluster_tail_spill(monkeypatch, slots):
    """The recovery's cluster tail keeps each CTA's ready vertices in its shared
    memory and spills the rest to a global list processed cluster-wide; with the
    slots capped (0: every vertex after the tail's first level spills) the
    colours must not change (R9)."""
    monkeypatch.setenv("MPLD_TAIL_SLOTS", slots)
    graphs, k, alpha = synth.config_graphs(1)
    b = synth.concat(graphs[:8])
    dev = torch.device("cuda:0")
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    ctx = mp.Context(0, b.n, b.n_layouts)  # reads MPLD_TAIL_SLOTS
    colors = torch.empty(b.n, dtype=torch.int32, device=dev)
    counts = torch.empty(2 * b.n_layouts, dtype=torch.int64, device=dev)
    cost = torch.empty(b.n_layouts, dtype=torch.float64, device=dev)
    stats = torch.empty(len(mp.STAT_NAMES), dtype=torch.int64, device=dev)
    ctx.decompose_device(T(b.layout_offsets), b.n, T(b.ce_rowptr), T(b.ce_col), T(b.se_rowptr), T(b.se_col),
                         k, alpha, 0, colors, counts, cost, stats, flags=mp.MPLD_FLAG_VALIDATE)
    torch.cuda.synchronize()
    ref = oracle.decompose(b, k, alpha, max_steps=0)
    assert np.array_equal(colors.cpu().numpy(), ref["colors"])
    c2 = counts.cpu().numpy().reshape(-1, 2)
    for li, (c, s_, cst) in enumerate(ref["per_layout"]):
        assert (int(c2[li, 0]), int(c2[li, 1]), float(cost[li])) == (c, s_, cst)
    ctx.close()


def test_bench_launch_config1_sampled():
    """configs[1] exactly as bench.py times it (bench.workload(0, 16): the ten
    ISCAS-85-shaped layouts x16 seeds in one batch, exact mode, validation on):
    Eq. (1) counts recomputed from the colours of every layout, and the oracle
    decomposes every layout on its own (layouts are independent, so each slice
    of the batch must equal its own oracle result element by element)."""
    graphs = []
    for r in range(16):
        gs, k, alpha = synth.config_graphs(1, seed=10 * r)
        graphs += gs
    b = synth.concat(graphs)
    got = mp.decompose_graph(b, k, alpha, max_steps=0, flags=mp.MPLD_FLAG_VALIDATE)
    colors = got["colors"]
    assert got["stats"]["error"] == 0 and got["stats"]["truncated"] == 0
    assert ((colors >= 0) & (colors < k)).all()
    offs = b.layout_offsets
    ce, se = b.ce_edges(), b.se_edges()
    lay_ce = np.searchsorted(offs, ce[:, 0], side="right") - 1
    lay_se = np.searchsorted(offs, se[:, 0], side="right") - 1
    nc = np.bincount(lay_ce, weights=(colors[ce[:, 0]] == colors[ce[:, 1]]), minlength=b.n_layouts)
    ns = np.bincount(lay_se, weights=(colors[se[:, 0]] != colors[se[:, 1]]), minlength=b.n_layouts)
    assert np.array_equal(nc.astype(np.int64), np.asarray(got["n_conflicts"], dtype=np.int64))
    assert np.array_equal(ns.astype(np.int64), np.asarray(got["n_stitches"], dtype=np.int64))
    parts = synth.split(b)
    for li in range(b.n_layouts):  # every layout (~0.2 s of oracle each)
        ref = oracle.decompose(parts[li], k, alpha, max_steps=0)
        a, e = int(offs[li]), int(offs[li + 1])
        assert np.array_equal(colors[a:e], ref["colors"]), li
        c, s_, cst = ref["per_layout"][0]
        assert (int(got["n_conflicts"][li]), int(got["n_stitches"][li]), float(got["cost"][li])) == (c, s_, cst)


def test_full_size_config3_element_by_element():
    """configs[3] at full size (10^6 polygons, one layout, k = 3) in exact mode,
    as bench.py --config 3 times it: full element-by-element parity (~20 s of
    oracle)."""
    graphs, k, alpha = synth.config_graphs(3)
    _assert_same(graphs[0], k, alpha, max_steps=0)


@pytest.mark.parametrize("k", [3, 4])
@pytest.mark.parametrize("size", [4, 8, 16, 24, 32, 48, 64])
def test_full_size_stress_sweep(size, k):
    """configs[4] at full size exactly as bench.py times it (bench.workload_items(4, 0, 1):
    10^5 components of `size` vertices in one launch, 500 distinct components
    repeated in 200 layouts; exact up to 16 vertices, the bench's budget above,
    DESIGN.md R13).  Every copy of a component must get the same colours
    wherever it lands (light lanes, heavy warps, work queue), the counts must be
    recomputable from the colours, and the oracle recomputes a sample of the
    distinct components one by one at the same budget."""
    import bench
    it = [i for i in bench.workload_items(4, 0, 1) if i.label == f"n{size}_k{k}"][0]
    g, budget = it.g, it.max_steps
    tmpl = bench.stress_template(size, k)
    assert g.n == bench.STRESS_COPIES * tmpl.n and np.array_equal(g.ce_col[: tmpl.ce_col.size], tmpl.ce_col)
    got = mp.decompose_graph(g, k, 0.1, max_steps=budget, flags=mp.MPLD_FLAG_VALIDATE)
    colors = got["colors"]
    ce_adj, se_adj = tmpl.ce_adj(), tmpl.se_adj()
    hround, _ = oracle.simplify(tmpl.n, ce_adj, se_adj, k)
    comps = oracle.components(tmpl.n, ce_adj, se_adj, hround)
    # a component of <= k vertices has every degree < k: the simplification hides it whole
    assert len(comps) == (bench.STRESS_TEMPLATES if size > k else 0)
    assert got["stats"]["components"] == bench.STRESS_COPIES * len(comps)
    assert ((colors >= 0) & (colors < k)).all()
    per = colors.reshape(bench.STRESS_COPIES, tmpl.n)
    assert (per == per[0]).all()
    ce = g.ce_edges()
    assert int((colors[ce[:, 0]] == colors[ce[:, 1]]).sum()) == int(got["n_conflicts"].sum())
    assert (got["n_conflicts"] == got["n_conflicts"][0]).all()
    assert (got["n_stitches"] == 0).all()
    assert np.allclose(got["cost"], got["n_conflicts"].astype(np.float64))
    if budget == 0:
        assert got["stats"]["truncated"] == 0
    else:  # the budget is per component and deterministic: every copy truncates alike
        assert got["stats"]["truncated"] % bench.STRESS_COPIES == 0
    w = oracle.alpha_units(0.1)
    trunc = 0
    for order in random.Random(size * 10 + k).sample(comps, min(len(comps), 6 if size >= 32 else 20)):
        r = oracle.solve_component(order, ce_adj, se_adj, k, w, budget)
        trunc += r["truncated"]
        for v, c in r["global_colors"].items():
            assert per[0, v] == c
    if not comps:  # everything recovered: the whole template equals the oracle's run
        assert np.array_equal(per[0], oracle.decompose(tmpl, k, 0.1, max_steps=0)["colors"])


@functools.lru_cache(maxsize=None)
def _solvable_stress_components(size, k):
    """Up to 4 components of the configs[4] template whose exact search the
    oracle finishes within 200,000 nodes, with the oracle's results."""
    import bench
    tmpl = bench.stress_template(size, k)
    ce_adj, se_adj = tmpl.ce_adj(), tmpl.se_adj()
    hround, _ = oracle.simplify(tmpl.n, ce_adj, se_adj, k)
    comps = oracle.components(tmpl.n, ce_adj, se_adj, hround)
    w = oracle.alpha_units(0.1)
    solved = []
    for order in comps[:40]:
        r = oracle.solve_component(order, ce_adj, se_adj, k, w, 200_000)
        if not r["truncated"]:
            solved.append((order, r))
        if len(solved) == 4:
            break
    return solved, ce_adj


@pytest.mark.parametrize("spill", [None, "64"])
@pytest.mark.parametrize("k", [3, 4])
@pytest.mark.parametrize("size", [32, 48, 64])
def test_exact_mode_large_stress_components(monkeypatch, size, k, spill):
    """Exact mode (max_steps = 0) on 32-64-vertex components (the 64-bit light
    lane, the 64-bit heavy search, its work queue and slots): the configs[4]
    components whose exact search the oracle finishes within 200,000 nodes,
    each repeated, must get the oracle's first optimal leaf, untruncated."""
    if spill:
        monkeypatch.setenv("MPLD_HEAVY_SPILL", spill)
    solved, ce_adj = _solvable_stress_components(size, k)
    assert len(solved) >= 2, "too few oracle-solvable components"
    parts = []
    for order, _ in solved:  # each solved component as its own layout (local ids in the template's order)
        loc = {v: i for i, v in enumerate(sorted(order))}
        es = {(min(loc[v], loc[u]), max(loc[v], loc[u])) for v in order for u in ce_adj[v] if u in loc}
        parts.append(from_edges(len(order), sorted(es)))
    b = synth.concat(parts * 16)
    ctx = mp.Context(0, b.n, b.n_layouts)  # reads MPLD_HEAVY_SPILL
    dev = torch.device("cuda:0")
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    colors = torch.empty(b.n, dtype=torch.int32, device=dev)
    counts = torch.empty(2 * b.n_layouts, dtype=torch.int64, device=dev)
    cost = torch.empty(b.n_layouts, dtype=torch.float64, device=dev)
    stats = torch.empty(len(mp.STAT_NAMES), dtype=torch.int64, device=dev)
    ctx.decompose_device(T(b.layout_offsets), b.n, T(b.ce_rowptr), T(b.ce_col), T(b.se_rowptr), T(b.se_col),
                         k, 0.1, 0, colors, counts, cost, stats, flags=mp.MPLD_FLAG_VALIDATE)
    torch.cuda.synchronize()
    st = dict(zip(mp.STAT_NAMES, stats.cpu().tolist()))
    assert st["error"] == 0 and st["truncated"] == 0
    got = colors.cpu().numpy()
    c2 = counts.cpu().numpy().reshape(-1, 2)
    offs = b.layout_offsets
    for li in range(b.n_layouts):
        order, r = solved[li % len(solved)]
        loc = {v: i for i, v in enumerate(sorted(order))}
        want = np.zeros(len(order), np.int32)
        for v, c in r["global_colors"].items():
            want[loc[v]] = c
        assert np.array_equal(got[offs[li]:offs[li + 1]], want), li
        assert int(c2[li, 0]) == r["n_conf"] and float(cost[li]) == r["n_conf"] + 0.1 * r["n_stitch"]
    ctx.close()


def test_host_staging_grows_with_layout_count():
    """Regression: a host call with more layouts than any earlier call must grow
    the device staging of layout offsets / counts / costs (it once sized them
    from the workspace capacity, already grown by then, and overflowed)."""
    small = synth.concat([synth.stress_components(6, 4, 3, seed=s) for s in range(2)])
    ref_s = oracle.decompose(small, 3, 0.1, max_steps=0)
    got = mp.decompose_graph(small, 3, 0.1, max_steps=0)
    assert np.array_equal(got["colors"], ref_s["colors"])
    tmpl = synth.stress_components(6, 4, 3, seed=9)
    ref_t = oracle.decompose(tmpl, 3, 0.1, max_steps=0)
    for n_lay in (300, 1000):
        big = synth.concat([tmpl] * n_lay)
        got = mp.decompose_graph(big, 3, 0.1, max_steps=0)
        assert np.array_equal(got["colors"].reshape(n_lay, tmpl.n), np.tile(ref_t["colors"], (n_lay, 1)))
        c, s_, cst = ref_t["per_layout"][0]
        assert (got["n_conflicts"] == c).all() and (got["n_stitches"] == s_).all() and (got["cost"] == cst).all()


def test_capacity_sequence_all_entry_points():
    """Batches that grow and shrink in vertices, edges and layout count, sent
    in turn through every entry point of ONE context that starts small (async,
    pairs, device, the sharded phases; and the process-wide host call): each result must be the oracle's, so no staging
    or workspace buffer may be sized from a capacity another buffer grew."""
    shapes = [(1, 150), (40, 50), (2, 1500), (1, 30), (150, 12), (3, 400), (300, 10), (1, 2500)]
    dev = torch.device("cuda:0")
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    ctx = mp.Context(0, 1 << 6, 1)
    for i, (n_lay, nv) in enumerate(shapes):
        b = synth.concat([synth.make_layout(nv, int(1.2 * nv), k=3, stitch_prob=0.5, comp_max=8, seed=50 * i + j)
                          for j in range(n_lay)])
        k, alpha = 3, 0.1
        ref = oracle.decompose(b, k, alpha, max_steps=0)
        want_c = np.array([p[0] for p in ref["per_layout"]], dtype=np.int64)
        want_s = np.array([p[1] for p in ref["per_layout"]], dtype=np.int64)
        want_cost = np.array([p[2] for p in ref["per_layout"]], dtype=np.float64)
        results = [mp.decompose_graph(b, k, alpha, max_steps=0, flags=mp.MPLD_FLAG_VALIDATE)]
        t1 = ctx.submit(b.layout_offsets, b.n, b.ce_rowptr, b.ce_col, b.se_rowptr, b.se_col, k, alpha, 0,
                        mp.MPLD_FLAG_VALIDATE)
        t2 = ctx.submit_pairs(b.layout_offsets, b.n, b.ce_rowptr, b.ce_col, _se_pairs(b), k, alpha, 0,
                              mp.MPLD_FLAG_VALIDATE)
        results += [ctx.wait(t1), ctx.wait(t2)]
        colors = torch.empty(b.n, dtype=torch.int32, device=dev)
        counts = torch.empty(2 * b.n_layouts, dtype=torch.int64, device=dev)
        cost = torch.empty(b.n_layouts, dtype=torch.float64, device=dev)
        ctx.decompose_device(T(b.layout_offsets), b.n, T(b.ce_rowptr), T(b.ce_col), T(b.se_rowptr), T(b.se_col),
                             k, alpha, 0, colors, counts, cost, flags=mp.MPLD_FLAG_VALIDATE)
        torch.cuda.synchronize()
        c2 = counts.cpu().numpy().reshape(-1, 2)
        results.append({"colors": colors.cpu().numpy(), "n_conflicts": c2[:, 0], "n_stitches": c2[:, 1],
                        "cost": cost.cpu().numpy()})
        # the phase-split path, two shards simulated on this GPU (combined by max)
        graph = [T(b.layout_offsets), T(b.ce_rowptr), T(b.ce_col), T(b.se_rowptr), T(b.se_col)]
        ctx.prepare_device(graph[0], b.n, *graph[1:], k, colors, counts, flags=mp.MPLD_FLAG_VALIDATE)
        parts = []
        for sh in range(2):
            c = colors.clone()
            ctx.search_device(alpha, 0, sh, 2, c)
            parts.append(c)
        combined = torch.stack(parts).amax(0).contiguous()
        ctx.finish_device(alpha, combined, counts, cost)
        torch.cuda.synchronize()
        c2 = counts.cpu().numpy().reshape(-1, 2)
        results.append({"colors": combined.cpu().numpy(), "n_conflicts": c2[:, 0], "n_stitches": c2[:, 1],
                        "cost": cost.cpu().numpy()})
        for path, r in zip(("host", "async", "pairs", "device", "sharded"), results):
            assert np.array_equal(r["colors"], ref["colors"]), (i, path)
            assert np.array_equal(np.asarray(r["n_conflicts"], np.int64), want_c), (i, path)
            assert np.array_equal(np.asarray(r["n_stitches"], np.int64), want_s), (i, path)
            assert np.array_equal(np.asarray(r["cost"], np.float64), want_cost), (i, path)
    ctx.close()


def test_phases_on_different_streams_and_a_fresh_counts_buffer():
    """A context's calls may be enqueued on different streams (each waits for
    the previous call's last operation), and mpld_finish_device may be given a
    counts buffer other than the one of mpld_prepare_device (it is reset and
    recomputed): results equal the oracle's."""
    graphs, k, alpha = synth.config_graphs(1)
    b = synth.concat(graphs[:5])
    b2 = synth.concat(graphs[5:])
    ref = oracle.decompose(b, k, alpha, max_steps=0)
    ref2 = oracle.decompose(b2, k, alpha, max_steps=0)
    dev = torch.device("cuda:0")
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    ctx = mp.Context(0, 1 << 10, 1)
    sa, sb, sc, sd = (torch.cuda.Stream(dev) for _ in range(4))
    graph = [T(b.layout_offsets), T(b.ce_rowptr), T(b.ce_col), T(b.se_rowptr), T(b.se_col)]
    torch.cuda.synchronize()
    colors = torch.empty(b.n, dtype=torch.int32, device=dev)
    counts1 = torch.empty(2 * b.n_layouts, dtype=torch.int64, device=dev)
    counts2 = torch.full((2 * b.n_layouts,), 987654321, dtype=torch.int64, device=dev)
    cost = torch.empty(b.n_layouts, dtype=torch.float64, device=dev)
    for one_shard_counts_buffer in (counts2, counts1):
        if one_shard_counts_buffer is counts2:
            counts2.fill_(987654321)
            torch.cuda.synchronize()
        ctx.prepare_device(graph[0], b.n, *graph[1:], k, colors, counts1, flags=mp.MPLD_FLAG_VALIDATE, stream=sa)
        ctx.search_device(alpha, 0, 0, 1, colors, stream=sb)
        ctx.finish_device(alpha, colors, one_shard_counts_buffer, cost, stream=sc)
        sc.synchronize()
        assert np.array_equal(colors.cpu().numpy(), ref["colors"])
        c2 = one_shard_counts_buffer.cpu().numpy().reshape(-1, 2)
        for li, (c, s_, cst) in enumerate(ref["per_layout"]):
            assert (int(c2[li, 0]), int(c2[li, 1]), float(cost[li])) == (c, s_, cst)
    # an asynchronous host submit (the context's own stream) followed at once by a
    # device call of another batch on another stream: both results intact
    t = ctx.submit(b.layout_offsets, b.n, b.ce_rowptr, b.ce_col, b.se_rowptr, b.se_col, k, alpha, 0,
                   mp.MPLD_FLAG_VALIDATE)
    g2 = [T(b2.layout_offsets), T(b2.ce_rowptr), T(b2.ce_col), T(b2.se_rowptr), T(b2.se_col)]
    col2 = torch.empty(b2.n, dtype=torch.int32, device=dev)
    cnt2 = torch.empty(2 * b2.n_layouts, dtype=torch.int64, device=dev)
    cost2 = torch.empty(b2.n_layouts, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    ctx.decompose_device(g2[0], b2.n, *g2[1:], k, alpha, 0, col2, cnt2, cost2, flags=mp.MPLD_FLAG_VALIDATE,
                         stream=sd)
    r = ctx.wait(t)
    sd.synchronize()
    assert np.array_equal(r["colors"], ref["colors"])
    assert np.array_equal(col2.cpu().numpy(), ref2["colors"])
    assert np.array_equal(cost2.cpu().numpy(), np.array([p[2] for p in ref2["per_layout"]]))
    ctx.close()


def test_binding_rejects_wrong_element_types():
    """The binding checks element types and contiguity (an int64 index tensor or
    a float32 cost buffer would otherwise be reinterpreted by the C ABI)."""
    g = synth.fixtures()["K4"]
    dev = torch.device("cuda:0")
    ctx = mp.Context(0, 16, 1)
    lo = torch.tensor(g.layout_offsets, dtype=torch.int32, device=dev)
    cr64 = torch.tensor(g.ce_rowptr, dtype=torch.int64, device=dev)
    args = [torch.tensor(a, dtype=torch.int32, device=dev) for a in (g.ce_rowptr, g.ce_col, g.se_rowptr, g.se_col)]
    colors = torch.empty(g.n, dtype=torch.int32, device=dev)
    counts = torch.empty(2, dtype=torch.int64, device=dev)
    cost = torch.empty(1, dtype=torch.float64, device=dev)
    with pytest.raises(TypeError):
        ctx.decompose_device(lo, g.n, cr64, *args[1:], 3, 0.1, 0, colors, counts, cost)
    with pytest.raises(TypeError):
        ctx.decompose_device(lo, g.n, *args, 3, 0.1, 0, colors, counts, cost.float())
    with pytest.raises(TypeError):
        mp.mpld_decompose_batch(g.layout_offsets, g.n, torch.tensor(g.ce_rowptr, dtype=torch.int64), g.ce_col,
                                g.se_rowptr, g.se_col, 3, 0.1)
    with pytest.raises(TypeError):
        mp.mpld_decompose_batch(g.layout_offsets, g.n, g.ce_rowptr, g.ce_col, g.se_rowptr, g.se_col, 3, 0.1,
                                out_colors=np.empty(g.n, dtype=np.int64))
    ctx.decompose_device(lo, g.n, *args, 3, 0.1, 0, colors, counts, cost)
    torch.cuda.synchronize()
    assert int(counts[0]) == 1
    ctx.close()


def _budget_trace_rows():
    import os
    rows = []
    for line in open(os.path.join(os.path.dirname(__file__), "golden", "k4_budget_trace.txt")):
        if line.startswith("budget"):
            _, b, steps, tr, cost, *col = line.split()
            rows.append((int(b), int(steps), int(tr), int(cost), [int(c) for c in col]))
    return rows


@pytest.mark.parametrize("budget,steps,truncated,cost,colors", _budget_trace_rows())
def test_k4_budget_hand_trace_through_the_c_abi(budget, steps, truncated, cost, colors):
    """The hand-traced node counts of tests/golden/k4_budget_trace.txt (K4,
    k = 3) at every budget: the GPU stops at exactly the traced node."""
    got = mp.decompose_graph(synth.fixtures()["K4"], 3, 0.1, max_steps=budget, flags=mp.MPLD_FLAG_VALIDATE)
    assert got["colors"].tolist() == colors
    assert (got["stats"]["steps"], got["stats"]["truncated"]) == (steps, truncated)
    assert int(got["n_conflicts"][0]) * 1000 == cost


def test_upper_triangle_entry_point():
    """mpld_decompose_batch_upper_async (conflict edges as the upper triangle
    of their CSR with uint8 row lengths, stitch candidates as pairs, the
    symmetric CSR built on the device) gives the oracle's colours and
    per-layout counts; malformed triangles are reported as MPLD_ERR_GRAPH and
    the context keeps working."""
    graphs, k, alpha = synth.config_graphs(1)
    b = synth.concat(graphs[:6])
    ref = oracle.decompose(b, k, alpha, max_steps=0)
    ctx = mp.Context(0, b.n, b.n_layouts)
    deg, col = synth.upper_csr(b)
    pairs = synth.stitch_pairs(b)
    for flags in (mp.MPLD_FLAG_VALIDATE, 0):
        r = ctx.wait(ctx.submit_upper(b.layout_offsets, b.n, deg, col, pairs, k, alpha, 0, flags))
        assert np.array_equal(r["colors"], ref["colors"])
        for li, (c, s_, cst) in enumerate(ref["per_layout"]):
            assert (int(r["n_conflicts"][li]), int(r["n_stitches"][li]), float(r["cost"][li])) == (c, s_, cst)
    # the device-built CSR equals the host one: a second graph with a denser triangle (k = 4 clusters)
    g2 = synth.config_graphs(2, scale=0.05)[0][0]
    ref2 = oracle.decompose(g2, 4, 0.1, max_steps=0)
    d2, c2 = synth.upper_csr(g2)
    r = ctx.wait(ctx.submit_upper(g2.layout_offsets, g2.n, d2, c2, synth.stitch_pairs(g2), 4, 0.1, 0,
                                  mp.MPLD_FLAG_VALIDATE))
    assert np.array_equal(r["colors"], ref2["colors"])
    bad_cases = []
    bc = col.copy()
    bc[5] = b.n  # out of range
    bad_cases.append((deg, bc))
    bc = col.copy()
    i = int(np.nonzero(deg > 1)[0][0])
    a = int(deg[:i].astype(np.int64).sum())
    bc[a], bc[a + 1] = bc[a + 1], bc[a]  # a row not ascending
    bad_cases.append((deg, bc))
    bd = deg.copy()
    bd[i] -= 1  # row lengths that do not sum to the entries sent
    bad_cases.append((bd, col))
    bc = col.copy()
    bc[a] = i  # a self loop / an entry below the row's vertex
    bad_cases.append((deg, bc))
    for dd, cc in bad_cases:
        with pytest.raises(mp.MPLDError) as ei:
            ctx.wait(ctx.submit_upper(b.layout_offsets, b.n, dd, cc, pairs, k, alpha, 0, 0))
        assert ei.value.code == 2
    r = ctx.wait(ctx.submit_upper(b.layout_offsets, b.n, deg, col, pairs, k, alpha, 0, mp.MPLD_FLAG_VALIDATE))
    assert np.array_equal(r["colors"], ref["colors"])
    ctx.close()


def test_compact_upload_degree_limits():
    """The device build of the compact uploads counts a vertex's stitch pairs
    in 8 bits: a vertex with 200 stitch pairs is rejected (MPLD_ERR_GRAPH),
    one with 60 (a 61-vertex component) is decomposed as the oracle does."""
    ctx = mp.Context(0, 1 << 10, 1)
    for d, ok in ((60, True), (200, False)):
        n = d + 1
        g = from_edges(n, [], [(0, i) for i in range(1, n)])
        lo = np.array([0, n], np.int32)
        deg, col = synth.upper_csr(g)
        t = ctx.submit_upper(lo, n, deg, col, synth.stitch_pairs(g), 3, 0.1, 0, mp.MPLD_FLAG_VALIDATE)
        if ok:
            r = ctx.wait(t)
            assert np.array_equal(r["colors"], oracle.decompose(g, 3, 0.1, max_steps=0)["colors"])
        else:
            with pytest.raises(mp.MPLDError) as ei:
                ctx.wait(t)
            assert ei.value.code == 2
    ctx.close()
