"""The tile pipeline (kernel_tile.cu, MPLD_FLAG_TILES) and its gate: parity with the CPU oracle
on inputs the tiles take (windows cut by their shared-memory capacity, pieces
crossing tile boundaries, the pending sub-tiles of exact mode) and on inputs
they must hand to the whole-graph pipeline (pieces not local in id space,
pieces longer than a window), plus the whole-graph pipeline alone
(the default) on the same inputs.  Device outputs of both pipelines
are compared element by element."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth
from synth import from_edges

mp = pytest.importorskip("paper_2303_14335_b200")
torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

BUDGET = 1 << 20
TILE = 1024  # vertex ids owned by a tile (kernel_tile.cu kTOwn)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    mp.lib()


def _device_run(g, k, alpha, max_steps, flags):
    """One call of mpld_decompose_device; returns outputs (host) and the tile gate."""
    dev = torch.device("cuda:0")
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    lo, cr, cc, sr, sc = (T(g.layout_offsets), T(g.ce_rowptr), T(g.ce_col), T(g.se_rowptr), T(g.se_col))
    L = g.n_layouts
    colors = torch.full((g.n,), -7, dtype=torch.int32, device=dev)
    counts = torch.full((2 * L,), -7, dtype=torch.int64, device=dev)
    cost = torch.full((L,), -7.0, dtype=torch.float64, device=dev)
    stats = torch.zeros(len(mp.STAT_NAMES), dtype=torch.int64, device=dev)
    ctx = mp.Context(0, max(g.n, 1), L)
    ctx.decompose_device(lo, g.n, cr, cc, sr, sc, k, alpha, max_steps, colors, counts, cost, stats, flags=flags)
    torch.cuda.synchronize()
    gate = int(ctx.debug()[88])
    ctx.close()
    return {"colors": colors.cpu().numpy(), "counts": counts.cpu().numpy(), "cost": cost.cpu().numpy(),
            "stats": dict(zip(mp.STAT_NAMES, stats.cpu().tolist()))}, gate


def _check(g, k, alpha, max_steps, expect_gate, ref=None):
    ref = ref or oracle.decompose(g, k, alpha, max_steps=max_steps)
    outs = {}
    for name, fl in (("tile", mp.MPLD_FLAG_VALIDATE | mp.MPLD_FLAG_TILES), ("whole", mp.MPLD_FLAG_VALIDATE)):
        got, gate = _device_run(g, k, alpha, max_steps, fl)
        if name == "tile":
            assert gate == expect_gate
        else:
            assert gate == -1
        assert np.array_equal(got["colors"], ref["colors"]), (name, np.nonzero(got["colors"] != ref["colors"])[0][:10])
        for li, (c, s, cost) in enumerate(ref["per_layout"]):
            assert int(got["counts"][2 * li]) == c, name
            assert int(got["counts"][2 * li + 1]) == s, name
            assert float(got["cost"][li]) == cost, name
        st = got["stats"]
        assert st["error"] == 0
        assert st["components"] == len(ref["components"]), name
        assert st["rounds"] == ref["n_rounds"], name
        assert st["hidden"] == int((ref["hround"] >= 0).sum()), name
        assert st["truncated"] == sum(c["truncated"] for c in ref["components"]), name
        if max_steps > 0:
            assert st["steps"] == sum(c["steps"] for c in ref["components"]), name
        outs[name] = got
    for key in ("colors", "counts", "cost"):
        assert np.array_equal(outs["tile"][key], outs["whole"][key])
    return outs, ref


def _relabel(g, perm):
    """The same graph with vertex v renamed perm[v] (one layout)."""
    ce = g.ce_edges()
    se = g.se_edges()
    return from_edges(g.n, perm[ce], perm[se], name=g.name + "_perm")


def test_tiles_take_the_iscas85_suite():
    graphs, k, alpha = synth.config_graphs(1)
    _check(synth.concat(graphs), k, alpha, BUDGET, expect_gate=0)


def test_tiles_exact_mode_pending_subtiles():
    """Exact mode on QPLD components: heavy components leave their sub-tiles
    pending until the warp-parallel search, then the finish launch recovers them."""
    graphs, k, alpha = synth.config_graphs(2, scale=0.1)
    outs, _ = _check(graphs[0], k, alpha, 0, expect_gate=0)
    assert outs["tile"]["stats"]["truncated"] == 0


def test_tiles_budgeted_wide_components():
    """Budgeted mode, components of 33-64 vertices: the 64-bit lane kernel after the tiles."""
    g = synth.stress_components(48, 40, 3, seed=5)
    _check(g, 3, 0.1, 3000, expect_gate=0)


def test_tiles_capacity_limited_windows():
    """Dense pieces (K10, 9 entries per row): a 2,048-vertex window exceeds the
    12,288 CE entries of shared memory, so tiles run in sub-passes of half a window."""
    K10 = [(a, b) for a in range(10) for b in range(a + 1, 10)]
    copies = 230
    ce = [(10 * c + a, 10 * c + b) for c in range(copies) for a, b in K10]
    g = from_edges(10 * copies, ce, [], name="k10x230")
    _check(g, 4, 0.1, 400, expect_gate=0)


def test_tiles_take_pieces_not_local_in_id_space():
    """Randomly renamed vertex ids: every piece spreads over the whole id range;
    the piece order makes them contiguous, the tiles take the input."""
    g = synth.iscas_layout("c2670", k=3, stitch_prob=0.5, seed=3)
    perm = np.random.default_rng(0).permutation(g.n).astype(np.int64)
    _check(_relabel(g, perm), 3, 0.1, BUDGET, expect_gate=0)


def test_gate_piece_longer_than_a_window():
    """One piece of 5,000 vertices (a wire) is larger than a window: gate bit 2."""
    n = 5000
    ce = [(v, v + 1) for v in range(n - 1)]
    g = from_edges(n, ce, [], name="long_piece")
    _check(g, 3, 0.1, BUDGET, expect_gate=2)


@pytest.mark.parametrize("offset", [TILE - 3, TILE - 1, TILE, 2 * TILE - 7])
def test_pieces_across_tile_boundaries(offset):
    """A 40-vertex kept piece starting just below / at a tile boundary (its owner's
    halo holds it) and a 300-vertex wire piece crossing the next boundary."""
    rng = np.random.default_rng(offset)
    n = offset + 40 + 300 + 200
    ce = []
    # a dense random piece of 40 vertices at [offset, offset + 40)
    for a in range(40):
        for b in range(a + 1, min(40, a + 6)):
            if rng.random() < 0.8:
                ce.append((offset + a, offset + b))
        if a:
            ce.append((offset + a - 1, offset + a))
    ce = sorted(set(ce))
    base = offset + 40
    ce += [(base + v, base + v + 1) for v in range(299)]  # a wire
    # isolated vertices and small triangles elsewhere
    for t in range(0, offset - 3, 97):
        ce += [(t, t + 1), (t + 1, t + 2), (t, t + 2)]
    g = from_edges(n, sorted(set(ce)), [], name=f"boundary{offset}")
    _check(g, 3, 0.1, BUDGET, expect_gate=0)


def test_device_outputs_identical_on_the_bench_batch():
    """configs[1] x16 (the headline bench batch): both pipelines, element by element."""
    graphs = []
    for r in range(16):
        gs, k, alpha = synth.config_graphs(1, seed=10 * r)
        graphs += gs
    b = synth.concat(graphs)
    a, gate = _device_run(b, k, alpha, 0, mp.MPLD_FLAG_VALIDATE | mp.MPLD_FLAG_TILES)
    assert gate == 0
    w, _ = _device_run(b, k, alpha, 0, mp.MPLD_FLAG_VALIDATE)
    for key in ("colors", "counts", "cost"):
        assert np.array_equal(a[key], w[key]), key
    for key in ("components", "hidden", "rounds", "max_component", "truncated", "error"):
        assert a["stats"][key] == w["stats"][key], key


def test_tiles_reject_invalid_input_like_the_whole_graph_pipeline():
    """An asymmetric CSR: the tiles gate (a neighbour outside its piece's window), the
    whole-graph pipeline reports MPLD_ERR_GRAPH."""
    g = from_edges(6, [(0, 1), (1, 2), (2, 0), (3, 4)], [])
    col = g.ce_col.copy()
    col[-1] = 5  # row 4 lists 5, row 5 does not list 4
    bad = synth.graph.DecompGraph(g.n, g.ce_rowptr.copy(), col, g.se_rowptr.copy(), g.se_col.copy(), name="asym")
    with pytest.raises(mp.MPLDError) as ei:
        mp.decompose_graph(bad, 3, 0.1, max_steps=BUDGET, flags=mp.MPLD_FLAG_VALIDATE | mp.MPLD_FLAG_TILES)
    assert ei.value.code == 2


@pytest.mark.parametrize("k", [2, 3, 4])
def test_tiles_every_k_with_stitches(k):
    """k = 2, 3, 4 with stitch candidates, budgeted and (small components)
    exact: tiles against the oracle and the default pipeline, 150 random
    layouts in one batch (windows hold several layouts)."""
    import random
    rng = random.Random(70 + k)
    graphs = []
    for _ in range(150):
        n = rng.randint(4, 14)
        ce, se = [], []
        for u in range(n):
            for v in range(u + 1, n):
                r = rng.random()
                if r < 0.06:
                    se.append((u, v))
                elif r < 0.06 + rng.choice([0.2, 0.35]):
                    ce.append((u, v))
        graphs.append(from_edges(n, ce, se))
    b = synth.concat(graphs)
    _check(b, k, 0.5, 300, expect_gate=0)
    _check(b, k, 0.1, 0, expect_gate=0)
