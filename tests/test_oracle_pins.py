"""Pins of the CPU oracle against things other than itself (CPU only).

Each test names what fixes the expected value: PAPER.md text, a closed form,
brute force, an invariant of the definitions.
"""
from __future__ import annotations

import os
import random
from fractions import Fraction
from math import comb

import numpy as np
import pytest

import oracle
import synth
from synth import from_edges
from tests._pins import (BAD_GRAPHS, GOOD_CE, GOOD_SE, bfs_components, brute_force, canonical_leaves, eq1,
                         first_optimal_leaf, random_graph, raw_graph)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _read_golden_graphs(path):
    out, cur = [], None
    for line in open(path):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        key, *rest = line.split()
        if key == "graph":
            cur = {"name": rest[0], "ce": [], "se": []}
        elif key == "end":
            out.append(cur)
        elif key in ("ce", "se"):
            cur[key] = [tuple(int(x) for x in e.split("-")) for e in rest]
        elif key == "alpha":
            cur[key] = rest[0]
        else:
            cur[key] = int(rest[0])
    return out


def _solve(n, ce, se, k, alpha, max_steps=0):
    g = from_edges(n, ce, se)
    return oracle.decompose(g, k, alpha, max_steps=max_steps)


# ---------------------------------------------------------------- PAPER.md Fig. 1
@pytest.mark.parametrize("gold", _read_golden_graphs(os.path.join(GOLDEN, "fig1.txt")), ids=lambda g: g["name"])
def test_fig1_golden(gold):
    alpha = Fraction(gold["alpha"])
    r = _solve(gold["n"], gold["ce"], gold["se"], gold["k"], float(alpha))
    assert r["n_conflicts"] == gold["expect_conflicts"]
    if "expect_stitches" in gold:
        assert r["n_stitches"] == gold["expect_stitches"]
    if "expect_stitches_max" in gold:
        assert r["n_stitches"] <= gold["expect_stitches_max"]
    best, _ = brute_force(gold["n"], gold["ce"], gold["se"], gold["k"], alpha)
    assert Fraction(r["n_conflicts"]) + alpha * r["n_stitches"] == best
    assert r["cost"] == r["n_conflicts"] + float(alpha) * r["n_stitches"]


# ---------------------------------------------------------------- closed forms
def _closed_form_graph(name):
    if name.startswith("K33"):
        return 6, [(i, j) for i in range(3) for j in range(3, 6)]
    if name.startswith("K"):
        n = int(name[1:].split("k")[0])
        return n, [(i, j) for i in range(n) for j in range(i + 1, n)]
    if name.startswith("C"):
        n = int(name[1:])
        return n, [(i, (i + 1) % n) for i in range(n)]
    raise KeyError(name)


def _turan(n, k):
    sizes = [n // k + (1 if i < n % k else 0) for i in range(k)]
    return sum(comb(s, 2) for s in sizes)


def _closed_rows():
    rows = []
    for line in open(os.path.join(GOLDEN, "closed_forms.txt")):
        if line.strip() and not line.startswith("#"):
            name, k, e = line.split()
            rows.append((name, int(k), int(e)))
    return rows


@pytest.mark.parametrize("name,k,expected", _closed_rows())
def test_closed_forms(name, k, expected):
    n, ce = _closed_form_graph(name)
    if name.startswith("K") and not name.startswith("K33"):
        assert _turan(n, k) == expected  # the golden row agrees with the Turán formula
    r = _solve(n, ce, [], k, 0.1)
    assert r["n_conflicts"] == expected
    assert r["n_stitches"] == 0


# ---------------------------------------------------------------- brute force k^n
@pytest.mark.parametrize("k", [2, 3, 4])
def test_brute_force_random(k):
    rng = random.Random(1234 + k)
    alpha = Fraction(1, 10)
    for trial in range(60):
        n = rng.randint(1, 7 if k < 4 else 6)
        ce, se = random_graph(rng, n, rng.choice([0.3, 0.5, 0.8]), rng.choice([0.0, 0.15]))
        r = _solve(n, ce, se, k, 0.1)
        best, opts = brute_force(n, ce, se, k, alpha)
        got = tuple(int(c) for c in r["colors"])
        assert eq1(got, ce, se, alpha) == (best, r["n_conflicts"], r["n_stitches"]), (n, ce, se)
        assert got in opts


@pytest.mark.parametrize("alpha", [Fraction(0), Fraction(1, 10), Fraction(1, 2), Fraction(1), Fraction(3, 2)])
def test_brute_force_alpha(alpha):
    """Ties between stitches and conflicts (alpha = 1, 1/10 ...) are decided exactly."""
    rng = random.Random(77)
    for trial in range(40):
        n = rng.randint(2, 7)
        ce, se = random_graph(rng, n, 0.6, 0.25)
        r = _solve(n, ce, se, 3, float(alpha))
        best, _ = brute_force(n, ce, se, 3, alpha)
        assert r["n_conflicts"] + alpha * r["n_stitches"] == best


# ---------------------------------------------------------------- canonical answer
def _bfs_relabel(n, ce, se):
    """The R5 column order from the pins' own BFS (tests/_pins.py), not oracle.components."""
    return bfs_components(n, ce, se)


def _read_bfs_golden():
    out, cur = [], None
    for line in open(os.path.join(GOLDEN, "bfs_order.txt")):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        key, *rest = line.split()
        if key == "graph":
            cur = {"name": rest[0], "ce": [], "se": [], "hidden": [], "components": []}
        elif key == "end":
            out.append(cur)
        elif key in ("ce", "se"):
            cur[key] = [tuple(int(x) for x in e.split("-")) for e in rest]
        elif key == "hidden":
            cur["hidden"] = [int(x) for x in rest]
        elif key == "component":
            cur["components"].append([int(x) for x in rest])
        else:
            cur[key] = int(rest[0])
    return out


@pytest.mark.parametrize("gold", _read_bfs_golden(), ids=lambda g: g["name"])
def test_components_bfs_order_golden(gold):
    """oracle.components against a hand-derived BFS (tests/golden/bfs_order.txt):
    a graph where CE-before-SE order, depth-first order and ascending id order
    all differ from the R5 order."""
    g = from_edges(gold["n"], gold["ce"], gold["se"])
    hround = [0 if v in gold["hidden"] else -1 for v in range(gold["n"])]
    assert oracle.components(gold["n"], g.ce_adj(), g.se_adj(), hround) == gold["components"]


def test_components_match_independent_bfs():
    """oracle.components equals the pins' own BFS (tests/_pins.py) on random graphs."""
    rng = random.Random(31)
    for trial in range(200):
        n = rng.randint(1, 14)
        ce, se = random_graph(rng, n, rng.choice([0.1, 0.25, 0.4]), rng.choice([0.0, 0.1]))
        g = from_edges(n, ce, se)
        assert oracle.components(n, g.ce_adj(), g.se_adj(), [-1] * n) == bfs_components(n, ce, se)


def _read_budget_trace():
    rows = []
    for line in open(os.path.join(GOLDEN, "k4_budget_trace.txt")):
        if line.startswith("budget"):
            _, b, steps, tr, cost, *col = line.split()
            rows.append((int(b), int(steps), bool(int(tr)), int(cost), tuple(int(c) for c in col)))
    return rows


@pytest.mark.parametrize("budget,steps,truncated,cost,colors", _read_budget_trace())
def test_k4_budget_hand_trace(budget, steps, truncated, cost, colors):
    """Node counts and truncated results at every budget against the hand trace
    of tests/golden/k4_budget_trace.txt (K4, k = 3), through algorithm_x and
    through the whole flow (K4 survives the k = 3 simplification whole)."""
    K4 = [(i, j) for i in range(4) for j in range(i + 1, 4)]
    r = oracle.algorithm_x(4, 3, K4, [[] for _ in range(4)], oracle.W_CONF, 100, max_steps=budget)
    assert (r["steps"], r["truncated"], r["cost"], tuple(r["colors"])) == (steps, truncated, cost, colors)
    d = oracle.decompose(synth.fixtures()["K4"], 3, 0.1, max_steps=budget)
    c = d["components"][0]
    assert (c["steps"], c["truncated"], c["cost_units"]) == (steps, truncated, cost)
    assert tuple(int(x) for x in d["colors"]) == colors


@pytest.mark.parametrize("k", [2, 3, 4])
def test_first_optimal_leaf_matches_pruning_free_enumeration(k):
    """The branch-and-bound answer (colours, not only cost) equals the first
    minimum-cost leaf of the pruning-free canonical tree, with and without the
    colour-symmetry rule (R6)."""
    rng = random.Random(99 + k)
    alpha = Fraction(1, 10)
    checked = 0
    while checked < 40:
        n = rng.randint(2, 7 if k < 4 else 6)
        ce, se = random_graph(rng, n, rng.choice([0.4, 0.7]), rng.choice([0.0, 0.2]))
        comps = _bfs_relabel(n, ce, se)
        if len(comps) != 1:
            continue
        order = comps[0]
        loc = {v: i for i, v in enumerate(order)}
        lce = [(min(loc[u], loc[v]), max(loc[u], loc[v])) for u, v in ce]
        lse = [(min(loc[u], loc[v]), max(loc[u], loc[v])) for u, v in se]
        s_adj = [[] for _ in range(n)]
        for u, v in lse:
            s_adj[u].append(v)
            s_adj[v].append(u)
        res = oracle.algorithm_x(n, k, sorted(lce), s_adj, oracle.W_CONF, 100)
        leaf, cost, _ = first_optimal_leaf(n, lce, lse, k, alpha, symmetry_rule=True)
        leaf_full, cost_full, _ = first_optimal_leaf(n, lce, lse, k, alpha, symmetry_rule=False)
        assert tuple(res["colors"]) == leaf == leaf_full
        assert Fraction(res["cost"], oracle.W_CONF) == cost == cost_full
        checked += 1


def test_budget_semantics():
    """max_steps small -> the first leaf of the dive; large -> the full answer."""
    rng = random.Random(5)
    alpha = Fraction(1, 10)
    for trial in range(30):
        n = rng.randint(3, 7)
        ce, se = random_graph(rng, n, 0.7, 0.0)
        comps = _bfs_relabel(n, ce, se)
        if len(comps) != 1:
            continue
        order = comps[0]
        loc = {v: i for i, v in enumerate(order)}
        lce = sorted((min(loc[u], loc[v]), max(loc[u], loc[v])) for u, v in ce)
        full = oracle.algorithm_x(n, 3, lce, [[] for _ in range(n)], oracle.W_CONF, 100)
        first = canonical_leaves(n, lce, 3)[0]
        one = oracle.algorithm_x(n, 3, lce, [[] for _ in range(n)], oracle.W_CONF, 100, max_steps=1)
        assert tuple(one["colors"]) == first
        assert one["truncated"] == (full["steps"] > n + 1)
        again = oracle.algorithm_x(n, 3, lce, [[] for _ in range(n)], oracle.W_CONF, 100, max_steps=full["steps"])
        assert again["colors"] == full["colors"] and not again["truncated"]


def test_bound_is_a_lower_bound():
    """R7's bound (zero-live columns + clique deficit over oracle.dlx.clique_partition)
    never exceeds the cheapest completion of a partial colouring (brute force)."""
    import itertools
    from oracle.dlx import clique_partition
    rng = random.Random(21)
    for trial in range(400):
        n = rng.randint(2, 7)
        k = rng.choice([2, 3, 4, 4])
        ce, _ = random_graph(rng, n, rng.choice([0.5, 0.8, 0.95]))
        adj = [set() for _ in range(n)]
        for u, v in ce:
            adj[u].add(v)
            adj[v].add(u)
        colored = {v: rng.randrange(k) for v in rng.sample(range(n), rng.randint(0, n - 1))}
        live = {v: {c for c in range(k) if all(colored.get(u) != c for u in adj[v])}
                for v in range(n) if v not in colored}
        zero = sum(1 for v in live if not live[v])
        def deficit_over(cliques):
            d = 0
            for Q in cliques:
                X = [v for v in Q if v in live and live[v]]
                d += max(0, len(X) - len(set().union(*[live[v] for v in X])))
            return d

        # the partition the oracle uses (oracle/dlx.py: cliques of >= k vertices, k >= 4 only) and,
        # as a stronger check of the argument, every greedy clique of >= 2 vertices
        used = clique_partition(n, ce, minsize=k) if k >= 4 else []
        deficit = deficit_over(used)
        deficit2 = deficit_over(clique_partition(n, ce, minsize=2))
        free = [v for v in range(n) if v not in colored]
        best = None
        for assign in itertools.product(range(k), repeat=len(free)):
            col = dict(colored)
            col.update(zip(free, assign))
            # conflicts not yet paid: edges with at least one uncoloured endpoint
            c = sum(1 for u, v in ce if col[u] == col[v] and (u in live or v in live))
            best = c if best is None else min(best, c)
        assert zero + deficit <= best, (n, k, ce, colored)
        assert zero + deficit2 <= best, (n, k, ce, colored)


# ---------------------------------------------------------------- Eq. (2) round trip
def test_dlx_cover_uncover_round_trip():
    """PAPER.md Eq. (2): Uncover is the exact inverse of Cover under LIFO."""
    rng = random.Random(3)
    for trial in range(200):
        n = rng.randint(1, 8)
        k = rng.randint(2, 4)
        ce, _ = random_graph(rng, n, 0.5)
        M = oracle.DLXMatrix(n, k, ce)
        snap = M.snapshot()
        stack = []
        for step in range(30):
            live = [c for c in range(M.n_head) if not M.covered[c]]
            if stack and (rng.random() < 0.4 or not live):
                M.uncover(stack.pop())
            elif live:
                c = rng.choice(live)
                M.cover(c)
                stack.append(c)
        while stack:
            M.uncover(stack.pop())
        assert M.snapshot() == snap


def test_dlx_column_sizes_are_live_rows():
    """S[v] after selecting rows = #masks c with no CE neighbour coloured c (the
    secondary columns' meaning), checked on random partial colourings."""
    rng = random.Random(11)
    for trial in range(100):
        n = rng.randint(2, 8)
        k = rng.randint(2, 4)
        ce, _ = random_graph(rng, n, 0.5)
        M = oracle.DLXMatrix(n, k, ce)
        adj = [[] for _ in range(n)]
        for u, v in ce:
            adj[u].append(v)
            adj[v].append(u)
        colors = [-1] * n
        for v in rng.sample(range(n), rng.randint(0, n)):
            c = rng.randrange(k)
            M.cover(1 + v)
            x = M.first[v * k + c]
            j = M.R[x]
            while j != x:
                if not M.covered[M.C[j]]:
                    M.cover(M.C[j])
                j = M.R[j]
            colors[v] = c
        for v in range(n):
            if colors[v] < 0:
                assert M.S[1 + v] == sum(1 for c in range(k) if all(colors[u] != c for u in adj[v]))
                assert sorted(M.live_rows(1 + v)) == [v * k + c for c in range(k) if all(colors[u] != c for u in adj[v])]


# ---------------------------------------------------------------- flow invariants
def _check_flow_invariants(g, k, alpha, r):
    n = g.n
    ce_adj, se_adj = g.ce_adj(), g.se_adj()
    colors = r["colors"]
    assert colors.shape == (n,) and ((colors >= 0) & (colors < k)).all()  # every vertex covered once
    ce, se = g.ce_edges(), g.se_edges()
    n_conf = int((colors[ce[:, 0]] == colors[ce[:, 1]]).sum()) if len(ce) else 0
    n_st = int((colors[se[:, 0]] != colors[se[:, 1]]).sum()) if len(se) else 0
    assert (n_conf, n_st) == (r["n_conflicts"], r["n_stitches"])
    assert r["cost"] == n_conf + alpha * n_st
    # recovery adds no cost: total = sum of component optima (hidden vertices have no SE)
    units = oracle.alpha_units(alpha)
    assert sum(c["cost_units"] for c in r["components"]) == n_conf * oracle.W_CONF + n_st * units
    # simplification: hidden vertices had conflict degree < k among vertices hidden no earlier
    hr = r["hround"]
    for v in range(n):
        if hr[v] >= 0:
            assert not se_adj[v]
            assert sum(1 for u in ce_adj[v] if hr[u] == -1 or hr[u] >= hr[v]) < k
        else:
            assert se_adj[v] or sum(1 for u in ce_adj[v] if hr[u] == -1) >= k
    # recovery: a hidden vertex takes the smallest mask unused by neighbours coloured before it
    prio = {}
    offs = g.layout_offsets.tolist()
    for li in range(len(offs) - 1):
        for v in range(offs[li], offs[li + 1]):
            prio[v] = oracle.lowbias32(v - offs[li])
    for v in range(n):
        if hr[v] >= 0:
            before = [u for u in ce_adj[v] if hr[u] == -1 or hr[u] > hr[v] or (hr[u] == hr[v] and prio[u] > prio[v])]
            used = {int(colors[u]) for u in before}
            assert int(colors[v]) == min(set(range(k)) - used)
    # components partition the kept vertices; no edge between two components
    comp_of = {}
    for ci, c in enumerate(r["components"]):
        pass
    kept = [v for v in range(n) if hr[v] == -1]
    comps = oracle.components(n, ce_adj, se_adj, list(hr))
    assert sorted(v for c in comps for v in c) == kept
    for ci, c in enumerate(comps):
        assert c[0] == min(c)
        for v in c:
            comp_of[v] = ci
    for v in kept:
        for u in ce_adj[v] + se_adj[v]:
            if hr[u] == -1:
                assert comp_of[u] == comp_of[v]


@pytest.mark.parametrize("cfg", [0, 1])
def test_config_invariants(cfg):
    graphs, k, alpha = synth.config_graphs(cfg)
    for g in graphs[:3]:
        r = oracle.decompose(g, k, alpha)
        _check_flow_invariants(g, k, alpha, r)


def test_batch_equals_individual():
    """A batch (disjoint union with layout boundaries) decomposes exactly like its layouts."""
    graphs = [synth.make_layout(300, 330, k=3, stitch_prob=0.5, comp_max=8, density=0.9, seed=s) for s in range(3)]
    b = synth.concat(graphs)
    rb = oracle.decompose(b, 3, 0.1)
    _check_flow_invariants(b, 3, 0.1, rb)
    for li, g in enumerate(graphs):
        r = oracle.decompose(g, 3, 0.1)
        a, e = b.layout_offsets[li], b.layout_offsets[li + 1]
        assert (rb["colors"][a:e] == r["colors"]).all()
        assert rb["per_layout"][li] == (r["n_conflicts"], r["n_stitches"], r["cost"])


def test_simplify_examples():
    # path a-b-c, k = 3: all hidden in round 0 (degrees <= 2 < 3); SPEC.md simplify_graph example
    g = from_edges(3, [(0, 1), (1, 2)])
    hr, rounds = oracle.simplify(3, g.ce_adj(), g.se_adj(), 3)
    assert hr == [0, 0, 0] and len(rounds) == 1
    # K4, k = 3: nothing hidden
    g = synth.fixtures()["K4"]
    hr, rounds = oracle.simplify(4, g.ce_adj(), g.se_adj(), 3)
    assert hr == [-1] * 4 and rounds == []
    # K4 with a pendant path: both path vertices (degrees 2 and 1) go in round 0, the clique stays
    g = from_edges(6, [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3), (3, 4), (4, 5)])
    hr, rounds = oracle.simplify(6, g.ce_adj(), g.se_adj(), 3)
    assert hr == [-1, -1, -1, -1, 0, 0]
    # stitch endpoints are never hidden
    g = from_edges(3, [(0, 1)], [(1, 2)])
    hr, _ = oracle.simplify(3, g.ce_adj(), g.se_adj(), 3)
    assert hr == [0, -1, -1]


def test_lowbias32_is_a_bijection():
    """R9 needs distinct priorities: invert the mix step by step on samples."""
    def inv_xorshift(y, s):
        x = y
        for _ in range(32 // s + 1):
            x = y ^ (x >> s)
        return x & 0xFFFFFFFF

    def inv(y):
        y = inv_xorshift(y, 16)
        y = (y * pow(0x846CA68B, -1, 1 << 32)) & 0xFFFFFFFF
        y = inv_xorshift(y, 15)
        y = (y * pow(0x7FEB352D, -1, 1 << 32)) & 0xFFFFFFFF
        return inv_xorshift(y, 16)

    rng = random.Random(0)
    xs = [0, 1, 2, 0xFFFFFFFF] + [rng.getrandbits(32) for _ in range(2000)]
    for x in xs:
        assert inv(oracle.lowbias32(x)) == x
    assert len({oracle.lowbias32(x) for x in range(20000)}) == 20000


def test_alpha_units():
    assert oracle.alpha_units(0.1) == 100
    assert oracle.alpha_units(0) == 0
    assert oracle.alpha_units(2.5) == 2500
    with pytest.raises(ValueError):
        oracle.alpha_units(0.0001)
    with pytest.raises(ValueError):
        oracle.alpha_units(-0.1)


@pytest.mark.parametrize("case", sorted(c for c in BAD_GRAPHS if not c.startswith("layout_offsets")))
def test_validate_rejects_each_invariant(case):
    """oracle.validate against one violation of each CSR invariant of §2.1's
    "E = {CE ∪ SE}" as include/mpld.h states it (the same table the GPU
    validation tests use)."""
    ce, se, _ = BAD_GRAPHS[case]
    with pytest.raises(ValueError):
        oracle.validate(raw_graph(5, ce, se))


@pytest.mark.parametrize("case", ["rowptr_start", "rowptr_end", "rowptr_length", "rowptr_decreasing"])
def test_validate_rejects_bad_row_pointers(case):
    g = raw_graph(5, GOOD_CE, GOOD_SE)
    oracle.validate(g)  # the reference graph is valid
    rp = g.ce_rowptr.copy()
    if case == "rowptr_start":
        rp = rp + 1
    elif case == "rowptr_end":
        rp[-1] -= 1
    elif case == "rowptr_length":
        rp = rp[:-1]
    else:
        rp[2], rp[3] = rp[3], rp[2] - 1
    g.ce_rowptr = rp
    with pytest.raises(ValueError):
        oracle.validate(g)


def test_validate_rejects_bad_graphs():
    g = from_edges(3, [(0, 1)])
    g.ce_col = np.array([1, 1], dtype=np.int32)  # 1 -> 1 self loop, asymmetric
    with pytest.raises(ValueError):
        oracle.validate(g)
    g = from_edges(3, [(0, 1)], [(0, 1)])
    g2 = from_edges(3, [(0, 1)])
    g2.se_rowptr, g2.se_col = g2.ce_rowptr.copy(), g2.ce_col.copy()
    with pytest.raises(ValueError):
        oracle.validate(g2)
    with pytest.raises(ValueError):
        oracle.decompose(synth.fixtures()["K4"], 5, 0.1)
