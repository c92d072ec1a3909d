"""The MPLD decomposition flow of PAPER.md §2.2 / Fig. 2, written plainly.

TEST INFRASTRUCTURE (see oracle/__init__.py): never imported by the product path.

decompose(G) = validate -> simplify (hide low-degree vertices) -> connected
components -> per-component exact-cover search (oracle/dlx.py) -> recover the
hidden vertices -> evaluate Eq. (1).  Readings R1..R10 are listed in DESIGN.md §2.
"""
from __future__ import annotations

import numpy as np

from .dlx import algorithm_x

# Eq. (1a) in integer cost units (R2): one conflict = W_CONF units,
# one stitch = round(alpha * W_CONF) units; alpha must be a multiple of 1/W_CONF.
W_CONF = 1000


def alpha_units(alpha: float) -> int:
    """§2.1 "alpha is a user-defined parameter ... set as 0.1 by default".
    Returns the stitch weight in cost units; raises for alpha outside
    [0, 1000] or not a multiple of 0.001 (R2)."""
    a = float(alpha) * W_CONF
    w = int(round(a))
    if not (0.0 <= alpha <= 1000.0) or abs(a - w) > 1e-6:
        raise ValueError(f"alpha={alpha!r} is not a multiple of 1/{W_CONF} in [0, 1000]")
    return w


def validate(g) -> None:
    """§2.1 "undirected layout graph G = {V, E}, E = {CE ∪ SE}": both edge sets
    symmetric, rows strictly ascending, no self loops, ids in range, CE ∩ SE = ∅."""
    n = g.n
    for name, rp, col in (("CE", g.ce_rowptr, g.ce_col), ("SE", g.se_rowptr, g.se_col)):
        if len(rp) != n + 1 or rp[0] != 0 or rp[-1] != len(col) or np.any(np.diff(rp) < 0):
            raise ValueError(f"{name}: bad row pointer")
        adj = [col[rp[v]:rp[v + 1]].tolist() for v in range(n)]
        for v in range(n):
            row = adj[v]
            for i, u in enumerate(row):
                if not (0 <= u < n) or u == v or (i and row[i - 1] >= u):
                    raise ValueError(f"{name}: row {v} not strictly ascending / self loop / out of range")
        es = {(v, u) for v in range(n) for u in adj[v]}
        if any((u, v) not in es for (v, u) in es):
            raise ValueError(f"{name}: not symmetric")
    ce = {(v, u) for v, u in zip(np.repeat(np.arange(n), np.diff(g.ce_rowptr)).tolist(), g.ce_col.tolist())}
    se = {(v, u) for v, u in zip(np.repeat(np.arange(n), np.diff(g.se_rowptr)).tolist(), g.se_col.tolist())}
    if ce & se:
        raise ValueError("CE and SE intersect")


def simplify(n: int, ce_adj, se_adj, k: int):
    """§2.2 "simplify the layout graph" (R8): in rounds r = 0, 1, ..., every
    not-yet-hidden vertex with no stitch edge whose conflict degree among
    not-yet-hidden vertices is < k is hidden, all at once.  Returns
    (hround[v] = round or -1 if kept, rounds = list of vertex lists)."""
    hidden = [False] * n
    hround = [-1] * n
    rounds = []
    while True:
        H = [v for v in range(n)
             if not hidden[v] and not se_adj[v]
             and sum(1 for u in ce_adj[v] if not hidden[u]) < k]
        if not H:
            break
        for v in H:
            hidden[v] = True
            hround[v] = len(rounds)
        rounds.append(H)
    return hround, rounds


def lowbias32(x: int) -> int:
    """Counter-based 32-bit integer mix (a bijection on [0, 2^32)) used as the
    recovery priority of R9; both sides implement it."""
    x &= 0xFFFFFFFF
    x ^= x >> 16
    x = (x * 0x7FEB352D) & 0xFFFFFFFF
    x ^= x >> 15
    x = (x * 0x846CA68B) & 0xFFFFFFFF
    x ^= x >> 16
    return x


def components(n: int, ce_adj, se_adj, hround):
    """Connected components of the kept vertices over CE ∪ SE (§2.2, Alg. 1
    lines 1-3 "the original DG will be decomposed into sub-graphs").  A
    component is listed in BFS order from its smallest vertex id, neighbours
    visited in ascending id (R5: "in BFS order of G"); components are returned
    in ascending order of that root."""
    seen = [False] * n
    comps = []
    for root in range(n):
        if hround[root] != -1 or seen[root]:
            continue
        seen[root] = True
        order = [root]
        i = 0
        while i < len(order):
            v = order[i]
            i += 1
            for u in sorted(ce_adj[v] + se_adj[v]):
                if hround[u] == -1 and not seen[u]:
                    seen[u] = True
                    order.append(u)
        comps.append(order)
    return comps


def solve_component(order, ce_adj, se_adj, k: int, w_stitch: int, max_steps: int = 0):
    """Build the exact-cover matrix of one component (columns = vertices in BFS
    order) and run the relaxed Algorithm X (oracle/dlx.py)."""
    loc = {v: i for i, v in enumerate(order)}
    n = len(order)
    ce_edges = sorted({(min(loc[v], loc[u]), max(loc[v], loc[u]))
                       for v in order for u in ce_adj[v] if u in loc})
    s_adj = [[loc[u] for u in se_adj[v] if u in loc] for v in order]
    res = algorithm_x(n, k, ce_edges, s_adj, W_CONF, w_stitch, max_steps)
    res["global_colors"] = {order[i]: c for i, c in enumerate(res["colors"])}
    return res


def recover(n: int, ce_adj, rounds, colors, k: int, layout_offsets=None):
    """§2.2 "the framework will recover the nodes removed in simplification step
    and assigns the coloring results": the hidden vertices are popped LIFO —
    rounds in reverse, inside a round in descending priority
    lowbias32(layout-local id) (R9) — and each takes the smallest mask not used
    by an already-coloured conflict neighbour.  Mutates and returns colors."""
    offs = [0, n] if layout_offsets is None else [int(x) for x in layout_offsets]
    base = [0] * n
    for li in range(len(offs) - 1):
        for v in range(offs[li], offs[li + 1]):
            base[v] = offs[li]
    for H in reversed(rounds):
        for v in sorted(H, key=lambda v: lowbias32(v - base[v]), reverse=True):
            used = {colors[u] for u in ce_adj[v] if colors[u] >= 0}
            c = 0
            while c in used:
                c += 1
            assert c < k, "simplification invariant broken"
            colors[v] = c
    return colors


def evaluate(colors, ce_edges, se_edges):
    """Eq. (1b)/(1c): conflicts = #{e_ij in CE : x_i == x_j},
    stitches = #{e_ij in SE : x_i != x_j}."""
    n_conf = sum(1 for u, v in ce_edges if colors[u] == colors[v])
    n_st = sum(1 for u, v in se_edges if colors[u] != colors[v])
    return n_conf, n_st


def decompose(g, k: int, alpha: float, max_steps: int = 0, check: bool = True):
    """Fig. 2 flow on one DecompGraph (possibly a batch of concatenated layouts).
    Returns a dict with colors (np.int32[n]), n_conflicts, n_stitches, cost
    (= n_conflicts + alpha * n_stitches, Eq. 1a), per-layout triples and the
    per-component results."""
    if not (2 <= k <= 4):
        raise ValueError("k must be in [2, 4]")
    w_st = alpha_units(alpha)
    if check:
        validate(g)
    n = g.n
    ce_adj, se_adj = g.ce_adj(), g.se_adj()
    hround, rounds = simplify(n, ce_adj, se_adj, k)
    comps = components(n, ce_adj, se_adj, hround)
    colors = [-1] * n
    comp_res = []
    for order in comps:
        r = solve_component(order, ce_adj, se_adj, k, w_st, max_steps)
        for v, c in r["global_colors"].items():
            colors[v] = c
        comp_res.append({"root": order[0], "size": len(order), "cost_units": r["cost"],
                         "n_conf": r["n_conf"], "n_stitch": r["n_stitch"],
                         "steps": r["steps"], "truncated": r["truncated"]})
    recover(n, ce_adj, rounds, colors, k, g.layout_offsets)
    ce_e = g.ce_edges().tolist()
    se_e = g.se_edges().tolist()
    n_conf, n_st = evaluate(colors, ce_e, se_e)
    per_layout = []
    offs = g.layout_offsets.tolist()
    for li in range(len(offs) - 1):
        a, b = offs[li], offs[li + 1]
        c1 = sum(1 for u, v in ce_e if a <= u < b and colors[u] == colors[v])
        s1 = sum(1 for u, v in se_e if a <= u < b and colors[u] != colors[v])
        per_layout.append((c1, s1, c1 + alpha * s1))
    return {"colors": np.array(colors, dtype=np.int32), "n_conflicts": n_conf, "n_stitches": n_st,
            "cost": n_conf + alpha * n_st, "per_layout": per_layout, "components": comp_res,
            "hround": np.array(hround, dtype=np.int32), "n_rounds": len(rounds)}
