"""Independent checkers used to pin the oracle (test code, not oracle code).

* `eq1` evaluates PAPER.md Eq. (1) from a colouring with exact rationals.
* `brute_force` enumerates all k^n colourings (the plain definition of the
  optimum of Eq. 1).
* `bfs_components` lists the components of a graph in the column order of
  DESIGN.md R5 with its own queue (collections.deque), for the pins that need
  the order without trusting oracle.components.
* `canonical_leaves` enumerates, WITHOUT any pruning, budget or dancing links,
  the leaves of the search tree DESIGN.md R4-R6 define (column rule of Alg. 1
  line 8, rows in index order), so the first minimum-cost leaf can be compared
  with the oracle's branch-and-bound answer colour by colour.
"""
from __future__ import annotations

import collections
import itertools
import random
from fractions import Fraction


def eq1(colors, ce, se, alpha: Fraction):
    conf = sum(1 for u, v in ce if colors[u] == colors[v])
    st = sum(1 for u, v in se if colors[u] != colors[v])
    return conf + alpha * st, conf, st


def brute_force(n, ce, se, k, alpha: Fraction):
    best, arg = None, []
    for col in itertools.product(range(k), repeat=n):
        c, _, _ = eq1(col, ce, se, alpha)
        if best is None or c < best:
            best, arg = c, [col]
        elif c == best:
            arg.append(col)
    return best, arg


def canonical_leaves(n, ce, k, symmetry_rule=True):
    adj = [[] for _ in range(n)]
    for u, v in ce:
        adj[u].append(v)
        adj[v].append(u)
    colors = [-1] * n
    out = []

    def rec(maxused):
        unc = [v for v in range(n) if colors[v] < 0]
        if not unc:
            out.append(tuple(colors))
            return
        live = {v: sum(1 for c in range(k) if all(colors[u] != c for u in adj[v])) for v in unc}
        zero = [v for v in unc if live[v] == 0]
        one = [v for v in unc if live[v] == 1]
        v = zero[0] if zero else (one[0] if one else unc[0])
        lim = min(k, maxused + 2) if symmetry_rule else k
        for c in range(lim):
            colors[v] = c
            rec(max(maxused, c))
            colors[v] = -1

    rec(-1)
    return out


def first_optimal_leaf(n, ce, se, k, alpha, symmetry_rule=True):
    leaves = canonical_leaves(n, ce, k, symmetry_rule)
    costs = [eq1(lf, ce, se, alpha)[0] for lf in leaves]
    m = min(costs)
    return leaves[costs.index(m)], m, leaves


def random_graph(rng: random.Random, n, p_ce, p_se=0.0):
    ce, se = [], []
    for u in range(n):
        for v in range(u + 1, n):
            r = rng.random()
            if r < p_se:
                se.append((u, v))
            elif r < p_se + p_ce:
                ce.append((u, v))
    return ce, se


def bfs_components(n, ce, se):
    """Components over CE ∪ SE, each in BFS order from its smallest vertex with
    neighbours in ascending id (R5), listed by ascending root."""
    nb = [set() for _ in range(n)]
    for u, v in list(ce) + list(se):
        nb[u].add(v)
        nb[v].add(u)
    seen = [False] * n
    out = []
    for r in range(n):
        if seen[r]:
            continue
        seen[r] = True
        q, order = collections.deque([r]), []
        while q:
            v = q.popleft()
            order.append(v)
            for u in sorted(nb[v]):
                if not seen[u]:
                    seen[u] = True
                    q.append(u)
        out.append(order)
    return out


def raw_graph(n, ce_rows, se_rows, layout_offsets=None):
    """A DecompGraph from explicit rows (may violate the CSR invariants on purpose)."""
    import numpy as np
    from synth.graph import DecompGraph

    def csr(rows):
        rp = np.zeros(n + 1, dtype=np.int32)
        rp[1:] = np.cumsum([len(r) for r in rows])
        col = np.array([u for r in rows for u in r], dtype=np.int32)
        return rp, col

    crp, ccol = csr(ce_rows)
    srp, scol = csr(se_rows)
    g = DecompGraph(n, crp, ccol, srp, scol)
    if layout_offsets is not None:
        g.layout_offsets = np.array(layout_offsets, dtype=np.int32)
    return g


# valid reference: path 0-1-2-3 in CE, stitch 3-4; then one violation of the
# CSR invariants of include/mpld.h per case (rows, symmetry, ids, CE ∩ SE)
GOOD_CE = [[1], [0, 2], [1, 3], [2], []]
GOOD_SE = [[], [], [], [4], [3]]
BAD_GRAPHS = {
    "asymmetric_ce": ([[1], [0, 2], [1, 3], [], []], GOOD_SE, None),
    "asymmetric_se": (GOOD_CE, [[], [], [], [4], []], None),
    "unsorted_row": ([[1], [2, 0], [1, 3], [2], []], GOOD_SE, None),
    "duplicate_entry": ([[1, 1], [0, 0, 2], [1, 3], [2], []], GOOD_SE, None),
    "self_loop": ([[1], [0, 2], [1, 2, 3], [2], []], GOOD_SE, None),
    "id_out_of_range": ([[1, 5], [0, 2], [1, 3], [2], []], GOOD_SE, None),
    "negative_id": ([[-1, 1], [0, 2], [1, 3], [2], []], GOOD_SE, None),
    "ce_and_se_overlap": (GOOD_CE, [[], [], [3], [2, 4], [3]], None),
    "layout_offsets_unsorted": (GOOD_CE, GOOD_SE, [0, 4, 2, 5]),
    "layout_offsets_short": (GOOD_CE, GOOD_SE, [0, 4]),  # rejected by the host entry point (MPLD_ERR_ARG)
}
