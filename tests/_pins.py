"""Independent checkers used to pin the oracle (test code, not oracle code).

* `eq1` evaluates PAPER.md Eq. (1) from a colouring with exact rationals.
* `brute_force` enumerates all k^n colourings (the plain definition of the
  optimum of Eq. 1).
* `canonical_leaves` enumerates, WITHOUT any pruning, budget or dancing links,
  the leaves of the search tree DESIGN.md R4-R6 define (column rule of Alg. 1
  line 8, rows in index order), so the first minimum-cost leaf can be compared
  with the oracle's branch-and-bound answer colour by colour.
"""
from __future__ import annotations

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
