"""Pins of the lower bound the exact-mode (heavy) search prunes with (CPU only).

Exact mode returns the canonical optimum of R7 whatever valid lower bound
prunes the tree, so the warp-parallel search adds a term to
R7's: a matching of adjacent uncovered columns whose only live row has the
same mask (each such pair costs at least one more conflict: either one of the
two takes a blocked row — a conflict with an already-coloured neighbour — or
both take the live one — the conflict on their own edge), the clique deficit
of R7 taken over the cliques' columns outside the matching.  The charged edge
sets are disjoint, so the sum is a lower bound.  Here the bound is written out
as the kernel computes it (kernel_search.cu warp_heavy_search) and checked
against brute force over every completion of random partial colourings.
"""
from __future__ import annotations

import itertools
import random

import pytest

from oracle.dlx import clique_partition
from tests._pins import random_graph


def exact_mode_bound(n, k, adj, colored):
    """#zero-live columns + greedy same-mask single-live matching (masks in
    order, columns ascending) + clique deficit over the cliques of >= k
    vertices (k >= 4) outside the matching, in conflicts."""
    ce = [(u, v) for u in range(n) for v in adj[u] if u < v]
    live = {v: {c for c in range(k) if all(colored.get(u) != c for u in adj[v])}
            for v in range(n) if v not in colored}
    zero = sum(1 for v in live if not live[v])
    matched, pairs = set(), 0
    for c in range(k):
        S = [v for v in sorted(live) if live[v] == {c}]
        T = list(S)
        while T:
            x = T.pop(0)
            N = sorted(u for u in adj[x] if u in S and u not in matched)
            if N:
                matched |= {x, N[0]}
                T = [t for t in T if t != N[0]]
                pairs += 1
    deficit = 0
    for Q in (clique_partition(n, ce, minsize=k) if k >= 4 else []):
        X = [v for v in Q if v in live and live[v] and v not in matched]
        deficit += max(0, len(X) - len(set().union(*[live[v] for v in X])))
    return zero + pairs + deficit


def cheapest_completion(n, k, adj, colored):
    """Brute force: fewest conflicts on edges with an uncoloured end."""
    free = [v for v in range(n) if v not in colored]
    ce = [(u, v) for u in range(n) for v in adj[u] if u < v and (u in free or v in free)]
    best = None
    for a in itertools.product(range(k), repeat=len(free)):
        col = dict(colored)
        col.update(zip(free, a))
        c = sum(1 for u, v in ce if col[u] == col[v])
        best = c if best is None else min(best, c)
    return best


@pytest.mark.parametrize("k", [2, 3, 4])
def test_exact_mode_bound_is_a_lower_bound(k):
    rng = random.Random(71 + k)
    tight = 0
    for trial in range(500):
        n = rng.randint(2, 8 if k < 4 else 7)
        ce, _ = random_graph(rng, n, rng.choice([0.4, 0.6, 0.9]))
        adj = [set() for _ in range(n)]
        for u, v in ce:
            adj[u].add(v)
            adj[v].add(u)
        colored = {v: rng.randrange(k) for v in rng.sample(range(n), rng.randint(0, n - 1))}
        lb = exact_mode_bound(n, k, adj, colored)
        best = cheapest_completion(n, k, adj, colored)
        assert lb <= best, (n, k, ce, colored, lb, best)
        tight += lb == best and lb > 0
    assert tight > 0  # the bound is not vacuous


def test_pair_term_example():
    """Path 0 - 1 - 2 - 3 with k = 2: colouring 0 with mask 0 and 3 with mask 1
    leaves 1 and 2 each with the single live mask 1 and 0 respectively: no pair
    (different masks), bound 0, and indeed 0-1-2-3 = 0,1,0,1 costs nothing.
    Colouring 3 with mask 0 instead leaves both 1 and 2 with mask 1 only: one
    pair, bound 1 = the cheapest completion."""
    adj = [{1}, {0, 2}, {1, 3}, {2}]
    assert exact_mode_bound(4, 2, adj, {0: 0, 3: 1}) == 0 == cheapest_completion(4, 2, adj, {0: 0, 3: 1})
    assert exact_mode_bound(4, 2, adj, {0: 0, 3: 0}) == 1 == cheapest_completion(4, 2, adj, {0: 0, 3: 0})
