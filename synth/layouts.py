"""Seeded synthetic decomposed graphs shaped like the paper's ISCAS benchmarks.

Recipe (restated in DESIGN.md §3 "Input recipe"):

* PAPER.md Table 1 gives, per ISCAS circuit, |V| and a second count we read as
  |E| (both columns are labelled "|V|"; SPEC.md layout_io "Open Questions"
  flags the same).  A synthetic layout for a circuit has exactly that |V| and
  an |E| within a few edges of the second count.
* Layout graphs are unit-disk-like (features within the minimum colouring
  spacing conflict, §2.1).  We emit two kinds of pieces, each on consecutive
  vertex ids (layout scan order locality):
    - *clusters* (dense regions: contact arrays, cell rows) — s points uniform in
      a square of side sqrt(s/density), a CE edge whenever two points are closer
      than 1 (the spacing).  Only these survive the low-degree simplification.
      configs[2] (QPLD, k = 4) draws 3/4 of its clusters as *lattice clusters*
      instead: track-aligned features on a jittered square lattice of pitch
      0.68 (jitter +-0.15), near-planar graphs whose k = 4 cores reach ~40
      vertices; its random clusters use density 1.0 (at 1.2, about one cluster
      in 500 has a sequential search of > 10^8 nodes at k = 4).
      Stitch candidates (Fig. 1(c)): a cluster vertex of conflict degree >= k is,
      with probability `stitch_prob`, split into two segments joined by an SE
      edge; neighbours left of its x-coordinate stay on segment 0, the rest move
      to segment 1 (no split if either side would be empty).
    - *wires* — chains of features (CE between consecutive ones), a few chords
      (i, i+2) and optional attachment of one end to a cluster vertex, plus short
      ladders (parallel wire pairs).  These model the routing fabric that
      dominates |V| and is removed by simplification.
* Cluster sizes are uniform in [comp_min, comp_max] before splitting, and
  splitting never grows a cluster past comp_max, so no component exceeds
  comp_max vertices.

No method arithmetic lives here (no simplification, search or cost).
"""
from __future__ import annotations

import numpy as np

from .graph import DecompGraph, from_edges, concat

# PAPER.md Table 1, "Graph Info" columns: name -> (|V|, second column read as |E|)
TABLE1 = {
    "c432": (1109, 1222), "c499": (2216, 2817), "c880": (2411, 2686),
    "c1355": (3262, 3326), "c1908": (5125, 5598), "c2670": (7933, 9336),
    "c3540": (10189, 11968), "c5315": (14603, 16881), "c6288": (14575, 15605),
    "c7552": (21253, 24372), "s1488": (4611, 5504), "s38417": (67696, 79527),
    "s35932": (157455, 186052), "s38584": (168319, 196072), "s15850": (159952, 190796),
}
ISCAS85 = ["c432", "c499", "c880", "c1355", "c1908", "c2670", "c3540", "c5315", "c6288", "c7552"]


def _points_graph(pts):
    """CE adjacency of features closer than the colouring spacing 1 (unit disk)."""
    s = len(pts)
    d2 = ((pts[:, None, :] - pts[None, :, :]) ** 2).sum(-1)
    iu, ju = np.nonzero(np.triu(d2 < 1.0, 1))
    adj = [set() for _ in range(s)]
    for a, b in zip(iu.tolist(), ju.tolist()):
        adj[a].add(b)
        adj[b].add(a)
    return adj


def _split_stitches(rng, adj, xs, k, stitch_prob, comp_max):
    """Stitch candidates (Fig. 1(c)): a vertex of conflict degree >= k is, with
    probability stitch_prob, split into two segments joined by an SE edge;
    neighbours left of its x-coordinate stay on segment 0, the rest move to
    segment 1 (no split if either side would be empty, none past comp_max)."""
    s = len(adj)
    se = []
    n = s
    if stitch_prob > 0:
        for v in range(s):
            if n >= comp_max:
                break
            nb = sorted(adj[v])
            if len(nb) < k or rng.random() >= stitch_prob:
                continue
            left = [u for u in nb if xs[u] < xs[v]]
            right = [u for u in nb if xs[u] >= xs[v]]
            if not left or not right:
                continue
            seg1 = n
            n += 1
            xs.append(xs[v])
            adj.append(set())
            for u in right:
                adj[v].discard(u)
                adj[u].discard(v)
                adj[u].add(seg1)
                adj[seg1].add(u)
            se.append((v, seg1))
    ce = [(a, b) for a in range(n) for b in adj[a] if a < b]
    return n, ce, se


def _cluster(rng, s, k, density, stitch_prob, comp_max):
    """One dense random cluster: s points uniform in a square of side
    sqrt(s/density); returns (n_vertices, ce_edges, se_edges) in local ids."""
    side = np.sqrt(s / density)
    pts = rng.random((s, 2)) * side
    adj = _points_graph(pts)
    return _split_stitches(rng, adj, pts[:, 0].tolist(), k, stitch_prob, comp_max)


def _lattice_cluster(rng, s, k, pitch, jitter, stitch_prob, comp_max):
    """One track-aligned cluster (a cell row / contact array on routing tracks):
    s features on a jittered square lattice of the given pitch (in units of the
    colouring spacing), row by row, ceil(sqrt(1.5 s)) per row, each coordinate
    offset uniformly in [-jitter, jitter].  At pitch 0.7 the orthogonal
    neighbours always conflict and about half the diagonals do: a near-planar
    graph of degree ~6 whose k = 4 core keeps most of the cluster."""
    cols = int(np.ceil(np.sqrt(1.5 * s)))
    pts = np.array([((i % cols) * pitch, (i // cols) * pitch) for i in range(s)], dtype=np.float64)
    pts += rng.uniform(-jitter, jitter, size=(s, 2))
    adj = _points_graph(pts)
    return _split_stitches(rng, adj, pts[:, 0].tolist(), k, stitch_prob, comp_max)


def make_layout(n_target: int, e_target: int, k: int = 3, stitch_prob: float = 0.0,
                comp_max: int = 8, comp_min: int = 4, cluster_frac: float = 0.1,
                density: float = 1.3, ladder_frac: float = 0.02, seed: int = 0,
                name: str = "layout", lattice_frac: float = 0.0, pitch: float = 0.7,
                jitter: float = 0.15) -> DecompGraph:
    """One synthetic layout with exactly n_target vertices and about e_target edges.
    A fraction lattice_frac of the clusters are track-aligned lattice clusters
    (_lattice_cluster), the rest random unit-disk clusters (_cluster)."""
    rng = np.random.default_rng(seed)
    pieces = []  # (size, ce, se, kind)
    nv = 0
    n_cluster = int(cluster_frac * n_target)
    while nv < n_cluster:
        s = int(rng.integers(comp_min, comp_max + 1))
        s = min(s, comp_max)
        if lattice_frac > 0 and rng.random() < lattice_frac:
            sz, ce, se = _lattice_cluster(rng, s, k, pitch, jitter, stitch_prob, comp_max)
        else:
            sz, ce, se = _cluster(rng, s, k, density, stitch_prob, comp_max)
        if nv + sz > n_target:
            break
        pieces.append((sz, ce, se, "cluster"))
        nv += sz
    n_ladder = int(ladder_frac * n_target)
    lv = 0
    while lv < n_ladder and nv + 8 <= n_target:
        L = int(rng.integers(3, 13))
        if nv + 2 * L > n_target:
            break
        ce = [(i, i + 1) for i in range(L - 1)] + [(L + i, L + i + 1) for i in range(L - 1)]
        ce += [(i, L + i) for i in range(L)]
        pieces.append((2 * L, ce, [], "ladder"))
        nv += 2 * L
        lv += 2 * L
    # wires fill the remaining vertices
    while nv < n_target:
        L = int(min(n_target - nv, 1 + rng.geometric(1 / 9.0)))
        ce = [(i, i + 1) for i in range(L - 1)]
        pieces.append((L, ce, [], "wire"))
        nv += L
    order = rng.permutation(len(pieces))
    base = 0
    bases = {}
    CE, SE = [], []
    for p in order:
        sz, ce, se, kind = pieces[p]
        perm = rng.permutation(sz)  # shuffle ids inside the piece
        bases[p] = (base, perm)
        CE += [(base + perm[a], base + perm[b]) for a, b in ce]
        SE += [(base + perm[a], base + perm[b]) for a, b in se]
        base += sz
    # match the edge target: chords (i, i+2) on wires every third position and
    # attachments of wire ends to cluster vertices add edges; cutting wire edges removes them
    e_cur = len(CE) + len(SE)
    wires = [p for p in range(len(pieces)) if pieces[p][3] == "wire"]
    clusters = [p for p in range(len(pieces)) if pieces[p][3] == "cluster"]
    extra = []
    if e_cur < e_target:
        cand = []
        for p in wires:
            sz = pieces[p][0]
            b, perm = bases[p]
            cand += [(b + perm[i], b + perm[i + 2]) for i in range(0, sz - 2, 3)]
            if clusters and sz >= 1:
                q = clusters[int(rng.integers(len(clusters)))]
                qb, qperm = bases[q]
                cv = qb + qperm[int(rng.integers(pieces[q][0]))]
                cand.append((b + perm[0], cv))
        idx = rng.permutation(len(cand))[: e_target - e_cur]
        extra = [cand[i] for i in idx]
        CE += extra
    elif e_cur > e_target:
        wire_edges = []
        for p in wires:
            sz = pieces[p][0]
            b, perm = bases[p]
            wire_edges += [(b + perm[i], b + perm[i + 1]) for i in range(sz - 1)]
        drop = set(rng.permutation(len(wire_edges))[: e_cur - e_target].tolist())
        dropset = {wire_edges[i] for i in drop}
        CE = [e for e in CE if e not in dropset]
    return from_edges(n_target, np.array(CE, dtype=np.int64).reshape(-1, 2),
                      np.array(SE, dtype=np.int64).reshape(-1, 2), name=name)


def iscas_layout(circuit: str, k: int = 3, stitch_prob: float = 0.5, comp_max: int = 12,
                 density: float = 0.8, seed: int = 0) -> DecompGraph:
    """A synthetic layout with the |V| / |E| of one PAPER.md Table 1 row."""
    nv, ne = TABLE1[circuit]
    return make_layout(nv, ne, k=k, stitch_prob=stitch_prob, comp_max=comp_max,
                       density=density, seed=seed, name=circuit)


def stress_components(size: int, count: int, k: int, seed: int = 0, extra_deg: float = 0.5) -> DecompGraph:
    """`count` disjoint components of exactly `size` vertices each, every vertex of
    conflict degree >= k (so the simplification keeps them whole): a random
    spanning path plus geometric-locality edges until the minimum degree is k."""
    rng = np.random.default_rng(seed)
    graphs = []
    for _ in range(count):
        pts = rng.random((size, 2))
        order = np.argsort(pts[:, 0] + 0.3 * pts[:, 1])
        edges = {(min(order[i], order[i + 1]), max(order[i], order[i + 1])) for i in range(size - 1)}
        d2 = ((pts[:, None, :] - pts[None, :, :]) ** 2).sum(-1)
        np.fill_diagonal(d2, np.inf)
        near = np.argsort(d2, axis=1)
        deg = np.zeros(size, np.int64)
        for a, b in edges:
            deg[a] += 1
            deg[b] += 1
        want = k + (rng.random(size) < extra_deg).astype(np.int64)
        for v in range(size):
            j = 0
            while deg[v] < min(want[v], size - 1) and j < size - 1:
                u = int(near[v, j])
                e = (min(v, u), max(v, u))
                if e not in edges:
                    edges.add(e)
                    deg[v] += 1
                    deg[u] += 1
                j += 1
        graphs.append(from_edges(size, np.array(sorted(edges), dtype=np.int64)))
    g = concat(graphs, name=f"stress_n{size}_k{k}")
    g.layout_offsets = np.array([0, g.n], dtype=np.int32)  # one layout
    return g


def config_graphs(config: int, seed: int = 0, scale: float = 1.0):
    """BASELINE.json configs -> (list of DecompGraph, k, alpha).

    0: TPLD k=3, 1,000 polygons, components <= 8 vertices, no stitches, seed 0
    1: TPLD k=3 + stitch candidates, alpha = 0.1, the ten ISCAS-85 rows (c432..c7552)
    2: QPLD k=4 on an s38584-scale layout, components up to ~40 vertices
    3: TPLD k=3 on a 10^6-polygon industrial-scale layout
    `scale` < 1 shrinks 2 and 3 for quick tests."""
    if config == 0:
        return [make_layout(1000, 1100, k=3, stitch_prob=0.0, comp_max=8, comp_min=4,
                            cluster_frac=0.3, density=1.4, seed=seed, name="cfg0")], 3, 0.1
    if config == 1:
        return [iscas_layout(c, k=3, seed=seed + i) for i, c in enumerate(ISCAS85)], 3, 0.1
    if config == 2:
        nv, ne = TABLE1["s38584"]
        nv, ne = int(nv * scale), int(ne * scale)
        return [make_layout(nv, ne, k=4, stitch_prob=0.2, comp_max=48, comp_min=24, cluster_frac=0.1,
                            density=1.0, lattice_frac=0.75, pitch=0.68, jitter=0.15, seed=seed,
                            name="s38584")], 4, 0.1
    if config == 3:
        nv = int(1_000_000 * scale)
        return [make_layout(nv, int(nv * 1.17), k=3, stitch_prob=0.5, comp_max=16,
                            cluster_frac=0.1, density=0.8, seed=seed, name="industrial1M")], 3, 0.1
    raise ValueError(config)


def fixtures():
    """Tiny named graphs used by the pins (tests/golden cites their sources)."""
    def K(n):
        return [(i, j) for i in range(n) for j in range(i + 1, n)]
    fx = {
        "K4": from_edges(4, K(4), name="K4"),
        "triangle": from_edges(3, K(3), name="triangle"),
        "C5": from_edges(5, [(i, (i + 1) % 5) for i in range(5)], name="C5"),
        "C6": from_edges(6, [(i, (i + 1) % 6) for i in range(6)], name="C6"),
        "K5": from_edges(5, K(5), name="K5"),
        "K7": from_edges(7, K(7), name="K7"),
        "W5": from_edges(6, [(i, (i + 1) % 5) for i in range(5)] + [(5, i) for i in range(5)], name="W5"),
        "single": from_edges(1, [], name="single"),
        "empty": from_edges(0, [], name="empty"),
        "stitch_pair": from_edges(2, [], [(0, 1)], name="stitch_pair"),
    }
    return fx
