"""CSR container for a decomposed graph (DG) — PAPER.md §2.1, "E = {CE ∪ SE}".

Both edge sets are stored as symmetric CSR with strictly ascending neighbour ids
per row, no self loops, and CE ∩ SE = ∅ (the layout the C-ABI `mpld_decompose`
expects, include/mpld.h).  Pure data plumbing: no method arithmetic.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class DecompGraph:
    n: int
    ce_rowptr: np.ndarray  # int32 [n+1]
    ce_col: np.ndarray     # int32 [2|CE|]
    se_rowptr: np.ndarray  # int32 [n+1]
    se_col: np.ndarray     # int32 [2|SE|]
    name: str = ""
    # layout boundaries when several layouts are concatenated into one batch
    layout_offsets: np.ndarray = field(default=None)  # int32 [L+1]

    def __post_init__(self):
        if self.layout_offsets is None:
            self.layout_offsets = np.array([0, self.n], dtype=np.int32)

    @property
    def n_ce(self) -> int:
        return int(self.ce_col.size // 2)

    @property
    def n_se(self) -> int:
        return int(self.se_col.size // 2)

    @property
    def n_layouts(self) -> int:
        return int(self.layout_offsets.size - 1)

    def ce_edges(self) -> np.ndarray:
        """Undirected CE edge list (u < v), shape [|CE|, 2]."""
        return _half(self.n, self.ce_rowptr, self.ce_col)

    def se_edges(self) -> np.ndarray:
        return _half(self.n, self.se_rowptr, self.se_col)

    def ce_adj(self):
        return [self.ce_col[self.ce_rowptr[v]:self.ce_rowptr[v + 1]].tolist() for v in range(self.n)]

    def se_adj(self):
        return [self.se_col[self.se_rowptr[v]:self.se_rowptr[v + 1]].tolist() for v in range(self.n)]

    def nbytes(self) -> int:
        return int(self.ce_rowptr.nbytes + self.ce_col.nbytes + self.se_rowptr.nbytes + self.se_col.nbytes)


def _half(n, rowptr, col):
    src = np.repeat(np.arange(n, dtype=np.int64), np.diff(rowptr.astype(np.int64)))
    m = src < col
    return np.stack([src[m], col[m].astype(np.int64)], axis=1)


def _csr(n: int, edges: np.ndarray):
    edges = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    if edges.size:
        a = np.minimum(edges[:, 0], edges[:, 1])
        b = np.maximum(edges[:, 0], edges[:, 1])
        keep = a != b
        a, b = a[keep], b[keep]
        key = np.unique(a * n + b)
        a, b = key // n, key % n
        src = np.concatenate([a, b])
        dst = np.concatenate([b, a])
        order = np.lexsort((dst, src))
        src, dst = src[order], dst[order]
    else:
        src = dst = np.zeros(0, dtype=np.int64)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rowptr, src + 1, 1)
    rowptr = np.cumsum(rowptr)
    return rowptr.astype(np.int32), dst.astype(np.int32)


def from_edges(n: int, ce_edges, se_edges=(), name: str = "") -> DecompGraph:
    """Build a DecompGraph from undirected edge lists; duplicates and self loops dropped.
    An edge present in both lists is kept as a stitch edge only (CE ∩ SE = ∅)."""
    ce = np.asarray(ce_edges, dtype=np.int64).reshape(-1, 2)
    se = np.asarray(se_edges, dtype=np.int64).reshape(-1, 2)
    if ce.size and se.size:
        skey = set((min(a, b) * n + max(a, b)) for a, b in se.tolist())
        ce = np.array([e for e in ce.tolist() if min(e) * n + max(e) not in skey], dtype=np.int64).reshape(-1, 2)
    cr, cc = _csr(n, ce)
    sr, sc = _csr(n, se)
    return DecompGraph(n, cr, cc, sr, sc, name=name)


def split(b: DecompGraph):
    """Inverse of concat: the layouts of a batch as separate DecompGraphs."""
    offs = b.layout_offsets.tolist()
    out = []
    for li in range(len(offs) - 1):
        a, e = offs[li], offs[li + 1]
        cr = b.ce_rowptr[a:e + 1].astype(np.int64)
        sr = b.se_rowptr[a:e + 1].astype(np.int64)
        out.append(DecompGraph(e - a, (cr - cr[0]).astype(np.int32), (b.ce_col[cr[0]:cr[-1]] - a).astype(np.int32),
                               (sr - sr[0]).astype(np.int32), (b.se_col[sr[0]:sr[-1]] - a).astype(np.int32),
                               name=f"{b.name}[{li}]"))
    return out


def concat(graphs, name: str = "batch") -> DecompGraph:
    """Disjoint union of several layouts (vertex ids offset), keeping layout boundaries."""
    offs = [0]
    cr, cc, sr, sc = [np.zeros(1, np.int64)], [], [np.zeros(1, np.int64)], []
    ce_base = se_base = 0
    for g in graphs:
        base = offs[-1]
        cr.append(g.ce_rowptr[1:].astype(np.int64) + ce_base)
        sr.append(g.se_rowptr[1:].astype(np.int64) + se_base)
        cc.append(g.ce_col.astype(np.int64) + base)
        sc.append(g.se_col.astype(np.int64) + base)
        ce_base += g.ce_col.size
        se_base += g.se_col.size
        offs.append(base + g.n)
    n = offs[-1]
    cat = lambda xs: np.concatenate(xs) if xs else np.zeros(0, np.int64)  # noqa: E731
    return DecompGraph(n, cat(cr).astype(np.int32), cat(cc).astype(np.int32),
                       cat(sr).astype(np.int32), cat(sc).astype(np.int32), name=name,
                       layout_offsets=np.array(offs, dtype=np.int32))


def upper_csr(g: DecompGraph):
    """The upper triangle of the CE CSR (the input of
    mpld_decompose_batch_upper_async): uint8 counts of the neighbours u > v of
    every vertex v and those neighbours, rows ascending.  Raises if a vertex
    has 256 or more larger neighbours."""
    n = g.n
    src = np.repeat(np.arange(n, dtype=np.int64), np.diff(g.ce_rowptr.astype(np.int64)))
    up = g.ce_col > src
    deg = np.bincount(src[up], minlength=n) if n else np.zeros(0, np.int64)
    if deg.size and deg.max() > 255:
        raise ValueError("a vertex has more than 255 larger conflict neighbours")
    return deg.astype(np.uint8), np.ascontiguousarray(g.ce_col[up], dtype=np.int32)


def stitch_pairs(g: DecompGraph):
    """Each stitch edge once, (u, v) with u < v, int32 [m, 2]."""
    e = g.se_edges()
    return np.ascontiguousarray(e, dtype=np.int32).reshape(-1, 2)
