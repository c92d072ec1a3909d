"""Algorithm X on dancing links for the relaxed exact-cover MPLD model.

TEST INFRASTRUCTURE (see oracle/__init__.py): never imported by the product path.

PAPER.md §2.3 ("The original layout will be ... translated into a binary matrix
of '0's and '1's ... finding a set of rows containing exactly one '1' in each
column"; Fig. 3) and Knuth's dancing links (§1, "doubly-linked circular lists
to represent the matrix"), with the cover/uncover pointer updates of Eq. (2):

    Cover:   L[R[x]] <- L[x],  R[L[x]] <- R[x]
    Uncover: L[R[x]] <- x,     R[L[x]] <- x

Exact-cover model of one component with n vertices (local ids in BFS order)
and k masks (BASELINE.json north_star; reading R3):
    row  r(v, c) = v*k + c                      vertex/segment v takes mask c
    primary column   1 + v                      every vertex covered exactly once
    secondary column (e, c), e = (u, w) in CE   hit by rows r(u, c) and r(w, c):
                                                at most one of them conflict-free
Conflict relaxation (Alg. 1 lines 10-12, "Mark (cl, cl') as one conflict
candidate"): a row whose secondary column is already covered stays selectable;
each already-covered secondary column of the selected row is one conflict
c_ij = 1 of Eq. (1b).  Stitch cost s_ij (Eq. 1c) of a row = number of stitch
neighbours already coloured differently.

Search (Alg. 1 lines 5-19, readings R4-R7):
  * a leaf is reached when no primary column remains (line 5);
  * column select (line 8): the lowest-index column with zero live rows, else
    the lowest-index column with exactly one live row ("only one related row"),
    else the lowest-index column, i.e. first in BFS order of G;
  * cover the column (line 9), then for each row of the column in index order
    (c = 0, 1, ...; line 13) include it, cover its not-yet-covered secondary
    columns ("Cover rw and its affected rows", line 15), recurse (16), uncover
    (17), exclude (18); finally uncover the column (20);
  * colour-symmetry rule: mask c is tried only if c <= 1 + (largest mask used so
    far) — colours are interchangeable in Eq. (1), this never removes the
    canonical optimum (R6);
  * branch and bound on the Eq. (1a) objective in integer cost units
    (W_CONF per conflict, W_STITCH per stitch): a node is pruned when
    cost + W_CONF * (#columns with zero live rows + clique deficit) >= best,
    the clique deficit (k >= 4 only) summing, over the greedy disjoint cliques
    of >= k vertices of the component (clique_partition below),
    max(0, |X| - |live masks of X|) for X = the clique's uncovered columns that
    still have a live row;
  * the result is the first minimum-cost leaf in this search order;
  * budget: every node entry is one step; once a leaf exists and steps exceed
    max_steps (> 0), the search stops and returns the best leaf so far.
"""
from __future__ import annotations


class _Abort(Exception):
    pass


class DLXMatrix:
    """Dancing-links matrix: node 0 is the root h, nodes 1..n primary column
    headers (linked in h's ring), then n_ce*k secondary headers (self-linked,
    never selected), then the row nodes, rows in index order r = v*k + c."""

    def __init__(self, n: int, k: int, ce_edges):
        self.n, self.k = n, k
        ce_edges = [tuple(e) for e in ce_edges]
        n_sec = len(ce_edges) * k
        n_head = 1 + n + n_sec
        L, R, U, D, C = [], [], [], [], []
        for x in range(n_head):
            L.append(x)
            R.append(x)
            U.append(x)
            D.append(x)
            C.append(x)
        # primary headers in the root ring, in column index order
        for x in range(n + 1):
            L[x] = (x - 1) % (n + 1)
            R[x] = (x + 1) % (n + 1)
        self.S = [0] * n_head
        incident = [[] for _ in range(n)]
        for ei, (u, w) in enumerate(ce_edges):
            incident[u].append(ei)
            incident[w].append(ei)
        self.first = []  # first (primary) node of each row
        self.row_of = []  # row id of each row node, indexed by node - n_head
        for v in range(n):
            for c in range(k):
                cols = [1 + v] + [1 + n + ei * k + c for ei in incident[v]]
                start = len(L)
                for t, col in enumerate(cols):
                    x = len(L)
                    L.append(start + (t - 1) % len(cols))
                    R.append(start + (t + 1) % len(cols))
                    # append at the bottom of column col
                    U.append(U[col])
                    D.append(col)
                    C.append(col)
                    D[U[col]] = x
                    U[col] = x
                    self.S[col] += 1
                    self.row_of.append(v * k + c)
                self.first.append(start)
        self.L, self.R, self.U, self.D, self.C = L, R, U, D, C
        self.n_head = n_head
        self.covered = [False] * n_head

    def secondary(self, e_index: int, c: int) -> int:
        return 1 + self.n + e_index * self.k + c

    def cover(self, c: int) -> None:
        """Eq. (2) Cover applied to column header c and, vertically, to every
        row that intersects c (Knuth's cover)."""
        L, R, U, D, C, S = self.L, self.R, self.U, self.D, self.C, self.S
        L[R[c]] = L[c]
        R[L[c]] = R[c]
        i = D[c]
        while i != c:
            j = R[i]
            while j != i:
                U[D[j]] = U[j]
                D[U[j]] = D[j]
                S[C[j]] -= 1
                j = R[j]
            i = D[i]
        self.covered[c] = True

    def uncover(self, c: int) -> None:
        """Eq. (2) Uncover: exact inverse of cover (LIFO discipline)."""
        L, R, U, D, C, S = self.L, self.R, self.U, self.D, self.C, self.S
        i = U[c]
        while i != c:
            j = L[i]
            while j != i:
                S[C[j]] += 1
                U[D[j]] = j
                D[U[j]] = j
                j = L[j]
            i = U[i]
        L[R[c]] = c
        R[L[c]] = c
        self.covered[c] = False

    def snapshot(self):
        return (tuple(self.L), tuple(self.R), tuple(self.U), tuple(self.D),
                tuple(self.S), tuple(self.covered))

    def live_rows(self, col: int):
        out, i = [], self.D[col]
        while i != col:
            out.append(self.row_of[i - self.n_head])
            i = self.D[i]
        return out


def clique_partition(n: int, ce_edges, minsize: int = 2):
    """Greedy disjoint maximal cliques of the component (bound of R7): for v in
    index order, if v is unused, Q = {v}; add the smallest unused vertex adjacent
    to all of Q while one exists; keep Q (and mark it used) if |Q| >= minsize."""
    nb = [set() for _ in range(n)]
    for u, w in ce_edges:
        nb[u].add(w)
        nb[w].add(u)
    used = [False] * n
    cliques = []
    for v in range(n):
        if used[v]:
            continue
        Q = [v]
        cand = {u for u in nb[v] if not used[u]}
        while cand:
            u = min(cand)
            Q.append(u)
            cand &= nb[u]
        if len(Q) >= minsize:
            cliques.append(Q)
            for u in Q:
                used[u] = True
    return cliques


def algorithm_x(n: int, k: int, ce_edges, se_adj, w_conf: int, w_stitch: int,
                max_steps: int = 0, matrix: DLXMatrix | None = None):
    """Relaxed Algorithm X with branch and bound (module docstring).

    n, ce_edges: component in local ids (BFS order); se_adj[v]: local stitch
    neighbours of v.  Returns dict(colors, cost, n_conf, n_stitch, steps,
    truncated, rows) where rows are the selected exact-cover rows."""
    M = matrix if matrix is not None else DLXMatrix(n, k, ce_edges)
    L, R, C, S, covered, first = M.L, M.R, M.C, M.S, M.covered, M.first
    h = 0
    color = [-1] * n
    INF = float("inf")
    st = {"best": INF, "colors": None, "n_conf": 0, "n_stitch": 0, "steps": 0, "truncated": False}
    # R7: the clique term is used for k >= 4, over cliques of >= k vertices
    cliques = clique_partition(n, ce_edges, minsize=k) if k >= 4 else []

    def clique_deficit():
        """sum over cliques of max(0, |X| - |live masks of X|), X = uncovered
        columns of the clique with at least one live row (R7)"""
        total = 0
        for Q in cliques:
            X = [v for v in Q if not covered[1 + v] and S[1 + v] > 0]
            masks = {r % k for v in X for r in M.live_rows(1 + v)}
            total += max(0, len(X) - len(masks))
        return total

    def search(cost, n_conf, n_stitch, maxused):
        st["steps"] += 1
        if st["best"] != INF and max_steps > 0 and st["steps"] > max_steps:
            st["truncated"] = True
            raise _Abort
        if R[h] == h:  # Alg. 1 line 5: all columns covered -> a solution
            if cost < st["best"]:
                st.update(best=cost, colors=list(color), n_conf=n_conf, n_stitch=n_stitch)
            return
        # column-count reduction over the live primary columns (S = live rows)
        zero = one = 0
        n_zero = 0
        col = R[h]
        while col != h:
            if S[col] == 0:
                n_zero += 1
                if not zero:
                    zero = col
            elif S[col] == 1 and not one:
                one = col
            col = R[col]
        if st["best"] != INF and cost + w_conf * (n_zero + clique_deficit()) >= st["best"]:  # bound (R7)
            return
        cl = zero or one or R[h]  # Alg. 1 line 8
        v = cl - 1
        M.cover(cl)  # line 9
        try:
            for c in range(min(k, maxused + 2)):  # line 13, rows in index order
                r = v * k + c
                x = first[r]
                newly = []
                conf = 0
                j = R[x]
                while j != x:  # line 15: cover rw's affected rows
                    if covered[C[j]]:
                        conf += 1  # secondary (e, c) already taken: c_ij = 1
                    else:
                        M.cover(C[j])
                        newly.append(C[j])
                    j = R[j]
                stitch = sum(1 for u in se_adj[v] if color[u] >= 0 and color[u] != c)
                color[v] = c  # line 14
                try:
                    search(cost + w_conf * conf + w_stitch * stitch, n_conf + conf,
                           n_stitch + stitch, max(maxused, c))  # line 16
                finally:
                    color[v] = -1  # line 18
                    for col2 in reversed(newly):  # line 17
                        M.uncover(col2)
        finally:
            M.uncover(cl)  # line 20

    try:
        search(0, 0, 0, -1)
    except _Abort:
        pass  # the finally-clauses restored the matrix on the way out
    colors = st["colors"]
    return {"colors": colors, "cost": st["best"], "n_conf": st["n_conf"], "n_stitch": st["n_stitch"],
            "steps": st["steps"], "truncated": st["truncated"],
            "rows": [v * k + c for v, c in enumerate(colors)] if colors is not None else None}
