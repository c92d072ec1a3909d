// The exact-cover search of PAPER.md §2.3 / Alg. 1 on bit-packed matrices.
//
// The exact-cover matrix of a component (rows r(v,c), primary columns =
// vertices, secondary columns = (e,c) for e in CE) is never materialised as a
// 0/1 array: with columns = bit positions of a machine word it is fully
// described by, per vertex v,
//     adj[v]  — CE neighbours (the secondary columns shared by r(v,c), r(u,c))
//     sadj[v] — SE neighbours (stitch cost of Eq. 1c)
// and the search state by, per mask c,
//     C[c] — vertices coloured c (selected rows of mask c)
//     B[c] — OR of adj[u] over u in C[c] = vertices whose row r(·,c) lost a
//            secondary column ("Cover rw and its affected rows", line 15)
// plus U = uncovered primary columns.  Then
//     live rows of column v          = #{c : v not in B[c]}        (bit-sliced below)
//     conflicts of selecting r(v,c)  = popc(adj[v] & C[c])         (already-covered secondary columns)
//     stitches of selecting r(v,c)   = popc(sadj[v] & coloured & ~C[c])
// Cover/uncover (Eq. 2) become mask AND/OR; backtracking pops a 32-byte frame.
// Components of <= 32 vertices run on 32-bit words, larger ones on 64-bit.
//
// Two kernels:
//   mpld_exact_cover_search<K>        one warp per component seed: warp-parallel
//                                     discovery of the component, relabelling to
//                                     the R5 column order, then the sequential DFS
//                                     on lane 0 (the oracle's exact node order and
//                                     budget, R7);
//   mpld_exact_cover_search_heavy<K>  exact mode (max_steps <= 0) only: one
//                                     128-thread CTA per component whose
//                                     sequential search needed more than the
//                                     light budget.  The canonical tree is split
//                                     level-synchronously into >= 128 subtrees
//                                     (DFS order kept, nodes stored as paths),
//                                     lanes search subtrees with a shared
//                                     incumbent keyed (cost, subtree index); the
//                                     first optimal leaf of R7 is recovered
//                                     exactly.
#include <climits>

#include "mpld_internal.cuh"

namespace mpld {

namespace {

constexpr unsigned kHeavyLaneCap = 1u << 22;  // exact mode safety cap: search nodes per lane per component

template <typename W>
struct WordOps;
template <>
struct WordOps<unsigned> {
  static __device__ __forceinline__ int popc(unsigned x) { return __popc(x); }
  static __device__ __forceinline__ int ffs(unsigned x) { return __ffs((int)x) - 1; }
  static __device__ __forceinline__ unsigned full(int n) { return n == 32 ? ~0u : ((1u << n) - 1u); }
};
template <>
struct WordOps<unsigned long long> {
  static __device__ __forceinline__ int popc(unsigned long long x) { return __popcll(x); }
  static __device__ __forceinline__ int ffs(unsigned long long x) { return __ffsll((long long)x) - 1; }
  static __device__ __forceinline__ unsigned long long full(int n) { return n == 64 ? ~0ull : ((1ull << n) - 1ull); }
};

// One level of the explicit backtrack stack (Alg. 1 recursion, lines 13-18).
template <typename W>
struct __align__(16) Frame {
  W saved;     // B[c] before r(v,c) was selected
  int cost;    // cost when the node was entered
  int packed;  // v | (c+1) << 8 | (maxused+1) << 16
};

template <int K, typename W>
__device__ __forceinline__ W pick(const W (&a)[K], int c) {
  W r = a[0];
#pragma unroll
  for (int i = 1; i < K; ++i) r = (c == i) ? a[i] : r;
  return r;
}

template <int K, typename W>
__device__ __forceinline__ void put(W (&a)[K], int c, W x) {
#pragma unroll
  for (int i = 0; i < K; ++i)
    if (c == i) a[i] = x;
}

// column-count reduction, bit-sliced over all columns: Z = no live row, O = one live row
template <int K, typename W>
__device__ __forceinline__ void live_counts(const W (&B)[K], W U, W& Z, W& O) {
  W s1 = 0, s2 = 0;
#pragma unroll
  for (int c = 0; c < K; ++c) {
    const W F = U & ~B[c];
    s2 |= s1 & F;
    s1 |= F;
  }
  Z = U & ~s1;
  O = s1 & ~s2;
}

// Greedy disjoint maximal cliques of a component (bound of R7, identical to
// oracle.dlx.clique_partition): for v in index order, if unused, Q = {v} grown
// by the smallest unused vertex adjacent to all of Q; kept if |Q| >= minsize.
// cl[q * cs] receives the clique masks; returns their number (<= n / 2).
template <typename W>
__device__ int clique_partition(const W* adj, int as, int n, W* cl, int cs, int minsize) {
  using O = WordOps<W>;
  W used = 0;
  int ncl = 0;
  for (int v = 0; v < n; ++v) {
    const W bv = W(1) << v;
    if (used & bv) continue;
    W Q = bv, cand = adj[v * as] & ~used;
    while (cand) {
      const int u = O::ffs(cand);
      Q |= W(1) << u;
      cand &= adj[u * as];
    }
    if (O::popc(Q) >= minsize) {
      cl[ncl * cs] = Q;
      ++ncl;
      used |= Q;
    }
  }
  return ncl;
}

// The clique term of the bound is used for k >= 4 only, over cliques of at
// least k vertices (R7; measured: for k = 3 it saves ~8 % of the nodes but costs
// more than that per node, for k = 4 it makes the hardest QPLD component of
// configs[2] finish — 16.7 M nodes instead of > 134 M).
template <int K>
__host__ __device__ constexpr int clique_min() {
  return K >= 4 ? K : 0;  // 0: no cliques
}

// Lower bound of R7 in conflicts: columns with no live row, plus, over the
// cliques, max(0, |X| - #masks live on X) for X = the clique's uncovered
// columns that still have a live row.
template <int K, typename W>
__device__ __forceinline__ int bound_conflicts(const W (&B)[K], W U, W Z, const W* cl, int cs, int ncl) {
  using O = WordOps<W>;
  int lb = O::popc(Z);
  if constexpr (clique_min<K>() > 0) {
    for (int q = 0; q < ncl; ++q) {
      const W X = cl[q * cs] & U & ~Z;
      if (!X) continue;
      int live = 0;
#pragma unroll
      for (int c = 0; c < K; ++c) live += (X & ~B[c]) ? 1 : 0;
      lb += max(0, O::popc(X) - live);
    }
  }
  return lb;
}

// Incumbent of the sequential search: strict improvement, prune on lb >= best.
struct SeqIncumbent {
  int best = INT_MAX;
  __device__ __forceinline__ bool has() const { return best != INT_MAX; }
  __device__ __forceinline__ bool prune(int lb) const { return lb >= best; }
  __device__ __forceinline__ bool improves(int cost) const { return cost < best; }
  __device__ __forceinline__ void take(int cost) { best = cost; }
};

// Incumbent of the warp-parallel search: keys (cost << 32 | subtree + 1),
// shared through a shared-memory atomicMin; a node of subtree f is pruned when
// (lb, f+1) >= the best key, so equal-cost leaves of earlier
// subtrees always win.
struct ParIncumbent {
  unsigned long long* shared_best;
  unsigned long long fkey;  // f + 1
  unsigned long long lane_best = ~0ull;
  __device__ __forceinline__ bool has() const { return true; }
  __device__ __forceinline__ bool prune(int lb) const {
    const unsigned long long g = *((volatile unsigned long long*)shared_best);
    return (((unsigned long long)lb << 32) | fkey) >= g;
  }
  __device__ __forceinline__ bool improves(int cost) const {
    return (((unsigned long long)cost << 32) | fkey) < lane_best;
  }
  __device__ __forceinline__ void take(int cost) {
    lane_best = ((unsigned long long)cost << 32) | fkey;
    atomicMin(shared_best, lane_best);
  }
};

// Relaxed Algorithm X with branch and bound (R4-R7) from the node
// (C, B, U, cost, maxused).  am_adj[i*as] / am_sadj[i*as] = masks of local
// vertex i; stack[d*ss] = frame of depth d (strides let a warp interleave its
// lanes' arrays in shared memory).  Returns the nodes entered; the best
// leaf's masks in bestC.
template <int K, typename W, typename Inc>
__device__ unsigned dfs(const W* __restrict__ am_adj, const W* __restrict__ am_sadj, int as, W (&C)[K], W (&B)[K],
                        W U, int cost, int maxused, int w_stitch, unsigned max_steps,
                        Frame<W>* __restrict__ stack, int ss, const W* __restrict__ cl, int cs, int ncl,
                        Inc& inc, W (&bestC)[K], bool& truncated) {
  using O = WordOps<W>;
  int depth = 0;
  unsigned steps = 0;
  truncated = false;
  bool enter = true;
  // the frame of the deepest expanded node lives in registers
  W f_saved = 0, f_adj = 0, f_sadj = 0;
  int f_cost = 0, f_v = 0, f_c = -1, f_mu = -1;
  while (true) {
    if (enter) {
      ++steps;
      if (inc.has() && steps > max_steps) { truncated = true; break; }
      if (U == 0) {  // Alg. 1 line 5: every column covered -> a solution
        if (inc.improves(cost)) {
          inc.take(cost);
#pragma unroll
          for (int c = 0; c < K; ++c) bestC[c] = C[c];
        }
      } else {
        W Z, Ol;
        live_counts<K, W>(B, U, Z, Ol);
        if (!inc.prune(cost + kCostUnits * bound_conflicts<K, W>(B, U, Z, cl, cs, ncl))) {  // bound (R7)
          const W cand = Z ? Z : (Ol ? Ol : U);  // Alg. 1 line 8 (R5)
          const int v = O::ffs(cand);
          if (depth > 0) {  // spill the parent frame
            Frame<W> f;
            f.saved = f_saved;
            f.cost = f_cost;
            f.packed = f_v | ((f_c + 1) << 8) | ((f_mu + 1) << 16);
            stack[(depth - 1) * ss] = f;
          }
          f_v = v;
          f_c = -1;
          f_mu = maxused;
          f_cost = cost;
          f_adj = am_adj[v * as];
          f_sadj = am_sadj[v * as];
          U &= ~(W(1) << v);  // cover column v (line 9)
          ++depth;
        }
      }
    }
    if (depth == 0) break;
    const W bit = W(1) << f_v;
    if (f_c >= 0) {  // uncover the previous row (line 17)
      put<K, W>(C, f_c, pick<K, W>(C, f_c) & ~bit);
      put<K, W>(B, f_c, f_saved);
    }
    const int c = f_c + 1;
    if (c > min(K - 1, f_mu + 1)) {  // rows exhausted (colour-symmetry limit R6): uncover column (line 20)
      U |= bit;
      --depth;
      if (depth > 0) {
        const Frame<W> f = stack[(depth - 1) * ss];
        f_saved = f.saved;
        f_cost = f.cost;
        f_v = f.packed & 0xff;
        f_c = ((f.packed >> 8) & 0xff) - 1;
        f_mu = ((f.packed >> 16) & 0xff) - 1;
        f_adj = am_adj[f_v * as];
        f_sadj = am_sadj[f_v * as];
      }
      enter = false;
      continue;
    }
    const W Cc = pick<K, W>(C, c);
    const W Bc = pick<K, W>(B, c);
    cost = f_cost + kCostUnits * O::popc(f_adj & Cc) + w_stitch * O::popc(f_sadj & ~U & ~Cc);
    f_saved = Bc;
    f_c = c;
    put<K, W>(C, c, Cc | bit);  // select r(v,c) (line 14) and cover its secondary columns (line 15)
    put<K, W>(B, c, Bc | f_adj);
    maxused = max(f_mu, c);
    enter = true;
  }
  return steps;
}

template <int K, typename W>
__device__ __forceinline__ int colour_of(const W (&bestC)[K], int i) {
  int c = 0;
#pragma unroll
  for (int cc = 1; cc < K; ++cc)
    if ((bestC[cc] >> i) & W(1)) c = cc;
  return c;
}

#ifndef MPLD_LDD
#define MPLD_LDD __ldg
#endif
constexpr int kCompWarps = 4;  // warps per CTA of the component kernel (one component per warp)

// Per-warp shared storage of the discovery kernel.
struct __align__(16) WarpDisc {
  unsigned long long dadj[kMaxComp];   // CE masks in discovery labels
  unsigned long long dsadj[kMaxComp];  // SE masks in discovery labels
  unsigned long long adj[kMaxComp];    // CE masks in BFS labels (R5); CE ∪ SE in rank labels while relabelling
  unsigned long long sadj[kMaxComp];   // SE masks in BFS labels
  int verts[kMaxComp];                 // discovery index -> vertex id
  int order[kMaxComp];                 // BFS position -> vertex id (the rank queue while relabelling)
  int rank[kMaxComp];                  // discovery index -> rank of its id inside the component
  int bpos[kMaxComp];                  // rank -> BFS position
};

// Per-warp shared storage of the search kernel.
struct __align__(16) WarpSearch {
  unsigned long long adj[kMaxComp];   // CE masks (BFS labels)
  unsigned long long sadj[kMaxComp];  // SE masks
  Frame<unsigned long long> stack[kMaxComp];
  unsigned long long cl[kMaxComp / 2];  // clique masks (R7); then the best leaf's C[c]
};

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ int warp_excl_scan(int x, int& total) {
  const int lane = threadIdx.x & 31;
  int y = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int z = __shfl_up_sync(0xffffffffu, y, o);
    if (lane >= o) y += z;
  }
  total = __shfl_sync(0xffffffffu, y, 31);
  return y - x;
}

// Discovers the component of a seed (a kept vertex without a smaller kept
// neighbour) with the whole warp: the CE and SE rows of up to 32 discovered
// vertices are concatenated and read 32 entries at a time, so one group costs
// three dependent memory round trips (row pointers, column ids, rounds)
// whatever its degree.  The masks come out in discovery labels (dadj/dsadj,
// verts).  Returns n, -1 when the component exceeds kMaxComp, or -2 as soon
// as it meets a kept vertex smaller than the seed: that component belongs to
// the seed that is its minimum.
__device__ int warp_discover(const GraphView& g, const Workspace& w, int seed, WarpDisc& s, int* diag = nullptr) {
  const int lane = threadIdx.x & 31;
  int n_groups = 0, n_chunks = 0;
  for (int i = lane; i < kMaxComp; i += 32) s.dadj[i] = s.dsadj[i] = 0ull;
  if (lane == 0) s.verts[0] = seed;
  __syncwarp();
  int n = 1;
  for (int head = 0; head < n;) {
    const int gsz = min(32, n - head);
    int ca = 0, cn = 0, sa = 0, sn = 0;
    if (lane < gsz) {
      const int v = s.verts[head + lane];
      ca = MPLD_LDD(&g.ce_rp[v]);
      cn = MPLD_LDD(&g.ce_rp[v + 1]) - ca;
      sa = MPLD_LDD(&g.se_rp[v]);
      sn = MPLD_LDD(&g.se_rp[v + 1]) - sa;
    }
    int total;
    const int excl = warp_excl_scan(cn + sn, total);
    ++n_groups;
    for (int b = 0; b < total; b += 32) {
      ++n_chunks;
      const int item = b + lane;
      int o = 0;  // owner: the last group lane whose row range starts at or before item
#pragma unroll
      for (int st = 16; st > 0; st >>= 1) {
        const int e = __shfl_sync(0xffffffffu, excl, o + st);
        if (e <= item) o += st;
      }
      const int off = item - __shfl_sync(0xffffffffu, excl, o);
      const int ocn = __shfl_sync(0xffffffffu, cn, o);
      const int oca = __shfl_sync(0xffffffffu, ca, o);
      const int osa = __shfl_sync(0xffffffffu, sa, o);
      int u = -1;
      const bool ce = off < ocn;
      if (item < total) u = ce ? MPLD_LDD(&g.ce_col[oca + off]) : MPLD_LDD(&g.se_col[osa + off - ocn]);
      const bool kept = u >= 0 && MPLD_LDD(&w.hround[u]) == -1;
      if (__any_sync(0xffffffffu, kept && u < seed)) return -2;
      int lu = -1;
      if (kept)
        for (int j = 0; j < n; ++j)
          if (s.verts[j] == u) {
            lu = j;
            break;
          }
      const bool fresh = kept && lu < 0;
      const unsigned grp = __match_any_sync(0xffffffffu, fresh ? u : -2 - lane);
      const int leader = __ffs(grp) - 1;
      const unsigned lead = __ballot_sync(0xffffffffu, fresh && leader == lane);
      if (n + __popc(lead) > kMaxComp) return -1;
      if (fresh && leader == lane) {
        lu = n + __popc(lead & lanemask_lt());
        s.verts[lu] = u;
      }
      const int lu_leader = __shfl_sync(0xffffffffu, lu, leader);
      if (fresh) lu = lu_leader;
      n += __popc(lead);
      if (kept) {  // one bit: a native 32-bit shared atomic on its half (the 64-bit one is a CAS loop)
        unsigned* word = (unsigned*)(ce ? &s.dadj[head + o] : &s.dsadj[head + o]) + (lu >> 5);
        atomicOr(word, 1u << (lu & 31));
      }
      __syncwarp();
    }
    head += gsz;
  }
  if (diag) *diag = n_groups | (n_chunks << 8);
  return n;
}

// Relabels the discovered component to the column order of R5 (BFS from the
// minimum vertex, neighbours over CE ∪ SE in ascending id): ranks of the ids,
// the BFS on rank-labelled masks (lane 0), then the final masks and order.
__device__ void warp_relabel(WarpDisc& s, int n) {
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < n; i += 32) {
    const int vi = s.verts[i];
    int r = 0;
    for (int j = 0; j < n; ++j) r += s.verts[j] < vi ? 1 : 0;
    s.rank[i] = r;
  }
  __syncwarp();
  for (int i = lane; i < n; i += 32) {
    unsigned long long m = s.dadj[i] | s.dsadj[i], x = 0ull;
    while (m) {
      x |= 1ull << s.rank[__ffsll((long long)m) - 1];
      m &= m - 1;
    }
    s.adj[s.rank[i]] = x;
  }
  __syncwarp();
  if (lane == 0) {  // BFS over ranks; rank 0 is the seed (the minimum)
    unsigned long long seen = 1ull;
    int tail = 1;
    s.order[0] = 0;
    s.bpos[0] = 0;
    for (int h = 0; h < tail; ++h) {
      unsigned long long m = s.adj[s.order[h]] & ~seen;
      seen |= m;
      while (m) {
        const int j = __ffsll((long long)m) - 1;
        m &= m - 1;
        s.bpos[j] = tail;
        s.order[tail++] = j;
      }
    }
  }
  __syncwarp();
  for (int i = lane; i < n; i += 32) {
    unsigned long long a = 0ull, b = 0ull, m = s.dadj[i];
    while (m) {
      a |= 1ull << s.bpos[s.rank[__ffsll((long long)m) - 1]];
      m &= m - 1;
    }
    m = s.dsadj[i];
    while (m) {
      b |= 1ull << s.bpos[s.rank[__ffsll((long long)m) - 1]];
      m &= m - 1;
    }
    const int p = s.bpos[s.rank[i]];
    s.adj[p] = a;  // every lane has read the rank-labelled masks before the barrier above
    s.sadj[p] = b;
    s.order[p] = s.verts[i];
  }
  __syncwarp();
}

// The sequential DFS of R4-R7 on lane 0 (the oracle's node order and budget).
// W = 32-bit words read the low halves of the 64-bit masks (stride 2).
template <int K, typename W>
__device__ unsigned comp_dfs(WarpSearch& s, int n, int w_stitch, unsigned budget, int& best_cost, bool& trunc) {
  constexpr int as = sizeof(unsigned long long) / sizeof(W);
  const W* a = (const W*)s.adj;
  const W* sa = (const W*)s.sadj;
  W* cl = (W*)s.cl;
  W C[K], B[K], bestC[K];
#pragma unroll
  for (int c = 0; c < K; ++c) C[c] = B[c] = bestC[c] = 0;
  SeqIncumbent inc;
  const int ncl = clique_min<K>() ? clique_partition<W>(a, as, n, cl, 1, clique_min<K>()) : 0;
  const unsigned steps = dfs<K, W, SeqIncumbent>(a, sa, as, C, B, WordOps<W>::full(n), 0, -1, w_stitch, budget,
                                                 (Frame<W>*)s.stack, 1, cl, 1, ncl, inc, bestC, trunc);
#pragma unroll
  for (int c = 0; c < K; ++c) s.cl[c] = (unsigned long long)bestC[c];
  best_cost = inc.best;
  return steps;
}

template <int K>
__device__ __forceinline__ int colour_of_mask(const unsigned long long* bestC, int i) {
  int c = 0;
#pragma unroll
  for (int cc = 1; cc < K; ++cc)
    if ((bestC[cc] >> i) & 1ull) c = cc;
  return c;
}

// One warp per component seed: discovery, relabelling to the R5 column order
// and the component's record in the pool (exactly one per component: the seed
// that is its minimum).  Low register use, so 64 warps per SM discover at once.
__global__ void __launch_bounds__(kCompWarps * 32, 16) mpld_component_discover(GraphView g, Workspace w,
                                                                              int shard_index, int shard_count) {
  __shared__ WarpDisc s_disc[kCompWarps];
  WarpDisc& s = s_disc[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  Control* ctl = w.ctl;
  const int n_seed = __ldcg(&ctl->err) ? 0 : __ldcg(&ctl->n_seed);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    ctl->t[14] = t;
  }
  unsigned acc_comp = 0;  // statistics, accumulated on lane 0
  int acc_maxn = 0;
  unsigned long long d_cyc = 0ull, d_n = 0ull;  // diagnostics: slowest seed of this warp
  const int nw = gridDim.x * kCompWarps;
  for (int ci = blockIdx.x * kCompWarps + (threadIdx.x >> 5); ci < n_seed; ci += nw) {
    const long long c0 = clock64();
    const int root = __ldg(&w.roots[ci]);
    if (shard_count > 1 && (int)(lowbias32((uint32_t)root) % (uint32_t)shard_count) != shard_index) continue;
#ifdef MPLD_DIAG_DISCOVER
    int dg = 0;
    const int n = warp_discover(g, w, root, s, &dg);
#else
    const int n = warp_discover(g, w, root, s);
#endif
    if (n == -2) continue;  // the seed is not its component's minimum
    ++acc_comp;
    if (n < 0) {
      if (lane == 0) {
        atomicOr(&ctl->err, kErrComponent);
        atomicMax(&ctl->max_comp, kMaxComp + 1);
      }
      continue;
    }
    // pool slot: the returning atomic is issued first, its latency hidden behind the relabelling
    unsigned long long old = 0ull;
    if (lane == 0) old = atomicAdd(&ctl->comp_pool, (1ull << 32) | (unsigned long long)n);
    warp_relabel(s, n);
    old = __shfl_sync(0xffffffffu, old, 0);
    const unsigned off = (unsigned)old;
    const unsigned c = (unsigned)(old >> 32);
    for (int i = lane; i < n; i += 32) {
      w.pmask[2 * ((size_t)off + i)] = s.adj[i];
      w.pmask[2 * ((size_t)off + i) + 1] = s.sadj[i];
      w.porder[off + i] = s.order[i];
    }
    if (lane == 0) {
      w.crec[c] = ((unsigned long long)off << 8) | (unsigned long long)n;
      acc_maxn = max(acc_maxn, n);
      const unsigned long long cyc = (unsigned long long)(clock64() - c0);
      if (cyc > d_cyc) {
        d_cyc = cyc;
#ifdef MPLD_DIAG_DISCOVER
        d_n = n | (dg << 8);
#else
        d_n = n;
#endif
      }
    }
    __syncwarp();
  }
  if (lane == 0 && acc_comp) atomicAdd(&ctl->n_comp, (int)acc_comp);
  if (lane == 0 && acc_maxn > 0) atomicMax(&ctl->max_comp, acc_maxn);
  if (lane == 0 && d_cyc > 0) atomicMax(&ctl->dbg[0], (d_cyc << 16) | (d_n & 0xffffull));  // diagnostics (no return)
}

// One warp per component of the pool: the budgeted sequential search on lane
// 0 (the oracle's node order and budget, R7), then the colours.  Exact mode
// hands components whose search exceeds the light budget to the CTA-parallel
// kernel below.
template <int K>
__global__ void __launch_bounds__(kCompWarps * 32, K >= 4 ? 6 : 8) mpld_exact_cover_search(GraphView g, Workspace w,
                                                                                           int w_stitch,
                                                                                           long long max_steps,
                                                                                           int* colors,
                                                                                           unsigned light_steps) {
  __shared__ WarpSearch s_search[kCompWarps];
  WarpSearch& s = s_search[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  Control* ctl = w.ctl;
  const int n_comp = __ldcg(&ctl->err) ? 0 : (int)(__ldcg(&ctl->comp_pool) >> 32);
  const bool exact = max_steps <= 0;
  const unsigned budget = exact ? light_steps
                                : (max_steps >= (long long)UINT_MAX ? UINT_MAX : (unsigned)max_steps);
  unsigned long long acc_steps = 0ull;  // statistics, accumulated on lane 0
  int acc_maxsteps = 0;
  unsigned acc_trunc = 0;
  unsigned long long d_cyc = 0ull, d_n = 0ull, d_steps = 0ull;  // diagnostics: slowest component of this warp
  const int nw = gridDim.x * kCompWarps;
  for (int ci = blockIdx.x * kCompWarps + (threadIdx.x >> 5); ci < n_comp; ci += nw) {
    const long long c0 = clock64();
    const unsigned long long rec = __ldcg(&w.crec[ci]);
    const size_t off = (size_t)(rec >> 8);
    const int n = (int)(rec & 0xffull);
    for (int i = lane; i < n; i += 32) {
      const ulonglong2 m = __ldcg((const ulonglong2*)&w.pmask[2 * (off + i)]);
      s.adj[i] = m.x;
      s.sadj[i] = m.y;
    }
    __syncwarp();
    unsigned steps = 0;
    bool trunc = false;
    int best_cost = 0;
    if (lane == 0) {
      if (n <= 32)
        steps = comp_dfs<K, unsigned>(s, n, w_stitch, budget, best_cost, trunc);
      else
        steps = comp_dfs<K, unsigned long long>(s, n, w_stitch, budget, best_cost, trunc);
    }
    __syncwarp();
    for (int i = lane; i < n; i += 32) colors[__ldcg(&w.porder[off + i])] = colour_of_mask<K>(s.cl, i);
    trunc = __shfl_sync(0xffffffffu, trunc, 0);
    if (lane == 0) {
      if (trunc && exact) {  // hand the component to the CTA-parallel search
        const int h = atomicAdd(&ctl->n_heavy, 1);
        w.hcomp[h] = ci;
        w.hcost[h] = best_cost;
      } else {
        acc_maxsteps = max(acc_maxsteps, (int)min(steps, (unsigned)INT_MAX));
        acc_trunc += trunc ? 1 : 0;
      }
      acc_steps += steps;
      const unsigned long long cyc = (unsigned long long)(clock64() - c0);
      if (cyc > d_cyc) {
        d_cyc = cyc;
        d_n = n;
        d_steps = steps;
      }
    }
    __syncwarp();
  }
  if (lane == 0 && d_cyc > 0)  // diagnostics (no return): cycles << 24 | steps << 8 | n
    atomicMax(&ctl->dbg[2], (d_cyc << 24) | (min(d_steps, 0xffffull) << 8) | (d_n & 0xffull));
  if (lane == 0 && acc_steps) {
    atomicAdd(&ctl->steps, acc_steps);
    atomicMax(&ctl->max_steps_comp, acc_maxsteps);
    if (acc_trunc) atomicAdd(&ctl->truncated, (int)acc_trunc);
  }
}

// ----------------------------------------------------------------------------
// Exact mode: CTA-parallel search of one heavy component (kHeavyThreads lanes,
// one warp per SM sub-partition, one shared incumbent).
//
// Split nodes are stored as their path from the root — the colour chosen at
// each level, 2 bits per level, depth in the top bits of a 64-bit word — and
// a lane rebuilds a node's state by replaying the path with the column rule
// of R5 (a few mask operations per level), so the level buffers cost 8 bytes
// per node.

#ifndef MPLD_HEAVY_THREADS
#define MPLD_HEAVY_THREADS 128
#endif
#ifndef MPLD_HEAVY_MULT
#define MPLD_HEAVY_MULT 1
#endif
constexpr int kHeavyThreads = MPLD_HEAVY_THREADS;
constexpr int kHeavyTargetNodes = MPLD_HEAVY_MULT * kHeavyThreads;  // subtrees wanted
constexpr int kHeavyCapNodes = 2 * kHeavyTargetNodes;  // level buffer capacity
#ifndef MPLD_HEAVY_STACK_KB
#define MPLD_HEAVY_STACK_KB 32
#endif
constexpr int kHeavyStackBytes = MPLD_HEAVY_STACK_KB * 1024;  // DFS stacks of the lanes (n frames each)
constexpr int kPathDepthShift = 58;
constexpr int kPathMaxDepth = 29;                      // 2 bits per level below the depth field

template <int K, typename W>
struct State {
  W C[K], B[K], U;
  int cost, mu;
};

template <int K, typename W>
__device__ __forceinline__ int select_column(const State<K, W>& s) {  // Alg. 1 line 8 (R5)
  W Z, Ol;
  live_counts<K, W>(s.B, s.U, Z, Ol);
  return WordOps<W>::ffs(Z ? Z : (Ol ? Ol : s.U));
}

// select row r(v, c): cover column v and the row's secondary columns (Alg. 1
// lines 9, 14-15), conflict and stitch cost as in dfs()
template <int K, typename W>
__device__ __forceinline__ void apply_row(State<K, W>& s, int v, int c, const W* adj, const W* sadj, int w_stitch) {
  using O = WordOps<W>;
  const W bit = W(1) << v;
  const W a = adj[v], sa = sadj[v];
  s.U &= ~bit;
  const W Cc = pick<K, W>(s.C, c);
  s.cost += kCostUnits * O::popc(a & Cc) + w_stitch * O::popc(sa & ~s.U & ~Cc);
  put<K, W>(s.C, c, Cc | bit);
  put<K, W>(s.B, c, pick<K, W>(s.B, c) | a);
  s.mu = max(s.mu, c);
}

template <int K, typename W>
__device__ __forceinline__ State<K, W> replay(unsigned long long path, int n, const W* adj, const W* sadj,
                                              int w_stitch) {
  State<K, W> s;
#pragma unroll
  for (int c = 0; c < K; ++c) s.C[c] = s.B[c] = 0;
  s.U = WordOps<W>::full(n);
  s.cost = 0;
  s.mu = -1;
  const int depth = (int)(path >> kPathDepthShift);
  for (int d = 0; d < depth; ++d) apply_row<K, W>(s, select_column<K, W>(s), (int)((path >> (2 * d)) & 3ull), adj, sadj, w_stitch);
  return s;
}

// children of a split node: 0 = pruned against the light-phase incumbent c1
// (its leaf precedes every subtree), 1 for a leaf (carried as itself), else
// min(K, mu + 2) (R4 with the colour-symmetry limit R6)
template <int K, typename W>
__device__ __forceinline__ int split_children(const State<K, W>& s, const W* cl, int ncl, int c1) {
  if (s.U == 0) return 1;
  W Z, Ol;
  live_counts<K, W>(s.B, s.U, Z, Ol);
  if (s.cost + kCostUnits * bound_conflicts<K, W>(s.B, s.U, Z, cl, 1, ncl) >= c1) return 0;
  return min(K - 1, s.mu + 1) + 1;
}

__device__ __forceinline__ int block_excl_scan(int x, int& total, int* s_tmp) {  // s_tmp: 32 ints
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int y = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int z = __shfl_up_sync(0xffffffffu, y, o);
    if (lane >= o) y += z;
  }
  if (lane == 31) s_tmp[wid] = y;
  __syncthreads();
  int base = 0;
  total = 0;
  for (int i = 0; i < nw; ++i) {
    const int t = s_tmp[i];
    if (i < wid) base += t;
    total += t;
  }
  __syncthreads();
  return base + y - x;
}

template <int K, typename W>
__device__ void heavy_component(int n, const int* s_order, const unsigned long long* s_adj64,
                                const unsigned long long* s_sadj64, unsigned char* smem, int w_stitch, int c1,
                                int* colors, Control* ctl) {
  const int tid = threadIdx.x;
  W* s_adj = (W*)smem;
  W* s_sadj = s_adj + kMaxComp;
  W* s_cl = s_sadj + kMaxComp;
  unsigned long long* lvl[2];
  lvl[0] = (unsigned long long*)(smem + 3 * kMaxComp * sizeof(unsigned long long));
  lvl[1] = lvl[0] + kHeavyCapNodes;
  Frame<W>* stack_base = (Frame<W>*)(lvl[1] + kHeavyCapNodes);
  __shared__ unsigned long long s_best;
  __shared__ unsigned long long s_win;
  __shared__ int s_next, s_ncl, s_flag, s_tmp[32];
  __shared__ unsigned long long s_red[32];
  for (int i = tid; i < n; i += blockDim.x) {
    s_adj[i] = (W)s_adj64[i];
    s_sadj[i] = (W)s_sadj64[i];
  }
  __syncthreads();
  if (tid == 0) {
    s_ncl = clique_min<K>() ? clique_partition<W>(s_adj, 1, n, s_cl, 1, clique_min<K>()) : 0;
    lvl[0][0] = 0ull;  // the root: depth 0
    s_best = (unsigned long long)c1 << 32;  // the light-phase leaf precedes every subtree (key f+1 = 0)
    s_next = 0;
  }
  __syncthreads();
  const int ncl = s_ncl;
  const long long hc0 = clock64();
  // level-synchronous split of the canonical tree, DFS order preserved
  int m = 1, cur = 0;
  unsigned expanded = 0;
#ifdef MPLD_HEAVY_DIAG_SEQ
  while (false) {
#else
  while (m < kHeavyTargetNodes) {
#endif
    int total = 0;
    if (tid == 0) s_flag = 0;  // bit 0: some node still has uncovered columns; bit 1: depth limit reached
    __syncthreads();
    for (int i0 = 0; i0 < m; i0 += blockDim.x) {
      const int i = i0 + tid;
      unsigned long long path = 0ull;
      int cnt = 0, depth = 0;
      State<K, W> st;
      if (i < m) {
        path = lvl[cur][i];
        depth = (int)(path >> kPathDepthShift);
        st = replay<K, W>(path, n, s_adj, s_sadj, w_stitch);
        cnt = split_children<K, W>(st, s_cl, ncl, c1);
        if (st.U != 0 && cnt > 0) atomicOr(&s_flag, depth + 1 >= kPathMaxDepth ? 3 : 1);
      }
      int t;
      const int off = block_excl_scan(cnt, t, s_tmp);
      if (total + t <= kHeavyCapNodes && cnt > 0) {
        unsigned long long* out = &lvl[cur ^ 1][total + off];
        if (st.U == 0) {
          out[0] = path;
        } else {
          const unsigned long long base = (path & ((1ull << kPathDepthShift) - 1)) |
                                          ((unsigned long long)(depth + 1) << kPathDepthShift);
          for (int c = 0; c < cnt; ++c) out[c] = base | ((unsigned long long)c << (2 * depth));
        }
      }
      total += t;
    }
    __syncthreads();
    const int flag = s_flag;
    if (total == 0) {
      m = 0;
      break;
    }
    if (total > kHeavyCapNodes || !(flag & 1) || (flag & 2)) break;
    expanded += m;
    cur ^= 1;
    m = total;
  }
  const long long hc1 = clock64();
  // lanes search the subtrees in DFS order with a shared incumbent; the stack
  // region holds n frames per active lane
#ifdef MPLD_HEAVY_DIAG_SEQ
  const int lanes = 1;
#else
  const int lanes = min((int)blockDim.x, (int)(kHeavyStackBytes / (n * (int)sizeof(Frame<W>))));
#endif
  W bestC[K];
#pragma unroll
  for (int c = 0; c < K; ++c) bestC[c] = 0;
  unsigned long long my_best = ~0ull;
  unsigned steps = 0;
  bool capped = false;
  if (tid < lanes) {
    while (true) {
      const int f = atomicAdd(&s_next, 1);
      if (f >= m) break;
      if (steps >= kHeavyLaneCap) {  // safety cap of exact mode: skip, flag as truncated
        capped = true;
        continue;
      }
      State<K, W> st = replay<K, W>(lvl[cur][f], n, s_adj, s_sadj, w_stitch);
      ParIncumbent inc;
      inc.shared_best = &s_best;
      inc.fkey = (unsigned long long)(f + 1);
      inc.lane_best = my_best;
      bool trunc;
      steps += dfs<K, W, ParIncumbent>(s_adj, s_sadj, 1, st.C, st.B, st.U, st.cost, st.mu, w_stitch,
                                       kHeavyLaneCap - steps, stack_base + tid, lanes, s_cl, 1, ncl, inc, bestC,
                                       trunc);
      my_best = inc.lane_best;
      capped |= trunc;
    }
  }
  // the minimum key over lanes is the canonical leaf
  const int lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  unsigned long long wmin = my_best;
  unsigned total_steps = steps;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long y = __shfl_xor_sync(0xffffffffu, wmin, o);
    wmin = y < wmin ? y : wmin;
    total_steps += __shfl_xor_sync(0xffffffffu, total_steps, o);
  }
  const int any_capped = __syncthreads_or(capped);
#ifdef MPLD_DIAG_LANESTEPS
  __shared__ unsigned s_maxsteps;
  if (tid == 0) s_maxsteps = 0;
  __syncthreads();
  atomicMax(&s_maxsteps, steps);
  __syncthreads();
#endif
  if (lane == 0) {
    s_red[wid] = wmin;
    s_tmp[wid] = (int)total_steps;
  }
  __syncthreads();
  if (tid == 0) {
    unsigned long long w = ~0ull;
    unsigned ts = 0;
    for (int i = 0; i < nw; ++i) {
      w = s_red[i] < w ? s_red[i] : w;
      ts += (unsigned)s_tmp[i];
    }
    s_win = w;
    if (any_capped) atomicAdd(&ctl->truncated, 1);
    atomicAdd(&ctl->steps, (unsigned long long)(ts + expanded));
    atomicMax(&ctl->max_steps_comp, (int)min(ts + expanded, (unsigned)INT_MAX));
    const long long hc2 = clock64();
    if ((unsigned long long)(hc2 - hc0) > ctl->dbg[5]) {  // diagnostics (racy by design)
      atomicMax(&ctl->dbg[5], (unsigned long long)(hc2 - hc0));
#ifdef MPLD_DIAG_LANESTEPS
      ctl->dbg[6] = ((unsigned long long)s_maxsteps << 32) | (unsigned)(ts + expanded);
#else
      ctl->dbg[6] = hc1 - hc0;
#endif
      ctl->dbg[7] = ((unsigned long long)m << 32) | (unsigned)n;
    }
  }
  __syncthreads();
  const unsigned long long win = s_win;
  if (win != ~0ull && my_best == win && win < ((unsigned long long)c1 << 32)) {  // keys are unique per subtree
    for (int i = 0; i < n; ++i) colors[s_order[i]] = colour_of<K, W>(bestC, i);
  }
}

template <int K>
__global__ void __launch_bounds__(kHeavyThreads) mpld_exact_cover_search_heavy(GraphView g, Workspace w, int w_stitch,
                                                                               int* colors) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_order[kMaxComp];
  __shared__ unsigned long long s_adj64[kMaxComp], s_sadj64[kMaxComp];
  Control* ctl = w.ctl;
  const int n_heavy = __ldcg(&ctl->n_heavy);
  for (int h = blockIdx.x; h < n_heavy; h += gridDim.x) {
    const int c1 = __ldcg(&w.hcost[h]);
    const unsigned long long rec = __ldcg(&w.crec[__ldcg(&w.hcomp[h])]);
    const size_t off = (size_t)(rec >> 8);
    const int n = (int)(rec & 0xffull);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      s_order[i] = __ldcg(&w.porder[off + i]);
      s_adj64[i] = __ldcg(&w.pmask[2 * (off + i)]);
      s_sadj64[i] = __ldcg(&w.pmask[2 * (off + i) + 1]);
    }
    __syncthreads();
    if (n <= 32)
      heavy_component<K, unsigned>(n, s_order, s_adj64, s_sadj64, smem, w_stitch, c1, colors, ctl);
    else
      heavy_component<K, unsigned long long>(n, s_order, s_adj64, s_sadj64, smem, w_stitch, c1, colors, ctl);
    __syncthreads();
  }
}

}  // namespace

cudaError_t launch_discover(const GraphView& g, Workspace ws, int shard_index, int shard_count, cudaStream_t s,
                            int blocks) {
  mpld_component_discover<<<blocks, kCompWarps * 32, 0, s>>>(g, ws, shard_index, shard_count);
  return cudaGetLastError();
}

cudaError_t launch_search(const GraphView& g, Workspace ws, int k, int w_stitch, long long max_steps, int* colors,
                          unsigned light_steps, cudaStream_t s, int blocks) {
  switch (k) {
    case 2:
      mpld_exact_cover_search<2><<<blocks, kCompWarps * 32, 0, s>>>(g, ws, w_stitch, max_steps, colors, light_steps);
      break;
    case 3:
      mpld_exact_cover_search<3><<<blocks, kCompWarps * 32, 0, s>>>(g, ws, w_stitch, max_steps, colors, light_steps);
      break;
    case 4:
      mpld_exact_cover_search<4><<<blocks, kCompWarps * 32, 0, s>>>(g, ws, w_stitch, max_steps, colors, light_steps);
      break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

size_t heavy_smem_bytes() {
  return 3 * kMaxComp * sizeof(unsigned long long) + 2 * kHeavyCapNodes * sizeof(unsigned long long) +
         kHeavyStackBytes;
}

cudaError_t launch_search_heavy(const GraphView& g, Workspace ws, int k, int w_stitch, int* colors, cudaStream_t s,
                                int blocks) {
  const size_t smem = heavy_smem_bytes();
  switch (k) {
    case 2: mpld_exact_cover_search_heavy<2><<<blocks, kHeavyThreads, smem, s>>>(g, ws, w_stitch, colors); break;
    case 3: mpld_exact_cover_search_heavy<3><<<blocks, kHeavyThreads, smem, s>>>(g, ws, w_stitch, colors); break;
    case 4: mpld_exact_cover_search_heavy<4><<<blocks, kHeavyThreads, smem, s>>>(g, ws, w_stitch, colors); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

int resident_blocks_heavy(int num_sms) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mpld_exact_cover_search_heavy<4>, kHeavyThreads,
                                                heavy_smem_bytes());
  return per_sm * num_sms;
}

cudaError_t configure_search_heavy() {
  const int smem = (int)heavy_smem_bytes();
  cudaError_t e = cudaSuccess;
  e = cudaFuncSetAttribute(mpld_exact_cover_search_heavy<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(mpld_exact_cover_search_heavy<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(mpld_exact_cover_search_heavy<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  return e;
}

int resident_blocks_discover(int num_sms) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mpld_component_discover, kCompWarps * 32, 0);
  return per_sm * num_sms;
}

int resident_blocks_search(int threads, int num_sms) {
  (void)threads;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mpld_exact_cover_search<4>, kCompWarps * 32, 0);
  return per_sm * num_sms;
}

}  // namespace mpld
