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
// Kernels:
//   mpld_component_discover           one warp per component seed: warp-parallel
//                                     discovery of the component and relabelling
//                                     to the R5 column order into the pool;
//   mpld_exact_cover_search<K>        the sequential DFS of R4-R7 (the oracle's
//                                     node order and budget), one component per
//                                     lane, 32 per warp (larger than 32 vertices:
//                                     lane 0 alone);
//   mpld_exact_cover_search_heavy<K,W> exact mode (max_steps <= 0) only: one warp
//                                     per component whose sequential search
//                                     needed more than the light budget; lanes
//                                     search disjoint parts of the canonical tree
//                                     with work donation and a (cost, leaf path)
//                                     incumbent, very large searches spill their
//                                     open work to a GPU-wide queue; the first
//                                     optimal leaf of R7 is recovered exactly
//                                     (DESIGN.md §1);
//   mpld_partition_*                  the cost-balanced shard partition (scan).
#include <algorithm>
#include <climits>

#include "mpld_internal.cuh"
#include "lane_search.cuh"

namespace mpld {

namespace {

constexpr unsigned kHeavyLaneCap = 1u << 22;  // exact mode safety cap: search nodes per lane per component

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

// Adds a component's Eq. (1b)/(1c) counts to its layout (the whole warp calls;
// nc, ns = per-lane sums over the vertices, each edge seen from both ends).
// The recovery never adds a conflict (R9) and stitch vertices are
// never hidden (R8), so these are the layout's final counts.
__device__ __forceinline__ void add_counts(const GraphView& g, int v0, int nc, int ns, long long* counts) {
  nc = __reduce_add_sync(0xffffffffu, nc) >> 1;
  ns = __reduce_add_sync(0xffffffffu, ns) >> 1;
  if ((threadIdx.x & 31) == 0 && (nc | ns)) {
    const int l = layout_of(g, v0);
    if (nc) atomicAdd((unsigned long long*)&counts[2 * l], (unsigned long long)nc);
    if (ns) atomicAdd((unsigned long long*)&counts[2 * l + 1], (unsigned long long)ns);
  }
}

// One warp per component seed: discovery, relabelling to the R5 column order
// and the component's record in the pool (exactly one per component: the seed
// that is its minimum).  Low register use, so 64 warps per SM discover at once.
__global__ void __launch_bounds__(kCompWarps * 32, 16) mpld_component_discover(GraphView g, Workspace w, int k,
                                                                              int sharded) {
  pdl_begin();
  if (gated_off(w)) return;
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

  int acc_maxn = 0;
  unsigned long long d_cyc = 0ull, d_n = 0ull;  // diagnostics: slowest seed of this warp
  const int nw = gridDim.x * kCompWarps;
  for (int ci = blockIdx.x * kCompWarps + (threadIdx.x >> 5); ci < n_seed; ci += nw) {
    const long long c0 = clock64();
    const int root = __ldg(&w.roots[ci]);
#ifdef MPLD_DIAG_DISCOVER
    int dg = 0;
    const int n = warp_discover(g, w, root, s, &dg);
#else
    const int n = warp_discover(g, w, root, s);
#endif
    if (n == -2) continue;  // the seed is not its component's minimum

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
      if (sharded) w.est[root] = partition_estimate(n, k);  // the balanced partition (scan, then light search)
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
  if (lane == 0 && acc_maxn > 0) atomicMax(&ctl->max_comp, acc_maxn);
  if (MPLD_DIAG && lane == 0 && d_cyc > 0) atomicMax(&ctl->dbg[0], (d_cyc << 16) | (d_n & 0xffffull));
}


// Cm: compact frames (no stored node cost; budgeted mode's long searches:
// more resident warps), else the stored cost (exact mode's 48-node searches:
// fewer instructions per pop)
template <int K, bool Cm>
__global__ void __launch_bounds__(kLaneWarps * 32) mpld_exact_cover_search(GraphView g, Workspace w, int w_stitch,
                                                                           long long max_steps, int* colors,
                                                                           unsigned light_steps, long long* counts,
                                                                           int shard_index, int shard_count) {
  pdl_begin();
  if (gated_off(w)) return;
  using Store = LaneStore<unsigned, 32, Cm>;
  __shared__ Store s_lane[kLaneWarps];
  Store& L = s_lane[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  Control* ctl = w.ctl;
  const int n_comp = __ldcg(&ctl->err) ? 0 : (int)(__ldcg(&ctl->comp_pool) >> 32);
  const bool exact = max_steps <= 0;
  const unsigned budget = light_budget(max_steps, light_steps);
  LightAcc acc;  // this lane's statistics
  const int nb = gridDim.x * kLaneWarps;
  for (int b = blockIdx.x * kLaneWarps + (threadIdx.x >> 5); b * 32 < n_comp; b += nb) {
    const int ci = b * 32 + lane;
    unsigned long long rec = 0ull;
    if (ci < n_comp) rec = __ldcg(&w.crec[ci]);
    const size_t off = (size_t)(rec >> 8);
    const int n = (int)(rec & 0xffull);
    const bool mine_c = ci < n_comp && in_shard(g, w, __ldcg(&w.porder[off]), n, K, shard_index, shard_count);
    acc.comps += mine_c ? 1 : 0;
    // components of more than 32 vertices: listed for the 64-bit lane kernel
    // (budgeted mode), or handed to the warp-parallel search unsearched (exact
    // mode: the light budget would not finish them; the heavy search starts
    // from a greedy colouring)
    const bool wide = mine_c && n > 32;
    if (wide && exact) light_handoff(g, w, ci, n, INT_MAX);
    const unsigned wm = __ballot_sync(0xffffffffu, wide && !exact);
    if (wm) {
      int base = 0;
      if (lane == 0) base = atomicAdd(&ctl->n_wide, __popc(wm));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (wide && !exact) w.wide[base + __popc(wm & lanemask_lt())] = ci;
    }
    lane_component<K, unsigned, 32, kStagedLight>(g, w, L, lane, ci < n_comp, mine_c && n <= 32, ci, rec, w_stitch,
                                                  budget, exact, colors, counts, acc);
    __syncwarp();
  }
  light_stats(ctl, acc);
}

// The components of more than 32 vertices (listed by the kernel above), one
// per lane on 64-bit words; one warp per CTA (LaneWide is 56 KB of shared memory: 4 per SM).
template <int K>
__global__ void __launch_bounds__(32) mpld_exact_cover_search_wide(GraphView g, Workspace w, int w_stitch,
                                                                   long long max_steps, int* colors,
                                                                   unsigned light_steps, long long* counts) {
  pdl_begin();
  if (gated_off(w)) return;
  extern __shared__ __align__(16) unsigned char smem[];
  LaneWide& L = *reinterpret_cast<LaneWide*>(smem);
  const int lane = threadIdx.x & 31;
  Control* ctl = w.ctl;
  const int n_wide = __ldcg(&ctl->err) ? 0 : __ldcg(&ctl->n_wide);
  const bool exact = max_steps <= 0;
  const unsigned budget = light_budget(max_steps, light_steps);
  LightAcc acc;
  for (int b = blockIdx.x; b * 32 < n_wide; b += gridDim.x) {
    const int j = b * 32 + lane;
    const int ci = j < n_wide ? __ldcg(&w.wide[j]) : -1;
    const unsigned long long rec = ci >= 0 ? __ldcg(&w.crec[ci]) : 0ull;
    lane_component<K, unsigned long long, kMaxComp, false>(g, w, L, lane, ci >= 0, ci >= 0, ci, rec, w_stitch,
                                                           budget, exact, colors, counts, acc);
    __syncwarp();
  }
  acc.comps = 0;  // counted by the kernel that listed them
  light_stats(ctl, acc);
}

// ----------------------------------------------------------------------------
// Exact mode: warp-parallel search of one heavy component with work donation.
//
// The result of R7 is the first minimum-cost leaf in the canonical (DFS) order.
// Every leaf sits at depth n and the DFS visits leaves in lexicographic order
// of their colour-choice sequences, so the result is the leaf with the minimum
// key (cost, path), path = the choices, 2 bits per level, level 0 most
// significant — whatever order the tree is explored in.  A node with lower
// bound lb and path prefix p can only hold leaves with keys >= (lb, p·00…0),
// so it is pruned iff that key >= the best key found: a leaf that beats the
// incumbent is never cut.
//
// The 32 lanes of a warp run independent DFSs over disjoint parts of the tree.
// Lane 0 starts at the root; at the top of every iteration each idle lane takes
// one node from a busy lane: the donor gives away the LAST untried child of its
// shallowest frame that still has one (shrinking that frame's child limit), as
// a path, and the thief rebuilds the node's state by replaying the path with
// the column rule of R5.  The best key is shared through warp shuffles whenever
// a lane finds a better leaf.  The light phase's best leaf (cost c1, found in
// the first light_steps nodes) is the starting incumbent: its path is rebuilt
// from the colours the light kernel wrote.
#ifndef MPLD_DONATE_MIN_LEVELS
#define MPLD_DONATE_MIN_LEVELS 0
#endif
constexpr int kDonateMinLevels = MPLD_DONATE_MIN_LEVELS;  // a frame is donated from only if n - depth >= this
#ifndef MPLD_STEAL_MIN_IDLE
#define MPLD_STEAL_MIN_IDLE 8
#endif
constexpr int kStealMinIdle = MPLD_STEAL_MIN_IDLE;  // donation rounds only when at least this many lanes are idle
#ifndef MPLD_SPILL
#define MPLD_SPILL 1
#endif
#ifndef MPLD_SPILL_LARGE
#define MPLD_SPILL_LARGE 64  // spill threshold of components of >= kHelpersMinN vertices
#endif
#ifndef MPLD_POLL_CAP
#define MPLD_POLL_CAP 512
#endif

#ifndef MPLD_QUEUE_LOW
#define MPLD_QUEUE_LOW 64
#endif
constexpr int kQueueLow = MPLD_QUEUE_LOW;
#ifndef MPLD_SEED_INCUMBENT
#define MPLD_SEED_INCUMBENT 1
#endif
constexpr bool kSeedIncumbent = MPLD_SEED_INCUMBENT != 0;  // greedy starting incumbent of heavy components
#ifndef MPLD_SEED_MIN_N
#define MPLD_SEED_MIN_N 0  // ... of at least this many vertices (smaller ones start from their light leaf)
#endif
#ifndef MPLD_PAIR_BOUND
#define MPLD_PAIR_BOUND 0  // measured slower (configs[2] 1.24-1.34 -> 1.56-1.62 ms, configs[1] +10 us): off
#endif
constexpr bool kPairBound = MPLD_PAIR_BOUND != 0;  // exact mode: the matching term of the lower bound  // the work queue is fed while it holds fewer items than this
#ifndef MPLD_HELPER_DIV
#define MPLD_HELPER_DIV 2  // helpers waiting for spilled work: gridDim.x / this
#endif
#ifndef MPLD_SPILL_CHECK
#define MPLD_SPILL_CHECK 64
#endif
constexpr unsigned kSpillCheck = MPLD_SPILL_CHECK;  // spill / slot-sync checks every this many iterations (power of two),
                                      // from Workspace::spill_iters on

struct Path {  // levels 0..31 in a, 32..63 in b; 2 bits per level, level 0 most significant
  unsigned long long a, b;
};

// kTwo: 64-level paths (components of more than 32 vertices); else only word a is used
template <bool kTwo = true>
__device__ __forceinline__ void path_put(Path& P, int d, int c) {
  const int sh = 62 - 2 * (d & 31);
  if (!kTwo || d < 32)
    P.a = (P.a & ~(3ull << sh)) | ((unsigned long long)c << sh);
  else
    P.b = (P.b & ~(3ull << sh)) | ((unsigned long long)c << sh);
}

template <bool kTwo = true>
__device__ __forceinline__ Path path_prefix(const Path& P, int j) {  // levels < j kept, the rest zero
  Path r;
  r.a = j <= 0 ? 0ull : (j >= 32 ? P.a : (P.a & (~0ull << (64 - 2 * j))));
  r.b = !kTwo || j <= 32 ? 0ull : (j >= 64 ? P.b : (P.b & (~0ull << (64 - 2 * (j - 32)))));
  return r;
}

template <bool kTwo = true>
__device__ __forceinline__ bool key_less(int c1, const Path& p1, int c2, const Path& p2) {
  if (c1 != c2) return c1 < c2;
  if (!kTwo || p1.a != p2.a) return p1.a < p2.a;
  return p1.b < p2.b;
}

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

// warp-wide minimum of the lanes' keys (cost, path), by 32-bit warp reductions
// (REDUX): the cost first, then each path word among the lanes still tied.
// Every lane receives the minimum; returns the lowest lane holding it.
template <bool kTwo>
__device__ __forceinline__ int warp_min_key(int& c, Path& p) {
  const int mc = (int)(__reduce_min_sync(0xffffffffu, (unsigned)c ^ 0x80000000u) ^ 0x80000000u);  // signed order
  bool tie = c == mc;
  unsigned words[4] = {(unsigned)(p.a >> 32), (unsigned)p.a, (unsigned)(p.b >> 32), (unsigned)p.b};
  unsigned best[4] = {0u, 0u, 0u, 0u};
#pragma unroll
  for (int i = 0; i < (kTwo ? 4 : 2); ++i) {
    best[i] = __reduce_min_sync(0xffffffffu, tie ? words[i] : 0xffffffffu);
    tie = tie && words[i] == best[i];
  }
  c = mc;
  p.a = ((unsigned long long)best[0] << 32) | best[1];
  p.b = kTwo ? (((unsigned long long)best[2] << 32) | best[3]) : 0ull;
  return __ffs(__ballot_sync(0xffffffffu, tie)) - 1;
}

// Frames of the lanes in shared memory, [field][depth][lane] (a lane only
// touches its own column: conflict-free).  Frame d is the node N_d at which
// column v_d was selected: saved = B[c] before its current child r(v_d, c)
// was selected, and the 16-bit state v | (c+1) << 6 | (maxused+1) << 9 |
// lim << 12 (current child c, child limit lim of R6).  The node's cost is not
// stored: popping back to N_d subtracts the cost of the row r(v_d, c) from
// the child's cost.  The masks and cost of N_j (for a donation or a spill) are
// rebuilt from the lane's current state by undoing the frames below j
// (node_at); the deepest frame lives in registers.
template <int K, typename W, int D>
struct LaneFrames {
  W saved[D][32];
  unsigned short pk[D][32];
};

__device__ __forceinline__ int pk16(int v, int c, int mu, int lim) {
  return v | ((c + 1) << 6) | ((mu + 1) << 9) | (lim << 12);
}
__device__ __forceinline__ int pk_v(int p) { return p & 63; }
__device__ __forceinline__ int pk_c(int p) { return ((p >> 6) & 7) - 1; }
__device__ __forceinline__ int pk_mu(int p) { return ((p >> 9) & 7) - 1; }
__device__ __forceinline__ int pk_lim(int p) { return p >> 12; }

// Eq. (1) cost of selecting row r(v, c) (Alg. 1 lines 14-15) with colour
// masks C and uncovered columns U: conflicts with neighbours coloured c,
// stitches to neighbours coloured otherwise.
template <typename W>
__device__ __forceinline__ int row_cost(W a, W sa, W Cc, W U, int w_stitch) {
  return kCostUnits * WordOps<W>::popc(a & Cc) + w_stitch * WordOps<W>::popc(sa & ~U & ~Cc);
}

// B, C, U and the cost at N_j from the lane's state at depth `depth` (frames
// j..depth-2 in shared memory, frame depth-1 in registers: f_saved, f_v, f_c,
// f_cost = cost of N_{depth-1}): undo the selected rows of frames depth-1 down
// to j, uncover their columns, subtract their row costs.
template <int K, typename W, int D>
__device__ __forceinline__ void node_at(int j, int depth, const W (&B)[K], const W (&C)[K], W U, W f_saved, int f_v,
                                        int f_c, int f_cost, const LaneFrames<K, W, D>& F, int lane, const W* adj,
                                        const W* sadj, int w_stitch, W (&jB)[K], W (&jC)[K], W& jU, int& jcost) {
#pragma unroll
  for (int c = 0; c < K; ++c) {
    jB[c] = B[c];
    jC[c] = C[c];
  }
  const W fbit = W(1) << f_v;
  if (f_c >= 0) {
    put<K, W>(jB, f_c, f_saved);
    put<K, W>(jC, f_c, pick<K, W>(jC, f_c) & ~fbit);
  }
  jU = U | fbit;
  jcost = f_cost;
  for (int d = depth - 2; d >= j; --d) {  // frames above the deepest always have a selected child
    const int pk = F.pk[d][lane];
    const int v = pk_v(pk), c = pk_c(pk);
    const W bit = W(1) << v;
    put<K, W>(jB, c, F.saved[d][lane]);
    const W Cc = pick<K, W>(jC, c) & ~bit;
    put<K, W>(jC, c, Cc);
    jU |= bit;
    jcost -= row_cost<W>(adj[v], sadj[v], Cc, jU, w_stitch);  // the row that led from N_d to N_{d+1}
  }
}

template <int K, typename W>
__host__ __device__ constexpr int heavy_depth() {
  return sizeof(W) == 4 ? 32 : 64;
}

template <int K, typename W>
__host__ __device__ constexpr size_t heavy_smem() {
  return 3 * kMaxComp * sizeof(W) + sizeof(LaneFrames<K, W, heavy_depth<K, W>()>);
}

// One work unit of the warp-parallel search: the subtree of one node (the root
// of a heavy component, or a spilled work item) searched by the warp's 32
// lanes with work donation.  The incumbent key (gcost, gP) is in/out; on
// return `mine` marks the lane that recorded the best leaf (bestC).  A unit
// that runs past kSpillIters iterations hands its open work to the work queue
// (`spilled`).
template <int K, typename W>
struct HeavyUnit {
  int n, ncl, w_stitch, cls, ci;
  int slot;  // spilled component's slot, -1 before the first spill
  const W* adj;
  const W* sadj;
  const W* cl;
  LaneFrames<K, W, heavy_depth<K, W>()>* F;
  int* pair;  // 32 ints: donor pairing table
  int c1;     // the light phase's leaf: key and colour masks (component units; slot initialisation)
  Path p1;
  W col[K];
  int hc;     // the starting incumbent's cost: min(c1, greedy seed) (a leaf of that cost exists)
};

__device__ __forceinline__ void slot_lock(HeavySlot* s) {
  while (atomicCAS(&s->lock, 0, 1) != 0) __nanosleep(32);
  __threadfence();
}
__device__ __forceinline__ void slot_unlock(HeavySlot* s) {
  __threadfence();
  atomicExch(&s->lock, 0);
}

template <int K, typename W>
__device__ void warp_heavy_search(HeavyUnit<K, W>& u, const Workspace& w, const W (&sC)[K], const W (&sB)[K], W sU,
                                  int scost, int smu, Path sP, int sdepth, int& gcost, Path& gP, bool& mine,
                                  W (&bestC)[K], unsigned& steps_out, bool& capped_out, bool& spilled,
                                  unsigned* iters_out = nullptr) {
  using O = WordOps<W>;
  constexpr bool kTwo = sizeof(W) == 8;
  const int lane = threadIdx.x & 31;
  const int n = u.n, ncl = u.ncl, w_stitch = u.w_stitch;
  const W* __restrict__ adj = u.adj;
  const W* __restrict__ sadj = u.sadj;
  const W* cl = u.cl;
  auto& F = *u.F;
  int* slot = u.pair;
  W clu = 0;  // the cliques' union (the clique term is summed only when it can change a decision)
  for (int q = 0; q < ncl; ++q) clu |= cl[q];
  const unsigned long long donatable = (n - kDonateMinLevels) >= 64 ? ~0ull
                                       : (n - kDonateMinLevels <= 0 ? 0ull : ((1ull << (n - kDonateMinLevels)) - 1ull));
  unsigned iters = 0;
  spilled = false;
  // large components (the ones idle warps stay for) feed the queue early
  const unsigned spill_at = n >= kHelpersMinN ? min(w.spill_iters, (unsigned)MPLD_SPILL_LARGE) : w.spill_iters;
  // lane DFS state: the node (C, B, U, cost, maxused) and its path P; frames
  // d0..depth-1, the deepest in registers; open bit d = frame d has an untried
  // child beyond its current one.  Lane 0 starts at the unit's node.
  W C[K], B[K], U = lane == 0 ? sU : W(0);
#pragma unroll
  for (int c = 0; c < K; ++c) {
    C[c] = lane == 0 ? sC[c] : W(0);
    B[c] = lane == 0 ? sB[c] : W(0);
  }
  int cost = scost, maxused = smu, depth = sdepth, d0 = sdepth;
  bool active = lane == 0, enter = lane == 0;
  W f_saved = 0, f_adj = 0, f_sadj = 0;
  int f_cost = 0, f_v = 0, f_c = -1, f_mu = -1, f_lim = 0;
  Path P = sP;
  unsigned long long open = 0ull;
  // incumbent: the warp's best key (identical in every lane); a lane records a
  // leaf only if it beats it, so only the lane that found the current best
  // holds colours for it
  mine = false;
#pragma unroll
  for (int c = 0; c < K; ++c) bestC[c] = 0;
  unsigned steps = 0;
  bool capped = false;
  bool all_idle = false;
  while (!all_idle) {
   // a compact inner loop of kSpillCheck iterations; the work-queue check between
   for (unsigned inner = 0; inner < kSpillCheck; ++inner) {
    const unsigned act = __ballot_sync(0xffffffffu, active);
    if (act == 0u) {
      all_idle = true;
      break;
    }
    ++iters;
    if (__popc(~act) >= kStealMinIdle) {  // work donation: the i-th idle lane takes a node from the i-th donor
      const unsigned don = __ballot_sync(0xffffffffu, active && (open & donatable) != 0ull);
      if (don) {

        const unsigned idle = ~act;
        const int np = min(__popc(don), __popc(idle));
        const unsigned lt = lanemask_lt();
        // donor: the last untried child of its shallowest open frame j, built
        // from the frame's masks (C at N_j = C & ~U_j)
        W xC[K], xB[K], xU = 0;
        int xcost = 0, xmu = 0, xd = 0;
        Path xP = {0ull, 0ull};
        if (((don >> lane) & 1u) && __popc(don & lt) < np) {
          const int j = __ffsll((long long)(open & donatable)) - 1;
          int pk, jc;
          W jU;
          node_at<K, W, heavy_depth<K, W>()>(j, depth, B, C, U, f_saved, f_v, f_c, f_cost, F, lane, adj, sadj,
                                             w_stitch, xB, xC, jU, jc);
          if (j == depth - 1) {
            pk = pk16(f_v, f_c, f_mu, f_lim);
            f_lim -= 1;
          } else {
            pk = F.pk[j][lane];
            F.pk[j][lane] = (unsigned short)(pk - (1 << 12));
          }
          const int v = pk_v(pk), cj = pk_c(pk), mu = pk_mu(pk), lim = pk_lim(pk);
          if (cj >= lim - 1) open &= ~(1ull << j);
          const W bit = W(1) << v;
          const W a = adj[v], sa = sadj[v];
          xU = jU & ~bit;
          const W Cc = pick<K, W>(xC, lim);
          xcost = jc + row_cost<W>(a, sa, Cc, xU, w_stitch);
          put<K, W>(xC, lim, Cc | bit);
          put<K, W>(xB, lim, pick<K, W>(xB, lim) | a);
          xmu = max(mu, lim);
          xP = path_prefix<kTwo>(P, j);
          path_put<kTwo>(xP, j, lim);
          xd = j + 1;
        }
        const bool take = !active && __popc(idle & lt) < np;
        // pair the i-th idle lane with the i-th donor through the warp's slot table
        if (((don >> lane) & 1u) && __popc(don & lt) < np) slot[__popc(don & lt)] = lane;
        __syncwarp();
        const int src = take ? slot[__popc(idle & lt)] : lane;
        __syncwarp();
#pragma unroll
        for (int c = 0; c < K; ++c) {
          xC[c] = __shfl_sync(0xffffffffu, xC[c], src);
          xB[c] = __shfl_sync(0xffffffffu, xB[c], src);
        }
        xU = __shfl_sync(0xffffffffu, xU, src);
        xcost = __shfl_sync(0xffffffffu, xcost, src);
        xmu = __shfl_sync(0xffffffffu, xmu, src);
        xd = __shfl_sync(0xffffffffu, xd, src);
        xP.a = __shfl_sync(0xffffffffu, xP.a, src);
        if (kTwo) xP.b = __shfl_sync(0xffffffffu, xP.b, src);
        if (take) {
#pragma unroll
          for (int c = 0; c < K; ++c) {
            C[c] = xC[c];
            B[c] = xB[c];
          }
          U = xU;
          cost = xcost;
          maxused = xmu;
          P = xP;
          depth = d0 = xd;
          open = 0ull;
          active = enter = true;
        }
      }
    }
    // One DFS event per lane, written branch-free (both outcomes computed,
    // committed with selects) so that lanes in different states do not
    // serialise: enter the pending node (leaf / prune / expand), then advance
    // the deepest frame (next child / exhausted: pop).
    bool found = false;
    const bool en = active && enter;
    if (en && ++steps > kHeavyLaneCap) {  // exact-mode safety cap: drop this lane's work, flag the component
      capped = true;
      active = false;
    }
    {
      W Z, Ol;
      live_counts<K, W>(B, U, Z, Ol);
      // bound (R7): the clique deficit is at most the live columns inside
      // cliques, so it is summed only when it can change the key comparison
      // exact mode may prune with any valid lower bound: R7's, plus (kPairBound)
      // a matching of adjacent columns whose only live row has the same mask
      // (each such pair costs >= one more conflict, on edges no other term
      // charges; pinned by brute force in tests/test_bound_pins.py)
      const int base = cost + kCostUnits * O::popc(Z);
      const W cliq_live = heavy_clique_min<K>() > 0 ? (U & ~Z & clu) : W(0);
      const int hi_terms = (kPairBound ? (O::popc(Ol) >> 1) : 0) + O::popc(cliq_live);
      const bool undecided = hi_terms > 0 && key_less<kTwo>(base, P, gcost, gP) &&
                             !key_less<kTwo>(base + kCostUnits * hi_terms, P, gcost, gP);
      int lb = base;
      if (undecided) {
        W M = 0;  // matched columns
        int pairs = 0;
        if (kPairBound) {
#pragma unroll
          for (int c = 0; c < K; ++c) {
            const W S = Ol & ~B[c];  // columns whose only live row is r(., c)
            W T = S;
            while (T) {
              const int x = O::ffs(T);
              T &= T - W(1);
              const W N = adj[x] & S & ~M;
              if (N) {
                const W pb = (W(1) << x) | (W(1) << O::ffs(N));
                M |= pb;
                T &= ~pb;
                ++pairs;
              }
            }
          }
        }
        lb = base + kCostUnits * (pairs + clique_deficit<K, W>(B, U & ~M, Z, cl, 1, ncl));
      }
      const bool leaf = U == 0;
      const bool better = active && en && leaf && key_less<kTwo>(cost, P, gcost, gP);  // Alg. 1 line 5
      const bool ex = active && en && !leaf && key_less<kTwo>(lb, P, gcost, gP);      // bound (R7)
      if (better) {
#pragma unroll
        for (int c = 0; c < K; ++c) bestC[c] = C[c];
        gcost = cost;  // provisional; the warp minimum below settles it
        gP = P;
        found = true;
      }
      const int v = ex ? O::ffs(Z ? Z : (Ol ? Ol : U)) : 0;  // Alg. 1 line 8 (R5)
      if (ex && depth > d0) {  // spill the parent frame
        const int d = depth - 1;
        F.saved[d][lane] = f_saved;
        F.pk[d][lane] = (unsigned short)pk16(f_v, f_c, f_mu, f_lim);
      }
      const W av = adj[v], sav = sadj[v];
      f_cost = ex ? cost : f_cost;
      f_v = ex ? v : f_v;
      f_c = ex ? -1 : f_c;
      f_mu = ex ? maxused : f_mu;
      f_lim = ex ? min(K - 1, maxused + 1) : f_lim;  // colour-symmetry limit (R6)
      f_adj = ex ? av : f_adj;
      f_sadj = ex ? sav : f_sadj;
      U = ex ? (U & ~(W(1) << v)) : U;  // cover column v (line 9)
      depth += ex ? 1 : 0;
    }
    {
      const bool adv = active && depth > d0;
      if (active && depth == d0) active = false;
      const W bit = W(1) << f_v;
      const bool unc = adv && f_c >= 0;  // uncover the previous row (line 17)
#pragma unroll
      for (int c = 0; c < K; ++c) {
        const bool mine_c = unc && c == f_c;
        C[c] = mine_c ? (C[c] & ~bit) : C[c];
        B[c] = mine_c ? f_saved : B[c];
      }
      const int c = f_c + 1;
      const int fd = depth - 1;
      const bool exh = adv && c > f_lim;  // rows exhausted (R6 limit)
      const bool nxt = adv && !exh;
      // next child: select r(v,c) (line 14), cover its secondary columns (line 15)
      const int cc = min(c, K - 1);
      const W Cc = pick<K, W>(C, cc);
      const W Bc = pick<K, W>(B, cc);
      const int ncost = f_cost + row_cost<W>(f_adj, f_sadj, Cc, U, w_stitch);
#pragma unroll
      for (int q = 0; q < K; ++q) {
        const bool sel = nxt && q == cc;
        C[q] = sel ? (C[q] | bit) : C[q];
        B[q] = sel ? (B[q] | f_adj) : B[q];
      }
      f_saved = nxt ? Bc : f_saved;
      cost = nxt ? ncost : cost;
      maxused = nxt ? max(f_mu, c) : maxused;
      if (adv) path_put<kTwo>(P, max(fd, 0), nxt ? c : 0);
      const unsigned long long fbit = 1ull << max(fd, 0);
      open = (nxt && c < f_lim) ? (open | fbit) : (adv ? (open & ~fbit) : open);
      // exhausted: uncover the column (line 20) and pop the parent frame
      U = exh ? (U | bit) : U;
      const bool pop = exh && fd > d0;
      const int pd = max(fd - 1, 0);
      const W ps = F.saved[pd][lane];
      const int ppk = F.pk[pd][lane];
      const int pv = pop ? pk_v(ppk) : f_v;
      const W pa = adj[pv], psa = sadj[pv];
      // cost of N_pd = cost of its child N_fd minus the row r(pv, pc) still applied in C
      const int pcc = max(pk_c(ppk), 0);
      const W pC = pick<K, W>(C, pcc) & ~(W(1) << pv);
      const int pinc = row_cost<W>(pa, psa, pC, U, w_stitch);
      f_saved = pop ? ps : f_saved;
      f_cost = pop ? f_cost - pinc : f_cost;
      f_v = pv;
      f_c = pop ? pk_c(ppk) : (nxt ? c : f_c);
      f_mu = pop ? pk_mu(ppk) : f_mu;
      f_lim = pop ? pk_lim(ppk) : f_lim;
      f_adj = pop ? pa : f_adj;
      f_sadj = pop ? psa : f_sadj;
      depth = exh ? fd : depth;
      if (exh && fd <= d0) active = false;
      enter = nxt;
    }
    if (__ballot_sync(0xffffffffu, found)) {  // settle the best key: the minimum over the lanes
      // the non-finding lanes hold the previous best, so a finding lane wins
      mine = warp_min_key<kTwo>(gcost, gP) == lane;
    }
   }
    if (MPLD_SPILL && !all_idle && iters >= spill_at) {
      // share the best cost with the other units of a spilled component (no
      // lock: their keys are merged when the units end)
      if (u.slot >= 0) {
        HeavySlot* hs = &w.hslot[u.slot];
        const int bc = *(volatile int*)&hs->bcost;
        if (bc < gcost) {  // a cheaper leaf exists: (bc, max path) is a valid, weaker incumbent
          gcost = bc;
          gP = Path{~0ull, ~0ull};
          mine = false;
        } else if (gcost < bc && __any_sync(0xffffffffu, mine)) {
          if (lane == 0) atomicMin(&hs->bcost, gcost);
        }
      }
      // feed the work queue when it runs low: every lane gives away the untried
      // children of its shallowest open frame (the largest subtrees it holds)
      int hungry = 0;
      if (lane == 0)
        hungry = *(volatile int*)&w.ctl->wq_tail[u.cls] - *(volatile int*)&w.ctl->wq_head[u.cls] < kQueueLow;  // < 0: warps wait
      if (__shfl_sync(0xffffffffu, hungry, 0)) {
        int cnt = 0, j = -1;
        if (active && (open & donatable)) {
          j = __ffsll((long long)(open & donatable)) - 1;
          const int pk = j == depth - 1 ? pk16(f_v, f_c, f_mu, f_lim) : F.pk[j][lane];
          cnt = pk_lim(pk) - pk_c(pk);
        }
        int tot = 0;
        const int excl = warp_excl_scan(cnt, tot);
        int base = -1;
        if (lane == 0 && tot > 0) {
          if (u.slot < 0) {  // the component's first spill: a slot holding the light leaf, one unit pending (this)
            const int sl = atomicAdd(&w.ctl->slot_next, 1);
            if (sl < kSlots) {
              HeavySlot* hs = &w.hslot[sl];
              hs->lock = 0;
              hs->pend = 1;
              hs->cost = hs->lcost = u.c1;
              hs->bcost = u.hc;
              hs->pa = hs->lpa = u.p1.a;
              hs->pb = hs->lpb = u.p1.b;
#pragma unroll
              for (int c = 0; c < K; ++c) hs->C[c] = (unsigned long long)u.col[c];
              hs->ci = u.ci;
              hs->ncl = ncl <= 16 ? ncl : -1;  // (more cliques: the items recompute them)
              for (int q = 0; q < ncl && q < 16; ++q) hs->cl[q] = (unsigned long long)cl[q];
              __threadfence();
              u.slot = sl;
            }
          }
          if (u.slot >= 0) {  // reserve tot ring positions while the ring has room (items not yet read)
            int t = *(volatile int*)&w.ctl->wq_tail[u.cls];
            while (t + tot - *(volatile int*)&w.ctl->wq_read[u.cls] <= kWQCap) {
              const int o = atomicCAS(&w.ctl->wq_tail[u.cls], t, t + tot);
              if (o == t) {
                base = t;
                break;
              }
              t = o;
            }
            if (base >= 0) atomicAdd(&w.hslot[u.slot].pend, tot);  // before any item is published
          }
          if (base < 0) atomicAdd(&w.ctl->spill_refused, 1);  // ring full or no slot: this unit goes on alone
        }
        u.slot = __shfl_sync(0xffffffffu, u.slot, 0);
        base = __shfl_sync(0xffffffffu, base, 0);
        if (base >= 0 && cnt > 0) {
          WorkItem* q = w.wq + (size_t)u.cls * kWQCap;
          unsigned long long* qf = w.wq_flag + (size_t)u.cls * kWQCap;
          int at = base + excl;
          W jB[K], jC[K], jU;
          int pk, jc;
          node_at<K, W, heavy_depth<K, W>()>(j, depth, B, C, U, f_saved, f_v, f_c, f_cost, F, lane, adj, sadj,
                                             w_stitch, jB, jC, jU, jc);
          if (j == depth - 1) {
            pk = pk16(f_v, f_c, f_mu, f_lim);
            f_lim = f_c;  // its children are in the queue now
          } else {
            pk = F.pk[j][lane];
            F.pk[j][lane] = (unsigned short)((pk & 0x0fff) | (pk_c(pk) << 12));
          }
          open &= ~(1ull << j);
          const int v = pk_v(pk), cj = pk_c(pk), mu = pk_mu(pk), lim = pk_lim(pk);
          const W bit = W(1) << v;
          const W a = adj[v], sa = sadj[v];
          for (int ch = cj + 1; ch <= lim; ++ch) {  // the untried children of frame j (C at N_j = C & ~U_j)
            W xC[K], xB[K];
#pragma unroll
            for (int c = 0; c < K; ++c) {
              xC[c] = jC[c];
              xB[c] = jB[c];
            }
            const W xU = jU & ~bit;
            const W Cc = pick<K, W>(xC, ch);
            const int xcost = jc + row_cost<W>(a, sa, Cc, xU, w_stitch);
            put<K, W>(xC, ch, Cc | bit);
            put<K, W>(xB, ch, pick<K, W>(xB, ch) | a);
            Path xP = path_prefix<kTwo>(P, j);
            path_put<kTwo>(xP, j, ch);
            WorkItem& it = q[at & (kWQCap - 1)];
            it.slot = u.slot;
            it.depth = j + 1;
            it.cost = xcost;
            it.mu = max(mu, ch);
            it.pa = xP.a;
            it.pb = xP.b;
#pragma unroll
            for (int c = 0; c < K; ++c) {
              it.C[c] = (unsigned long long)xC[c];
              it.B[c] = (unsigned long long)xB[c];
            }
            it.U = (unsigned long long)xU;
            __threadfence();
            *(volatile unsigned long long*)&qf[at & (kWQCap - 1)] = wq_tag(w.epoch, at);
            ++at;
          }
        }
        if (base >= 0) spilled = true;
      }
    }
  }
  unsigned tot = steps;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
  steps_out = tot;
  capped_out = __any_sync(0xffffffffu, capped);
  if (iters_out) *iters_out = iters;
}

// A starting incumbent for the exact search ("seeded
// incumbent"): every lane builds one colouring greedily — the uncovered
// column with the fewest live rows (a random one among ties), the row of least
// Eq. (1) cost (random tie order) — then improves it by single-vertex moves
// (three sweeps); the warp's minimum cost is returned.  Masks are
// interchangeable, so a colouring of cost c is (after renaming masks into
// first-use order along its own column sequence) a leaf of the canonical tree:
// (c, maximal path) is a valid incumbent key that never cuts the canonical
// optimum (its key is <= (c, path of any leaf of cost c)).
template <int K, typename W>
__device__ int warp_greedy_once(const W* adj, const W* sadj, int n, int w_stitch, unsigned seed, W (&best)[K]) {
  using O = WordOps<W>;
  const int lane = threadIdx.x & 31;
  unsigned r = lowbias32(seed * 32u + (unsigned)lane + 0x9e3779b9u);
  W C[K], B[K];
#pragma unroll
  for (int c = 0; c < K; ++c) C[c] = B[c] = 0;
  W U = O::full(n);
  for (int d = 0; d < n; ++d) {
    // live-row count of every uncovered column, bit-sliced (3 bits: 0..4)
    W b0 = 0, b1 = 0, b2 = 0;
#pragma unroll
    for (int c = 0; c < K; ++c) {
      const W F = U & ~B[c];
      const W c0 = b0 & F;
      b0 ^= F;
      const W c1 = b1 & c0;
      b1 ^= c0;
      b2 |= c1;
    }
    W cand = U & ~b0 & ~b1 & ~b2;                         // 0 live rows
    if (!cand) cand = b0 & ~b1 & ~b2;                     // 1
    if (!cand) cand = ~b0 & b1 & ~b2 & U;                 // 2
    if (!cand) cand = b0 & b1 & ~b2;                      // 3
    if (!cand) cand = U;                                  // 4
    r = r * 1664525u + 1013904223u;
    const int sh = (int)((r >> 8) % (unsigned)n);
    const W rot = sh ? (((cand >> sh) | (cand << (n - sh))) & O::full(n)) : cand;
    int v = O::ffs(rot) + sh;
    v = v >= n ? v - n : v;
    const W bit = W(1) << v;
    const W a = adj[v], sa = sadj[v];
    const int off = (int)((r >> 24) % (unsigned)K);
    int bc = 0, bcost = INT_MAX;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const int c = (i + off) % K;
      const W Cc = pick<K, W>(C, c);
      const int cc = kCostUnits * O::popc(a & Cc) + w_stitch * O::popc(sa & ~U & ~Cc);
      if (cc < bcost) {
        bcost = cc;
        bc = c;
      }
    }
    U &= ~bit;
#pragma unroll
    for (int c = 0; c < K; ++c) {
      C[c] = c == bc ? (C[c] | bit) : C[c];
      B[c] = c == bc ? (B[c] | a) : B[c];
    }
  }
  for (int sweep = 0; sweep < 3; ++sweep)
    for (int v = 0; v < n; ++v) {
      const W bit = W(1) << v;
      const W a = adj[v], sa = sadj[v];
      int cur = 0, bc = 0, bcost = INT_MAX;
#pragma unroll
      for (int c = 0; c < K; ++c) {
        const int cc = kCostUnits * O::popc(a & C[c]) + w_stitch * O::popc(sa & ~C[c]);
        if (C[c] & bit) cur = cc;
        if (cc < bcost) {
          bcost = cc;
          bc = c;
        }
      }
      if (bcost < cur) {
#pragma unroll
        for (int c = 0; c < K; ++c) C[c] = c == bc ? (C[c] | bit) : (C[c] & ~bit);
      }
    }
  int nc = 0, ns = 0;
  for (int v = 0; v < n; ++v) {
    const W bit = W(1) << v;
    W Cv = C[0];
#pragma unroll
    for (int c = 1; c < K; ++c) Cv = (C[c] & bit) ? C[c] : Cv;
    nc += O::popc(adj[v] & Cv);
    ns += O::popc(sadj[v] & ~Cv);
  }
  const int cost = kCostUnits * (nc >> 1) + w_stitch * (ns >> 1);
  const int mc = (int)__reduce_min_sync(0xffffffffu, (unsigned)cost);
  const int src = __ffs(__ballot_sync(0xffffffffu, cost == mc)) - 1;
#pragma unroll
  for (int c = 0; c < K; ++c) best[c] = __shfl_sync(0xffffffffu, C[c], src);
  return mc;
}

// `rounds` x 32 randomized greedy colourings (Workspace::greedy_rounds), the cheapest kept
template <int K, typename W>
__device__ int warp_greedy_seed(const W* adj, const W* sadj, int n, int w_stitch, unsigned seed, int rounds,
                                W (&best)[K]) {
  int bc = warp_greedy_once<K, W>(adj, sadj, n, w_stitch, seed, best);
  for (int i = 1; i < rounds && bc > 0; ++i) {
    W t[K];
    const int c = warp_greedy_once<K, W>(adj, sadj, n, w_stitch, seed + 0x10000u * (unsigned)i, t);
    if (c < bc) {
      bc = c;
#pragma unroll
      for (int q = 0; q < K; ++q) best[q] = t[q];
    }
  }
  return bc;
}

// The canonical leaf of a colouring: follow the column rule of R5 and take
// each selected column's colour, masks renamed into first-use order along
// that column sequence (R6: masks are interchangeable and the live counts that
// drive R5 do not depend on their names, so the renamed colouring is a leaf of
// the canonical tree with the same cost).  col is renamed in place; returns
// the leaf's path and its cost.
template <int K, typename W>
__device__ __forceinline__ Path leaf_path(W (&col)[K], int n, const W* adj, const W* sadj, int w_stitch, int& cost) {
  State<K, W> s;
#pragma unroll
  for (int c = 0; c < K; ++c) s.C[c] = s.B[c] = 0;
  s.U = WordOps<W>::full(n);
  s.cost = 0;
  s.mu = -1;
  Path P = {0ull, 0ull};
  int perm = 0;  // 3 bits per original mask: 0 = not seen yet, else new name + 1
  for (int d = 0; d < n; ++d) {
    const int v = select_column<K, W>(s);
    const int c0 = colour_of<K, W>(col, v);
    int c = ((perm >> (3 * c0)) & 7) - 1;
    if (c < 0) {
      c = s.mu + 1;
      perm |= (c + 1) << (3 * c0);
    }
    apply_row<K, W>(s, v, c, adj, sadj, w_stitch);
    path_put(P, d, c);
  }
#pragma unroll
  for (int c = 0; c < K; ++c) col[c] = s.C[c];
  cost = s.cost;
  return P;
}

// Eq. (1b)/(1c) counts of a component's final colouring (whole warp)
template <int K, typename W>
__device__ __forceinline__ void heavy_counts(const GraphView& g, const W* adj, const W* sadj, int n, const W (&fin)[K],
                                             int v0, long long* counts) {
  if (!counts) return;
  int nc = 0, ns = 0;
  for (int i = threadIdx.x & 31; i < n; i += 32) {
    const W Ci = pick<K, W>(fin, colour_of<K, W>(fin, i));
    nc += WordOps<W>::popc(adj[i] & Ci);
    ns += WordOps<W>::popc(sadj[i] & ~Ci);
  }
  add_counts(g, v0, nc, ns, counts);
}

// The end of a unit of a spilled component: merge the unit's best leaf into
// the slot; the last unit of the component writes its colours and counts.
template <int K, typename W>
__device__ void heavy_unit_done(const GraphView& g, const Workspace& w, const HeavyUnit<K, W>& u, int gcost,
                                const Path& gP, bool mine, const W (&bestC)[K], const int* porder, int* colors,
                                long long* counts) {
  constexpr bool kTwo = sizeof(W) == 8;
  const int lane = threadIdx.x & 31;
  const unsigned owner = __ballot_sync(0xffffffffu, mine);
  const int src = owner ? __ffs(owner) - 1 : 0;
  W oc[K];
#pragma unroll
  for (int c = 0; c < K; ++c) oc[c] = __shfl_sync(0xffffffffu, bestC[c], src);
  HeavySlot* hs = &w.hslot[u.slot];
  int last = 0;
  if (lane == 0) {
    if (owner && gcost <= *(volatile int*)&hs->bcost) {  // a leaf that may beat the slot's key
      atomicMin(&hs->bcost, gcost);
      slot_lock(hs);
      const Path cur = {__ldcg(&hs->pa), __ldcg(&hs->pb)};
      if (key_less<kTwo>(gcost, gP, __ldcg(&hs->cost), cur)) {
        hs->cost = gcost;
        hs->pa = gP.a;
        hs->pb = gP.b;
#pragma unroll
        for (int c = 0; c < K; ++c) hs->C[c] = (unsigned long long)oc[c];
      }
      slot_unlock(hs);
    }
    __threadfence();
    last = atomicSub(&hs->pend, 1) == 1;
    __threadfence();
  }
  if (!__shfl_sync(0xffffffffu, last, 0)) return;
  W fin[K];  // the component's final colouring
#pragma unroll
  for (int c = 0; c < K; ++c) fin[c] = (W)__ldcg(&hs->C[c]);
  for (int i = lane; i < u.n; i += 32) colors[__ldcg(&porder[i])] = colour_of<K, W>(fin, i);
  heavy_counts<K, W>(g, u.adj, u.sadj, u.n, fin, __ldcg(&porder[0]), counts);
}

// A heavy component's pool record -> shared memory (masks, clique partition).
template <int K, typename W>
__device__ void heavy_load(const Workspace& w, size_t off, int n, W* s_adj, W* s_sadj, W* s_cl, int& ncl,
                           const int* colors, W (&col)[K], const HeavySlot* hs = nullptr) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int c = 0; c < K; ++c) col[c] = 0;
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int i = i0 + lane;
    int ci = -1;
    if (i < n) {
      const ulonglong2 m = __ldcg((const ulonglong2*)&w.pmask[2 * (off + i)]);
      s_adj[i] = (W)m.x;
      s_sadj[i] = (W)m.y;
      if (colors) ci = __ldcg(&colors[__ldcg(&w.porder[off + i])]);  // the light phase's best leaf
    }
#pragma unroll
    for (int c = 0; c < K; ++c) {
      const unsigned b = __ballot_sync(0xffffffffu, ci == c);
      col[c] |= (W)b << i0;
    }
  }
  __syncwarp();
  const int cached = hs ? __ldcg(&hs->ncl) : -1;
  if (cached >= 0) {  // a spilled item: the partition its component's first unit stored in the slot
    ncl = cached;
    if (lane < ncl) s_cl[lane] = (W)__ldcg(&hs->cl[lane]);
  } else {
    ncl = heavy_clique_min<K>() ? clique_partition<W>(s_adj, 1, n, s_cl, 1, heavy_clique_min<K>()) : 0;
  }
  __syncwarp();
}

// The units of the warp-parallel search: a heavy component (its light leaf or
// a cheaper greedy colouring as the starting incumbent), or a spilled work
// item.  W = 32-bit words for components of <= 32 vertices, 64-bit words for
// larger ones; both word classes share the warp's shared memory (sized for
// the 64-bit class).
struct HeavyAcc {
  unsigned long long steps = 0ull;
  int max = 0, capped = 0;
};

// A unit is finished: count it; the unit that completes the last pending work
// (every heavy component and every item reserved so far — no unit runs, so no
// item can be added) raises heavy_finished for the warps waiting for items.
__device__ __forceinline__ void heavy_unit_finished(Control* ctl, int cls, int n_heavy0, int n_heavy1) {
  __threadfence();
  const int d = atomicAdd(&ctl->wq_done[cls], 1) + 1;
  if (!*(volatile int*)&ctl->may_spill) return;  // no warp waits for spilled work (set before this kernel)
  __threadfence();
  const int d0 = cls == 0 ? d : *(volatile int*)&ctl->wq_done[0];
  const int d1 = cls == 1 ? d : *(volatile int*)&ctl->wq_done[1];
  const int t0 = *(volatile int*)&ctl->wq_tail[0], t1 = *(volatile int*)&ctl->wq_tail[1];
  if (d0 >= n_heavy0 + t0 && d1 >= n_heavy1 + t1) atomicExch(&ctl->heavy_finished, 1);
}

// MPLD_DIAG_HEAVY builds: one trace record per heavy unit (component or spilled
// item) in Workspace::est (free outside sharded runs): ci | n << 32 | item << 48,
// nodes, start / end %globaltimer; read back by mpld_context_debug out[96..]
#ifndef MPLD_DIAG_HEAVY
#define MPLD_DIAG_HEAVY 0
#endif
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void heavy_trace(const Workspace& w, int ci, int n, int item, unsigned long long steps,
                                            unsigned long long t0) {
  if (!MPLD_DIAG_HEAVY || (threadIdx.x & 31) != 0) return;
  const unsigned long long i = atomicAdd(&w.ctl->dbg[7], 1ull);
  if (4 * i + 3 >= (unsigned long long)w.diag_cap) return;
  w.est[4 * i] = (unsigned)ci | ((unsigned long long)n << 32) | ((unsigned long long)item << 48);
  w.est[4 * i + 1] = steps;
  w.est[4 * i + 2] = t0;
  w.est[4 * i + 3] = gtimer();
}

template <int K, typename W>
__device__ void heavy_component(const GraphView& g, const Workspace& w, int h, int w_stitch, int* colors,
                                long long* counts, unsigned char* smem, int* s_pair, int& cur_ci, int& cur_ncl,
                                HeavyAcc& acc) {
  constexpr int cls = sizeof(W) == 4 ? 0 : 1;
  constexpr bool kTwo = sizeof(W) == 8;
  const int lane = threadIdx.x & 31;
  W* s_adj = (W*)smem;
  W* s_sadj = s_adj + kMaxComp;
  W* s_cl = s_sadj + kMaxComp;
  const unsigned long long t0 = MPLD_DIAG_HEAVY ? gtimer() : 0ull;
  HeavyUnit<K, W> u;
  u.w_stitch = w_stitch;
  u.cls = cls;
  u.adj = s_adj;
  u.sadj = s_sadj;
  u.cl = s_cl;
  u.F = (LaneFrames<K, W, heavy_depth<K, W>()>*)(smem + 3 * kMaxComp * sizeof(unsigned long long));
  u.pair = s_pair;
  const int idx = cls ? g.n - 1 - h : h;
  u.ci = __ldcg(&w.hcomp[idx]);
  const unsigned long long rec = __ldcg(&w.crec[u.ci]);
  const size_t off = (size_t)(rec >> 8);
  u.n = (int)(rec & 0xffull);
  u.c1 = __ldcg(&w.hcost[idx]);
  u.slot = -1;
  const bool light_leaf = u.c1 != INT_MAX;  // exact mode hands components of > 32 vertices over unsearched
  heavy_load<K, W>(w, off, u.n, s_adj, s_sadj, s_cl, u.ncl, light_leaf ? colors : nullptr, u.col);
  cur_ci = u.ci;
  cur_ncl = u.ncl;
  W gcol[K];
  const int hc = ((kSeedIncumbent && u.n >= MPLD_SEED_MIN_N) || !light_leaf) ? warp_greedy_seed<K, W>(s_adj, s_sadj, u.n, w_stitch,
                                                                          (unsigned)u.ci + w.greedy_salt,
                                                                          w.greedy_rounds, gcol)
                                                 : INT_MAX;
  if (!light_leaf) {  // the greedy colouring (renamed into a canonical leaf by leaf_path) is the starting leaf
#pragma unroll
    for (int c = 0; c < K; ++c) u.col[c] = gcol[c];
  }
  int lc = 0;  // the leaf's cost
  u.p1 = leaf_path<K, W>(u.col, u.n, s_adj, s_sadj, w_stitch, lc);
  if (!light_leaf) u.c1 = lc;
  int gcost = u.c1;
  Path gP = u.p1;
  u.hc = u.c1;
  if (hc < u.c1) {  // a cheaper greedy colouring: (its cost, maximal path) is a valid incumbent key
    u.hc = hc;
    gcost = hc;
    gP = Path{~0ull, ~0ull};
  }
  W zero[K], bestC[K];
#pragma unroll
  for (int c = 0; c < K; ++c) zero[c] = 0;
  bool mine, capped, spilled;
  unsigned steps;
  unsigned iters = 0;
  warp_heavy_search<K, W>(u, w, zero, zero, WordOps<W>::full(u.n), 0, -1, Path{0ull, 0ull}, 0, gcost, gP, mine,
                          bestC, steps, capped, spilled, &iters);
  const int* porder = w.porder + off;
  if (u.slot < 0) {  // searched whole: the final colouring is the warp's best (or the light leaf)
    W fin[K];
#pragma unroll
    for (int c = 0; c < K; ++c) fin[c] = u.col[c];
    const unsigned owner = __ballot_sync(0xffffffffu, mine);
    const bool better = owner && key_less<kTwo>(gcost, gP, u.c1, u.p1);
    if (better) {
#pragma unroll
      for (int c = 0; c < K; ++c) fin[c] = __shfl_sync(0xffffffffu, bestC[c], __ffs(owner) - 1);
    }
    if (better || !light_leaf)
      for (int i = lane; i < u.n; i += 32) colors[__ldcg(&porder[i])] = colour_of<K, W>(fin, i);
    heavy_counts<K, W>(g, s_adj, s_sadj, u.n, fin, __ldcg(&porder[0]), counts);
  } else {
    heavy_unit_done<K, W>(g, w, u, gcost, gP, mine, bestC, porder, colors, counts);
  }
  heavy_trace(w, u.ci, u.n, 0, steps | ((unsigned long long)iters << 32), t0);
  acc.steps += steps;
  acc.max = max(acc.max, (int)min(steps, (unsigned)INT_MAX));
  acc.capped += capped ? 1 : 0;  // per unit (a spilled component may count more than once)
  __syncwarp();
  if (lane == 0) heavy_unit_finished(w.ctl, cls, __ldcg(&w.ctl->n_heavy[0]), __ldcg(&w.ctl->n_heavy[1]));
}

template <int K, typename W>
__device__ void heavy_item(const GraphView& g, const Workspace& w, int pos, int w_stitch, int* colors,
                           long long* counts, unsigned char* smem, int* s_pair, int& cur_ci, int& cur_ncl,
                           HeavyAcc& acc) {
  constexpr int cls = sizeof(W) == 4 ? 0 : 1;
  const int lane = threadIdx.x & 31;
  const unsigned long long t0 = MPLD_DIAG_HEAVY ? gtimer() : 0ull;
  W* s_adj = (W*)smem;
  W* s_sadj = s_adj + kMaxComp;
  W* s_cl = s_sadj + kMaxComp;
  HeavyUnit<K, W> u;
  u.w_stitch = w_stitch;
  u.cls = cls;
  u.adj = s_adj;
  u.sadj = s_sadj;
  u.cl = s_cl;
  u.F = (LaneFrames<K, W, heavy_depth<K, W>()>*)(smem + 3 * kMaxComp * sizeof(unsigned long long));
  u.pair = s_pair;
  u.hc = INT_MAX;
  const WorkItem* q = w.wq + (size_t)cls * kWQCap + (pos & (kWQCap - 1));
  u.slot = __ldcg(&q->slot);
  HeavySlot* hs = &w.hslot[u.slot];
  u.ci = __ldcg(&hs->ci);
  const unsigned long long rec = __ldcg(&w.crec[u.ci]);
  const size_t off = (size_t)(rec >> 8);
  u.n = (int)(rec & 0xffull);
  W sC[K], sB[K];
#pragma unroll
  for (int c = 0; c < K; ++c) {
    sC[c] = (W)__ldcg(&q->C[c]);
    sB[c] = (W)__ldcg(&q->B[c]);
  }
  const Path sP = {__ldcg(&q->pa), __ldcg(&q->pb)};
  const W sU = (W)__ldcg(&q->U);
  const int scost = __ldcg(&q->cost), smu = __ldcg(&q->mu), sdepth = __ldcg(&q->depth);
  __syncwarp();
  if (lane == 0) {  // the ring slot may be reused from now on
    __threadfence();
    atomicAdd(&w.ctl->wq_read[cls], 1);
  }
  if (u.ci != cur_ci) {  // items of one component mostly follow each other: keep its masks
    heavy_load<K, W>(w, off, u.n, s_adj, s_sadj, s_cl, u.ncl, nullptr, u.col, hs);
    cur_ci = u.ci;
    cur_ncl = u.ncl;
  }
  u.ncl = cur_ncl;
  // the best cost known as the starting incumbent, (bcost, max path): a valid
  // key no smaller than the slot's
  int sc = 0;
  if (lane == 0) sc = *(volatile int*)&hs->bcost;
  int gcost = __shfl_sync(0xffffffffu, sc, 0);
  Path gP = Path{~0ull, ~0ull};
  W bestC[K];
  bool mine, capped, spilled;
  unsigned steps;
  unsigned iters = 0;
  warp_heavy_search<K, W>(u, w, sC, sB, sU, scost, smu, sP, sdepth, gcost, gP, mine, bestC, steps, capped, spilled,
                          &iters);
  heavy_unit_done<K, W>(g, w, u, gcost, gP, mine, bestC, w.porder + off, colors, counts);
  heavy_trace(w, u.ci, u.n, 1 + sdepth, steps | ((unsigned long long)iters << 32), t0);
  acc.steps += steps;
  acc.capped += capped ? 1 : 0;
  __syncwarp();
  if (lane == 0) heavy_unit_finished(w.ctl, cls, __ldcg(&w.ctl->n_heavy[0]), __ldcg(&w.ctl->n_heavy[1]));
}

// One warp per heavy component, both word classes in one launch: the 64-bit
// class first (the longest searches), then the 32-bit class, then spilled
// work items of either class (a warp claims a ring position only once a
// producer has reserved it, so no warp waits on one class while the other
// has work), until every unit of both classes is done.
template <int K>
__global__ void __launch_bounds__(32, 8) mpld_exact_cover_search_heavy(GraphView g, Workspace w, int w_stitch,
                                                                    int* colors, long long* counts) {
  pdl_begin();
  if (gated_off(w)) return;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_pair[32];
  const int lane = threadIdx.x & 31;
  Control* ctl = w.ctl;
  const int n_heavy0 = __ldcg(&ctl->n_heavy[0]), n_heavy1 = __ldcg(&ctl->n_heavy[1]);
  HeavyAcc acc;
  int cur_ci = -1, cur_ncl = 0;  // the component whose masks are in shared memory
  while (true) {  // the 64-bit class first (the longest searches)
    int h = 0;
    if (lane == 0) h = atomicAdd(&ctl->heavy_next[1], 1);
    h = __shfl_sync(0xffffffffu, h, 0);
    if (h >= n_heavy1) break;
    heavy_component<K, unsigned long long>(g, w, h, w_stitch, colors, counts, smem, s_pair, cur_ci, cur_ncl, acc);
  }
  while (true) {
    int h = 0;
    if (lane == 0) h = atomicAdd(&ctl->heavy_next[0], 1);
    h = __shfl_sync(0xffffffffu, h, 0);
    if (h >= n_heavy0) break;
    heavy_component<K, unsigned>(g, w, h, w_stitch, colors, counts, smem, s_pair, cur_ci, cur_ncl, acc);
  }
  // no component left: stay for spilled work only if some may come (small
  // components never run long; a spill without helpers is still drained by the
  // warps that are running, the spilling one included)
  // Only the first gridDim.x / MPLD_HELPER_DIV warps stay as helpers: every
  // waiting warp polls the ring's counters, and a thousand pollers on those
  // lines slow down the running units' own spill checks and finish counts.
  int leave = 0;
  if (lane == 0)
    leave = (*(volatile int*)&ctl->may_spill == 0 || (int)blockIdx.x >= (int)gridDim.x / MPLD_HELPER_DIV) &&
            *(volatile int*)&ctl->wq_tail[0] == 0 && *(volatile int*)&ctl->wq_tail[1] == 0;
  unsigned backoff = 32;
  while (!__shfl_sync(0xffffffffu, leave, 0)) {
    int pos = -1, pcls = 0;
    if (lane == 0) {
      // claim a reserved position (64-bit class first).  Claims are CAS on the
      // head and only below the reserved tail (measured: one-atomic tickets
      // that may run past the tail made the idle warps take items faster and
      // the producers spill more, 0.8 M -> 2.5-2.9 M nodes on configs[2])
      for (int c = 1; c >= 0 && pos < 0; --c) {
        int hd = *(volatile int*)&ctl->wq_head[c];
        while (hd < *(volatile int*)&ctl->wq_tail[c]) {
          const int o = atomicCAS(&ctl->wq_head[c], hd, hd + 1);
          if (o == hd) {
            pos = hd;
            pcls = c;
            break;
          }
          hd = o;
        }
      }
      if (pos >= 0) {  // its producer publishes the item right after reserving it
        const unsigned long long tag = wq_tag(w.epoch, pos);
        const volatile unsigned long long* f = &w.wq_flag[(size_t)pcls * kWQCap + (pos & (kWQCap - 1))];
        while (*f != tag) __nanosleep(20);
        __threadfence();
      }
    }
    pos = __shfl_sync(0xffffffffu, pos, 0);
    pcls = __shfl_sync(0xffffffffu, pcls, 0);
    if (pos >= 0) {
      backoff = 32;
      if (pcls)
        heavy_item<K, unsigned long long>(g, w, pos, w_stitch, colors, counts, smem, s_pair, cur_ci, cur_ncl, acc);
      else
        heavy_item<K, unsigned>(g, w, pos, w_stitch, colors, counts, smem, s_pair, cur_ci, cur_ncl, acc);
      continue;
    }
    // done when every unit (heavy components + items) of both classes has
    // finished (raised by the unit that finished last: heavy_unit_finished)
    if (lane == 0) leave = *(volatile int*)&ctl->heavy_finished;
    if (!__shfl_sync(0xffffffffu, leave, 0)) {
      __nanosleep(backoff);
      backoff = min(backoff * 2u, (unsigned)MPLD_POLL_CAP);
    }
  }
  if (lane == 0 && acc.steps) {
    atomicAdd(&ctl->steps, acc.steps);
    atomicAdd(&ctl->steps_heavy, acc.steps);
    atomicMax(&ctl->max_steps_comp, acc.max);
  }
  if (lane == 0 && acc.capped) atomicAdd(&ctl->truncated, acc.capped);
}

}  // namespace

cudaError_t launch_discover(const GraphView& g, Workspace ws, int k, int sharded, cudaStream_t s, int blocks, bool pdl) {
  return launch_ex(mpld_component_discover, dim3(blocks), dim3(kCompWarps * 32), 0, s, pdl, false, g, ws, k, sharded);
}

// Inclusive prefix sum of ws.est[0..n) (the balanced shard partition): block
// sums, one block scanning them, every block rescanning its tile.
__device__ __forceinline__ unsigned long long block_scan_u64(unsigned long long x, unsigned long long* s_w,
                                                             unsigned long long& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  unsigned long long y = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long z = __shfl_up_sync(0xffffffffu, y, o);
    if (lane >= o) y += z;
  }
  if (lane == 31) s_w[wid] = y;
  __syncthreads();
  if (wid == 0) {
    unsigned long long t = lane < nw ? s_w[lane] : 0ull;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long z = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += z;
    }
    if (lane < nw) s_w[lane] = t;
  }
  __syncthreads();
  total = s_w[nw - 1];
  const unsigned long long r = y + (wid ? s_w[wid - 1] : 0ull);  // inclusive
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(1024) mpld_partition_sums(int n, const unsigned long long* est,
                                                            unsigned long long* bsum) {
  __shared__ unsigned long long s_w[32];
  const size_t base = (size_t)blockIdx.x * kScanTile;
  unsigned long long x = 0ull;
  for (int j = 0; j < kScanTile / 1024; ++j) {
    const size_t i = base + (size_t)j * 1024 + threadIdx.x;
    if (i < (size_t)n) x += __ldcg(&est[i]);
  }
  unsigned long long total;
  block_scan_u64(x, s_w, total);
  if (threadIdx.x == 0) bsum[blockIdx.x] = total;
}

__global__ void __launch_bounds__(1024) mpld_partition_offsets(int nb, unsigned long long* bsum) {
  __shared__ unsigned long long s_w[32];
  unsigned long long carry = 0ull;
  for (int b0 = 0; b0 < nb; b0 += 1024) {  // exclusive scan of the block sums, in place
    const int i = b0 + threadIdx.x;
    const unsigned long long x = i < nb ? bsum[i] : 0ull;
    unsigned long long total;
    const unsigned long long inc = block_scan_u64(x, s_w, total);
    if (i < nb) bsum[i] = carry + inc - x;
    carry += total;
  }
}

__global__ void __launch_bounds__(1024) mpld_partition_apply(int n, unsigned long long* est,
                                                             const unsigned long long* bsum) {
  __shared__ unsigned long long s_w[32];
  const size_t base = (size_t)blockIdx.x * kScanTile;
  unsigned long long carry = bsum[blockIdx.x];
  for (int j = 0; j < kScanTile / 1024; ++j) {
    const size_t i = base + (size_t)j * 1024 + threadIdx.x;
    const unsigned long long x = i < (size_t)n ? est[i] : 0ull;
    unsigned long long total;
    const unsigned long long inc = block_scan_u64(x, s_w, total);
    if (i < (size_t)n) est[i] = carry + inc;
    carry += total;
  }
}

cudaError_t launch_partition_scan(const GraphView& g, Workspace ws, cudaStream_t s) {
  if (g.n <= 0) return cudaSuccess;
  const int nb = (g.n + kScanTile - 1) / kScanTile;
  mpld_partition_sums<<<nb, 1024, 0, s>>>(g.n, ws.est, ws.bsum);
  mpld_partition_offsets<<<1, 1024, 0, s>>>(nb, ws.bsum);
  mpld_partition_apply<<<nb, 1024, 0, s>>>(g.n, ws.est, ws.bsum);
  return cudaGetLastError();
}

int g_light_per_sm[2] = {0, 0};  // resident CTAs per SM of the light kernel: [compact frames]

template <int K>
cudaError_t launch_search_k(const GraphView& g, Workspace ws, int w_stitch, long long max_steps, int* colors,
                            unsigned light_steps, long long* counts, int shard_index, int shard_count, cudaStream_t s,
                            int blocks, bool pdl) {
  if (max_steps > 0) {  // budgeted: compact frames, its own resident grid (blocks is the stored-cost kernel's)
    const int nb = g_light_per_sm[0] > 0 ? blocks / g_light_per_sm[0] * g_light_per_sm[1] : blocks;
    return launch_ex(mpld_exact_cover_search<K, true>, dim3(nb), dim3(kLaneWarps * 32), 0, s, pdl, false, g, ws,
                     w_stitch, max_steps, colors, light_steps, counts, shard_index, shard_count);
  }
  return launch_ex(mpld_exact_cover_search<K, false>, dim3(blocks), dim3(kLaneWarps * 32), 0, s, pdl, false, g, ws,
                   w_stitch, max_steps, colors, light_steps, counts, shard_index, shard_count);
}

cudaError_t launch_search(const GraphView& g, Workspace ws, int k, int w_stitch, long long max_steps, int* colors,
                          unsigned light_steps, long long* counts, int shard_index, int shard_count, cudaStream_t s,
                          int blocks, bool pdl) {
  switch (k) {
    case 2: return launch_search_k<2>(g, ws, w_stitch, max_steps, colors, light_steps, counts, shard_index,
                                      shard_count, s, blocks, pdl);
    case 3: return launch_search_k<3>(g, ws, w_stitch, max_steps, colors, light_steps, counts, shard_index,
                                      shard_count, s, blocks, pdl);
    case 4: return launch_search_k<4>(g, ws, w_stitch, max_steps, colors, light_steps, counts, shard_index,
                                      shard_count, s, blocks, pdl);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_search_wide(const GraphView& g, Workspace ws, int k, int w_stitch, long long max_steps,
                               int* colors, unsigned light_steps, long long* counts, cudaStream_t s, int blocks) {
  const size_t smem = sizeof(LaneWide);
  switch (k) {
    case 2: return launch_ex(mpld_exact_cover_search_wide<2>, dim3(blocks), dim3(32), smem, s, true, false, g, ws,
                             w_stitch, max_steps, colors, light_steps, counts);
    case 3: return launch_ex(mpld_exact_cover_search_wide<3>, dim3(blocks), dim3(32), smem, s, true, false, g, ws,
                             w_stitch, max_steps, colors, light_steps, counts);
    case 4: return launch_ex(mpld_exact_cover_search_wide<4>, dim3(blocks), dim3(32), smem, s, true, false, g, ws,
                             w_stitch, max_steps, colors, light_steps, counts);
    default: return cudaErrorInvalidValue;
  }
}

template <int K>
cudaError_t configure_wide_k(int num_sms, int* blocks) {
  cudaError_t e = cudaFuncSetAttribute(mpld_exact_cover_search_wide<K>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LaneWide));
  if (e == cudaSuccess)  // the whole unified L1 as shared memory (see configure_heavy_k)
    e = cudaFuncSetAttribute(mpld_exact_cover_search_wide<K>, cudaFuncAttributePreferredSharedMemoryCarveout,
                             (int)cudaSharedmemCarveoutMaxShared);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mpld_exact_cover_search_wide<K>, 32, sizeof(LaneWide));
  *blocks = per_sm * num_sms;
  return cudaSuccess;
}

// shared-memory limit and resident grid of the 64-bit lane kernels (the same for every k)
cudaError_t configure_search_wide(int num_sms, int* blocks) {
  int b2 = 0, b3 = 0, b4 = 0;
  cudaError_t e = configure_wide_k<2>(num_sms, &b2);
  if (e == cudaSuccess) e = configure_wide_k<3>(num_sms, &b3);
  if (e == cudaSuccess) e = configure_wide_k<4>(num_sms, &b4);
  *blocks = std::min(b2, std::min(b3, b4));
  return e;
}

constexpr size_t heavy_smem_all(int k) {
  // masks + clique words (64-bit) and the frames of the 64-bit class (the 32-bit class needs less)
  return 3 * kMaxComp * sizeof(unsigned long long) +
         (k == 2 ? sizeof(LaneFrames<2, unsigned long long, 64>)
                 : (k == 3 ? sizeof(LaneFrames<3, unsigned long long, 64>) : sizeof(LaneFrames<4, unsigned long long, 64>)));
}
static_assert(sizeof(LaneFrames<4, unsigned, 32>) <= sizeof(LaneFrames<4, unsigned long long, 64>),
              "the 32-bit class fits the shared memory of the 64-bit class");

cudaError_t launch_search_heavy(const GraphView& g, Workspace ws, int k, int w_stitch, int* colors, long long* counts,
                                cudaStream_t s, const int* blocks, bool pdl) {
  switch (k) {
    case 2: return launch_ex(mpld_exact_cover_search_heavy<2>, dim3(blocks[0]), dim3(32), heavy_smem_all(2), s, pdl,
                             false, g, ws, w_stitch, colors, counts);
    case 3: return launch_ex(mpld_exact_cover_search_heavy<3>, dim3(blocks[1]), dim3(32), heavy_smem_all(3), s, pdl,
                             false, g, ws, w_stitch, colors, counts);
    case 4: return launch_ex(mpld_exact_cover_search_heavy<4>, dim3(blocks[2]), dim3(32), heavy_smem_all(4), s, pdl,
                             false, g, ws, w_stitch, colors, counts);
    default: return cudaErrorInvalidValue;
  }
}

template <int K>
cudaError_t configure_heavy_k(int num_sms, int* blocks) {
  cudaError_t e = cudaFuncSetAttribute(mpld_exact_cover_search_heavy<K>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)heavy_smem_all(K));
  // the whole unified L1 as shared memory: the resident-grid size below assumes it, and without
  // the preference the SM keeps the carveout of the kernel before (measured: configs[2] after the
  // light kernel 0.93-0.99 ms, after a kernel that had set the maximum 0.45-0.50 ms)
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(mpld_exact_cover_search_heavy<K>, cudaFuncAttributePreferredSharedMemoryCarveout,
                             (int)cudaSharedmemCarveoutMaxShared);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mpld_exact_cover_search_heavy<K>, 32, heavy_smem_all(K));
  *blocks = per_sm * num_sms;
  return cudaSuccess;
}

// sets the shared-memory limits of the heavy kernels and their resident grid sizes blocks[k - 2]
cudaError_t configure_search_heavy(int num_sms, int* blocks) {
  cudaError_t e = configure_heavy_k<2>(num_sms, blocks + 0);
  if (e == cudaSuccess) e = configure_heavy_k<3>(num_sms, blocks + 1);
  if (e == cudaSuccess) e = configure_heavy_k<4>(num_sms, blocks + 2);
  return e;
}

int resident_blocks_discover(int num_sms) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mpld_component_discover, kCompWarps * 32, 0);
  return per_sm * num_sms;
}

int resident_blocks_search(int threads, int num_sms) {
  (void)threads;
  for (auto f : {mpld_exact_cover_search<2, false>, mpld_exact_cover_search<3, false>, mpld_exact_cover_search<4, false>,
                 mpld_exact_cover_search<2, true>, mpld_exact_cover_search<3, true>, mpld_exact_cover_search<4, true>})
    cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
  int per_sm = 0, per_sm_c = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mpld_exact_cover_search<4, false>, kLaneWarps * 32, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_c, mpld_exact_cover_search<4, true>, kLaneWarps * 32, 0);
  g_light_per_sm[0] = per_sm;
  g_light_per_sm[1] = per_sm_c > 0 ? per_sm_c : per_sm;
  return per_sm * num_sms;
}

}  // namespace mpld
