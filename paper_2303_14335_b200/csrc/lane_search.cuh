// The lane-parallel search of PAPER.md §2.3 / Alg. 1 (one component per lane)
// and the bit-sliced helpers it shares with the warp-parallel search: word
// operations, the column-count reduction (Alg. 1 line 8), the clique term of
// the R7 bound, the component staging and the light-search epilogue.  Used by
// kernel_search.cu (light / wide / heavy kernels) and kernel_tile.cu (the
// fused tile pipeline).  Internal: not part of the C ABI.
#pragma once

#include <climits>

#include "mpld_internal.cuh"

namespace mpld {
namespace {

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

// Exact mode's warp-parallel search may use any valid bound (its result is
// the canonical leaf whatever it prunes); the clique term pays off there for
// k = 3 as well (cliques of >= MPLD_HEAVY_CLIQUE vertices, 0 = as the light search).
#ifndef MPLD_HEAVY_CLIQUE
#define MPLD_HEAVY_CLIQUE 0
#endif
// Lower bound of R7 in conflicts: columns with no live row (popc(Z), summed by
// the callers), plus this clique term: over the cliques, max(0, |X| - #masks
// live on X) for X = the clique's uncovered columns that still have a live row.
template <int K, typename W>
__device__ __forceinline__ int clique_deficit(const W (&B)[K], W U, W Z, const W* cl, int cs, int ncl) {
  using O = WordOps<W>;
  int d = 0;
  for (int q = 0; q < ncl; ++q) {
    const W X = cl[q * cs] & U & ~Z;
    if (!X) continue;
    int live = 0;
#pragma unroll
    for (int c = 0; c < K; ++c) live += (X & ~B[c]) ? 1 : 0;
    d += max(0, O::popc(X) - live);
  }
  return d;
}

// The same clique term with the cliques in registers (the lane searches: at
// most N / 4 cliques of >= 4 vertices, zero masks past ncl contribute 0), the
// loop unrolled up to the warp's largest clique count (no shared-memory loads,
// no per-clique branch).
template <int K, typename W, int NQ>
__device__ __forceinline__ int clique_deficit_reg(const W (&B)[K], W U, W Z, const W (&clr)[NQ], int nq_warp) {
  using O = WordOps<W>;
  int d = 0;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    if (q < nq_warp) {
      const W X = clr[q] & U & ~Z;
      int live = 0;
#pragma unroll
      for (int c = 0; c < K; ++c) live += (X & ~B[c]) ? 1 : 0;
      d += max(0, O::popc(X) - live);
    }
  }
  return d;
}

template <int K>
__host__ __device__ constexpr int heavy_clique_min() {
  return MPLD_HEAVY_CLIQUE > 0 ? MPLD_HEAVY_CLIQUE : clique_min<K>();
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

// The budgeted sequential search (the oracle's node order and budget, R7) of
// one component per LANE: a warp takes 32 consecutive components of the pool
// and every lane runs the DFS of lane_dfs() on its own component, written
// branch-free so that the lanes issue one instruction stream.  Masks and
// frames are [index][lane] in shared memory (a lane only touches its own
// column).  mpld_exact_cover_search<K> runs the components of <= 32 vertices
// on 32-bit words and lists the larger ones; mpld_exact_cover_search_wide<K>
// runs those, again one per lane, on 64-bit words.  Exact mode hands
// components whose search exceeds the light budget to the warp-parallel
// kernel below.
constexpr int kLaneWarps = 2;  // warps per CTA of the light search (32-bit words)
#ifndef MPLD_STAGED_LIGHT
#define MPLD_STAGED_LIGHT 1
#endif
constexpr bool kStagedLight = MPLD_STAGED_LIGHT != 0;  // coalesced warp staging of the light kernel's records

// A frame holds the word B[c] saved before its row was selected and 12 bits
// of state.  For 64-bit words (kCompact) the node cost is not stored either:
// popping back to a frame subtracts its row's cost from the child's (56 KB
// per warp: four 64-bit lane warps per SM instead of three; the 32-bit light
// kernel keeps the cost, measured faster there).  After the search the saved
// rows hold the staged vertex ids.
template <typename W, int N, bool Cm = (N > 32)>
struct __align__(16) LaneStore {
  static constexpr bool kCompact = Cm;
  W A[N][32];                        // adj[v][lane]
  W S[N][32];                        // sadj[v][lane]
  W saved[N][32];                    // frame d: B[c] before r(v,c) was selected; then vertex ids (warp_stage)
  int cost[kCompact ? 1 : N][32];    // frame d: cost when the node was entered (not kCompact)
  unsigned short pk[N][32];          // frame d: v | (c+1) << 6 | (maxused+1) << 9
  W cl[N / 4][32];                   // clique masks (R7, k >= 4: cliques of >= 4 vertices)
};
using LaneLight = LaneStore<unsigned, 32>;
using LaneWide = LaneStore<unsigned long long, kMaxComp>;

// The relaxed Algorithm X of R4-R7 with branch and bound, one component per
// lane (the oracle's node order, incumbent rule and budget); returns the nodes
// entered and the best leaf's colour masks in bestC.
template <int K, typename W, int N, bool Cm>
__device__ unsigned lane_dfs(LaneStore<W, N, Cm>& L, int lane, bool valid, int n, int w_stitch, unsigned budget, int ncl,
                             W clu, W (&bestC)[K], int& best, bool& trunc) {
  using O = WordOps<W>;
  W C[K], B[K];
#pragma unroll
  for (int c = 0; c < K; ++c) C[c] = B[c] = bestC[c] = 0;
  W U = valid ? O::full(n) : 0;
  int cost = 0, maxused = -1, depth = 0;
  best = INT_MAX;
  trunc = false;
  unsigned steps = 0;
  bool active = valid, enter = valid;
  W f_saved = 0, f_adj = 0, f_sadj = 0;
  int f_cost = 0, f_v = 0, f_c = -1, f_mu = -1;
  constexpr int kNQ = N / 4;  // cliques in registers (clique_deficit_reg)
  W clr[kNQ];
#pragma unroll
  for (int q = 0; q < kNQ; ++q) clr[q] = (clique_min<K>() > 0 && q < ncl) ? L.cl[q][lane] : W(0);
  const int nq_warp = clique_min<K>() > 0 ? (int)__reduce_max_sync(0xffffffffu, (unsigned)ncl) : 0;
  while (__any_sync(0xffffffffu, active)) {
    const bool en = active && enter;
    if (en && ++steps > budget && best != INT_MAX) {  // budget (R7): stop at exactly the oracle's node
      trunc = true;
      active = false;
    }
    {  // enter the pending node: leaf / prune / expand
      W Z, Ol;
      live_counts<K, W>(B, U, Z, Ol);
      // bound (R7): cost + zero-live columns + clique deficit.  The deficit is at
      // most the number of live columns inside cliques (clu), so it is summed
      // only when it can change the decision lb < best (same decisions, same
      // node order as the oracle; most nodes skip the clique loop)
      const int base = cost + kCostUnits * O::popc(Z);
      const bool undecided = clique_min<K>() > 0 && base < best && base + kCostUnits * O::popc(U & ~Z & clu) >= best;
      const int lb =
          undecided ? base + kCostUnits * clique_deficit_reg<K, W, kNQ>(B, U, Z, clr, nq_warp) : base;
      const bool leaf = U == 0;
      const bool better = active && en && leaf && cost < best;  // Alg. 1 line 5, strict improvement
      const bool ex = active && en && !leaf && lb < best;       // bound (R7)
      if (better) {
        best = cost;
#pragma unroll
        for (int c = 0; c < K; ++c) bestC[c] = C[c];
      }
      const int v = ex ? O::ffs(Z ? Z : (Ol ? Ol : U)) : 0;  // Alg. 1 line 8 (R5)
      if (ex && depth > 0) {  // spill the parent frame
        const int d = depth - 1;
        L.saved[d][lane] = f_saved;
        if (!Cm) L.cost[d][lane] = f_cost;
        L.pk[d][lane] = (unsigned short)(f_v | ((f_c + 1) << 6) | ((f_mu + 1) << 9));
      }
      const W av = L.A[v][lane], sav = L.S[v][lane];
      f_v = ex ? v : f_v;
      f_c = ex ? -1 : f_c;
      f_mu = ex ? maxused : f_mu;
      f_cost = ex ? cost : f_cost;
      f_adj = ex ? av : f_adj;
      f_sadj = ex ? sav : f_sadj;
      U = ex ? (U & ~(W(1) << v)) : U;  // cover column v (line 9)
      depth += ex ? 1 : 0;
    }
    {  // advance the deepest frame: next row, or exhausted -> pop
      const bool adv = active && depth > 0;
      if (active && depth == 0) active = false;
      const W bit = W(1) << f_v;
      const bool unc = adv && f_c >= 0;  // uncover the previous row (line 17)
#pragma unroll
      for (int c = 0; c < K; ++c) {
        const bool mc = unc && c == f_c;
        C[c] = mc ? (C[c] & ~bit) : C[c];
        B[c] = mc ? f_saved : B[c];
      }
      const int c = f_c + 1;
      const int fd = depth - 1;
      const bool exh = adv && c > min(K - 1, f_mu + 1);  // rows exhausted (colour-symmetry limit R6)
      const bool nxt = adv && !exh;
      const int cc = min(c, K - 1);
      const W Cc = pick<K, W>(C, cc), Bc = pick<K, W>(B, cc);
      const int ncost = f_cost + kCostUnits * O::popc(f_adj & Cc) + w_stitch * O::popc(f_sadj & ~U & ~Cc);
#pragma unroll
      for (int q = 0; q < K; ++q) {  // select r(v,c) (line 14), cover its secondary columns (line 15)
        const bool sel = nxt && q == cc;
        C[q] = sel ? (C[q] | bit) : C[q];
        B[q] = sel ? (B[q] | f_adj) : B[q];
      }
      f_saved = nxt ? Bc : f_saved;
      cost = nxt ? ncost : cost;
      maxused = nxt ? max(f_mu, c) : maxused;
      U = exh ? (U | bit) : U;  // exhausted: uncover the column (line 20)
      const bool pop = exh && fd > 0;
      const int pd = max(fd - 1, 0);
      const W ps = L.saved[pd][lane];
      const int ppk = L.pk[pd][lane];
      const int pv = pop ? (ppk & 63) : f_v;
      const int pcol = max(((ppk >> 6) & 7) - 1, 0);
      const W pa = L.A[pv][lane], psa = L.S[pv][lane];
      // the parent's cost: the child's minus the parent's row r(pv, pcol), whose
      // column set C[pcol] \ {pv} and uncovered set U are as when it was selected
      int pc;
      if (Cm) {
        const W pCc = pick<K, W>(C, pcol) & ~(W(1) << pv);
        pc = f_cost - kCostUnits * O::popc(pa & pCc) - w_stitch * O::popc(psa & ~U & ~pCc);
      } else {
        pc = L.cost[pd][lane];
      }
      f_saved = pop ? ps : f_saved;
      f_cost = pop ? pc : f_cost;
      f_v = pv;
      f_c = pop ? ((ppk >> 6) & 7) - 1 : (nxt ? c : f_c);
      f_mu = pop ? ((ppk >> 9) & 7) - 1 : f_mu;
      f_adj = pop ? pa : f_adj;
      f_sadj = pop ? psa : f_sadj;
      depth = exh ? fd : depth;
      if (exh && fd == 0) active = false;
      enter = nxt;
    }
  }
  return steps;
}

// The component's epilogue: colours, Eq. (1b)/(1c) counts, statistics, hand-off.
struct LightAcc {
  unsigned long long steps = 0ull;
  int maxsteps = 0;
  unsigned trunc = 0;
  unsigned comps = 0;  // components searched (this shard's)
  unsigned handoff = 0;  // components handed to the warp-parallel search (exact mode)
};

__device__ __forceinline__ void light_handoff(const GraphView& g, const Workspace& w, int ci, int n, int best_cost) {
  const int cls = n > 32 ? 1 : 0;
  if (n >= kHelpersMinN) atomicOr(&w.ctl->may_spill, 1);
  const int h = atomicAdd(&w.ctl->n_heavy[cls], 1);
  const int idx = cls ? g.n - 1 - h : h;
  w.hcomp[idx] = ci;
  w.hcost[idx] = best_cost;
}

// Sharded search: the component rooted at `root` belongs to the
// shard in which its cost interval [prefix - est, prefix) starts (contiguous
// root-id ranges of equal estimated cost; the same on every rank).
__device__ __forceinline__ bool in_shard(const GraphView& g, const Workspace& w, int root, int n, int k,
                                         int shard_index, int shard_count) {
  if (shard_count <= 1) return true;
  const unsigned long long total = __ldcg(&w.est[g.n - 1]);
  const unsigned long long start = __ldcg(&w.est[root]) - partition_estimate(n, k);
  int s = (int)((double)start / (double)total * (double)shard_count);
  s = min(max(s, 0), shard_count - 1);
  return s == shard_index;
}

// Staging of the warp's 32 CONSECUTIVE pool records (the light kernel's lanes
// take components b*32 + lane; the discovery kernel hands out component index
// and pool offset from one atomic, so lane l's rows are pool entries
// [off_l, off_l + n_l), contiguous and increasing with l): the warp reads the
// whole range with coalesced loads, entry e going to the lane that owns it
// (binary search over the lanes' start offsets by shuffles), transposed into
// the [row][lane] layout of shared memory.  Lanes with `has` = false hold no
// record; rows of lanes with `store` = false are read but not kept.
__device__ __forceinline__ int warp_owner(unsigned rel, unsigned e) {
  int o = 0;
#pragma unroll
  for (int st = 16; st > 0; st >>= 1) {
    const unsigned r = __shfl_sync(0xffffffffu, rel, o + st);
    if (r <= e) o += st;
  }
  return o;
}

template <typename W, int N, bool kOrder, bool Cm>
__device__ __forceinline__ void warp_stage(const Workspace& w, LaneStore<W, N, Cm>& L, int lane, bool has, bool store,
                                           size_t off, int n) {
  __syncwarp();  // the lanes' earlier accesses to the rows written below (frames / masks) are complete
  const size_t base = __shfl_sync(0xffffffffu, off, 0);  // lane 0 always holds a record
  const unsigned rel = has ? (unsigned)(off - base) : 0xffffffffu;
  const unsigned end = __reduce_max_sync(0xffffffffu, has ? rel + (unsigned)n : 0u);
  for (unsigned e0 = 0; e0 < end; e0 += 32) {
    const unsigned e = e0 + lane;
    const int o = warp_owner(rel, e);
    const unsigned ro = __shfl_sync(0xffffffffu, rel, o);
    const bool so = __shfl_sync(0xffffffffu, store, o);
    if (e < end) {
      if (kOrder) {  // vertex ids (after the search: the frames' saved rows are free)
        const int v = __ldcg(&w.porder[base + e]);
        if (so) L.saved[e - ro][o] = (W)(unsigned)v;
      } else {  // adj / sadj words
        const ulonglong2 m = __ldcg((const ulonglong2*)&w.pmask[2 * (base + e)]);
        if (so) {
          L.A[e - ro][o] = (W)m.x;
          L.S[e - ro][o] = (W)m.y;
        }
      }
    }
  }
  __syncwarp();
}

// One component per lane (lane `valid` with pool record `rec`): staging of its
// masks, clique partition, the DFS, then colours / counts / statistics, or the
// hand-off to the warp-parallel search (exact mode, light budget exceeded).
// kStaged: the warp's records are consecutive (warp_stage), `has` = the lane
// holds a record; else each lane reads its own record.
template <int K, typename W, int N, bool kStaged, bool Cm>
__device__ __forceinline__ void lane_component(const GraphView& g, const Workspace& w, LaneStore<W, N, Cm>& L, int lane,
                                               bool has, bool valid, int ci, unsigned long long rec, int w_stitch,
                                               unsigned budget, bool exact, int* colors, long long* counts,
                                               LightAcc& acc) {
  const size_t off = (size_t)(rec >> 8);
  const int n = (int)(rec & 0xffull);
  if (kStaged) {
    warp_stage<W, N, false>(w, L, lane, has, valid, off, n);
  } else if (valid) {
    for (int i = 0; i < n; ++i) {
      const ulonglong2 m = __ldcg((const ulonglong2*)&w.pmask[2 * (off + i)]);
      L.A[i][lane] = (W)m.x;
      L.S[i][lane] = (W)m.y;
    }
  }
  const int ncl = valid && clique_min<K>() ? clique_partition<W>(&L.A[0][lane], 32, n, &L.cl[0][lane], 32,
                                                                  clique_min<K>())
                                           : 0;
  W clu = 0;  // the cliques' union
  for (int q = 0; q < ncl; ++q) clu |= L.cl[q][lane];
  W bestC[K];
  int best_cost = 0;
  bool trunc = false;
  const unsigned steps = lane_dfs<K, W, N>(L, lane, valid, n, w_stitch, budget, ncl, clu, bestC, best_cost, trunc);
  if (kStaged) warp_stage<W, N, true>(w, L, lane, has, valid, off, n);
  if (!valid) return;
  for (int i = 0; i < n; ++i)
    colors[kStaged ? (int)L.saved[i][lane] : __ldcg(&w.porder[off + i])] = colour_of<K, W>(bestC, i);
  if (trunc && exact) {
    light_handoff(g, w, ci, n, best_cost);
    acc.handoff += 1;
  } else {
    if (counts) {  // final colouring: Eq. (1b)/(1c) counts of the component
      int nc = 0, ns = 0;
      for (int i = 0; i < n; ++i) {
        const W Ci = pick<K, W>(bestC, colour_of<K, W>(bestC, i));
        nc += WordOps<W>::popc(L.A[i][lane] & Ci);
        ns += WordOps<W>::popc(L.S[i][lane] & ~Ci);
      }
      nc >>= 1;
      ns >>= 1;
      if (nc | ns) {
        const int l = layout_of(g, kStaged ? (int)L.saved[0][lane] : __ldcg(&w.porder[off]));
        if (nc) atomicAdd((unsigned long long*)&counts[2 * l], (unsigned long long)nc);
        if (ns) atomicAdd((unsigned long long*)&counts[2 * l + 1], (unsigned long long)ns);
      }
    }
    acc.maxsteps = max(acc.maxsteps, (int)min(steps, (unsigned)INT_MAX));
    acc.trunc += trunc ? 1 : 0;
  }
  acc.steps += steps;
}

// statistics of a light kernel: one atomic per warp
__device__ __forceinline__ void light_stats(Control* ctl, const LightAcc& acc) {
  const int lane = threadIdx.x & 31;
  unsigned long long st = acc.steps;
  int mx = acc.maxsteps;
  unsigned tr = acc.trunc, nc = acc.comps;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    st += __shfl_xor_sync(0xffffffffu, st, o);
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    tr += __shfl_xor_sync(0xffffffffu, tr, o);
    nc += __shfl_xor_sync(0xffffffffu, nc, o);
  }
  if (lane == 0 && nc) atomicAdd(&ctl->n_comp, (int)nc);
  if (lane == 0 && st) {
    atomicAdd(&ctl->steps, st);
    atomicMax(&ctl->max_steps_comp, mx);
    if (tr) atomicAdd(&ctl->truncated, (int)tr);
  }
}

__host__ __device__ constexpr unsigned light_budget(long long max_steps, unsigned light_steps) {
  return max_steps <= 0 ? light_steps : (max_steps >= (long long)UINT_MAX ? UINT_MAX : (unsigned)max_steps);
}

}  // namespace
}  // namespace mpld
