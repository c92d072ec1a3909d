// Graph-level kernels of the MPLD hot path (§2.2 / Fig. 2 flow):
//   mpld_simplify_components simplification (R8), component seeds (Alg. 1
//                            lines 1-3), recovery pop keys and its level 0
//   mpld_recover             recovery of the hidden vertices (R9)
//   mpld_evaluate            Eq. (1) conflict / stitch counts and cost per layout
//
// The two persistent kernels are launched cooperatively (one wave of resident
// CTAs, grid-wide barriers between rounds) so that the whole path is enqueued
// without a host synchronisation.  Queue appends reserve space with one atomic
// per CTA (a single hot counter serialises at the L2).
//
// Every pass is bound by chains of dependent loads (row pointer -> column ids
// -> the neighbours' data), not by bandwidth: the neighbours of an item are
// read in batches of kNb independent loads, items are tiled kP per thread
// (measured on B200: kP = 1, kNb = 4 and one 1024-thread CTA per SM are the
// fastest; lockstep tiles of 2-3 items per thread lengthen every level).
#include <algorithm>
#include <climits>
#include <cooperative_groups.h>

#include "mpld_internal.cuh"

namespace cg = cooperative_groups;

namespace mpld {

namespace {

bool g_pdl = true;

#ifndef MPLD_GRAPH_P
#define MPLD_GRAPH_P 1
#endif
#ifndef MPLD_GRAPH_NB
#define MPLD_GRAPH_NB 4
#endif
#ifndef MPLD_EVAL_P
#define MPLD_EVAL_P 1
#endif
#ifndef MPLD_GRAPH_MINB
#define MPLD_GRAPH_MINB 1
#endif
#ifndef MPLD_GRAPH_PF
#define MPLD_GRAPH_PF 1
#endif
constexpr int kP = MPLD_GRAPH_P;    // items per thread and tile (frontier rounds, recovery levels)
constexpr int kPF = MPLD_GRAPH_PF;  // items per thread and tile of the full passes over all vertices
constexpr int kNb = MPLD_GRAPH_NB;  // neighbours per item and batch of independent memory operations
#ifndef MPLD_TAIL
#define MPLD_TAIL 1024
#endif
constexpr int kTail = MPLD_TAIL;  // frontiers up to this size are finished by CTA 0 alone
#ifndef MPLD_GROUP
#define MPLD_GROUP 16
#endif
#ifndef MPLD_CLUSTER_TAIL
#define MPLD_CLUSTER_TAIL 1
#endif
#ifndef MPLD_CLUSTER
#define MPLD_CLUSTER 16
#endif
#ifndef MPLD_TAIL_LOCAL
#define MPLD_TAIL_LOCAL 1
#endif
#ifndef MPLD_CLUSTER_ROUNDS
#define MPLD_CLUSTER_ROUNDS 0  // measured slower in the PDL chain: off
#endif
constexpr int kTC = MPLD_CLUSTER;                // CTAs of the recovery's cluster tail
#ifndef MPLD_CLUSTER_TAIL_ITEMS
#define MPLD_CLUSTER_TAIL_ITEMS 1
#endif
constexpr int kClusterTailMax = MPLD_CLUSTER_TAIL_ITEMS * kTC * 1024;  // levels up to this size go to the cluster tail
constexpr int kGroup = MPLD_GROUP;  // frontiers up to kGroup * blockDim items: the first kGroup CTAs, group barriers
constexpr int kStitchDeg = 1 << 29;  // live degree of stitch vertices: never reaches k (never hidden, R8)
#ifndef MPLD_PACKED_PRED
#define MPLD_PACKED_PRED 1
#endif
// Recovery state of a hidden vertex v.  Packed (default): ONE 32-bit word in
// deg[v] = (hidden predecessors still uncoloured) | popped-before bits << 8,
// bit t = CE entry t of the row (t < 24) pops before v or is kept.  The count
// fits 8 bits: v had < k live neighbours when it was hidden and every
// predecessor is one of them, so it is < k <= 4.  Unpacked: the count in
// deg[v] and 64 bits in bmask[v].  Entries past the mask compare pop keys.
constexpr bool kPackedPred = MPLD_PACKED_PRED != 0;
constexpr int kPredBits = kPackedPred ? 24 : 64;

__device__ __forceinline__ void stamp(Control* ctl, int i) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    ctl->t[i] = t;
  }
}

__device__ __forceinline__ void dstamp(Control* ctl, int i, int cnt) {
  if (blockIdx.x == 0 && threadIdx.x == 0 && i < 32) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    ctl->tr[i] = t;
    ctl->nr[i] = cnt;
  }
}

// Recovery pop-order key (R9): kept vertices (coloured by the search) sort above
// every hidden vertex; hidden ones by (round, priority) — u is popped before v
// iff key(u) > key(v).
__device__ __forceinline__ unsigned long long pop_key(int h, uint32_t p) {
  return h < 0 ? ~0ull : (((unsigned long long)(h + 1) << 32) | p);
}

// Layout of a vertex (binary search in layout_off), cached per thread: the
// tiles of a thread are consecutive ids, so the search rarely runs.
struct LayoutCache {
  int lo = 0, begin = 0, end = -1;  // layout lo covers [begin, end)
  __device__ __forceinline__ int get(const GraphView& g, int v) {
    if (g.n_layouts <= 1) return 0;
    if (v < begin || v >= end) {
      int a = 0, b = g.n_layouts;  // off[a] <= v < off[a+1]
      while (b - a > 1) {
        const int m = (a + b) >> 1;
        if (__ldg(&g.layout_off[m]) <= v) a = m; else b = m;
      }
      lo = a;
      begin = __ldg(&g.layout_off[a]);
      end = __ldg(&g.layout_off[a + 1]);
    }
    return lo;
  }
  __device__ __forceinline__ int local(const GraphView& g, int v) {  // layout-local id (R10)
    if (g.n_layouts <= 1) return v;
    get(g, v);
    return v - begin;
  }
};

// CTA queues in shared memory: items are pushed with one shared atomic per
// coalesced group of lanes (no CTA barrier inside a pass, so the warps of a CTA
// progress independently through their tiles) and flushed once at the end of
// the pass with one global atomic per CTA.  Items beyond kQCap go straight to
// the global queue (warp-aggregated atomics).
#ifndef MPLD_QCAP
#define MPLD_QCAP 4096
#endif
constexpr int kQCap = MPLD_QCAP;
struct CtaQueues {
  int n[2], m[2], base[2];
  int item[2][kQCap];
};

__device__ __forceinline__ void cq_init(CtaQueues& Q) {
  if (threadIdx.x < 2) Q.n[threadIdx.x] = 0;
  __syncthreads();
}

__device__ __forceinline__ void cq_push(CtaQueues& Q, int q, int v, int* gcnt, int* gout) {
  const cg::coalesced_group grp = cg::coalesced_threads();
  int base = 0;
  if (grp.thread_rank() == 0) base = atomicAdd(&Q.n[q], (int)grp.size());
  const int i = grp.shfl(base, 0) + (int)grp.thread_rank();
  if (i < kQCap) {
    Q.item[q][i] = v;
  } else {  // overflow: direct global append
    const cg::coalesced_group ov = cg::coalesced_threads();
    int gb = 0;
    if (ov.thread_rank() == 0) gb = atomicAdd(gcnt, (int)ov.size());
    gout[ov.shfl(gb, 0) + (int)ov.thread_rank()] = v;
  }
}

// Every thread of the CTA must call it (uniform control flow).
__device__ __forceinline__ void cq_flush(CtaQueues& Q, int q, int* gcnt, int* gout) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const int m = min(Q.n[q], kQCap);
    Q.m[q] = m;
    Q.base[q] = m ? atomicAdd(gcnt, m) : 0;
    Q.n[q] = 0;
  }
  __syncthreads();
  const int m = Q.m[q], b = Q.base[q];
  for (int i = threadIdx.x; i < m; i += blockDim.x) gout[b + i] = Q.item[q][i];
  __syncthreads();
}

// Item i of a frontier whose first s_cnt items sit in shared memory (a CTA
// queue of the single-CTA tail) and the rest in global memory.
__device__ __forceinline__ int frontier_item(const int* s_in, int s_cnt, const int* g_in, int i) {
  return i < s_cnt ? s_in[i] : __ldcg(&g_in[i - s_cnt]);
}

// The single-CTA tail of a level-synchronous loop (simplification rounds,
// recovery levels): the frontier stays in the CTA's two shared queues (items
// beyond kQCap spill to the global queue that is not being read), so a level
// costs its dependent loads plus two block barriers.
struct TailFrontier {
  int in_slot = -1;  // shared slot holding the input's first items (-1: input all global)
  int s_cnt = 0;
  const int* g_in;
  int out_slot = 0;
  __device__ __forceinline__ const int* s_in(const CtaQueues& Q) const { return in_slot >= 0 ? Q.item[in_slot] : nullptr; }
  __device__ __forceinline__ int* g_out(const Workspace& w) const { return g_in == w.q0 ? w.q1 : w.q0; }
  // after the level: the output becomes the input; returns its size
  __device__ __forceinline__ int advance(CtaQueues& Q, const Workspace& w) {
    __syncthreads();
    const int c = Q.n[out_slot];
    __syncthreads();
    if (threadIdx.x == 0 && in_slot >= 0) Q.n[in_slot] = 0;
    g_in = g_out(w);
    in_slot = out_slot;
    s_cnt = min(c, kQCap);
    out_slot ^= 1;
    __syncthreads();
    return c;
  }
  __device__ __forceinline__ void finish(CtaQueues& Q) {
    if (threadIdx.x < 2) Q.n[threadIdx.x] = 0;
    __syncthreads();
  }
};

// ---------------------------------------------------------------------------
// Input validation (MPLD_FLAG_VALIDATE, include/mpld.h invariants), fused into
// the first pass over the CSR: row pointers inside [0, nnz], rows strictly
// ascending, ids in range, no self loop, CE ∩ SE = ∅ are checked exactly per
// row.  Symmetry — every entry (v, u) has its transpose (u, v) — is checked as
// the multiset identity sum H(v, u) == sum H(u, v) over all entries (rows are
// strictly ascending, so entries are distinct): one 64-bit sum per direction,
// no lookups; an asymmetric graph passes with probability ~2^-64.
__device__ __forceinline__ unsigned long long pair_hash(int x, int y) {
  unsigned long long z = ((unsigned long long)(unsigned)x << 32) | (unsigned)y;  // splitmix64 finaliser
  z ^= z >> 30;
  z *= 0xbf58476d1ce4e5b9ull;
  z ^= z >> 27;
  z *= 0x94d049bb133111ebull;
  z ^= z >> 31;
  return z;
}

// One simplification round r >= 1: push the decrements of the frontier
// cur[0..cnt), tiles of kP * blockDim items starting at first, step stride.
// A neighbour enters round r+1 exactly when its live degree crosses k -> k-1.
// The decrement is unconditional (no load of the neighbour's round first):
// hidden vertices already sit below k (round-0 vertices at 0, later rounds at
// their degree when hidden) and stitch vertices at kStitchDeg, so only a live
// vertex can cross k -> k-1.
// The frontier is item i = frontier_item(s_in, s_cnt, g_in, i); hidden
// neighbours are pushed into CTA queue slot qo (overflow: ocnt / oarr).
__device__ void peel_round(const GraphView& g, const Workspace& w, int k, int r, int cnt, int first, int stride,
                           const int* s_in, int s_cnt, const int* g_in, CtaQueues& Q, int qo, int* ocnt, int* oarr) {
  for (int t0 = first; t0 < cnt; t0 += stride) {
    int e[kP], e1[kP];
#pragma unroll
    for (int j = 0; j < kP; ++j) {
      const int i = t0 + j * blockDim.x + threadIdx.x;
      const int v = i < cnt ? frontier_item(s_in, s_cnt, g_in, i) : -1;
      e[j] = v >= 0 ? __ldg(&g.ce_rp[v]) : 0;
      e1[j] = v >= 0 ? __ldg(&g.ce_rp[v + 1]) : 0;
    }
    while (true) {
      bool open = false;
#pragma unroll
      for (int j = 0; j < kP; ++j) open |= e[j] < e1[j];
      if (!open) break;
      int u[kP][kNb], old[kP][kNb];
#pragma unroll
      for (int j = 0; j < kP; ++j)
#pragma unroll
        for (int t = 0; t < kNb; ++t) u[j][t] = e[j] + t < e1[j] ? __ldg(&g.ce_col[e[j] + t]) : -1;
#pragma unroll
      for (int j = 0; j < kP; ++j)
#pragma unroll
        for (int t = 0; t < kNb; ++t) old[j][t] = u[j][t] >= 0 ? atomicSub(&w.deg[u[j][t]], 1) : 0;
#pragma unroll
      for (int j = 0; j < kP; ++j) {
#pragma unroll
        for (int t = 0; t < kNb; ++t) {
          if (old[j][t] == k) {
            w.hround[u[j][t]] = r + 1;
            cq_push(Q, qo, u[j][t], ocnt, oarr);
          }
        }
        e[j] += kNb;
      }
    }
  }
}

// The final pass of the simplification (the rounds are final): see the
// comment at its call in mpld_simplify_components.
// mode bit 1: the component seeds (kept vertices); bit 2: the recovery's
// predecessor counts, "popped before" bitmasks and level 0 (hidden vertices).
__device__ void final_pass(const GraphView& g, const Workspace& w, CtaQueues& Q, int mode) {
  const int n = g.n;
  const int nth = gridDim.x * blockDim.x;
  const int tile0f = blockIdx.x * blockDim.x * kPF, tstridef = nth * kPF;
  Control* ctl = w.ctl;
  // One batched walk over the CE row of every vertex: a hidden vertex counts
  // its predecessors, a kept one looks for a kept neighbour of smaller id
  // (rows ascending: the walk stops at the first larger id).
  for (int t0 = tile0f; t0 < n; t0 += tstridef) {
    int v[kPF], e0[kPF], e[kPF], e1[kPF], cnt[kPF];
    unsigned long long kv[kPF], bm[kPF];
    bool seed[kPF];
#pragma unroll
    for (int j = 0; j < kPF; ++j) {
      v[j] = t0 + j * blockDim.x + threadIdx.x;
      const int hv = v[j] < n ? __ldcg(&w.hround[v[j]]) : -1;
      kv[j] = v[j] < n ? pop_key(hv, __ldcg(&w.prio[v[j]])) : ~0ull;
      const bool walk = v[j] < n && (mode & (kv[j] == ~0ull ? 1 : 2));
      e[j] = e0[j] = walk ? __ldg(&g.ce_rp[v[j]]) : 0;
      e1[j] = walk ? __ldg(&g.ce_rp[v[j] + 1]) : 0;
      cnt[j] = 0;
      bm[j] = 0ull;
      seed[j] = true;
    }
    while (true) {
      bool open = false;
#pragma unroll
      for (int j = 0; j < kPF; ++j) open |= e[j] < e1[j];
      if (!open) break;
      int u[kPF][kNb], hu[kPF][kNb];
      unsigned pu[kPF][kNb];
#pragma unroll
      for (int j = 0; j < kPF; ++j)
#pragma unroll
        for (int t = 0; t < kNb; ++t) u[j][t] = e[j] + t < e1[j] ? __ldg(&g.ce_col[e[j] + t]) : -1;
#pragma unroll
      for (int j = 0; j < kPF; ++j)
#pragma unroll
        for (int t = 0; t < kNb; ++t) {
          hu[j][t] = u[j][t] >= 0 ? __ldcg(&w.hround[u[j][t]]) : -1;
          pu[j][t] = u[j][t] >= 0 && kv[j] != ~0ull ? __ldcg(&w.prio[u[j][t]]) : 0u;
        }
#pragma unroll
      for (int j = 0; j < kPF; ++j) {
        bool past = false;  // kept v: a neighbour above v was seen
#pragma unroll
        for (int t = 0; t < kNb; ++t) {
          if (u[j][t] < 0) continue;
          if (kv[j] != ~0ull) {
            const bool before = pop_key(hu[j][t], pu[j][t]) > kv[j];  // popped before v, or kept
            cnt[j] += (hu[j][t] >= 0 && before) ? 1 : 0;
            const int rel = e[j] + t - e0[j];
            if (rel < kPredBits && before) bm[j] |= 1ull << rel;
          } else {
            if (u[j][t] < v[j] && hu[j][t] == -1) seed[j] = false;
            past |= u[j][t] > v[j];
          }
        }
        e[j] = (kv[j] == ~0ull && (past || !seed[j])) ? e1[j] : e[j] + kNb;
      }
    }
#pragma unroll
    for (int j = 0; j < kPF; ++j) {
      if (v[j] >= n || !(mode & (kv[j] == ~0ull ? 1 : 2))) continue;
      if (kv[j] != ~0ull) {
        if (kPackedPred) {
          w.deg[v[j]] = cnt[j] | (int)((unsigned)bm[j] << 8);
        } else {
          w.deg[v[j]] = cnt[j];
          w.bmask[v[j]] = bm[j];
        }
        if (cnt[j] == 0) cq_push(Q, 1, v[j], &ctl->rq[0], w.q0);
      } else {
        // stitch neighbours (stitch vertices only; rows ascending)
        if (seed[j])
          for (int x = __ldg(&g.se_rp[v[j]]), x1 = __ldg(&g.se_rp[v[j] + 1]); x < x1; ++x) {
            const int u = __ldg(&g.se_col[x]);
            if (u > v[j]) break;
            if (__ldcg(&w.hround[u]) == -1) {
              seed[j] = false;
              break;
            }
          }
        if (seed[j]) cq_push(Q, 0, v[j], &ctl->n_seed, w.roots);
      }
    }
  }
  if (mode & 1) cq_flush(Q, 0, &ctl->n_seed, w.roots);
  if (mode & 2) cq_flush(Q, 1, &ctl->rq[0], w.q0);
  if (mode & 1) stamp(w.ctl, 3);
}

// ---------------------------------------------------------------------------
// Simplification (R8, §2.2 "simplify the layout graph"):
// round r hides every not-yet-hidden vertex without stitch edges whose
// conflict degree among not-yet-hidden vertices is < k.
//   * rounds 0 and 1 need no barrier: round 0 is a property of each vertex,
//     and the degree after round 0 is pulled from the neighbours' static data;
//   * a vertex enters round r+1 (r >= 1) exactly when its live degree crosses
//     k -> k-1 while round r is pushed, so each round only touches the
//     neighbours of the previous round (frontier queue).
// Then one pass over all vertices writes the recovery pop keys, the search
// seeds and the recovery's predecessor counts and level 0.
__global__ void __launch_bounds__(1024, MPLD_GRAPH_MINB) mpld_simplify_components(GraphView g, Workspace w, int k,
                                                                    int* colors, long long* counts, int validate,
                                                                    int cluster_rounds, int separate_prep) {
  if (gated_off(w)) return;  // after the tile pipeline, which took the input
  GridBarrier grid(&w.ctl->bar0);
  __shared__ CtaQueues Q;
  cq_init(Q);
  stamp(w.ctl, 12);
  const int n = g.n;
  const int nth = gridDim.x * blockDim.x;
  const int tile0 = blockIdx.x * blockDim.x * kP, tstride = nth * kP;
  const int tile0f = blockIdx.x * blockDim.x * kPF, tstridef = nth * kPF;
  Control* ctl = w.ctl;
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < 2 * g.n_layouts; l += nth) counts[l] = 0;

  // rounds 0 and 1, recovery priorities, colours = -1 (and the optional
  // validation of the input, fused into this first pass over the CSR)
  const int nnz_ce = __ldg(&g.ce_rp[n]), nnz_se = __ldg(&g.se_rp[n]);
  int hidden0 = 0;
  bool bad = false;
  unsigned long long hs[4] = {0ull, 0ull, 0ull, 0ull};  // sum H(v,u), H(u,v) over CE, then over SE
  if (blockIdx.x == 0 && threadIdx.x == 0 && w.build_err && *w.build_err) {  // CSR built on the device from bad input
    bad = true;
    *w.build_err = 0;
  }
  if (validate && blockIdx.x == 0 && threadIdx.x == 0) {
    if (g.layout_off[0] != 0 || g.layout_off[g.n_layouts] != g.n || g.ce_rp[0] != 0 || g.se_rp[0] != 0) bad = true;
    for (int l = 0; l < g.n_layouts; ++l)
      if (g.layout_off[l] > g.layout_off[l + 1]) bad = true;
  }
  LayoutCache lc;
  for (int t0 = tile0f; t0 < n; t0 += tstridef) {
    int v[kPF], e[kPF], e1[kPF], d[kPF], hr[kPF], prev[kPF];
    bool need[kPF], scan[kPF];
#pragma unroll
    for (int j = 0; j < kPF; ++j) {
      v[j] = t0 + j * blockDim.x + threadIdx.x;
      int a = 0, b = 0, sa = 0, sb = 0;
      if (v[j] < n) {
        a = __ldg(&g.ce_rp[v[j]]);
        b = __ldg(&g.ce_rp[v[j] + 1]);
        sa = __ldg(&g.se_rp[v[j]]);
        sb = __ldg(&g.se_rp[v[j] + 1]);
      }
      if (validate && v[j] < n) {
        if (a < 0 || a > b || b > nnz_ce) {  // never read outside the column arrays
          bad = true;
          b = a = 0;
        }
        if (sa < 0 || sa > sb || sb > nnz_se) {
          bad = true;
          sb = sa = 0;
        }
        // stitch rows (rare): exact per-entry checks, CE ∩ SE by binary search in the CE row
        for (int x = sa, pu = -1; x < sb; ++x) {
          const int u = __ldg(&g.se_col[x]);
          if (u < 0 || u >= n || u == v[j] || u <= pu) bad = true;
          pu = u;
          hs[2] += pair_hash(v[j], u);
          hs[3] += pair_hash(u, v[j]);
          int lo = a, hi = b;
          while (lo < hi) {
            const int m = (lo + hi) >> 1;
            const int y = __ldg(&g.ce_col[m]);
            if (y == u) bad = true;
            if (y < u) lo = m + 1; else hi = m;
          }
        }
      }
      e[j] = a;
      e1[j] = b;
      d[j] = 0;
      hr[j] = -1;
      prev[j] = -1;
      need[j] = false;
      if (v[j] < n) {
        w.prio[v[j]] = lowbias32((uint32_t)lc.local(g, v[j]));
        colors[v[j]] = -1;  // every vertex is coloured later by exactly one search shard or the recovery
        if (sb > sa) {
          w.deg[v[j]] = kStitchDeg;
        } else if (b - a < k) {
          hr[j] = 0;
          ++hidden0;
        } else {
          need[j] = true;
        }
      }
      scan[j] = need[j] || (validate && v[j] < n);
    }
    // the CE rows: live degree after round 0 of the vertices that survive it
    // (pulled from the neighbours' row pointers), validation of every row
    while (true) {
      bool open = false;
#pragma unroll
      for (int j = 0; j < kPF; ++j) open |= scan[j] && e[j] < e1[j];
      if (!open) break;
      int u[kPF][kNb], r0[kPF][kNb], r1[kPF][kNb], s0[kPF][kNb], s1[kPF][kNb];
#pragma unroll
      for (int j = 0; j < kPF; ++j)
#pragma unroll
        for (int t = 0; t < kNb; ++t) u[j][t] = scan[j] && e[j] + t < e1[j] ? __ldg(&g.ce_col[e[j] + t]) : -1;
#pragma unroll
      for (int j = 0; j < kPF; ++j)
#pragma unroll
        for (int t = 0; t < kNb; ++t) {
          const bool ok = need[j] && (unsigned)u[j][t] < (unsigned)n;  // invalid ids are flagged by the validation
          r0[j][t] = ok ? __ldg(&g.ce_rp[u[j][t]]) : 0;
          r1[j][t] = ok ? __ldg(&g.ce_rp[u[j][t] + 1]) : 0;
          s0[j][t] = ok ? __ldg(&g.se_rp[u[j][t]]) : 0;
          s1[j][t] = ok ? __ldg(&g.se_rp[u[j][t] + 1]) : 0;
        }
#pragma unroll
      for (int j = 0; j < kPF; ++j) {
#pragma unroll
        for (int t = 0; t < kNb; ++t) {
          if (e[j] + t >= e1[j]) continue;
          if (need[j]) d[j] += (s1[j][t] > s0[j][t] || r1[j][t] - r0[j][t] >= k) ? 1 : 0;
          if (validate) {
            if (u[j][t] < 0 || u[j][t] >= n || u[j][t] == v[j] || u[j][t] <= prev[j]) bad = true;
            prev[j] = u[j][t];
            hs[0] += pair_hash(v[j], u[j][t]);
            hs[1] += pair_hash(u[j][t], v[j]);
          }
        }
        e[j] += kNb;
      }
    }
#pragma unroll
    for (int j = 0; j < kPF; ++j) {
      if (need[j]) {
        w.deg[v[j]] = d[j];
        if (d[j] < k) {
          hr[j] = 1;
          cq_push(Q, 0, v[j], &ctl->qcnt[1], w.q1);
        }
      } else if (hr[j] == 0) {
        w.deg[v[j]] = 0;  // below k for good: later rounds decrement without checking (peel_round)
      }
      if (v[j] < n) w.hround[v[j]] = hr[j];
    }
  }
  cq_flush(Q, 0, &ctl->qcnt[1], w.q1);
  hidden0 = __reduce_add_sync(0xffffffffu, hidden0);
  if ((threadIdx.x & 31) == 0 && hidden0) atomicAdd(&ctl->n_hidden, hidden0);
  if (bad) atomicOr(&ctl->err, kErrGraph);
  if (validate) {  // CTA sums of the symmetry hashes, one atomic per CTA and direction
    __shared__ unsigned long long s_h[32][4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) hs[q] += __shfl_xor_sync(0xffffffffu, hs[q], o);
      if ((threadIdx.x & 31) == 0) s_h[threadIdx.x >> 5][q] = hs[q];
    }
    __syncthreads();
    if (threadIdx.x < 4) {
      unsigned long long x = 0ull;
      for (int i = 0; i < (int)(blockDim.x >> 5); ++i) x += s_h[i][threadIdx.x];
      atomicAdd(&ctl->vh[threadIdx.x], x);
    }
  }
  grid.sync();
  stamp(w.ctl, 0);
  if (validate && (__ldcg(&ctl->vh[0]) != __ldcg(&ctl->vh[1]) || __ldcg(&ctl->vh[2]) != __ldcg(&ctl->vh[3]))) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&ctl->err, kErrGraph);  // not symmetric
    return;  // every CTA sees the same sums
  }
  if (__ldcg(&ctl->err)) return;  // invalid input: every later kernel exits too

  // rounds r >= 1: push the frontier's decrements.  Large frontiers: every
  // CTA, one grid barrier per round; up to kGroup * blockDim items: the first
  // kGroup CTAs with their own barrier; up to kTail items: CTA 0 alone with
  // block barriers (a barrier over fewer CTAs is cheaper; the rounds only need
  // the dependent-load latency).  Everyone meets at one grid barrier after.
  int r = 1;
  int cnt = __ldcg(&ctl->qcnt[1]);
  const int grid_min = cluster_rounds ? kClusterTailMax : kGroup * (int)blockDim.x;
  while (cnt > grid_min) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      ctl->qcnt[(r + 2) % 3] = 0;
      ctl->n_hidden += cnt;
    }
    dstamp(ctl, r, cnt);
    {
      const int* cur = (r & 1) ? w.q1 : w.q0;
      int* nxt = (r & 1) ? w.q0 : w.q1;
      int* ncnt = &ctl->qcnt[(r + 1) % 3];
      peel_round(g, w, k, r, cnt, tile0, tstride, nullptr, 0, cur, Q, 0, ncnt, nxt);
      cq_flush(Q, 0, ncnt, nxt);
    }
    ++r;
    grid.sync();
    stamp(w.ctl, 2);
    cnt = __ldcg(&ctl->qcnt[r % 3]);
  }
  if (cluster_rounds) {  // the remaining rounds: mpld_simplify_tail, then mpld_final_pass
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl->n_rounds = r;
    return;
  }
  if (cnt > kTail && (int)blockIdx.x < kGroup) {  // group rounds (every CTA read the same cnt)
    GridBarrier grp(&ctl->bar0g, kGroup);
    while (cnt > kTail) {
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctl->qcnt[(r + 2) % 3] = 0;
        ctl->n_hidden += cnt;
      }
      dstamp(ctl, r, cnt);
      const int* cur = (r & 1) ? w.q1 : w.q0;
      int* nxt = (r & 1) ? w.q0 : w.q1;
      int* ncnt = &ctl->qcnt[(r + 1) % 3];
      peel_round(g, w, k, r, cnt, blockIdx.x * blockDim.x * kP, kGroup * blockDim.x * kP, nullptr, 0, cur, Q, 0,
                 ncnt, nxt);
      cq_flush(Q, 0, ncnt, nxt);
      ++r;
      grp.sync();
      cnt = __ldcg(&ctl->qcnt[r % 3]);
    }
  }
  if (blockIdx.x == 0) {
    if (cnt > 0) {  // the single-CTA tail, frontier in shared memory
      int c = cnt;
      TailFrontier tf;
      tf.g_in = (r & 1) ? w.q1 : w.q0;
      while (c > 0) {
        if (threadIdx.x == 0) {
          ctl->tcnt[0] = 0;  // own overflow counter
          ctl->n_hidden += c;
        }
        dstamp(ctl, r, c);
        __syncthreads();
        peel_round(g, w, k, r, c, 0, blockDim.x * kP, tf.s_in(Q), tf.s_cnt, tf.g_in, Q, tf.out_slot,
                   &ctl->tcnt[0], tf.g_out(w));
        ++r;
        c = tf.advance(Q, w);
      }
      tf.finish(Q);
    }
    if (threadIdx.x == 0) ctl->n_rounds = r;
  }
  grid.sync();
  r = __ldcg(&ctl->n_rounds);
  if (blockIdx.x == 0 && threadIdx.x == 0) ctl->n_rounds = __ldcg(&ctl->n_hidden) ? r : 0;
  stamp(w.ctl, 1);

  // Final pass (rounds are final now):
  //  * the "popped before" bitmask of every hidden vertex (pop keys, R9);
  //  * component-search seeds: a kept vertex with no kept neighbour (CE ∪ SE)
  //    of smaller id.  Every component has at least one seed (its minimum);
  //    the search kernel keeps a seed only if it is its component's minimum,
  //    so no union-find and no further grid barrier are needed here;
  //  * recovery: hidden predecessors of every hidden vertex (conflict
  //    neighbours popped before it) and level 0 = the vertices without one.
  final_pass(g, w, Q, separate_prep ? 1 : 3);
}

// ---------------------------------------------------------------------------
// The last simplification rounds (<= kClusterTailMax hidden vertices) on ONE
// thread-block cluster: every CTA pushes the decrements of the vertices its
// own threads hid (frontier slots in its shared memory, no global queue), the
// rounds are separated by the hardware cluster barrier.  Then
// mpld_final_pass runs the final pass on the whole GPU.
template <typename Push>
__device__ __forceinline__ void peel_vertex(const GraphView& g, const Workspace& w, int k, int r, int v, Push push) {
  const int e1 = __ldg(&g.ce_rp[v + 1]);
  for (int e = __ldg(&g.ce_rp[v]); e < e1; e += kNb) {
    int u[kNb], old[kNb];
#pragma unroll
    for (int t = 0; t < kNb; ++t) u[t] = e + t < e1 ? __ldg(&g.ce_col[e + t]) : -1;
#pragma unroll
    for (int t = 0; t < kNb; ++t) old[t] = u[t] >= 0 ? atomicSub(&w.deg[u[t]], 1) : 0;
#pragma unroll
    for (int t = 0; t < kNb; ++t)
      if (old[t] == k) {  // live degree k -> k-1: hidden in round r + 1 (see peel_round)
        w.hround[u[t]] = r + 1;
        push(u[t]);
      }
  }
}

constexpr int kTQ = 4096;  // frontier slots per CTA and parity of the cluster tails

__global__ void __launch_bounds__(1024) mpld_simplify_tail(GraphView g, Workspace w, int k) {
  pdl_begin();
  if (gated_off(w)) return;
  cg::cluster_group cl = cg::this_cluster();
  __shared__ int s_item[2][kTQ];
  const int tq = min(max(w.tail_slots, 0), kTQ);  // slots in use (MPLD_TAIL_SLOTS lowers it: tests)
  __shared__ int s_n[2];
  __shared__ int s_tot;
  const int rank = (int)cl.block_rank(), nc = (int)cl.num_blocks();
  Control* ctl = w.ctl;
  if (threadIdx.x < 2) s_n[threadIdx.x] = 0;
  cl.sync();
  const bool ok = !__ldcg(&ctl->err);
  int r = ok ? __ldcg(&ctl->n_rounds) : 0;  // the first round the grid kernel left
  int total = ok ? __ldcg(&ctl->qcnt[r % 3]) : 0;
  const int* g_first = (r & 1) ? w.q1 : w.q0;
  int* const ovf[2] = {w.q0 == g_first ? w.q1 : w.q0, w.roots};  // spill lists (not the first frontier)
  int n_ovf = 0;
  for (int t = 0; total > 0; ++t) {
    const int in = t & 1, outs = in ^ 1;
    if (threadIdx.x == 0) s_n[outs] = 0;
    if (rank == 0 && threadIdx.x == 0) {
      ctl->tovf[outs] = 0;
      ctl->n_hidden += total;
    }
    __syncthreads();
    auto push = [&](int u) {
      const int i = atomicAdd(&s_n[outs], 1);
      if (i < tq) s_item[outs][i] = u;
      else ovf[outs][atomicAdd(&ctl->tovf[outs], 1)] = u;
    };
    if (t == 0) {
      for (int i = rank * (int)blockDim.x + threadIdx.x; i < total; i += nc * (int)blockDim.x)
        peel_vertex(g, w, k, r, __ldcg(&g_first[i]), push);
    } else {
      const int mine = min(s_n[in], tq);
      for (int i = threadIdx.x; i < mine; i += blockDim.x) peel_vertex(g, w, k, r, s_item[in][i], push);
      for (int i = rank * (int)blockDim.x + threadIdx.x; i < n_ovf; i += nc * (int)blockDim.x)
        peel_vertex(g, w, k, r, __ldcg(&ovf[in][i]), push);
    }
    cl.sync();  // the round's decrements are done; every CTA's output slot is complete
    if (threadIdx.x < 32) {
      const int x = (int)threadIdx.x < nc ? min(*cl.map_shared_rank(&s_n[outs], (int)threadIdx.x), tq) : 0;
      const int sum = __reduce_add_sync(0xffffffffu, x);
      if (threadIdx.x == 0) s_tot = sum;
    }
    __syncthreads();
    n_ovf = __ldcg(&ctl->tovf[outs]);
    total = s_tot + n_ovf;
    ++r;
  }
  cl.sync();  // no CTA leaves while others may still read its shared memory
  if (rank == 0 && threadIdx.x == 0) ctl->n_rounds = __ldcg(&ctl->n_hidden) ? r : 0;
}

__global__ void __launch_bounds__(1024, MPLD_GRAPH_MINB) mpld_final_pass(GraphView g, Workspace w, int separate_prep) {
  pdl_begin();
  if (gated_off(w)) return;
  __shared__ CtaQueues Q;
  cq_init(Q);
  if (__ldcg(&w.ctl->err)) return;
  final_pass(g, w, Q, separate_prep ? 1 : 3);
}

// The recovery's share of the final pass (predecessor counts, bitmasks, level
// 0) as its own kernel, on a second stream while the search runs.
__global__ void __launch_bounds__(1024, MPLD_GRAPH_MINB) mpld_recover_prep(GraphView g, Workspace w) {
  if (gated_off(w)) return;
  __shared__ CtaQueues Q;
  cq_init(Q);
  if (__ldcg(&w.ctl->err)) return;
  final_pass(g, w, Q, 2);
}

// ---------------------------------------------------------------------------
// Recovery (R9, §2.2 "recover the nodes removed in
// simplification step"): the hidden stack is popped LIFO — rounds in reverse,
// inside a round in descending lowbias32(layout-local id) — and each vertex
// takes the smallest mask unused by its already-coloured conflict neighbours.
//
// Only the relative order of conflict-adjacent hidden vertices matters, so the
// LIFO order is realised level-synchronously over the DAG "u before v" (u, v
// adjacent, u popped first): level 0 = hidden vertices without a hidden
// predecessor (listed by the simplification kernel); a vertex joins the next
// level when its last predecessor is coloured.  Every level is coloured in
// parallel, one grid barrier per level (DAG depth ~ 10-20 on layout graphs);
// the result equals the sequential pop.
// One recovery level: colour the ready vertices cur[0..cnt) (tiles as in
// peel_round), queue the successors whose last predecessor this was.
__device__ void recover_level(const GraphView& g, const Workspace& w, int k, int* colors, int cnt, int first,
                              int stride, const int* s_in, int s_cnt, const int* g_in, CtaQueues& Q, int qo,
                              int* ocnt, int* oarr) {
  for (int t0 = first; t0 < cnt; t0 += stride) {
    int v[kP], e0[kP], e[kP], e1[kP];
    unsigned long long bm[kP], kv[kP];
    unsigned used[kP];
#pragma unroll
    for (int j = 0; j < kP; ++j) {
      const int i = t0 + j * blockDim.x + threadIdx.x;
      v[j] = i < cnt ? frontier_item(s_in, s_cnt, g_in, i) : -1;
      bm[j] = v[j] < 0 ? 0ull
                       : (kPackedPred ? (unsigned long long)((unsigned)__ldcg(&w.deg[v[j]]) >> 8) : __ldcg(&w.bmask[v[j]]));
      e[j] = e0[j] = v[j] >= 0 ? __ldg(&g.ce_rp[v[j]]) : 0;
      e1[j] = v[j] >= 0 ? __ldg(&g.ce_rp[v[j] + 1]) : 0;
      kv[j] = e1[j] - e0[j] > kPredBits ? pop_key(__ldcg(&w.hround[v[j]]), __ldcg(&w.prio[v[j]])) : 0ull;  // long rows
      used[j] = 0u;
    }
    while (true) {
      bool open = false;
#pragma unroll
      for (int j = 0; j < kP; ++j) open |= e[j] < e1[j];
      if (!open) break;
      int u[kP][kNb], x[kP][kNb];
      bool before[kP][kNb];
#pragma unroll
      for (int j = 0; j < kP; ++j)
#pragma unroll
        for (int t = 0; t < kNb; ++t) u[j][t] = e[j] + t < e1[j] ? __ldg(&g.ce_col[e[j] + t]) : -1;
#pragma unroll
      for (int j = 0; j < kP; ++j)
#pragma unroll
        for (int t = 0; t < kNb; ++t) {  // popped before v (or kept): the final pass's bit, past 64 the keys
          const int rel = e[j] + t - e0[j];
          before[j][t] = u[j][t] >= 0 && (rel < kPredBits ? ((bm[j] >> rel) & 1ull) != 0ull
                                                   : pop_key(__ldcg(&w.hround[u[j][t]]), __ldcg(&w.prio[u[j][t]])) > kv[j]);
        }
#pragma unroll
      for (int j = 0; j < kP; ++j)
#pragma unroll
        for (int t = 0; t < kNb; ++t)
          x[j][t] = u[j][t] < 0 ? -1 : (before[j][t] ? __ldcg(&colors[u[j][t]]) : atomicSub(&w.deg[u[j][t]], 1));
#pragma unroll
      for (int j = 0; j < kP; ++j) {
#pragma unroll
        for (int t = 0; t < kNb; ++t) {
          if (u[j][t] < 0) continue;
          if (before[j][t]) {
            if (x[j][t] >= 0) used[j] |= 1u << x[j][t];
          } else if ((x[j][t] & 0xff) == 1) {  // v was u's last predecessor
            cq_push(Q, qo, u[j][t], ocnt, oarr);
          }
        }
        e[j] += kNb;
      }
    }
#pragma unroll
    for (int j = 0; j < kP; ++j) {
      if (v[j] < 0) continue;
      const int c = __ffs(~used[j]) - 1;
      colors[v[j]] = c < k ? c : 0;  // c < k by the simplification invariant
    }
  }
}

// Eq. (1a) cost per layout and the statistics, by the last CTA of a kernel
// to finish (counter `done`; the caller's threads have all finished their part).
__device__ void finalize_outputs(const GraphView& g, const Workspace& w, const Outputs& out, int* done) {
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(done, 1) == (int)gridDim.x - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int l = threadIdx.x; l < g.n_layouts; l += blockDim.x) {
    const long long nc = __ldcg(&out.counts[2 * l]);
    const long long ns = __ldcg(&out.counts[2 * l + 1]);
    out.cost[l] = __dadd_rn(__dmul_rn(out.alpha, (double)ns), (double)nc);
  }
  if (threadIdx.x == 0 && out.stats) {
    Control* ctl = w.ctl;
    out.stats[MPLD_STAT_COMPONENTS] = __ldcg(&ctl->n_comp);
    out.stats[MPLD_STAT_HIDDEN] = __ldcg(&ctl->n_hidden);
    out.stats[MPLD_STAT_ROUNDS] = __ldcg(&ctl->n_rounds);
    out.stats[MPLD_STAT_MAX_COMP] = __ldcg(&ctl->max_comp);
    out.stats[MPLD_STAT_STEPS] = (long long)__ldcg(&ctl->steps);
    out.stats[MPLD_STAT_TRUNCATED] = __ldcg(&ctl->truncated);
    out.stats[MPLD_STAT_ERROR] = __ldcg(&ctl->err);
    out.stats[MPLD_STAT_LAUNCHES] = out.launches;
    out.stats[MPLD_STAT_MAX_STEPS] = __ldcg(&ctl->max_steps_comp);
    out.stats[MPLD_STAT_SPILL_REFUSED] = __ldcg(&ctl->spill_refused);
  }
}

__device__ void recover_levels(const GraphView& g, const Workspace& w, int k, int* colors, GridBarrier& grid,
                               CtaQueues& Q, int cluster_tail);

// With out.enabled the search kernels have accumulated the counts (one shard)
// and the last CTA of the recovery writes the costs and statistics.
__global__ void __launch_bounds__(1024, MPLD_GRAPH_MINB) mpld_recover(GraphView g, Workspace w, int k, int* colors,
                                                                    Outputs out) {
  pdl_begin();
  if (gated_off(w)) return;
  GridBarrier grid(&w.ctl->bar1);
  __shared__ CtaQueues Q;
  cq_init(Q);
  stamp(w.ctl, 13);
  if (!__ldcg(&w.ctl->err)) recover_levels(g, w, k, colors, grid, Q, out.cluster_tail);
  if (out.enabled && !out.cluster_tail) finalize_outputs(g, w, out, &w.ctl->done_recover);
}

__device__ void recover_levels(const GraphView& g, const Workspace& w, int k, int* colors, GridBarrier& grid,
                               CtaQueues& Q, int cluster_tail) {
  const int nth = gridDim.x * blockDim.x;
  Control* ctl = w.ctl;
  const int tile0 = blockIdx.x * blockDim.x * kP, tstride = nth * kP;
  // as the simplification rounds: every CTA for large levels, the first
  // kGroup CTAs with their own barrier for levels up to kGroup * blockDim
  // items, CTA 0 alone (frontier in shared memory) for the last small levels
  int L = 0;
  int cnt = __ldcg(&ctl->rq[0]);
  const int grid_min = cluster_tail ? kClusterTailMax : kGroup * (int)blockDim.x;
  while (cnt > grid_min) {
    dstamp(ctl, 16 + L, cnt);
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl->rq[(L + 2) % 3] = 0;
    {
      const int* cur = (L & 1) ? w.q1 : w.q0;
      int* nxt = (L & 1) ? w.q0 : w.q1;
      int* ncnt = &ctl->rq[(L + 1) % 3];
      recover_level(g, w, k, colors, cnt, tile0, tstride, nullptr, 0, cur, Q, 0, ncnt, nxt);
      cq_flush(Q, 0, ncnt, nxt);
    }
    ++L;
    grid.sync();
    stamp(w.ctl, 9);
    cnt = __ldcg(&ctl->rq[L % 3]);
  }
  if (cluster_tail) {  // the remaining levels: mpld_recover_tail (one thread-block cluster)
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl->n_levels = L;
    return;
  }
  if (cnt > kTail && (int)blockIdx.x < kGroup) {  // group levels (every CTA read the same cnt)
    GridBarrier grp(&ctl->bar1g, kGroup);
    while (cnt > kTail) {
      dstamp(ctl, 16 + L, cnt);
      if (blockIdx.x == 0 && threadIdx.x == 0) ctl->rq[(L + 2) % 3] = 0;
      const int* cur = (L & 1) ? w.q1 : w.q0;
      int* nxt = (L & 1) ? w.q0 : w.q1;
      int* ncnt = &ctl->rq[(L + 1) % 3];
      recover_level(g, w, k, colors, cnt, blockIdx.x * blockDim.x * kP, kGroup * blockDim.x * kP, nullptr, 0, cur,
                    Q, 0, ncnt, nxt);
      cq_flush(Q, 0, ncnt, nxt);
      ++L;
      grp.sync();
      cnt = __ldcg(&ctl->rq[L % 3]);
    }
  }
  if (blockIdx.x == 0) {
    if (cnt > 0) {  // the single-CTA tail
      int c = cnt;
      TailFrontier tf;
      tf.g_in = (L & 1) ? w.q1 : w.q0;
      while (c > 0) {
        if (threadIdx.x == 0) ctl->trq[0] = 0;  // own overflow counter, as in the simplification tail
        __syncthreads();
        recover_level(g, w, k, colors, c, 0, blockDim.x * kP, tf.s_in(Q), tf.s_cnt, tf.g_in, Q, tf.out_slot,
                      &ctl->trq[0], tf.g_out(w));
        ++L;
        c = tf.advance(Q, w);
      }
    }
    if (threadIdx.x == 0) ctl->n_levels = L;
  }
}

// ---------------------------------------------------------------------------
// The last recovery levels (<= kClusterTailMax ready vertices) on ONE
// thread-block cluster of kTC CTAs: the frontier lives in the CTAs' shared
// memory (read across the cluster through distributed shared memory) and the
// levels are separated by the hardware cluster barrier — no global counter,
// flush or grid barrier per level.  Ready vertices beyond a CTA's kTQ slots
// spill to a global list per level parity (roots / hcomp, free after the
// search).  The last CTA writes the Eq. (1a) costs and the statistics.
template <typename Push>
__device__ __forceinline__ void recover_vertex(const GraphView& g, const Workspace& w, int k, int* colors, int v,
                                               Push push) {
  const int e0 = __ldg(&g.ce_rp[v]), e1 = __ldg(&g.ce_rp[v + 1]);
  const unsigned long long bm =
      kPackedPred ? (unsigned long long)((unsigned)__ldcg(&w.deg[v]) >> 8) : __ldcg(&w.bmask[v]);
  const unsigned long long kv = e1 - e0 > kPredBits ? pop_key(__ldcg(&w.hround[v]), __ldcg(&w.prio[v])) : 0ull;
  unsigned used = 0u;
  for (int e = e0; e < e1; e += kNb) {
    int u[kNb], x[kNb];
    bool before[kNb];
#pragma unroll
    for (int t = 0; t < kNb; ++t) u[t] = e + t < e1 ? __ldg(&g.ce_col[e + t]) : -1;
#pragma unroll
    for (int t = 0; t < kNb; ++t) {  // popped before v (or kept): the final pass's bit, past 64 the keys
      const int rel = e + t - e0;
      before[t] = u[t] >= 0 && (rel < kPredBits ? ((bm >> rel) & 1ull) != 0ull
                                         : pop_key(__ldcg(&w.hround[u[t]]), __ldcg(&w.prio[u[t]])) > kv);
    }
#pragma unroll
    for (int t = 0; t < kNb; ++t) x[t] = u[t] < 0 ? -1 : (before[t] ? __ldcg(&colors[u[t]]) : atomicSub(&w.deg[u[t]], 1));
#pragma unroll
    for (int t = 0; t < kNb; ++t) {
      if (u[t] < 0) continue;
      if (before[t]) {
        if (x[t] >= 0) used |= 1u << x[t];
      } else if ((x[t] & 0xff) == 1) {  // v was u's last predecessor
        push(u[t]);
      }
    }
  }
  const int c = __ffs(~used) - 1;
  colors[v] = c < k ? c : 0;  // c < k by the simplification invariant
}

__global__ void __launch_bounds__(1024) mpld_recover_tail(GraphView g, Workspace w, int k, int* colors, Outputs out) {
  pdl_begin();
  if (gated_off(w)) return;
  cg::cluster_group cl = cg::this_cluster();
  __shared__ int s_item[2][kTQ];
  const int tq = min(max(w.tail_slots, 0), kTQ);  // slots in use (MPLD_TAIL_SLOTS lowers it: tests)
  __shared__ int s_n[2];
  __shared__ int s_pref[kTC + 1];
  const int rank = (int)cl.block_rank(), nc = (int)cl.num_blocks();
  Control* ctl = w.ctl;
  if (threadIdx.x < 2) s_n[threadIdx.x] = 0;
  cl.sync();
  int L = __ldcg(&ctl->n_levels);  // the first level the grid kernel left
  int total = __ldcg(&ctl->err) ? 0 : __ldcg(&ctl->rq[L % 3]);
  const int* g_first = (L & 1) ? w.q1 : w.q0;
  int* const ovf[2] = {w.roots, w.hcomp};
  int n_local = 0, n_ovf = 0;  // input level: items in the CTAs' slots, then in the global spill list
  for (int t = 0; total > 0; ++t) {
    const int in = t & 1, outs = in ^ 1;
    if (threadIdx.x == 0) s_n[outs] = 0;  // read by the other CTAs two levels ago
    if (rank == 0 && threadIdx.x == 0) ctl->tovf[outs] = 0;  // read two levels ago, written from the next level on
    __syncthreads();
    auto push = [&](int u) {
      const int i = atomicAdd(&s_n[outs], 1);
      if (i < tq) s_item[outs][i] = u;
      else ovf[outs][atomicAdd(&ctl->tovf[outs], 1)] = u;
    };
#if MPLD_TAIL_LOCAL
    // every CTA colours the vertices its own threads made ready (no remote
    // reads), plus a strided share of the first level and of the spill list
    if (t == 0) {
      for (int i = rank * (int)blockDim.x + threadIdx.x; i < total; i += nc * (int)blockDim.x)
        recover_vertex(g, w, k, colors, __ldcg(&g_first[i]), push);
    } else {
      const int mine = min(s_n[in], tq);
      for (int i = threadIdx.x; i < mine; i += blockDim.x) recover_vertex(g, w, k, colors, s_item[in][i], push);
      for (int i = rank * (int)blockDim.x + threadIdx.x; i < n_ovf; i += nc * (int)blockDim.x)
        recover_vertex(g, w, k, colors, __ldcg(&ovf[in][i]), push);
    }
#else
    for (int i = rank * (int)blockDim.x + threadIdx.x; i < total; i += nc * (int)blockDim.x) {
      int v;
      if (t == 0) {
        v = __ldcg(&g_first[i]);
      } else if (i < n_local) {
        int lo = 0, hi = nc - 1;  // the CTA holding item i: s_pref[lo] <= i < s_pref[lo + 1]
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (s_pref[mid] <= i) lo = mid; else hi = mid - 1;
        }
        v = *cl.map_shared_rank(&s_item[in][i - s_pref[lo]], lo);
      } else {
        v = __ldcg(&ovf[in][i - n_local]);
      }
      recover_vertex(g, w, k, colors, v, push);
    }
#endif
    cl.sync();  // the level is coloured; every CTA's output slot is complete
    if (threadIdx.x < 32) {  // one remote count per lane, a warp scan
      const int lane = threadIdx.x;
      const int x = lane < nc ? min(*cl.map_shared_rank(&s_n[outs], lane), tq) : 0;
      int y = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int z = __shfl_up_sync(0xffffffffu, y, o);
        if (lane >= o) y += z;
      }
      if (lane < nc) s_pref[lane] = y - x;
      if (lane == nc - 1) s_pref[nc] = y;
    }
    __syncthreads();
    n_local = s_pref[nc];
    n_ovf = __ldcg(&ctl->tovf[outs]);
    total = n_local + n_ovf;
    ++L;
  }
  if (rank == 0 && threadIdx.x == 0) ctl->n_levels = L;
  cl.sync();  // no CTA leaves while others may still read its shared memory
  if (out.enabled) finalize_outputs(g, w, out, &ctl->done_recover);
}

// ---------------------------------------------------------------------------
// Eq. (1b)/(1c) per layout; the last CTA writes cost (Eq. 1a) and the stats.
__global__ void __launch_bounds__(256) mpld_evaluate(GraphView g, Workspace w, const int* colors, double alpha,
                                                     long long* counts, double* cost, long long* stats,
                                                     int launches) {
  constexpr int P = MPLD_EVAL_P;
  const int nth = gridDim.x * blockDim.x;
  stamp(w.ctl, 15);
  const int vend = __ldcg(&w.ctl->err) ? 0 : g.n;
  LayoutCache lc;
  for (int t0 = blockIdx.x * blockDim.x * P; t0 < vend; t0 += nth * P) {
    int v[P], e[P], e1[P], cv[P], nc[P], ns[P];
#pragma unroll
    for (int j = 0; j < P; ++j) {
      v[j] = t0 + j * blockDim.x + threadIdx.x;
      const bool ok = v[j] < vend;
      e[j] = ok ? __ldg(&g.ce_rp[v[j]]) : 0;
      e1[j] = ok ? __ldg(&g.ce_rp[v[j] + 1]) : 0;
      cv[j] = ok ? __ldcg(&colors[v[j]]) : 0;
      nc[j] = ns[j] = 0;
    }
    while (true) {
      bool open = false;
#pragma unroll
      for (int j = 0; j < P; ++j) open |= e[j] < e1[j];
      if (!open) break;
      int u[P][kNb];
#pragma unroll
      for (int j = 0; j < P; ++j)
#pragma unroll
        for (int t = 0; t < kNb; ++t) u[j][t] = e[j] + t < e1[j] ? __ldg(&g.ce_col[e[j] + t]) : -1;
#pragma unroll
      for (int j = 0; j < P; ++j) {
#pragma unroll
        for (int t = 0; t < kNb; ++t)  // each conflict edge counted once, from its smaller end
          if (u[j][t] > v[j] && __ldcg(&colors[u[j][t]]) == cv[j]) ++nc[j];
        e[j] += kNb;
      }
    }
#pragma unroll
    for (int j = 0; j < P; ++j) {
      if (v[j] >= vend) continue;
      for (int x = __ldg(&g.se_rp[v[j]]), x1 = __ldg(&g.se_rp[v[j] + 1]); x < x1; ++x) {
        const int u = __ldg(&g.se_col[x]);
        if (u > v[j] && __ldcg(&colors[u]) != cv[j]) ++ns[j];
      }
      if (nc[j] | ns[j]) {
        const int l = lc.get(g, v[j]);
        if (nc[j]) atomicAdd((unsigned long long*)&counts[2 * l], (unsigned long long)nc[j]);
        if (ns[j]) atomicAdd((unsigned long long*)&counts[2 * l + 1], (unsigned long long)ns[j]);
      }
    }
  }
  Outputs out;
  out.counts = counts;
  out.cost = cost;
  out.stats = stats;
  out.alpha = alpha;
  out.launches = launches;
  out.enabled = 1;
  finalize_outputs(g, w, out, &w.ctl->done_blocks);
}

// ---------------------------------------------------------------------------
// Sharded runs: the colours one shard's search wrote, as a
// compact list of (vertex, colour) pairs (every vertex a search coloured; -1
// everywhere else), and the scatter of the lists of all shards.  Appends are
// warp-aggregated: one atomic per warp and chunk.
__global__ void __launch_bounds__(256) mpld_shard_export(int n, const int* __restrict__ colors, int* pairs,
                                                         unsigned long long* count) {
  const int lane = threadIdx.x & 31;
  const int stride = gridDim.x * blockDim.x;
  for (int v0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31); v0 < n; v0 += stride) {
    const int v = v0 + lane;
    const int c = v < n ? __ldg(&colors[v]) : -1;
    const unsigned m = __ballot_sync(0xffffffffu, c >= 0);
    if (!m) continue;
    unsigned long long base = 0ull;
    if (lane == 0) base = atomicAdd(count, (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (c >= 0) {
      const unsigned long long at = base + __popc(m & ((1u << lane) - 1u));
      pairs[2 * at] = v;
      pairs[2 * at + 1] = c;
    }
  }
}

__global__ void __launch_bounds__(256) mpld_shard_import(long long m, const int* __restrict__ pairs, int n,
                                                         int* colors) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
    const int v = __ldg(&pairs[2 * i]);
    if (v >= 0 && v < n) colors[v] = __ldg(&pairs[2 * i + 1]);  // v < 0: padding of a shorter list
  }
}

// ---------------------------------------------------------------------------
// The graph build of the compact uploads in ONE cooperative launch (two
// 1024-thread CTAs per SM, five grid barriers).  CTA c owns the vertex range
// [c n / G, (c+1) n / G); each of its warps a contiguous sub-range, walked in
// chunks of 32 consecutive vertices (coalesced, warp scans).  One counter word
// per vertex holds both degree counts (CE in the low 24 bits, SE above).
//   P1 zero the counters; warp / CTA sums of deg_up
//   P2 scan of deg_up -> rp_up; the chunk's upper entries 32 at a time
//      (coalesced; row by a search over the lanes' offsets): an entry (v, u)
//      is valid iff v < u < n and it is larger than its row predecessor; every
//      valid one counts the lower entry of row u and one entry of row v
//      (aggregated per row); stitch pairs (grid-stride): count both ends
//   P3 warp / CTA sums of both degree counts
//   P4 scans -> ce_rp, se_rp
//   P5 scatter (entry-parallel as P2): lower CE entries and SE entries by
//      atomics on the fill word, the upper CE entries in order after the lower
//      ones
//   P6 sort the lower part of every CE row with >= 2 of them, every SE row
//      with >= 2 entries (insertion sort: rows are short)
// Rows of up to 8 entries are sorted in registers (all loads issued at once),
// longer ones in place.
__device__ __forceinline__ void build_row_sort(int* col, int a, int b) {
  constexpr int kR = 8;
  if (b - a > kR) {
    for (int i = a + 1; i < b; ++i) {
      const int x = col[i];
      int j = i - 1;
      while (j >= a && col[j] > x) {
        col[j + 1] = col[j];
        --j;
      }
      col[j + 1] = x;
    }
    return;
  }
  int r[kR];
#pragma unroll
  for (int i = 0; i < kR; ++i) r[i] = a + i < b ? col[a + i] : INT_MAX;
#pragma unroll
  for (int i = 1; i < kR; ++i)  // insertion network on registers
#pragma unroll
    for (int j = i; j > 0; --j) {
      const int lo = min(r[j - 1], r[j]), hi = max(r[j - 1], r[j]);
      r[j - 1] = lo;
      r[j] = hi;
    }
#pragma unroll
  for (int i = 0; i < kR; ++i)
    if (a + i < b) col[a + i] = r[i];
}

__device__ __forceinline__ int warp_scan_excl(int x, int& total) {
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

// Row of entry i of a warp's chunk: the first lane whose inclusive entry
// offset exceeds i (lanes without entries are skipped); 32 when i >= total.
__device__ __forceinline__ int warp_row_of(int incl, int i) {
  int o = 0;
#pragma unroll
  for (int st = 16; st > 0; st >>= 1)
    if (__shfl_sync(0xffffffffu, incl, o + st - 1) <= i) o += st;
  return min(o, 31);
}

constexpr int kCeMask = (1 << 24) - 1;  // CE count in a build counter word; SE count << 24

__global__ void __launch_bounds__(1024, 1) mpld_graph_build(GraphBuild b) {
  __shared__ int s_w[32];
  __shared__ int s_base[3];
  GridBarrier grid(b.bar, gridDim.x, b.epoch0);
  const int G = gridDim.x, c = blockIdx.x, n = b.n;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int v0 = (int)((long long)n * c / G), v1 = (int)((long long)n * (c + 1) / G);
  const int wper = (((v1 - v0) + nw - 1) / nw + 31) & ~31;  // vertices per warp, whole chunks
  const int w0 = min(v0 + wid * wper, v1), w1 = min(w0 + wper, v1);
  const bool ce = b.deg_up != nullptr, se = b.m_se >= 0;
  int* cnt = b.cnt_ce;   // CE | SE << 24
  int* fill = b.fill_ce;
  // P1
  int s_up = 0;
  for (int v = w0 + lane; v < w1; v += 32) {
    cnt[v] = 0;
    fill[v] = 0;
    if (ce) s_up += b.deg_up[v];
  }
  s_up = __reduce_add_sync(0xffffffffu, s_up);
  if (lane == 0) s_w[wid] = s_up;
  __syncthreads();
  int wbase_up = 0;  // this warp's offset inside the CTA
  if (threadIdx.x < 32) {
    int t;
    const int e = warp_scan_excl(lane < nw ? s_w[lane] : 0, t);
    if (lane < nw) s_w[lane] = e;
    if (lane == 0) b.tot[c] = t;
  }
  __syncthreads();
  wbase_up = s_w[wid];
  __syncthreads();
  grid.sync();
  // P2
  if (ce) {
    if (threadIdx.x < 32) {
      int base = 0;
      for (int i = lane; i < c; i += 32) base += __ldcg(&b.tot[i]);
      base = __reduce_add_sync(0xffffffffu, base);
      if (lane == 0) s_base[0] = base;
    }
    __syncthreads();
    int carry = s_base[0] + wbase_up;
    bool bad = false;
    for (int vv = w0; vv < w1; vv += 32) {
      const int v = vv + lane;
      const int d = v < w1 ? (int)b.deg_up[v] : 0;
      int t;
      const int ex = warp_scan_excl(d, t);
      const int a = carry + ex;
      const int base = carry;
      carry += t;
      if (v < w1) {
        b.rp_up[v] = a;
        bad |= a + d > b.m_up;
        if (v == n - 1) {  // the last vertex closes the upper row pointer
          b.rp_up[n] = a + d;
          if (a + d != b.m_up) bad = true;
        }
      }
      // the chunk's entries 32 at a time (coalesced), each with its row found
      // by a search over the lanes' inclusive offsets
      const int incl = ex + d;
      const int tl = min(t, max(b.m_up - base, 0));
      for (int i0 = 0; i0 < tl; i0 += 32) {
        const int i = i0 + lane;
        const int o = warp_row_of(incl, i);
        const int ov = vv + o, oex = __shfl_sync(0xffffffffu, ex, o);
        const int u = i < tl ? __ldg(&b.col_up[base + i]) : 0;
        int pu = __shfl_up_sync(0xffffffffu, u, 1);
        if (lane == 0 && i < tl && i > oex) pu = __ldg(&b.col_up[base + i - 1]);
        const bool ok = i < tl && u > ov && u < n && (i == oex || u > pu);
        bad |= i < tl && !ok;
        if (ok) atomicAdd(&cnt[u], 1);  // the lower entry ov of row u
        const unsigned grp = __match_any_sync(0xffffffffu, i < tl ? ov : -1 - lane);
        const int k = __popc(__ballot_sync(0xffffffffu, ok) & grp);
        if (k && lane == __ffs(grp) - 1) atomicAdd(&cnt[ov], k);
      }
    }
    if (bad) atomicOr(b.err, 1);
  }
  if (se)
    for (int i = c * blockDim.x + threadIdx.x; i < b.m_se; i += G * blockDim.x) {
      atomicAdd(&cnt[__ldg(&b.se_pairs[2 * i])], 1 << 24);
      atomicAdd(&cnt[__ldg(&b.se_pairs[2 * i + 1])], 1 << 24);
    }
  grid.sync();
  // P3
  int sc = 0, ss = 0;
  for (int v = w0 + lane; v < w1; v += 32) {
    const int x = __ldcg(&cnt[v]);
    sc += x & kCeMask;
    ss += x >> 24;
  }
  sc = __reduce_add_sync(0xffffffffu, sc);
  ss = __reduce_add_sync(0xffffffffu, ss);
  __shared__ int s_w2[32];
  if (lane == 0) {
    s_w[wid] = sc;
    s_w2[wid] = ss;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    int t;
    int e = warp_scan_excl(lane < nw ? s_w[lane] : 0, t);
    if (lane < nw) s_w[lane] = e;
    if (lane == 0) b.tot[G + c] = t;
    e = warp_scan_excl(lane < nw ? s_w2[lane] : 0, t);
    if (lane < nw) s_w2[lane] = e;
    if (lane == 0) b.tot[2 * G + c] = t;
  }
  __syncthreads();
  const int wbase_ce = s_w[wid], wbase_se = s_w2[wid];
  grid.sync();
  // P4
  if (threadIdx.x < 64) {  // warp q: the earlier CTAs' sums of count q
    const int q = threadIdx.x >> 5;
    int base = 0;
    for (int i = lane; i < c; i += 32) base += __ldcg(&b.tot[(1 + q) * G + i]);
    base = __reduce_add_sync(0xffffffffu, base);
    if (lane == 0) s_base[1 + q] = base;
    // the last CTA checks the totals: a count that overflowed its field (a CE
    // degree >= 2^24, an SE degree >= 128) cannot leave both sums intact
    if (c == G - 1 && lane == 0) {
      const int all = base + __ldcg(&b.tot[(1 + q) * G + c]);
      if (q == 0 && ce && all != 2 * b.m_up) atomicOr(b.err, 1);
      if (q == 1 && se && all != 2 * b.m_se) atomicOr(b.err, 1);
    }
  }
  __syncthreads();
  {
    int cc = s_base[1] + wbase_ce, cs = s_base[2] + wbase_se;
    for (int vv = w0; vv < w1; vv += 32) {
      const int v = vv + lane;
      const int x = v < w1 ? __ldcg(&cnt[v]) : 0;
      int tc, ts;
      const int ac = cc + warp_scan_excl(x & kCeMask, tc);
      const int as = cs + warp_scan_excl(x >> 24, ts);
      cc += tc;
      cs += ts;
      if (v < w1) {
        if (ce) b.ce_rp[v] = ac;
        if (se) b.se_rp[v] = as;
        if (v == n - 1) {
          if (ce) b.ce_rp[n] = ac + (x & kCeMask);
          if (se) b.se_rp[n] = as + (x >> 24);
        }
      }
    }
  }
  grid.sync();
  // P5 (invalid input: an empty CSR instead, so that nothing reads past it;
  // the error is reported through the simplification)
  const bool failed = __ldcg(b.err) != 0;
  if (failed) {
    for (int v = w0 + lane; v < w1; v += 32) {
      if (ce) b.ce_rp[v] = 0;
      if (se) b.se_rp[v] = 0;
    }
    if (c == G - 1 && threadIdx.x == 0) {
      if (ce) b.ce_rp[n] = 0;
      if (se) b.se_rp[n] = 0;
    }
  }
  if (ce && !failed)  // every entry is valid here (else the build failed): upper part at the end of row v
    for (int vv = w0; vv < w1; vv += 32) {
      const int v = vv + lane;
      const int d = v < w1 ? (int)b.deg_up[v] : 0;
      const int a = v < w1 ? __ldcg(&b.rp_up[v]) : 0;
      const int up0 = v < w1 ? __ldcg(&b.ce_rp[v + 1]) - d : 0;
      int t;
      const int ex = warp_scan_excl(d, t);
      const int incl = ex + d;
      const int base = __shfl_sync(0xffffffffu, a - ex, 0);  // lane 0 always holds a vertex
      for (int i0 = 0; i0 < t; i0 += 32) {
        const int i = i0 + lane;
        const int o = warp_row_of(incl, i);
        const int ov = vv + o;
        const int orow = __shfl_sync(0xffffffffu, up0, o), oex = __shfl_sync(0xffffffffu, ex, o);
        if (i < t) {
          const int u = __ldg(&b.col_up[base + i]);
          b.ce_col[orow + (i - oex)] = u;
          b.ce_col[__ldcg(&b.ce_rp[u]) + (atomicAdd(&fill[u], 1) & kCeMask)] = ov;
        }
      }
    }
  if (se && !failed)
    for (int i = c * blockDim.x + threadIdx.x; i < b.m_se; i += G * blockDim.x) {
      const int u = __ldg(&b.se_pairs[2 * i]), v = __ldg(&b.se_pairs[2 * i + 1]);
      b.se_col[__ldcg(&b.se_rp[u]) + (atomicAdd(&fill[u], 1 << 24) >> 24)] = v;
      b.se_col[__ldcg(&b.se_rp[v]) + (atomicAdd(&fill[v], 1 << 24) >> 24)] = u;
    }
  grid.sync();  // every CTA passes all kBuildBarriers barriers
  // P6
  if (failed) return;
  for (int v = w0 + lane; v < w1; v += 32) {
    const int f = __ldcg(&fill[v]);
    if (ce && (f & kCeMask) >= 2) {
      const int a = __ldcg(&b.ce_rp[v]);
      build_row_sort(b.ce_col, a, a + (f & kCeMask));
    }
    if (se && (f >> 24) >= 2) build_row_sort(b.se_col, __ldcg(&b.se_rp[v]), __ldcg(&b.se_rp[v + 1]));
  }
}

}  // namespace

cudaError_t launch_graph_build(const GraphBuild& b, cudaStream_t s, int blocks) {
  if (b.n <= 0) {
    cudaError_t e = cudaSuccess;
    if (b.deg_up) e = cudaMemsetAsync(b.ce_rp, 0, sizeof(int), s);
    if (e == cudaSuccess && b.m_se >= 0) e = cudaMemsetAsync(b.se_rp, 0, sizeof(int), s);
    return e;
  }
  return launch_ex(mpld_graph_build, dim3(blocks), dim3(1024), 0, s, false, true, b);
}

int coop_blocks_build(int num_sms) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mpld_graph_build, 1024, 0);
  return std::min(per_sm, 2) * num_sms;
}

bool pdl_enabled() { return g_pdl; }

void set_pdl(bool enable) { g_pdl = enable; }

bool g_tail_ok = false;

// one thread-block cluster of kTC CTAs (the cluster tails), after the previous kernel (PDL)
template <typename... KArgs, typename... Args>
cudaError_t launch_cluster(void (*kern)(KArgs...), cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kTC);
  cfg.blockDim = dim3(1024);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kTC;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  unsigned na = 1;
  if (pdl_enabled()) {
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    na = 2;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

cudaError_t launch_simplify_components(const GraphView& g, Workspace ws, int k, int* colors, long long* counts,
                                       int validate, cudaStream_t s, int blocks, int threads, int separate_prep) {
  const int cluster = g_tail_ok && MPLD_CLUSTER_ROUNDS ? 1 : 0;
  cudaError_t e = launch_ex(mpld_simplify_components, dim3(blocks), dim3(threads), 0, s, false, true, g, ws, k, colors,
                            counts, validate, cluster, separate_prep);
  if (e != cudaSuccess || !cluster) return e;
  e = launch_cluster(mpld_simplify_tail, s, g, ws, k);
  if (e != cudaSuccess) return e;
  return launch_ex(mpld_final_pass, dim3(blocks), dim3(threads), 0, s, true, false, g, ws, separate_prep);
}
int simplify_launches() { return g_tail_ok && MPLD_CLUSTER_ROUNDS ? 3 : 1; }

cudaError_t launch_recover_prep(const GraphView& g, Workspace ws, cudaStream_t s, int blocks, int threads) {
  return launch_ex(mpld_recover_prep, dim3(blocks), dim3(threads), 0, s, false, false, g, ws);
}
cudaError_t configure_recover_tail() {
  g_tail_ok = false;
  if (!MPLD_CLUSTER_TAIL) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(mpld_recover_tail, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(mpld_simplify_tail, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return cudaSuccess;  // no cluster tail: the grid kernel finishes every level
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kTC);
  cfg.blockDim = dim3(1024);
  cudaLaunchAttribute at;
  at.id = cudaLaunchAttributeClusterDimension;
  at.val.clusterDim.x = kTC;
  at.val.clusterDim.y = 1;
  at.val.clusterDim.z = 1;
  cfg.attrs = &at;
  cfg.numAttrs = 1;
  int nclusters = 0;
  e = cudaOccupancyMaxActiveClusters(&nclusters, mpld_recover_tail, &cfg);
  if (e != cudaSuccess) cudaGetLastError();
  g_tail_ok = e == cudaSuccess && nclusters >= 1;
  return cudaSuccess;
}
bool recover_tail_available() { return g_tail_ok; }

cudaError_t launch_recover(const GraphView& g, Workspace ws, int k, int* colors, Outputs out, cudaStream_t s,
                           int blocks, int threads, bool pdl) {
  out.cluster_tail = g_tail_ok ? 1 : 0;
  cudaError_t e = launch_ex(mpld_recover, dim3(blocks), dim3(threads), 0, s, pdl, true, g, ws, k, colors, out);
  if (e != cudaSuccess || !out.cluster_tail) return e;
  return launch_cluster(mpld_recover_tail, s, g, ws, k, colors, out);
}

cudaError_t launch_evaluate(const GraphView& g, Workspace ws, const int* colors, double alpha, long long* counts,
                            double* cost, long long* stats, int launches, cudaStream_t s, int blocks) {
  mpld_evaluate<<<blocks, 256, 0, s>>>(g, ws, colors, alpha, counts, cost, stats, launches);
  return cudaGetLastError();
}

cudaError_t launch_shard_export(int n, const int* colors, int* pairs, unsigned long long* count, cudaStream_t s,
                                int blocks) {
  cudaError_t e = cudaMemsetAsync(count, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess || n <= 0) return e;
  mpld_shard_export<<<std::min(blocks, (n + 255) / 256), 256, 0, s>>>(n, colors, pairs, count);
  return cudaGetLastError();
}

cudaError_t launch_shard_import(long long m, const int* pairs, int n, int* colors, cudaStream_t s, int blocks) {
  if (m <= 0) return cudaSuccess;
  mpld_shard_import<<<(int)std::min<long long>(blocks, (m + 255) / 256), 256, 0, s>>>(m, pairs, n, colors);
  return cudaGetLastError();
}

int coop_blocks_simplify(int threads, int num_sms) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mpld_simplify_components, threads, 0);
  return per_sm * num_sms;
}

int coop_blocks_recover(int threads, int num_sms) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mpld_recover, threads, 0);
  return per_sm * num_sms;
}

int resident_blocks_evaluate(int num_sms) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mpld_evaluate, 256, 0);
  return per_sm * num_sms;
}

}  // namespace mpld
