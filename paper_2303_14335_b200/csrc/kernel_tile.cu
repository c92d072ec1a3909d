// The fused tile pipeline: the whole flow of PAPER.md §2.2 / Fig. 2 —
// simplification, sub-graphs (Alg. 1 lines 1-3), the exact-cover search
// (Alg. 1 lines 4-19) and the recovery — for the PIECES of the decomposed
// graph (connected components of CE ∪ SE), a window of whole pieces per CTA,
// held in shared memory.
//
// Every step of the flow is local to a piece: a vertex's simplification round
// (R8) depends only on its piece, the sub-graphs of Alg. 1 line 1 lie inside
// pieces, and the recovery order (R9) only relates adjacent vertices.  Layout
// graphs are unions of many small pieces (conflict clusters with the wires
// hanging off them: configs[1] has 5,721 pieces of at most 168 vertices), so
// the level-synchronous whole-graph kernels — one grid barrier per
// simplification round and per recovery level, ~40 global round trips per
// call — are replaced by:
//
//   mpld_piece_order     one cooperative kernel (4 grid barriers): the pieces
//                        by union-find over CE ∪ SE (random-priority roots), then
//                        positions with every piece contiguous (t_perm /
//                        t_pos; the order inside a piece is irrelevant: every
//                        tie-break below compares original ids)
//   mpld_tile_decompose  tile t owns the pieces starting at positions
//                        [t·kTOwn, (t+1)·kTOwn); its CTA gathers them (a window
//                        of <= kTMaxV vertices, rows as 16-bit window indices)
//                        and runs, in shared memory with block barriers:
//     simplification rounds   frontier queues (R8)
//     kept sub-graphs         union-find with minimum-id roots, BFS from the
//                             minimum in ascending id (R5 column order) ->
//                             bit-packed matrices in the component pool
//     relaxed Algorithm X     one component per lane of warp 0 (lane_search.cuh),
//                             the oracle's node order and budget, while the
//                             other warps count the recovery predecessors
//     recovery                level-synchronous over the pop-order DAG (R9)
//   Windows with more than 32 components defer them to the light kernel; the
//   components the light search hands on (heavy in exact mode, > 32 vertices
//   in budgeted mode) are searched by the warp-parallel / 64-bit lane kernels;
//   such windows are recovered by the finish launch of mpld_tile_decompose
//   (gathered and peeled again: deterministic), whose last CTA writes the
//   Eq. (1a) costs and the statistics.
//
// Anything the tiles cannot take — a piece larger than a window, input that
// fails validation (or a row pointer / id out of range), a component of more
// than 64 vertices — sets the gate: the whole-graph kernels (kernels_graph.cu,
// kernel_search.cu), enqueued after the finish launch and idle otherwise, then
// recompute every output from scratch and report MPLD_ERR_GRAPH /
// MPLD_ERR_COMPONENT exactly as alone.  Both pipelines compute identical
// results.
#include <cooperative_groups.h>

#include <algorithm>

#include "lane_search.cuh"
#include "mpld_internal.cuh"

namespace mpld {

namespace {

constexpr int kTT = 512;        // threads per tile CTA (two CTAs per SM)
constexpr int kTOwn = 1024;     // positions owned by a tile (pieces starting there)
constexpr int kTMaxV = 2048;    // vertices of a window
constexpr int kTMaxCE = 12288;  // CE entries of a window
constexpr int kTMaxSE = 2048;   // SE entries of a window
constexpr int kTBig = 1 << 29;  // live degree of a stitch vertex (never hidden, R8)
constexpr int kTWarps = kTT / 32;
constexpr int kPieceThreads = 1024;

struct __align__(16) TileSmem {
  LaneLight L;                    // the light search of warp 0
  int uf[kTMaxV + 1];             // CE row starts (scan); union-find parents; component offsets
  int cnt[kTMaxV + 1];            // SE row starts (scan); live degree; component sizes; recovery predecessors
  int orig[kTMaxV];               // window index -> vertex id
  unsigned prio[kTMaxV];          // lowbias32(layout-local id) (R9)
  unsigned short rc[kTMaxV + 2];  // CE row offsets in colC
  unsigned short rs[kTMaxV + 2];  // SE row offsets in colS
  unsigned short colC[kTMaxCE];   // CE rows as window indices
  unsigned short colS[kTMaxSE];   // SE rows
  short hr[kTMaxV];               // simplification round, -1 kept; <= -3: BFS position (-3 - p)
  short q[2][kTMaxV];             // frontier queues; component roots / ordinals / BFS orders
  signed char col8[kTMaxV];       // colours (recovery)
  int nq[3];
  int m, bad, ncomp, pending, tile, maxn;
  unsigned cb, ob;
  int wsum[2][kTWarps];
};

// ---------------------------------------------------------------------------
// The piece order.  Union-find on parent offsets (t_par[v] = parent - v, 0 for
// a root), so a zeroed array is the initial forest; the root of larger
// priority lowbias32(id) is hooked under the other (any root will do: it only
// names the piece).
__device__ __forceinline__ int pfind(int* par, int x) {
  while (true) {
    const int d = __ldcg(&par[x]);
    if (d == 0) return x;
    const int y = x + d;
    const int d2 = __ldcg(&par[y]);
    if (d2 != 0) par[x] = y + d2 - x;  // path halving (parents only move to smaller ancestors)
    x = y;
  }
}

// find without path halving: the compress phase stores every vertex's root,
// and a halving store racing with it could put back a non-root ancestor
__device__ __forceinline__ int pfind_ro(const int* par, int x) {
  while (true) {
    const int d = __ldcg(&par[x]);
    if (d == 0) return x;
    x += d;
  }
}

__device__ __forceinline__ void punion(int* par, int a, int b) {
  while (true) {
    a = pfind(par, a);
    b = pfind(par, b);
    if (a == b) return;
    if (lowbias32((uint32_t)a) < lowbias32((uint32_t)b)) {  // random priorities: trees of expected
      const int t = a;                                      // logarithmic depth (minimum-id roots
      a = b;                                                // chain up along wires)
      b = t;
    }
    if (atomicCAS(&par[a], 0, b - a) == 0) return;
  }
}

// gate reasons (mpld_context_debug out[88])
enum GateBits : int {
  kGateRows = 1,        // a row pointer or id out of range (piece order)
  kGateWindow = 2,      // a piece larger than a window
  kGateOpen = 4,        // a neighbour outside its piece's window (asymmetric input)
  kGateInvalid = 8,     // validation: a row not strictly ascending, a self loop, CE ∩ SE
  kGateSymmetry = 16,   // validation: symmetry hashes differ
  kGateComponent = 32,  // a component of more than 64 vertices
  kGateBuild = 64,      // the device CSR build saw invalid input
  kGateLayouts = 128,   // validation: layout offsets / first row pointers
};
__device__ __forceinline__ void set_gate(Control* ctl, int why) { atomicOr(&ctl->gate, why); }

__global__ void __launch_bounds__(kPieceThreads, 2) mpld_piece_order(GraphView g, Workspace w) {
  Control* ctl = w.ctl;
  GridBarrier grid(&ctl->bar_piece);
  const int n = g.n;
  const int nth = gridDim.x * blockDim.x;
  const int t0 = blockIdx.x * blockDim.x + threadIdx.x;
  const int nnz_ce = __ldg(&g.ce_rp[n]), nnz_se = __ldg(&g.se_rp[n]);
  for (int v = t0; v < n; v += nth) {
    w.t_par[v] = 0;
    w.t_cnt[v] = 0;
  }
  grid.sync();
  // the pieces: union over every CE / SE entry (v, u > v); rows out of range gate the call
  bool bad = false;
  for (int v = t0; v < n; v += nth) {
    const int a = __ldg(&g.ce_rp[v]), b = __ldg(&g.ce_rp[v + 1]);
    const int c = __ldg(&g.se_rp[v]), d = __ldg(&g.se_rp[v + 1]);
    if (a < 0 || a > b || b > nnz_ce || c < 0 || c > d || d > nnz_se) {
      bad = true;
      continue;
    }
    for (int e = a; e < b; ++e) {
      const int u = __ldg(&g.ce_col[e]);
      if ((unsigned)u >= (unsigned)n) bad = true;
      else if (u > v) punion(w.t_par, v, u);
    }
    for (int e = c; e < d; ++e) {
      const int u = __ldg(&g.se_col[e]);
      if ((unsigned)u >= (unsigned)n) bad = true;
      else if (u > v) punion(w.t_par, v, u);
    }
  }
  if (bad) set_gate(ctl, kGateRows);
  grid.sync();
  for (int v = t0; v < n; v += nth) {  // compress, piece sizes at the roots
    const int r = pfind_ro(w.t_par, v);
    w.t_par[v] = r - v;
    atomicAdd(&w.t_cnt[r], 1);
  }
  grid.sync();
  // piece ranges: one atomic per CTA and chunk (the order of the pieces is free)
  __shared__ int s_w[32];
  __shared__ int s_base;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int c0 = blockIdx.x * blockDim.x; c0 < n; c0 += nth) {
    const int v = c0 + threadIdx.x;
    const int sz = (v < n && __ldcg(&w.t_par[v]) == 0) ? __ldcg(&w.t_cnt[v]) : 0;
    int y = sz;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int z = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= o) y += z;
    }
    if (lane == 31) s_w[wid] = y;
    __syncthreads();
    if (threadIdx.x < 32) {
      const int x = threadIdx.x < (int)(blockDim.x >> 5) ? s_w[threadIdx.x] : 0;
      int z = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int q = __shfl_up_sync(0xffffffffu, z, o);
        if (lane >= o) z += q;
      }
      s_w[threadIdx.x] = z - x;
      if (threadIdx.x == 31) s_base = z ? atomicAdd(&ctl->piece_cursor, z) : 0;
    }
    __syncthreads();
    if (sz) w.t_end[v] = s_base + s_w[wid] + y;  // exclusive prefix + size
    __syncthreads();
  }
  grid.sync();
  for (int v = t0; v < n; v += nth) {  // positions: pieces contiguous
    const int r = v + __ldcg(&w.t_par[v]);
    const int e = __ldcg(&w.t_end[r]);
    const int p = e - atomicSub(&w.t_cnt[r], 1);
    w.t_pos[v] = p;
    w.t_perm[p] = v;
    w.t_pend[p] = e;
  }
}

// ---------------------------------------------------------------------------
__device__ __forceinline__ int uf_find(int* p, int x) {
  while (true) {
    const int y = p[x];
    if (y == x) return x;
    const int z = p[y];
    if (z != y) p[x] = z;  // path halving
    x = y;
  }
}

// hook the root with the larger vertex id under the other: roots are minima (ids)
__device__ __forceinline__ void uf_union_id(int* p, const int* id, int a, int b) {
  while (true) {
    a = uf_find(p, a);
    b = uf_find(p, b);
    if (a == b) return;
    if (id[a] < id[b]) {
      const int t = a;
      a = b;
      b = t;
    }
    const int old = atomicCAS(&p[a], a, b);
    if (old == a) return;
    a = old;
  }
}

__device__ __forceinline__ unsigned long long tkey(const TileSmem& S, int i) {  // pop key (R9): kept above all
  const int h = S.hr[i];
  return h < 0 ? ~0ull : (((unsigned long long)(h + 1) << 32) | S.prio[i]);
}

// symmetry check of the validation: multiset hash of the (row, column) pairs
__device__ __forceinline__ unsigned long long edge_hash(int x, int y) {
  unsigned long long z = ((unsigned long long)(unsigned)x << 32) | (unsigned)y;
  z ^= z >> 30;
  z *= 0xbf58476d1ce4e5b9ull;
  z ^= z >> 27;
  z *= 0x94d049bb133111ebull;
  z ^= z >> 31;
  return z;
}

// exclusive scans of a[0..cnt) and b[0..cnt) (cnt <= kTMaxV; in place allowed)
// into oa / ob, totals at oa[cnt] / ob[cnt]; S.maxn = max of a
__device__ void block_scan2(TileSmem& S, const int* a, int* oa, const int* b, int* ob, int cnt) {
  constexpr int kPer = kTMaxV / kTT;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  int x[kPer], y[kPer], sx = 0, sy = 0, mx = 0;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int c = tid * kPer + j;
    x[j] = c < cnt ? a[c] : 0;
    y[j] = (b && c < cnt) ? b[c] : 0;
    sx += x[j];
    sy += y[j];
    mx = max(mx, x[j]);
  }
  int ix = sx, iy = sy;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int zx = __shfl_up_sync(0xffffffffu, ix, o), zy = __shfl_up_sync(0xffffffffu, iy, o);
    if (lane >= o) {
      ix += zx;
      iy += zy;
    }
  }
  mx = __reduce_max_sync(0xffffffffu, mx);
  if (lane == 31) {
    S.wsum[0][wid] = ix;
    S.wsum[1][wid] = iy;
  }
  if (lane == 0) atomicMax(&S.maxn, mx);
  __syncthreads();
  int bx = 0, by = 0, tx = 0, ty = 0;
  for (int i = 0; i < kTWarps; ++i) {
    const int vx = S.wsum[0][i], vy = S.wsum[1][i];
    bx += i < wid ? vx : 0;
    by += i < wid ? vy : 0;
    tx += vx;
    ty += vy;
  }
  int rx = bx + ix - sx, ry = by + iy - sy;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int c = tid * kPer + j;
    if (c < cnt) {
      oa[c] = rx;
      if (b) ob[c] = ry;
    }
    rx += x[j];
    ry += y[j];
  }
  if (tid == 0) {
    oa[cnt] = tx;
    if (b) ob[cnt] = ty;
  }
  __syncthreads();
}

struct TileArgs {
  int w_stitch;
  long long max_steps;
  unsigned light_steps;
  int* colors;
  long long* counts;
  double* cost;
  long long* stats;
  double alpha;
  int launches;
  int validate;
  int finish;  // 0: decompose; 1: recover the pending windows and write the outputs
};

// Layout-local id (R10) of vertex v: binary search in the layout offsets.
__device__ __forceinline__ int local_id(const GraphView& g, int v) {
  if (g.n_layouts <= 1) return v;
  return v - __ldg(&g.layout_off[layout_of(g, v)]);
}

// first piece start at or after position x (x in [0, n])
__device__ __forceinline__ int piece_start_from(const Workspace& w, int n, int x) {
  if (x <= 0 || x >= n) return x <= 0 ? 0 : n;
  return __ldcg(&w.t_pend[x - 1]) == x ? x : __ldcg(&w.t_pend[x]);
}

// One window: the whole pieces at positions [s0, s0 + m), m as large as the
// capacity allows below `hi` (m_given in the finish launch).  Returns s0 + m,
// or -1 when the gate was set (the caller stops).
template <int K>
__device__ int tile_pass(TileSmem& S, const GraphView& g, const Workspace& w, const TileArgs& a, int s0, int hi,
                         int m_given, LightAcc& acc, unsigned long long (&hs)[4]) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int n = g.n;
  Control* ctl = w.ctl;
  const bool finish = a.finish != 0;
  // ---- 1. the window's vertices, row lengths, extent m (ends on a piece end)
  const int nmax = finish ? m_given : min(kTMaxV, hi - s0);
  if (tid == 0) {
    S.m = 0;
    S.bad = 0;
    S.ncomp = 0;
    S.maxn = 0;
    S.pending = 0;
  }
  // row starts in the CSR arrays, until the rows are gathered (prio and the
  // queues are free until step 3)
  int* gcs = reinterpret_cast<int*>(S.prio);
  int* gss = reinterpret_cast<int*>(&S.q[0][0]);
  {
    constexpr int kPer = kTMaxV / kTT;
    int vv[kPer], a0[kPer], a1[kPer], b0[kPer], b1[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int i = tid + j * kTT;
      vv[j] = i < nmax ? __ldcg(&w.t_perm[s0 + i]) : -1;
    }
#pragma unroll
    for (int j = 0; j < kPer; ++j) {  // (row pointers range-checked by the piece order)
      const int v = max(vv[j], 0);
      a0[j] = vv[j] >= 0 ? __ldg(&g.ce_rp[v]) : 0;
      a1[j] = vv[j] >= 0 ? __ldg(&g.ce_rp[v + 1]) : 0;
      b0[j] = vv[j] >= 0 ? __ldg(&g.se_rp[v]) : 0;
      b1[j] = vv[j] >= 0 ? __ldg(&g.se_rp[v + 1]) : 0;
    }
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int i = tid + j * kTT;
      if (vv[j] < 0) continue;
      S.orig[i] = vv[j];
      S.uf[i] = a1[j] - a0[j];
      S.cnt[i] = b1[j] - b0[j];
      gcs[i] = a0[j];
      gss[i] = b0[j];
      S.hr[i] = -1;
    }
  }
  __syncthreads();
  block_scan2(S, S.uf, S.uf, S.cnt, S.cnt, nmax);  // in place: row starts, totals at [nmax]
  for (int i = tid; i < nmax; i += kTT)  // the last piece end that fits the capacity
    if (__ldcg(&w.t_pend[s0 + i]) == s0 + i + 1 && S.uf[i + 1] <= kTMaxCE && S.cnt[i + 1] <= kTMaxSE)
      atomicMax(&S.m, i + 1);
  __syncthreads();
  const int m = finish ? m_given : S.m;
  if (m == 0) {  // one piece larger than a window
    if (tid == 0) set_gate(ctl, kGateWindow);
    return -1;
  }
  for (int i = tid; i <= m; i += kTT) {
    S.rc[i] = (unsigned short)S.uf[i];
    S.rs[i] = (unsigned short)S.cnt[i];
  }
  __syncthreads();
  // ---- 2. the rows, as window indices (every neighbour lies in the window:
  // pieces are closed), gathered entry by entry (consecutive entries of a row
  // on consecutive threads); validation (MPLD_FLAG_VALIDATE) on the raw ids
  for (int i = tid; i < m; i += kTT) {  // each entry's row, in the entry's slot
    for (int o = S.rc[i], o1 = S.rc[i + 1]; o < o1; ++o) S.colC[o] = (unsigned short)i;
    for (int o = S.rs[i], o1 = S.rs[i + 1]; o < o1; ++o) S.colS[o] = (unsigned short)i;
  }
  __syncthreads();
  const bool val = a.validate && !finish;
  const int nce = S.rc[m], nse = S.rs[m];
  for (int o0 = 0; o0 < nce; o0 += 4 * kTT) {
    int row[4], e[4], u[4], p[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int o = o0 + t * kTT + tid;
      row[t] = o < nce ? S.colC[o] : -1;
      e[t] = row[t] >= 0 ? gcs[row[t]] + (o - S.rc[row[t]]) : 0;
      u[t] = row[t] >= 0 ? __ldg(&g.ce_col[e[t]]) : 0;
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) p[t] = row[t] >= 0 ? __ldcg(&w.t_pos[u[t]]) - s0 : 0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int o = o0 + t * kTT + tid;
      if (row[t] < 0) continue;
      if ((unsigned)p[t] >= (unsigned)m) atomicOr(&S.bad, kGateOpen);  // asymmetric input
      S.colC[o] = (unsigned short)min(max(p[t], 0), m - 1);
      if (val) {
        const int v = S.orig[row[t]];
        const bool first = o == S.rc[row[t]];
        if (u[t] == v || (!first && u[t] <= __ldg(&g.ce_col[e[t] - 1]))) atomicOr(&S.bad, kGateInvalid);
        hs[0] += edge_hash(v, u[t]);
        hs[1] += edge_hash(u[t], v);
      }
    }
  }
  for (int o = tid; o < nse; o += kTT) {
    const int r = S.colS[o];
    const int e = gss[r] + (o - S.rs[r]);
    const int u = __ldg(&g.se_col[e]);
    const int p = __ldcg(&w.t_pos[u]) - s0;
    if ((unsigned)p >= (unsigned)m) atomicOr(&S.bad, kGateOpen);
    S.colS[o] = (unsigned short)min(max(p, 0), m - 1);
    if (val) {
      const int v = S.orig[r];
      if (u == v || (o > S.rs[r] && u <= __ldg(&g.se_col[e - 1]))) atomicOr(&S.bad, kGateInvalid);
      hs[2] += edge_hash(v, u);
      hs[3] += edge_hash(u, v);
      int lo = gcs[r], hi2 = gcs[r] + (S.rc[r + 1] - S.rc[r]);  // CE ∩ SE: binary search in the CE row
      while (lo < hi2) {
        const int mid = (lo + hi2) >> 1;
        const int y = __ldg(&g.ce_col[mid]);
        if (y == u) atomicOr(&S.bad, kGateInvalid);
        if (y < u) lo = mid + 1; else hi2 = mid;
      }
    }
  }
  if (tid < 3) S.nq[tid] = 0;
  __syncthreads();
  if (S.bad) {
    if (tid == 0) set_gate(ctl, S.bad);
    return -1;
  }
  // ---- 3. simplification (R8): frontier rounds in shared memory
  int hidden = 0;
  for (int i = tid; i < m; i += kTT) {
    const bool st = S.rs[i + 1] > S.rs[i];
    const int d = S.rc[i + 1] - S.rc[i];
    S.prio[i] = lowbias32((uint32_t)local_id(g, S.orig[i]));
    S.cnt[i] = st ? kTBig : d;
    if (!st && d < K) {
      S.hr[i] = 0;
      S.q[0][atomicAdd(&S.nq[0], 1)] = (short)i;
    }
  }
  __syncthreads();
  int r = 0;
  while (true) {
    const int c = S.nq[r % 3];
    if (c == 0) break;
    hidden += c;
    if (tid == 0) S.nq[(r + 2) % 3] = 0;
    const short* cur = S.q[r & 1];
    short* nxt = S.q[(r + 1) & 1];
    int* ncnt = &S.nq[(r + 1) % 3];
    for (int x = tid; x < c; x += kTT) {
      const int v = cur[x];
      for (int e = S.rc[v], e1 = S.rc[v + 1]; e < e1; ++e) {
        const int u = S.colC[e];
        if (atomicSub(&S.cnt[u], 1) == K) {  // its live degree crosses k -> k-1: hidden next round
          S.hr[u] = (short)(r + 1);
          nxt[atomicAdd(ncnt, 1)] = (short)u;
        }
      }
    }
    ++r;
    __syncthreads();
  }
  if (tid < 3) S.nq[tid] = 0;  // the rounds leave stale counts behind
  __syncthreads();
  // ---- 4. (decompose) kept sub-graphs (Alg. 1 lines 1-3) -> pool, light search
  if (!finish) {
    for (int i = tid; i < m; i += kTT) S.uf[i] = i;
    __syncthreads();
    for (int i = tid; i < m; i += kTT) {
      if (S.hr[i] != -1) continue;
      for (int e = S.rc[i], e1 = S.rc[i + 1]; e < e1; ++e) {
        const int u = S.colC[e];
        if (u > i && S.hr[u] == -1) uf_union_id(S.uf, S.orig, i, u);
      }
      for (int e = S.rs[i], e1 = S.rs[i + 1]; e < e1; ++e) {
        const int u = S.colS[e];
        if (u > i && S.hr[u] == -1) uf_union_id(S.uf, S.orig, i, u);
      }
    }
    __syncthreads();
    for (int i = tid; i < m; i += kTT)
      if (S.hr[i] == -1) S.uf[i] = uf_find(S.uf, i);
    __syncthreads();
    for (int i = tid; i < m; i += kTT)
      if (S.hr[i] == -1 && S.uf[i] == i) {
        const int c = atomicAdd(&S.ncomp, 1);
        S.q[1][i] = (short)c;  // ordinal of the component (at its root)
        S.q[0][c] = (short)i;  // component root (its minimum id: the BFS start of R5)
      }
    __syncthreads();
    const int nk = S.ncomp;
    for (int c = tid; c < nk; c += kTT) S.cnt[c] = 0;
    if (tid == 0) S.maxn = 0;
    __syncthreads();
    for (int i = tid; i < m; i += kTT)
      if (S.hr[i] == -1) atomicAdd(&S.cnt[S.q[1][S.uf[i]]], 1);
    __syncthreads();
    block_scan2(S, S.cnt, S.uf, nullptr, nullptr, nk);  // S.uf[c] = offset of component c, S.uf[nk] = total
    const int maxn = S.maxn, tk = S.uf[nk];
    if (maxn > kMaxComp) {  // MPLD_ERR_COMPONENT: reported by the whole-graph pipeline
      if (tid == 0) set_gate(ctl, kGateComponent);
      return -1;
    }
    // more than one lane batch: the light kernel searches them (all its warps), the
    // finish launch recovers the window; else warp 0 searches them here
    const bool defer = nk > 32;
    if (tid == 0 && nk > 0) {
      if (defer) {
        const unsigned long long old = atomicAdd(&ctl->comp_pool, ((unsigned long long)nk << 32) | (unsigned)tk);
        S.cb = (unsigned)(old >> 32);
        S.ob = (unsigned)old;
        S.pending = 1;
      } else {  // the tiles' own records from the top of the pool
        const unsigned long long old =
            atomicAdd(&ctl->comp_pool_tile, ((unsigned long long)nk << 32) | (unsigned)tk);
        S.cb = (unsigned)n - (unsigned)(old >> 32) - (unsigned)nk;
        S.ob = (unsigned)n - (unsigned)old - (unsigned)tk;
      }
      atomicMax(&ctl->max_comp, maxn);
    }
    __syncthreads();
    const unsigned cb = S.cb, ob = S.ob;
    // one lane per component: BFS from the minimum over CE ∪ SE in ascending id
    // (R5 column order), then the adj / sadj words in that order
    for (int c = tid; c < nk; c += kTT) {
      const int root = S.q[0][c], off = S.uf[c], nc = S.cnt[c];
      short* ord = &S.q[1][off];
      ord[0] = (short)root;
      S.hr[root] = -3;
      int t = 1;
      for (int h = 0; h < t; ++h) {
        const int v = ord[h];
        int x = S.rc[v], xe = S.rc[v + 1], y = S.rs[v], ye = S.rs[v + 1];
        while (x < xe || y < ye) {  // both rows ascending in id: merge
          const int ux = x < xe ? S.colC[x] : -1, uy = y < ye ? S.colS[y] : -1;
          const bool takex = uy < 0 || (ux >= 0 && S.orig[ux] < S.orig[uy]);
          const int u = takex ? ux : uy;
          if (takex) ++x; else ++y;
          if (S.hr[u] == -1 && t < nc) {
            S.hr[u] = (short)(-3 - t);
            ord[t++] = (short)u;
          }
        }
      }
      for (int h = 0; h < t; ++h) {
        const int v = ord[h];
        unsigned long long adj = 0ull, sadj = 0ull;
        for (int e = S.rc[v], e1 = S.rc[v + 1]; e < e1; ++e) {
          const int x = S.hr[S.colC[e]];
          if (x <= -3) adj |= 1ull << (-3 - x);
        }
        for (int e = S.rs[v], e1 = S.rs[v + 1]; e < e1; ++e) {
          const int x = S.hr[S.colS[e]];
          if (x <= -3) sadj |= 1ull << (-3 - x);
        }
        const size_t p = (size_t)ob + off + h;
        *(ulonglong2*)&w.pmask[2 * p] = make_ulonglong2(adj, sadj);
        w.porder[p] = S.orig[v];
      }
      w.crec[cb + c] = ((unsigned long long)(ob + off) << 8) | (unsigned long long)t;
      for (int h = 0; h < t; ++h) S.hr[ord[h]] = -1;
    }
    __threadfence();  // the pool records are read by warp 0 through L2 (warp_stage)
    __syncthreads();
    if (wid == 0 && !defer && nk > 0) {
      // the light search: one component per lane (the oracle's node order and budget)
      const bool exact = a.max_steps <= 0;
      const unsigned budget = light_budget(a.max_steps, a.light_steps);
      const unsigned h0 = acc.handoff;
      const bool valid = lane < nk;
      const int ci = (int)cb + lane;
      const unsigned long long rec = valid ? __ldcg(&w.crec[ci]) : 0ull;
      const int nn = (int)(rec & 0xffull);
      acc.comps += valid ? 1 : 0;
      const bool wide = valid && nn > 32;
      if (wide && exact) {
        light_handoff(g, w, ci, nn, INT_MAX);
        acc.handoff += 1;
      }
      const unsigned wm = __ballot_sync(0xffffffffu, wide && !exact);
      if (wm) {
        int base = 0;
        if (lane == 0) base = atomicAdd(&ctl->n_wide, __popc(wm));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (wide && !exact) {
          w.wide[base + __popc(wm & lanemask_lt())] = ci;
          acc.handoff += 1;
        }
      }
      lane_component<K, unsigned, 32, kStagedLight>(g, w, S.L, lane, valid, valid && nn <= 32, ci, rec, a.w_stitch,
                                                    budget, exact, a.colors, a.counts, acc);
      const unsigned dh = __reduce_add_sync(0xffffffffu, acc.handoff - h0);
      if (lane == 0 && dh > 0) S.pending = 1;
      __threadfence();  // the colours written by the search, read below by the other warps
    }
  }
  // ---- 5. recovery (R9): predecessor counts and level 0 (beside the search:
  // warps 1.. in decompose mode), then the levels once the kept colours are final
  {
    const int first = finish ? tid : tid - 32, stride = finish ? kTT : kTT - 32;
    if (first >= 0)
      for (int i = first; i < m; i += stride) {
        if (S.hr[i] < 0) continue;
        const unsigned long long kv = tkey(S, i);
        int c = 0;
        for (int e = S.rc[i], e1 = S.rc[i + 1]; e < e1; ++e) {
          const int u = S.colC[e];
          c += (S.hr[u] >= 0 && tkey(S, u) > kv) ? 1 : 0;
        }
        S.cnt[i] = c;
        if (c == 0) S.q[0][atomicAdd(&S.nq[0], 1)] = (short)i;
      }
  }
  __syncthreads();
  if (!finish && S.pending) {  // the search is not over for this window: recovery in the finish launch
    if (tid == 0) {
      const int p = atomicAdd(&ctl->n_pending, 1);
      w.q0[p] = s0;
      w.q1[p] = m;
    }
  } else {
    for (int i = tid; i < m; i += kTT)
      if (S.hr[i] == -1) S.col8[i] = (signed char)a.colors[S.orig[i]];
    __syncthreads();
    int L = 0;
    while (true) {
      const int c = S.nq[L % 3];
      if (c == 0) break;
      if (tid == 0) S.nq[(L + 2) % 3] = 0;
      const short* cur = S.q[L & 1];
      short* nxt = S.q[(L + 1) & 1];
      int* ncnt = &S.nq[(L + 1) % 3];
      for (int x = tid; x < c; x += kTT) {
        const int v = cur[x];
        const unsigned long long kv = tkey(S, v);
        unsigned used = 0u;
        for (int e = S.rc[v], e1 = S.rc[v + 1]; e < e1; ++e) {
          const int u = S.colC[e];
          if (tkey(S, u) > kv) {  // kept, or popped before v: already coloured
            used |= 1u << (S.col8[u] & 7);
          } else if (atomicSub(&S.cnt[u], 1) == 1) {  // v was u's last predecessor
            nxt[atomicAdd(ncnt, 1)] = (short)u;
          }
        }
        const int col = __ffs(~used) - 1;
        S.col8[v] = (signed char)(col < K ? col : 0);  // col < k by the simplification invariant
      }
      ++L;
      __syncthreads();
    }
    for (int i = tid; i < m; i += kTT)
      if (S.hr[i] >= 0) a.colors[S.orig[i]] = S.col8[i];
  }
  if (!finish && tid == 0) {  // every thread counted the same rounds
    if (hidden) atomicAdd(&ctl->n_hidden, hidden);
    if (r) atomicMax(&ctl->n_rounds, r);
  }
  __syncthreads();
  return s0 + m;
}

template <int K>
__global__ void __launch_bounds__(kTT, 2) mpld_tile_decompose(GraphView g, Workspace w, TileArgs a) {
  pdl_begin();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TileSmem& S = *reinterpret_cast<TileSmem*>(smem_raw);
  Control* ctl = w.ctl;
  const int tid = threadIdx.x;
  const int n = g.n;
  if (!a.finish && blockIdx.x == 0 && tid == 0) {
    if (w.build_err && *(volatile int*)w.build_err) set_gate(ctl, kGateBuild);  // reported by the whole-graph pipeline
    if (a.validate) {
      bool bad = g.layout_off[0] != 0 || g.layout_off[g.n_layouts] != n || g.ce_rp[0] != 0 || g.se_rp[0] != 0;
      for (int l = 0; l < g.n_layouts; ++l) bad |= g.layout_off[l] > g.layout_off[l + 1];
      if (bad) set_gate(ctl, kGateLayouts);
    }
  }
  LightAcc acc;
  unsigned long long hs[4] = {0ull, 0ull, 0ull, 0ull};
  const int count = a.finish ? __ldcg(&ctl->n_pending) : (n + kTOwn - 1) / kTOwn;
  int* next = a.finish ? &ctl->finish_next : &ctl->tile_next;
  while (true) {
    if (tid == 0) S.tile = *(volatile int*)&ctl->gate ? count : atomicAdd(next, 1);
    __syncthreads();
    const int t = S.tile;
    __syncthreads();
    if (t >= count) break;
    if (a.finish) {
      if (tile_pass<K>(S, g, w, a, __ldcg(&w.q0[t]), n, __ldcg(&w.q1[t]), acc, hs) < 0) break;
    } else {
      int s0 = piece_start_from(w, n, t * kTOwn);
      const int hi = piece_start_from(w, n, min(n, (t + 1) * kTOwn));
      while (s0 >= 0 && s0 < hi) s0 = tile_pass<K>(S, g, w, a, s0, hi, 0, acc, hs);
      if (s0 < 0) break;
    }
  }
  if (!a.finish) {
    if (tid < 32) light_stats(ctl, acc);
    if (a.validate) {  // CTA sums of the symmetry hashes
      __shared__ unsigned long long s_h[kTWarps][4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) hs[q] += __shfl_xor_sync(0xffffffffu, hs[q], o);
        if ((tid & 31) == 0) s_h[tid >> 5][q] = hs[q];
      }
      __syncthreads();
      if (tid < 4) {
        unsigned long long x = 0ull;
        for (int i = 0; i < kTWarps; ++i) x += s_h[i][tid];
        atomicAdd(&ctl->vh[tid], x);
      }
    }
    return;
  }
  // finish launch: the last CTA checks the symmetry sums and writes Eq. (1a) and the statistics
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(&ctl->done_tiles, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (tid == 0 && a.validate &&
      (__ldcg(&ctl->vh[0]) != __ldcg(&ctl->vh[1]) || __ldcg(&ctl->vh[2]) != __ldcg(&ctl->vh[3])))
    set_gate(ctl, kGateSymmetry);
  __syncthreads();
  if (*(volatile int*)&ctl->gate) return;  // the whole-graph pipeline writes every output
  for (int l = tid; l < g.n_layouts; l += kTT) {
    const long long nc = __ldcg(&a.counts[2 * l]);
    const long long ns = __ldcg(&a.counts[2 * l + 1]);
    a.cost[l] = __dadd_rn(__dmul_rn(a.alpha, (double)ns), (double)nc);
  }
  if (tid == 0 && a.stats) {
    a.stats[MPLD_STAT_COMPONENTS] = __ldcg(&ctl->n_comp);
    a.stats[MPLD_STAT_HIDDEN] = __ldcg(&ctl->n_hidden);
    a.stats[MPLD_STAT_ROUNDS] = __ldcg(&ctl->n_rounds);
    a.stats[MPLD_STAT_MAX_COMP] = __ldcg(&ctl->max_comp);
    a.stats[MPLD_STAT_STEPS] = (long long)__ldcg(&ctl->steps);
    a.stats[MPLD_STAT_TRUNCATED] = __ldcg(&ctl->truncated);
    a.stats[MPLD_STAT_ERROR] = 0;
    a.stats[MPLD_STAT_LAUNCHES] = a.launches;
    a.stats[MPLD_STAT_MAX_STEPS] = __ldcg(&ctl->max_steps_comp);
    a.stats[MPLD_STAT_SPILL_REFUSED] = __ldcg(&ctl->spill_refused);
  }
}

template <int K>
cudaError_t launch_tile_k(const GraphView& g, const Workspace& w, const TileArgs& a, cudaStream_t s, int blocks,
                          bool pdl) {
  return launch_ex(mpld_tile_decompose<K>, dim3(blocks), dim3(kTT), sizeof(TileSmem), s, pdl, false, g, w, a);
}

}  // namespace

cudaError_t configure_tile() {
  cudaError_t e = cudaSuccess;
  const int sz = (int)sizeof(TileSmem);
  for (auto f : {mpld_tile_decompose<2>, mpld_tile_decompose<3>, mpld_tile_decompose<4>})
    if (e == cudaSuccess) e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, sz);
  for (auto f : {mpld_tile_decompose<2>, mpld_tile_decompose<3>, mpld_tile_decompose<4>})
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
  return e;
}

int resident_blocks_tile(int num_sms) {
  int per = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, mpld_tile_decompose<4>, kTT, sizeof(TileSmem)) != cudaSuccess)
    return 0;
  return per * num_sms;
}

int coop_blocks_piece(int num_sms) {
  int per = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, mpld_piece_order, kPieceThreads, 0) != cudaSuccess)
    return 0;
  return std::min(per, 2) * num_sms;
}

cudaError_t launch_piece_order(const GraphView& g, const Workspace& w, cudaStream_t s, int blocks) {
  return launch_ex(mpld_piece_order, dim3(blocks), dim3(kPieceThreads), 0, s, false, true, g, w);
}

cudaError_t launch_tile(const GraphView& g, const Workspace& w, int k, const TileLaunch& t, cudaStream_t s,
                        int blocks, bool pdl) {
  TileArgs a{t.w_stitch, t.max_steps, t.light_steps, t.colors, t.counts, t.cost, t.stats, t.alpha, t.launches,
             t.validate, t.finish};
  switch (k) {
    case 2: return launch_tile_k<2>(g, w, a, s, blocks, pdl);
    case 3: return launch_tile_k<3>(g, w, a, s, blocks, pdl);
    default: return launch_tile_k<4>(g, w, a, s, blocks, pdl);
  }
}

}  // namespace mpld
