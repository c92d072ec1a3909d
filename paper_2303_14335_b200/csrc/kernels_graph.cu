// Graph-level kernels of the MPLD hot path (§2.2 / Fig. 2 flow):
//   mpld_simplify_components simplification (R8) + component seeds (Alg. 1 lines 1-3)
//   mpld_recover             recovery of the hidden vertices (R9)
//   mpld_evaluate            Eq. (1) conflict / stitch counts and cost per layout
//
// The two persistent kernels are launched cooperatively (one wave of resident
// CTAs, grid-wide barriers between rounds) so that the whole path is enqueued
// without a host synchronisation.  Queue appends reserve space with one atomic
// per CTA (a single hot counter serialises at the L2).
#include "mpld_internal.cuh"

namespace mpld {

namespace {

constexpr int kAppend = 8;   // items one thread may append per call before spilling to direct atomics
constexpr int kNb = 4;       // neighbours processed per batch of independent memory operations
constexpr int kTail = 1024;  // frontiers up to one item per thread of a CTA are finished by that CTA alone

__device__ __forceinline__ bool row_contains(const int* __restrict__ col, int a, int b, int x) {
  // binary search in the strictly ascending row col[a..b)
  while (a < b) {
    int m = (a + b) >> 1;
    int y = col[m];
    if (y == x) return true;
    if (y < x) a = m + 1; else b = m;
  }
  return false;
}

__device__ __forceinline__ int layout_index(const GraphView& g, int v) {
  if (g.n_layouts <= 1) return 0;
  int lo = 0, hi = g.n_layouts;  // off[lo] <= v < off[lo+1]
  while (hi - lo > 1) {
    int m = (lo + hi) >> 1;
    if (__ldg(&g.layout_off[m]) <= v) lo = m; else hi = m;
  }
  return lo;
}

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

// Block-wide append: thread i contributes cnt_i items; the CTA reserves its
// range with one atomicAdd.  Every thread of the CTA must call it (uniform
// control flow); blockDim.x must be a multiple of 32.
__device__ __forceinline__ void cta_append(int cnt, const int* items, int* counter, int* out) {
  __shared__ int s_warp[32];
  __shared__ int s_base;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int x = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[wid] = x;
  __syncthreads();
  if (wid == 0) {
    const int t = lane < nw ? s_warp[lane] : 0;
    int y = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int z = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= o) y += z;
    }
    if (lane < nw) s_warp[lane] = y - t;  // exclusive prefix of the warp totals
    if (lane == 31) s_base = y ? atomicAdd(counter, y) : 0;
  }
  __syncthreads();
  const int pos = s_base + s_warp[wid] + x - cnt;
  for (int i = 0; i < cnt; ++i) out[pos + i] = items[i];
  __syncthreads();
}

// push into a per-thread append list, spilling to a direct atomic when full
__device__ __forceinline__ void list_push(int* items, int& cnt, int v, int* counter, int* out) {
  if (cnt < kAppend) items[cnt++] = v;
  else out[atomicAdd(counter, 1)] = v;
}

// ---------------------------------------------------------------------------
// Input invariants of include/mpld.h for vertex v (MPLD_FLAG_VALIDATE): both
// rows strictly ascending, ids in range, no self loop, symmetric (binary search
// in the neighbour's row), CE ∩ SE = ∅.
__device__ bool vertex_invalid(const GraphView& g, int v) {
  for (int pass = 0; pass < 2; ++pass) {
    const int* rp = pass ? g.se_rp : g.ce_rp;
    const int* col = pass ? g.se_col : g.ce_col;
    const int* orp = pass ? g.ce_rp : g.se_rp;
    const int* ocol = pass ? g.ce_col : g.se_col;
    const int a = rp[v], b = rp[v + 1];
    if (a > b) return true;
    int prev = -1;
    for (int e = a; e < b; ++e) {
      const int u = col[e];
      if (u < 0 || u >= g.n || u == v || u <= prev) return true;
      prev = u;
      if (!row_contains(col, rp[u], rp[u + 1], v)) return true;   // symmetric
      if (row_contains(ocol, orp[v], orp[v + 1], u)) return true;  // CE ∩ SE = ∅
    }
  }
  return false;
}

// One simplification round r >= 1: push the decrements of the frontier
// (items [first, cnt) with the given stride; every thread of the CTA calls it).
__device__ void peel_round(const GraphView& g, const Workspace& w, int k, int r, int cnt, int first, int stride,
                           int* qc) {
  const int* cur = (r & 1) ? w.q1 : w.q0;
  int* nxt = (r & 1) ? w.q0 : w.q1;
  int* ncnt = &qc[(r + 1) % 3];
  for (int i0 = first; i0 < cnt; i0 += stride) {
    const int i = i0 + threadIdx.x;
    int items[kAppend];
    int m = 0;
    if (i < cnt) {
      const int v = __ldcg(&cur[i]);
      const int e1 = g.ce_rp[v + 1];
      // neighbours in batches of kNb: ids, rounds and decrements of a batch are
      // independent and in flight together (a few memory round trips per batch
      // instead of three per neighbour)
      for (int e0 = g.ce_rp[v]; e0 < e1; e0 += kNb) {
        int u[kNb], hu[kNb], old[kNb];
#pragma unroll
        for (int j = 0; j < kNb; ++j) u[j] = e0 + j < e1 ? g.ce_col[e0 + j] : -1;
#pragma unroll
        for (int j = 0; j < kNb; ++j) hu[j] = u[j] >= 0 ? __ldcg(&w.hround[u[j]]) : 0;
#pragma unroll
        for (int j = 0; j < kNb; ++j)  // already-hidden neighbours' degrees no longer matter
          old[j] = hu[j] == -1 ? atomicSub(&w.deg[u[j]], 1) : 0;
#pragma unroll
        for (int j = 0; j < kNb; ++j) {
          if (old[j] == k && g.se_rp[u[j] + 1] == g.se_rp[u[j]]) {
            w.hround[u[j]] = r + 1;
            list_push(items, m, u[j], ncnt, nxt);
          }
        }
      }
    }
    cta_append(m, items, ncnt, nxt);
  }
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
// Then the seeds of the component search (see below).
__global__ void __launch_bounds__(1024, 2) mpld_simplify_components(GraphView g, Workspace w, int k,
                                                                    int* colors, long long* counts, int validate) {
  GridBarrier grid(&w.ctl->bar[0]);
  stamp(w.ctl, 12);
  const int n = g.n;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int nth = gridDim.x * blockDim.x;
  Control* ctl = w.ctl;
  for (int l = tid; l < 2 * g.n_layouts; l += nth) counts[l] = 0;

  // rounds 0 and 1, recovery priorities, union-find init (and the optional
  // validation of the input, fused into this first pass over the CSR)
  int hidden0 = 0;
  bool bad = false;
  if (validate && tid == 0) {
    if (g.layout_off[0] != 0 || g.layout_off[g.n_layouts] != g.n) bad = true;
    for (int l = 0; l < g.n_layouts; ++l)
      if (g.layout_off[l] > g.layout_off[l + 1]) bad = true;
  }
  for (int v0 = blockIdx.x * blockDim.x; v0 < n; v0 += nth) {
    const int v = v0 + threadIdx.x;
    int take = 0;
    if (v < n) {
      if (validate) bad |= vertex_invalid(g, v);
      const int a = g.ce_rp[v], b = g.ce_rp[v + 1];
      const bool st = g.se_rp[v + 1] > g.se_rp[v];
      const int lo = layout_index(g, v);
      w.prio[v] = lowbias32((uint32_t)(v - (g.n_layouts > 1 ? __ldg(&g.layout_off[lo]) : 0)));
      colors[v] = -1;  // every vertex is coloured later by exactly one search shard or the recovery
      int hr = -1;
      if (!st && b - a < k) {
        hr = 0;
        ++hidden0;
      } else {
        int d0 = 0;  // live degree after round 0
        for (int e = a; e < b; ++e) {
          const int u = g.ce_col[e];
          if ((unsigned)u >= (unsigned)n) continue;  // invalid input (flagged when validating)
          d0 += (g.se_rp[u + 1] > g.se_rp[u] || g.ce_rp[u + 1] - g.ce_rp[u] >= k) ? 1 : 0;
        }
        w.deg[v] = d0;
        if (!st && d0 < k) { hr = 1; take = 1; }
      }
      w.hround[v] = hr;
    }
    int item = v;
    cta_append(take, &item, &ctl->qcnt[1], w.q1);
  }
  hidden0 = __reduce_add_sync(0xffffffffu, hidden0);
  if ((threadIdx.x & 31) == 0 && hidden0) atomicAdd(&ctl->n_hidden, hidden0);
  if (bad) atomicOr(&ctl->err, kErrGraph);
  grid.sync();
  stamp(w.ctl, 0);
  if (__ldcg(&ctl->err)) return;  // invalid input: every later kernel exits too

  // rounds r >= 1: push the frontier's decrements
  int r = 1;
  while (true) {
    const int cnt = __ldcg(&ctl->qcnt[r % 3]);
    if (cnt == 0) break;
    if (cnt <= kTail) {
      // small frontier: CTA 0 runs the remaining rounds alone with block
      // barriers (a grid barrier costs ~1.5 µs; the rounds only need the
      // dependent-load latency)
      if (blockIdx.x == 0) {
        int rr = r, c = cnt;
        while (c > 0) {
          // own counters: the other CTAs may still be reading qcnt[r % 3] to
          // take this branch, so the tail must never reset that slot
          if (threadIdx.x == 0) {
            ctl->tcnt[(rr + 2) % 3] = 0;
            ctl->n_hidden += c;
          }
          dstamp(ctl, rr, c);
          peel_round(g, w, k, rr, c, 0, blockDim.x, ctl->tcnt);
          ++rr;
          __syncthreads();
          c = __ldcg(&ctl->tcnt[rr % 3]);
        }
        if (threadIdx.x == 0) ctl->n_rounds = rr;
      }
      grid.sync();
      r = __ldcg(&ctl->n_rounds);
      break;
    }
    if (tid == 0) {
      ctl->qcnt[(r + 2) % 3] = 0;
      ctl->n_hidden += cnt;
    }
    dstamp(ctl, r, cnt);
    peel_round(g, w, k, r, cnt, blockIdx.x * blockDim.x, nth, ctl->qcnt);
    ++r;
    grid.sync();
    stamp(w.ctl, 2);
  }
  if (tid == 0) ctl->n_rounds = __ldcg(&ctl->n_hidden) ? r : 0;
  stamp(w.ctl, 1);

  // Pop keys, and the component search seeds: a kept vertex with no kept
  // neighbour (CE ∪ SE) of smaller id.  Every component has at least one seed
  // (its minimum); the search kernel's BFS from a seed keeps the component only
  // if the seed is the component's minimum, so no union-find and no further
  // grid barrier are needed here.
  for (int v0 = blockIdx.x * blockDim.x; v0 < n; v0 += nth) {
    const int v = v0 + threadIdx.x;
    int seed = 0;
    if (v < n) {
      const int hv = __ldcg(&w.hround[v]);
      w.key[v] = pop_key(hv, w.prio[v]);
      if (hv == -1) {
        seed = 1;
        for (int pass = 0; pass < 2 && seed; ++pass) {
          const int* rp = pass ? g.se_rp : g.ce_rp;
          const int* col = pass ? g.se_col : g.ce_col;
          const int e0 = rp[v];
          // rows are ascending: only the first neighbours can be smaller than v
          for (int e = e0, e1 = rp[v + 1]; e < e1; ++e) {
            const int u = col[e];
            if (u > v) break;
            if (__ldcg(&w.hround[u]) == -1) {
              seed = 0;
              break;
            }
          }
        }
      }
    }
    int item = v;
    cta_append(seed, &item, &ctl->n_seed, w.roots);
  }
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
// predecessor; a vertex joins the next level when its last predecessor is
// coloured.  Every level is coloured in parallel, one grid barrier per level
// (DAG depth ~ 10-20 on layout graphs); the result equals the sequential pop.
// One recovery level: colour the ready vertices cur[first..cnt) (stride),
// queue the successors whose last predecessor this was.
__device__ void recover_level(const GraphView& g, const Workspace& w, int k, int* colors, int L, int cnt, int first,
                              int stride, int* qc) {
  const int* cur = (L & 1) ? w.q1 : w.q0;
  int* nxt = (L & 1) ? w.q0 : w.q1;
  int* ncnt = &qc[(L + 1) % 3];
  for (int i0 = first; i0 < cnt; i0 += stride) {
    const int i = i0 + threadIdx.x;
    int items[kAppend];
    int m = 0;
    if (i < cnt) {
      const int v = __ldcg(&cur[i]);
      const unsigned long long kv = w.key[v];
      unsigned used = 0;
      const int e1 = g.ce_rp[v + 1];
      for (int e0 = g.ce_rp[v]; e0 < e1; e0 += kNb) {  // batches with independent loads / atomics
        int u[kNb], x[kNb];
        bool before[kNb];
#pragma unroll
        for (int j = 0; j < kNb; ++j) u[j] = e0 + j < e1 ? g.ce_col[e0 + j] : -1;
#pragma unroll
        for (int j = 0; j < kNb; ++j) before[j] = u[j] >= 0 && w.key[u[j]] > kv;  // popped before v (or kept)
#pragma unroll
        for (int j = 0; j < kNb; ++j)
          x[j] = u[j] < 0 ? -1 : (before[j] ? __ldcg(&colors[u[j]]) : atomicSub(&w.deg[u[j]], 1));
#pragma unroll
        for (int j = 0; j < kNb; ++j) {
          if (u[j] < 0) continue;
          if (before[j]) {
            if (x[j] >= 0) used |= 1u << x[j];
          } else if (x[j] == 1) {  // v was u's last predecessor
            list_push(items, m, u[j], ncnt, nxt);
          }
        }
      }
      const int c = __ffs(~used) - 1;
      colors[v] = c < k ? c : 0;  // c < k by the simplification invariant
    }
    cta_append(m, items, ncnt, nxt);
  }
}

__global__ void __launch_bounds__(1024, 2) mpld_recover(GraphView g, Workspace w, int k, int* colors) {
  GridBarrier grid(&w.ctl->bar[1]);
  stamp(w.ctl, 13);
  if (__ldcg(&w.ctl->err)) return;
  const int nth = gridDim.x * blockDim.x;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  Control* ctl = w.ctl;
  // level 0 and predecessor counts
  for (int v0 = blockIdx.x * blockDim.x; v0 < g.n; v0 += nth) {
    const int v = v0 + threadIdx.x;
    int ready = 0;
    if (v < g.n) {
      const unsigned long long kv = w.key[v];
      if (kv != ~0ull) {
        int cnt = 0;
        const int e1 = g.ce_rp[v + 1];
        for (int e0 = g.ce_rp[v]; e0 < e1; e0 += kNb) {
          int u[kNb];
#pragma unroll
          for (int j = 0; j < kNb; ++j) u[j] = e0 + j < e1 ? g.ce_col[e0 + j] : -1;
#pragma unroll
          for (int j = 0; j < kNb; ++j) {
            if (u[j] < 0) continue;
            const unsigned long long ku = w.key[u[j]];
            cnt += (ku > kv && ku != ~0ull) ? 1 : 0;
          }
        }
        w.deg[v] = cnt;
        ready = cnt == 0;
      }
    }
    int item = v;
    cta_append(ready, &item, &ctl->rq[0], w.q0);
  }
  grid.sync();
  stamp(w.ctl, 8);
  int L = 0;
  while (true) {
    const int cnt = __ldcg(&ctl->rq[L % 3]);
    dstamp(ctl, 16 + L, cnt);
    if (cnt == 0) {
      if (tid == 0) ctl->n_levels = L;
      break;
    }
    if (cnt <= kTail) {  // small level: CTA 0 finishes the remaining levels with block barriers
      if (blockIdx.x == 0) {
        int LL = L, c = cnt;
        while (c > 0) {
          if (threadIdx.x == 0) ctl->trq[(LL + 2) % 3] = 0;  // own counters, as in the simplification tail
          recover_level(g, w, k, colors, LL, c, 0, blockDim.x, ctl->trq);
          ++LL;
          __syncthreads();
          c = __ldcg(&ctl->trq[LL % 3]);
        }
        if (threadIdx.x == 0) ctl->n_levels = LL;
      }
      break;  // no grid barrier needed: the kernel ends here
    }
    if (tid == 0) ctl->rq[(L + 2) % 3] = 0;
    recover_level(g, w, k, colors, L, cnt, blockIdx.x * blockDim.x, nth, ctl->rq);
    ++L;
    grid.sync();
    stamp(w.ctl, 9);
  }
}

// ---------------------------------------------------------------------------
// Eq. (1b)/(1c) per layout; the last CTA writes cost (Eq. 1a) and the stats.
__global__ void __launch_bounds__(256) mpld_evaluate(GraphView g, Workspace w, const int* colors, double alpha,
                                                     long long* counts, double* cost, long long* stats,
                                                     int launches) {
  const int nth = gridDim.x * blockDim.x;
  stamp(w.ctl, 15);
  const int vend = __ldcg(&w.ctl->err) ? 0 : g.n;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < vend; v += nth) {
    const int cv = colors[v];
    int nc = 0, ns = 0;
    const int e1 = g.ce_rp[v + 1];
    for (int e0 = g.ce_rp[v]; e0 < e1; e0 += kNb) {
      int u[kNb];
#pragma unroll
      for (int j = 0; j < kNb; ++j) u[j] = e0 + j < e1 ? g.ce_col[e0 + j] : -1;
#pragma unroll
      for (int j = 0; j < kNb; ++j)
        if (u[j] > v && colors[u[j]] == cv) ++nc;
    }
    for (int e = g.se_rp[v], e1 = g.se_rp[v + 1]; e < e1; ++e) {
      const int u = g.se_col[e];
      if (u > v && colors[u] != cv) ++ns;
    }
    if (nc | ns) {
      const int l = layout_index(g, v);
      if (nc) atomicAdd((unsigned long long*)&counts[2 * l], (unsigned long long)nc);
      if (ns) atomicAdd((unsigned long long*)&counts[2 * l + 1], (unsigned long long)ns);
    }
  }
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(&w.ctl->done_blocks, 1) == (int)gridDim.x - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int l = threadIdx.x; l < g.n_layouts; l += blockDim.x) {
    const long long nc = __ldcg(&counts[2 * l]);
    const long long ns = __ldcg(&counts[2 * l + 1]);
    cost[l] = __dadd_rn(__dmul_rn(alpha, (double)ns), (double)nc);
  }
  if (threadIdx.x == 0 && stats) {
    Control* ctl = w.ctl;
    stats[MPLD_STAT_COMPONENTS] = __ldcg(&ctl->n_comp);
    stats[MPLD_STAT_HIDDEN] = __ldcg(&ctl->n_hidden);
    stats[MPLD_STAT_ROUNDS] = __ldcg(&ctl->n_rounds);
    stats[MPLD_STAT_MAX_COMP] = __ldcg(&ctl->max_comp);
    stats[MPLD_STAT_STEPS] = (long long)__ldcg(&ctl->steps);
    stats[MPLD_STAT_TRUNCATED] = __ldcg(&ctl->truncated);
    stats[MPLD_STAT_ERROR] = __ldcg(&ctl->err);
    stats[MPLD_STAT_LAUNCHES] = launches;
    stats[MPLD_STAT_MAX_STEPS] = __ldcg(&ctl->max_steps_comp);
  }
}

}  // namespace

cudaError_t launch_simplify_components(const GraphView& g, Workspace ws, int k, int* colors, long long* counts,
                                       int validate, cudaStream_t s, int blocks, int threads) {
  GraphView gg = g;
  void* args[] = {&gg, &ws, &k, &colors, &counts, &validate};
  return cudaLaunchCooperativeKernel((void*)mpld_simplify_components, dim3(blocks), dim3(threads), args, 0, s);
}

cudaError_t launch_recover(const GraphView& g, Workspace ws, int k, int* colors, cudaStream_t s, int blocks,
                           int threads) {
  GraphView gg = g;
  void* args[] = {&gg, &ws, &k, &colors};
  return cudaLaunchCooperativeKernel((void*)mpld_recover, dim3(blocks), dim3(threads), args, 0, s);
}

cudaError_t launch_evaluate(const GraphView& g, Workspace ws, const int* colors, double alpha, long long* counts,
                            double* cost, long long* stats, int launches, cudaStream_t s, int blocks) {
  mpld_evaluate<<<blocks, 256, 0, s>>>(g, ws, colors, alpha, counts, cost, stats, launches);
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

}  // namespace mpld
