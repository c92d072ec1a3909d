// Graph-level kernels of the MPLD hot path (§2.2 / Fig. 2 flow):
//   mpld_validate            input CSR invariants (optional)
//   mpld_simplify_components simplification (R8) + connected components (Alg. 1 lines 1-3)
//   mpld_recover             recovery of the hidden vertices (R9)
//   mpld_evaluate            Eq. (1) conflict / stitch counts and cost per layout
//
// The two persistent kernels are launched cooperatively (one wave of resident
// CTAs, grid-wide barriers between rounds) so that the whole path is enqueued
// without a host synchronisation.
#include <cooperative_groups.h>

#include "mpld_internal.cuh"

namespace cg = cooperative_groups;

namespace mpld {

namespace {

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

__device__ __forceinline__ int layout_base(const GraphView& g, int v) {
  if (g.n_layouts <= 1) return 0;
  int lo = 0, hi = g.n_layouts;  // find l with off[l] <= v < off[l+1]
  while (hi - lo > 1) {
    int m = (lo + hi) >> 1;
    if (__ldg(&g.layout_off[m]) <= v) lo = m; else hi = m;
  }
  return __ldg(&g.layout_off[lo]);
}

__device__ __forceinline__ int layout_index(const GraphView& g, int v) {
  if (g.n_layouts <= 1) return 0;
  int lo = 0, hi = g.n_layouts;
  while (hi - lo > 1) {
    int m = (lo + hi) >> 1;
    if (__ldg(&g.layout_off[m]) <= v) lo = m; else hi = m;
  }
  return lo;
}

__device__ __forceinline__ int find_root(int* parent, int x) {
  int p = __ldcg(&parent[x]);
  while (p != x) {
    x = p;
    p = __ldcg(&parent[x]);
  }
  return x;
}

// Lock-free union: the larger root is hooked under the smaller one, so every
// final root is the minimum vertex id of its component.
__device__ __forceinline__ void unite(int* parent, int a, int b) {
  while (true) {
    a = find_root(parent, a);
    b = find_root(parent, b);
    if (a == b) return;
    if (a < b) { int t = a; a = b; b = t; }
    int old = atomicCAS(&parent[a], a, b);
    if (old == a) return;
  }
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) mpld_validate(GraphView g, Workspace w) {
  const int nth = gridDim.x * blockDim.x;
  int bad = 0;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < g.n; v += nth) {
    for (int pass = 0; pass < 2; ++pass) {
      const int* rp = pass ? g.se_rp : g.ce_rp;
      const int* col = pass ? g.se_col : g.ce_col;
      const int* orp = pass ? g.ce_rp : g.se_rp;
      const int* ocol = pass ? g.ce_col : g.se_col;
      int a = rp[v], b = rp[v + 1];
      if (a > b) { bad = 1; break; }
      int prev = -1;
      for (int e = a; e < b; ++e) {
        int u = col[e];
        if (u < 0 || u >= g.n || u == v || u <= prev) { bad = 1; break; }
        prev = u;
        if (!row_contains(col, rp[u], rp[u + 1], v)) bad = 1;         // symmetric
        if (row_contains(ocol, orp[v], orp[v + 1], u)) bad = 1;       // CE ∩ SE = ∅
      }
    }
  }
  if (g.n_layouts > 0 && blockIdx.x == 0 && threadIdx.x == 0) {
    if (g.layout_off[0] != 0 || g.layout_off[g.n_layouts] != g.n) bad = 1;
    for (int l = 0; l < g.n_layouts; ++l)
      if (g.layout_off[l] > g.layout_off[l + 1]) bad = 1;
  }
  if (bad) atomicOr(&w.ctl->err, kErrGraph);
}

// ---------------------------------------------------------------------------
// Simplification (R8, §2.2 "simplify the layout graph"):
// round r hides every not-yet-hidden vertex without stitch edges whose
// conflict degree among not-yet-hidden vertices is < k.  A vertex enters round
// r+1 exactly when its live degree crosses k -> k-1 during round r, so each
// round only touches the neighbours of the previous round (frontier queue).
// Then union-find connected components over CE ∪ SE of the kept vertices.
__global__ void __launch_bounds__(256) mpld_simplify_components(GraphView g, Workspace w, int k,
                                                                int* colors, long long* counts) {
  cg::grid_group grid = cg::this_grid();
  const int n = g.n;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int nth = gridDim.x * blockDim.x;
  Control* ctl = w.ctl;

  // phase A: reset the workspace
  for (int v = tid; v < n + 2; v += nth) w.rcnt[v] = 0;
  for (int v = tid; v < n; v += nth) {
    w.deg[v] = g.ce_rp[v + 1] - g.ce_rp[v];
    w.hround[v] = -1;
    w.parent[v] = v;
    w.loc[v] = -1;
    colors[v] = -1;
  }
  for (int l = tid; l < 2 * g.n_layouts; l += nth) counts[l] = 0;
  if (tid == 0) {
    ctl->n_rounds = 0;
    ctl->n_hidden = 0;
    ctl->n_comp = 0;
    ctl->next_comp = 0;
    ctl->max_comp = 0;
    ctl->truncated = 0;
    ctl->done_blocks = 0;
    ctl->left[0] = ctl->left[1] = ctl->left[2] = 0;
    ctl->steps = 0ull;
  }
  grid.sync();

  // phase B: round 0 = all low-degree vertices without stitch edges
  for (int v = tid; v < n; v += nth) {
    if (g.se_rp[v + 1] == g.se_rp[v] && w.deg[v] < k) {
      w.hround[v] = 0;
      int p = atomicAdd(&w.rcnt[0], 1);
      w.hid[p] = v;
    }
  }
  grid.sync();

  // phase C: rounds 1, 2, ... (frontier = vertices whose degree crossed k -> k-1)
  int off = 0, r = 0;
  while (true) {
    const int cnt = __ldcg(&w.rcnt[r]);
    if (cnt == 0) break;
    if (tid == 0) w.roff[r] = off;
    const int next_off = off + cnt;
    for (int i = tid; i < cnt; i += nth) {
      const int v = __ldcg(&w.hid[off + i]);
      const int e1 = g.ce_rp[v + 1];
      for (int e = g.ce_rp[v]; e < e1; ++e) {
        const int u = g.ce_col[e];
        if (__ldcg(&w.hround[u]) != -1) continue;  // already hidden: its degree no longer matters
        const int old = atomicSub(&w.deg[u], 1);
        if (old == k && g.se_rp[u + 1] == g.se_rp[u]) {
          w.hround[u] = r + 1;
          const int p = atomicAdd(&w.rcnt[r + 1], 1);
          w.hid[next_off + p] = u;
        }
      }
    }
    off = next_off;
    ++r;
    grid.sync();
  }
  if (tid == 0) {
    ctl->n_rounds = r;
    ctl->n_hidden = off;
    w.roff[r] = off;
  }

  // phase D: union-find hooking over CE ∪ SE between kept vertices
  for (int v = tid; v < n; v += nth) {
    if (__ldcg(&w.hround[v]) != -1) continue;
    for (int pass = 0; pass < 2; ++pass) {
      const int* rp = pass ? g.se_rp : g.ce_rp;
      const int* col = pass ? g.se_col : g.ce_col;
      const int e1 = rp[v + 1];
      for (int e = rp[v]; e < e1; ++e) {
        const int u = col[e];
        if (u < v && __ldcg(&w.hround[u]) == -1) unite(w.parent, u, v);
      }
    }
  }
  grid.sync();

  // phase E: compress, list the roots (component order is irrelevant to the result)
  for (int v = tid; v < n; v += nth) {
    if (__ldcg(&w.hround[v]) != -1) continue;
    const int root = find_root(w.parent, v);
    w.parent[v] = root;
    if (root == v) {
      const int p = atomicAdd(&ctl->n_comp, 1);
      w.roots[p] = v;
    }
  }
}

// ---------------------------------------------------------------------------
// Recovery (R9, §2.2 "recover the nodes removed in
// simplification step"): the hidden stack is popped LIFO — rounds in reverse,
// inside a round in descending lowbias32(layout-local id) — and each vertex
// takes the smallest mask unused by its already-coloured conflict neighbours.
// Inside a round the order is realised Jones-Plassmann style: a vertex is
// coloured as soon as every same-round neighbour of higher priority is, which
// yields exactly the sequential result.
__global__ void __launch_bounds__(256) mpld_recover(GraphView g, Workspace w, int k, int* colors) {
  cg::grid_group grid = cg::this_grid();
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int nth = gridDim.x * blockDim.x;
  Control* ctl = w.ctl;
  const int R = __ldcg(&ctl->n_rounds);
  int it = 0;
  for (int r = R - 1; r >= 0; --r) {
    const int off = __ldcg(&w.roff[r]);
    const int cnt = __ldcg(&w.rcnt[r]);
    while (true) {
      if (tid == 0) ctl->left[(it + 1) % 3] = 0;
      int left = 0;
      for (int i = tid; i < cnt; i += nth) {
        const int v = __ldcg(&w.hid[off + i]);
        if (__ldcg(&colors[v]) >= 0) continue;
        const int base = layout_base(g, v);
        const uint32_t pv = lowbias32((uint32_t)(v - base));
        bool ready = true;
        unsigned used = 0;
        const int e1 = g.ce_rp[v + 1];
        for (int e = g.ce_rp[v]; e < e1; ++e) {
          const int u = g.ce_col[e];
          const int hu = __ldcg(&w.hround[u]);
          if (hu == r) {
            if (lowbias32((uint32_t)(u - base)) > pv) {
              const int cu = *((volatile int*)&colors[u]);
              if (cu < 0) { ready = false; break; }
              used |= 1u << cu;
            }
          } else if (hu == -1 || hu > r) {
            const int cu = __ldcg(&colors[u]);
            if (cu >= 0) used |= 1u << cu;
          }
        }
        if (ready) {
          const int c = __ffs(~used) - 1;
          colors[v] = c < k ? c : 0;  // c < k by the simplification invariant
        } else {
          ++left;
        }
      }
      if (left) atomicAdd(&ctl->left[it % 3], left);
      grid.sync();
      const int remaining = __ldcg(&ctl->left[it % 3]);
      ++it;
      if (remaining == 0) break;
    }
  }
}

// ---------------------------------------------------------------------------
// Eq. (1b)/(1c) per layout; the last CTA writes cost (Eq. 1a) and the stats.
__global__ void __launch_bounds__(256) mpld_evaluate(GraphView g, Workspace w, const int* colors, double alpha,
                                                     long long* counts, double* cost, long long* stats,
                                                     int launches) {
  const int nth = gridDim.x * blockDim.x;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < g.n; v += nth) {
    const int cv = colors[v];
    int nc = 0, ns = 0;
    for (int e = g.ce_rp[v], e1 = g.ce_rp[v + 1]; e < e1; ++e) {
      const int u = g.ce_col[e];
      if (u > v && colors[u] == cv) ++nc;
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
  if (threadIdx.x == 0) {
    Control* ctl = w.ctl;
    if (stats) {
      stats[MPLD_STAT_COMPONENTS] = __ldcg(&ctl->n_comp);
      stats[MPLD_STAT_HIDDEN] = __ldcg(&ctl->n_hidden);
      stats[MPLD_STAT_ROUNDS] = __ldcg(&ctl->n_rounds);
      stats[MPLD_STAT_MAX_COMP] = __ldcg(&ctl->max_comp);
      stats[MPLD_STAT_STEPS] = (long long)__ldcg(&ctl->steps);
      stats[MPLD_STAT_TRUNCATED] = __ldcg(&ctl->truncated);
      stats[MPLD_STAT_ERROR] = __ldcg(&ctl->err);
      stats[MPLD_STAT_LAUNCHES] = launches;
    }
    ctl->err = 0;  // the control block resets itself for the next call
  }
}

}  // namespace

cudaError_t launch_validate(const GraphView& g, Workspace ws, cudaStream_t s, int blocks) {
  mpld_validate<<<blocks, 256, 0, s>>>(g, ws);
  return cudaGetLastError();
}

cudaError_t launch_simplify_components(const GraphView& g, Workspace ws, int k, int* colors,
                                       long long* counts, cudaStream_t s, int blocks, int threads) {
  GraphView gg = g;
  void* args[] = {&gg, &ws, &k, &colors, &counts};
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
