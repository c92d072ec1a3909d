// The exact-cover search of PAPER.md §2.3 / Alg. 1 on bit-packed matrices.
//
// One thread owns one component (n <= 64 vertices).  The exact-cover matrix
// (rows r(v,c), primary columns = vertices, secondary columns = (e,c) for
// e in CE) is never materialised as a 0/1 array: with columns = bit positions
// of a machine word it is fully described by, per vertex v,
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
// The search order, bound and budget are DESIGN.md R4-R7, identical to the
// oracle's dancing-links Algorithm X, so the result is bit-identical.
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

// One level of the explicit backtrack stack (Alg. 1 recursion, lines 13-18).
template <typename W>
struct __align__(16) Frame {
  W saved;   // B[c] before r(v,c) was selected
  W adj;     // adj[v]
  W sadj;    // sadj[v]
  int cost;  // cost when the node was entered
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

// Relaxed Algorithm X with branch and bound (R4-R7).  am[i] =
// (adj, sadj) of local vertex i.  Returns the steps taken; the best masks in bestC.
template <int K, typename W>
__device__ unsigned search_component(const W* __restrict__ am_adj, const W* __restrict__ am_sadj, int n,
                                     int w_stitch, unsigned max_steps, Frame<W>* __restrict__ stack,
                                     W (&bestC)[K], bool& truncated) {
  using O = WordOps<W>;
  W C[K], B[K];
#pragma unroll
  for (int c = 0; c < K; ++c) { C[c] = 0; B[c] = 0; bestC[c] = 0; }
  W U = O::full(n);
  int cost = 0, maxused = -1, depth = 0;
  int best = INT_MAX;
  unsigned steps = 0;
  truncated = false;
  bool enter = true;
  // the frame of the deepest expanded node lives in registers
  W f_saved = 0, f_adj = 0, f_sadj = 0;
  int f_cost = 0, f_v = 0, f_c = -1, f_mu = -1;
  while (true) {
    if (enter) {
      ++steps;
      if (best != INT_MAX && steps > max_steps) { truncated = true; break; }
      if (U == 0) {  // Alg. 1 line 5: every column covered -> a solution
        if (cost < best) {
          best = cost;
#pragma unroll
          for (int c = 0; c < K; ++c) bestC[c] = C[c];
        }
      } else {
        // column-count reduction, bit-sliced over all columns at once
        W s1 = 0, s2 = 0;
#pragma unroll
        for (int c = 0; c < K; ++c) {
          const W F = U & ~B[c];  // live rows of mask c
          s2 |= s1 & F;
          s1 |= F;
        }
        const W Z = U & ~s1;  // columns with no live row
        const W Ol = s1 & ~s2;  // columns with exactly one live row
        if (cost + kCostUnits * O::popc(Z) < best) {  // bound (R7)
          const W cand = Z ? Z : (Ol ? Ol : U);  // Alg. 1 line 8 (R5)
          const int v = O::ffs(cand);
          if (depth > 0) {  // spill the parent frame
            Frame<W> f;
            f.saved = f_saved;
            f.adj = f_adj;
            f.sadj = f_sadj;
            f.cost = f_cost;
            f.packed = f_v | ((f_c + 1) << 8) | ((f_mu + 1) << 16);
            stack[depth - 1] = f;
          }
          f_v = v;
          f_c = -1;
          f_mu = maxused;
          f_cost = cost;
          f_adj = am_adj[v];
          f_sadj = am_sadj[v];
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
        const Frame<W> f = stack[depth - 1];
        f_saved = f.saved;
        f_adj = f.adj;
        f_sadj = f.sadj;
        f_cost = f.cost;
        f_v = f.packed & 0xff;
        f_c = ((f.packed >> 8) & 0xff) - 1;
        f_mu = ((f.packed >> 16) & 0xff) - 1;
      }
      enter = false;
      continue;
    }
    const W Cc = pick<K, W>(C, c);
    const W Bc = pick<K, W>(B, c);
    const int inc = kCostUnits * O::popc(f_adj & Cc) + w_stitch * O::popc(f_sadj & ~U & ~Cc);
    f_saved = Bc;
    f_c = c;
    put<K, W>(C, c, Cc | bit);  // select r(v,c) (line 14) and cover its secondary columns (line 15)
    put<K, W>(B, c, Bc | f_adj);
    cost = f_cost + inc;
    maxused = max(f_mu, c);
    enter = true;
  }
  return steps;
}

template <int K>
__global__ void __launch_bounds__(128) mpld_exact_cover_search(GraphView g, Workspace w, int w_stitch,
                                                               long long max_steps, int* colors) {
  Control* ctl = w.ctl;
  const int n_comp = __ldcg(&ctl->n_comp);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    ctl->t[14] = t;
  }
  const unsigned budget = (max_steps <= 0 || max_steps >= (long long)UINT_MAX) ? UINT_MAX : (unsigned)max_steps;
  int order[kMaxComp];
  unsigned long long adjm[kMaxComp], sadjm[kMaxComp];
  union {
    Frame<unsigned> f32[32];
    Frame<unsigned long long> f64[kMaxComp];
  } stack;
  for (int ci = blockIdx.x * blockDim.x + threadIdx.x; ci < n_comp; ci += gridDim.x * blockDim.x) {
    const int root = w.roots[ci];
    // build the component's bit-packed matrix: BFS from the root (column order
    // = BFS order of G, neighbours in ascending id, R5)
    int n = 1, head = 0;
    bool too_big = false;
    order[0] = root;
    w.loc[root] = 0;
    while (head < n) {
      const int v = order[head];
      unsigned long long adj = 0ull, sadj = 0ull;
      int a = g.ce_rp[v], ae = g.ce_rp[v + 1], b = g.se_rp[v], be = g.se_rp[v + 1];
      while (a < ae || b < be) {
        int u;
        bool is_ce;
        if (b >= be || (a < ae && g.ce_col[a] < g.se_col[b])) { u = g.ce_col[a++]; is_ce = true; }
        else { u = g.se_col[b++]; is_ce = false; }
        if (w.hround[u] != -1) continue;
        int lu = w.loc[u];
        if (lu < 0) {
          if (n == kMaxComp) { too_big = true; break; }
          lu = n;
          w.loc[u] = n;
          order[n++] = u;
        }
        if (is_ce) adj |= 1ull << lu; else sadj |= 1ull << lu;
      }
      if (too_big) break;
      adjm[head] = adj;
      sadjm[head] = sadj;
      ++head;
    }
    if (too_big) {
      atomicOr(&ctl->err, kErrComponent);
      atomicMax(&ctl->max_comp, kMaxComp + 1);
      continue;
    }
    unsigned steps;
    bool trunc;
    int cval[kMaxComp];
    if (n <= 32) {
      unsigned a32[32], s32[32];
      for (int i = 0; i < n; ++i) { a32[i] = (unsigned)adjm[i]; s32[i] = (unsigned)sadjm[i]; }
      unsigned bestC[K];
      steps = search_component<K, unsigned>(a32, s32, n, w_stitch, budget, stack.f32, bestC, trunc);
      for (int i = 0; i < n; ++i) {
        int c = 0;
#pragma unroll
        for (int cc = 1; cc < K; ++cc)
          if ((bestC[cc] >> i) & 1u) c = cc;
        cval[i] = c;
      }
    } else {
      unsigned long long bestC[K];
      steps = search_component<K, unsigned long long>(adjm, sadjm, n, w_stitch, budget, stack.f64, bestC, trunc);
      for (int i = 0; i < n; ++i) {
        int c = 0;
#pragma unroll
        for (int cc = 1; cc < K; ++cc)
          if ((bestC[cc] >> i) & 1ull) c = cc;
        cval[i] = c;
      }
    }
    for (int i = 0; i < n; ++i) colors[order[i]] = cval[i];
    atomicAdd(&ctl->steps, (unsigned long long)steps);
    atomicMax(&ctl->max_comp, n);
    atomicMax(&ctl->max_steps_comp, (int)min(steps, (unsigned)INT_MAX));
    if (trunc) atomicAdd(&ctl->truncated, 1);
  }
}

}  // namespace

cudaError_t launch_search(const GraphView& g, Workspace ws, int k, int w_stitch, long long max_steps, int* colors,
                          cudaStream_t s, int blocks, int threads) {
  switch (k) {
    case 2: mpld_exact_cover_search<2><<<blocks, threads, 0, s>>>(g, ws, w_stitch, max_steps, colors); break;
    case 3: mpld_exact_cover_search<3><<<blocks, threads, 0, s>>>(g, ws, w_stitch, max_steps, colors); break;
    case 4: mpld_exact_cover_search<4><<<blocks, threads, 0, s>>>(g, ws, w_stitch, max_steps, colors); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

int resident_blocks_search(int threads, int num_sms) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mpld_exact_cover_search<4>, threads, 0);
  return per_sm * num_sms;
}

}  // namespace mpld
