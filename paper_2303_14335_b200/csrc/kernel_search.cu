// The exact-cover search of PAPER.md §2.3 / Alg. 1 on bit-packed matrices.
//
// One thread owns one component (n <= 64 vertices).  The exact-cover matrix
// (rows r(v,c), primary columns = vertices, secondary columns = (e,c) for
// e in CE) is never materialised as a 0/1 array: with columns = bit positions
// of a 64-bit word it is fully described by, per vertex v,
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
// Cover/uncover (Eq. 2) become mask AND/OR on a 16-byte stack frame per level.
// The search order, bound and budget are DESIGN.md R4-R7, identical to the
// oracle's dancing-links Algorithm X, so the result is bit-identical.
#include <climits>

#include "mpld_internal.cuh"

namespace mpld {

namespace {

struct __align__(16) Frame {
  unsigned long long savedB;  // B[c] before r(v,c) was selected
  int cost;                   // cost when the node was entered
  int packed;                 // v | (c+1) << 8 | (maxused+1) << 16
};

template <int K>
__device__ __forceinline__ unsigned long long pick(const unsigned long long (&a)[K], int c) {
  unsigned long long r = a[0];
#pragma unroll
  for (int i = 1; i < K; ++i) r = (c == i) ? a[i] : r;
  return r;
}

template <int K>
__device__ __forceinline__ void put(unsigned long long (&a)[K], int c, unsigned long long x) {
#pragma unroll
  for (int i = 0; i < K; ++i)
    if (c == i) a[i] = x;
}

// Relaxed Algorithm X with branch and bound (R4-R7).  Returns the
// best masks in bestC; steps and truncation through references.
template <int K>
__device__ void search_component(const ulonglong2* __restrict__ am, int n, int w_stitch, long long max_steps,
                                 Frame* __restrict__ stack, unsigned long long (&bestC)[K], long long& steps_out,
                                 bool& truncated) {
  unsigned long long C[K], B[K];
#pragma unroll
  for (int c = 0; c < K; ++c) { C[c] = 0ull; B[c] = 0ull; bestC[c] = 0ull; }
  unsigned long long U = (n == 64) ? ~0ull : ((1ull << n) - 1ull);
  int cost = 0, maxused = -1, depth = 0;
  int best = INT_MAX;
  long long steps = 0;
  truncated = false;
  bool enter = true;
  while (true) {
    if (enter) {
      ++steps;
      if (best != INT_MAX && max_steps > 0 && steps > max_steps) { truncated = true; break; }
      if (U == 0ull) {  // Alg. 1 line 5: every column covered -> a solution
        if (cost < best) {
          best = cost;
#pragma unroll
          for (int c = 0; c < K; ++c) bestC[c] = C[c];
        }
      } else {
        // column-count reduction, bit-sliced over all 64 columns at once
        unsigned long long s1 = 0ull, s2 = 0ull;
#pragma unroll
        for (int c = 0; c < K; ++c) {
          const unsigned long long F = U & ~B[c];  // live rows of mask c
          s2 |= s1 & F;
          s1 |= F;
        }
        const unsigned long long Z = U & ~s1;  // columns with no live row
        const unsigned long long O = s1 & ~s2; // columns with exactly one live row
        if (cost + kCostUnits * __popcll(Z) < best) {  // bound (R7)
          const unsigned long long cand = Z ? Z : (O ? O : U);  // Alg. 1 line 8 (R5)
          const int v = __ffsll((long long)cand) - 1;
          Frame f;
          f.savedB = 0ull;
          f.cost = cost;
          f.packed = v | ((maxused + 1) << 16);  // c = -1 (stored as 0)
          stack[depth] = f;
          U &= ~(1ull << v);  // cover column v (line 9)
          ++depth;
        }
      }
    }
    if (depth == 0) break;
    Frame f = stack[depth - 1];
    const int v = f.packed & 0xff;
    const int cprev = ((f.packed >> 8) & 0xff) - 1;
    const int mu = ((f.packed >> 16) & 0xff) - 1;
    const unsigned long long bit = 1ull << v;
    if (cprev >= 0) {  // uncover the previous row (line 17)
      put<K>(C, cprev, pick<K>(C, cprev) & ~bit);
      put<K>(B, cprev, f.savedB);
    }
    const int c = cprev + 1;
    if (c > min(K - 1, mu + 1)) {  // rows exhausted (colour-symmetry limit R6): uncover column (line 20)
      U |= bit;
      --depth;
      enter = false;
      continue;
    }
    const ulonglong2 a = am[v];
    const unsigned long long Cc = pick<K>(C, c);
    const unsigned long long Bc = pick<K>(B, c);
    const int inc = kCostUnits * __popcll(a.x & Cc) + w_stitch * __popcll(a.y & ~U & ~Cc);
    f.savedB = Bc;
    f.packed = v | ((c + 1) << 8) | ((mu + 1) << 16);
    stack[depth - 1] = f;
    put<K>(C, c, Cc | bit);  // select r(v,c) (line 14) and cover its secondary columns (line 15)
    put<K>(B, c, Bc | a.x);
    cost = f.cost + inc;
    maxused = max(mu, c);
    enter = true;
  }
  steps_out = steps;
}

template <int K>
__global__ void __launch_bounds__(128) mpld_exact_cover_search(GraphView g, Workspace w, int w_stitch,
                                                               long long max_steps, int* colors) {
  Control* ctl = w.ctl;
  const int n_comp = __ldcg(&ctl->n_comp);
  int order[kMaxComp];
  ulonglong2 am[kMaxComp];
  Frame stack[kMaxComp];
  while (true) {
    const int ci = atomicAdd(&ctl->next_comp, 1);
    if (ci >= n_comp) break;
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
      am[head] = make_ulonglong2(adj, sadj);
      ++head;
    }
    if (too_big) {
      atomicOr(&ctl->err, kErrComponent);
      atomicMax(&ctl->max_comp, kMaxComp + 1);
      continue;
    }
    unsigned long long bestC[K];
    long long steps;
    bool trunc;
    search_component<K>(am, n, w_stitch, max_steps, stack, bestC, steps, trunc);
    for (int i = 0; i < n; ++i) {
      int c = 0;
#pragma unroll
      for (int cc = 1; cc < K; ++cc)
        if ((bestC[cc] >> i) & 1ull) c = cc;
      colors[order[i]] = c;
    }
    atomicAdd(&ctl->steps, (unsigned long long)steps);
    atomicMax(&ctl->max_comp, n);
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
