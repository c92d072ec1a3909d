// Internal declarations of the MPLD CUDA library (not part of the C ABI).
//
// Data layout in HBM:
//   graph     : caller's CSR arrays (int32), read-only.
//   per vertex: deg, hround, prio (int32), bmask (u64) — indexed by vertex id
//   queues    : q0, q1 (int32 [n]) — simplification frontiers, then recovery levels
//   seeds     : roots (int32 [n])
//   component pool (filled by the discovery kernel, one record per component):
//               crec (u64 [n]) = pool offset << 8 | size; pmask (u64 [2n]) = adj/sadj
//               words of every component vertex in BFS column order (R5),
//               interleaved; porder (int32 [n]) = their vertex ids
//   heavy list: hcomp, hcost (int32 [n]) — exact mode's warp-parallel components
//   Control   : one control block (counters, barrier arrivals, error bits,
//               diagnostics) per context, zeroed at the start of every call.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "mpld.h"

namespace mpld {

constexpr int kMaxComp = MPLD_MAX_COMPONENT;  // one 64-bit word per mask
constexpr int kCostUnits = MPLD_COST_UNITS;

enum ErrBits : int { kErrGraph = 1, kErrComponent = 2 };

// Device-resident control block, zeroed by one memset node at the start of
// every call (before the optional validation kernel).
// Counters that are hit by atomics from many warps in the same kernel sit on
// their own 128-byte lines (one L2 slice each), away from the polled barrier
// counters and from each other.
struct Control {
  int n_rounds;     // simplification rounds R (R8)
  int n_hidden;     // |hidden vertices|
  int n_seed;       // component-search seeds listed in roots[]
  int err;          // ErrBits
  int done_blocks;  // last-block detection of the evaluation kernel
  int done_recover; // last-block detection of the recovery kernel (finalisation)
  int n_levels;     // recovery levels (DAG depth + 1)
  alignas(128) int qcnt[3];  // simplification frontier sizes (rotating by round)
  int rq[3];                 // recovery level sizes (rotating by level)
  int tcnt[3];               // ... the same, for the single-CTA tails (never read by other CTAs)
  int trq[3];
  alignas(128) unsigned bar0;  // grid-barrier arrival counter of mpld_simplify_components
  alignas(128) unsigned bar1;  // ... of mpld_recover
  alignas(128) unsigned bar0g; // group barriers (the first kGroup CTAs) of the two kernels
  alignas(128) unsigned bar1g;
  alignas(128) int tovf[2];    // recovery cluster tail: ready vertices spilled to global memory per level parity
  alignas(128) int n_comp;     // components found (counted by the discovery kernel)
  int max_comp;                // largest component
  alignas(128) int truncated;  // components whose search hit max_steps
  int max_steps_comp;          // largest per-component step count
  unsigned long long steps;    // search nodes entered
  unsigned long long steps_heavy;  // ... by the warp-parallel (heavy) search
  alignas(128) int n_heavy[2]; // exact mode: components handed to the warp-parallel search, per word class
                               // (32-bit: hcomp[0..), 64-bit: hcomp[n-1], hcomp[n-2], ...; reset per search call)
  int slot_next;               // spilled-component slots handed out (reset with n_heavy)
  int may_spill;               // a heavy component of >= kHelpersMinN vertices was handed off: idle heavy
                               // warps stay for spilled work instead of leaving (reset with n_heavy)
  int n_wide;                  // components of > 32 vertices listed for the 64-bit lane kernel (reset with n_heavy)
  alignas(128) int heavy_next[2];  // exact mode: next heavy component to take per word class (reset with n_heavy)
  alignas(128) int wq_head[2];     // spilled work items (a ring per word class): positions claimed by consumers
  alignas(128) int wq_tail[2];     // ... positions reserved by producers (polled)
  int wq_done[2];                  // work units (heavy components + items) finished per word class (polled)
  alignas(128) int wq_read[2];     // ... items copied out by their consumers (ring slots free again)
  int spill_refused;               // spills refused (ring full or no slot left): those units ran on alone
  alignas(128) int heavy_finished; // set by the unit that finishes the last pending work: waiting warps leave
  alignas(128) unsigned long long comp_pool;  // components << 32 | pool words used by this search call (reset with n_heavy)
  alignas(128) unsigned long long vh[4];  // validation: symmetry hashes (CE forward / transposed, SE forward / transposed)
  unsigned long long t[16];  // diagnostics: %globaltimer at phase boundaries (ns)
  unsigned long long tr[32];  // diagnostics: per round / level start time (ns)
  int nr[32];                // diagnostics: per round / level frontier size
  alignas(128) unsigned long long dbg[8];  // diagnostics (MPLD_DIAG builds): slowest discovery / search / heavy search
  // the fused tile pipeline (kernel_tile.cu; its own Control block)
  alignas(128) int tile_next;  // next tile to take (dynamic tile assignment)
  alignas(128) int n_pending;  // sub-tiles whose recovery waits for the heavy / wide search (w.q0 / w.q1)
  int done_tiles;              // last-CTA detection of the finish launch
  int finish_next;             // next pending sub-tile of the finish launch
  alignas(128) unsigned long long comp_pool_tile;  // components << 32 | pool words of the tiles' own searches
                                                   // (taken from the top of the pool; comp_pool: deferred ones)
  alignas(128) int piece_cursor;  // piece order: positions handed out to pieces
  alignas(128) unsigned bar_piece;  // grid-barrier arrivals of mpld_piece_order
  alignas(128) int gate;       // 1: the tile pipeline could not take the input (a piece not closed inside
                               // its tile's window, a window over capacity, invalid input): the
                               // whole-graph pipeline runs after it and rewrites every output
};

#ifndef MPLD_DIAG
#define MPLD_DIAG 0  // per-warp diagnostics atomics (tools/kernel_times.py); off in production builds
#endif

// Grid-wide barrier for the cooperatively launched persistent kernels.  Each
// CTA arrives once per barrier on a monotonically increasing counter and polls
// it with relaxed loads (no L1 invalidation inside the spin loop; one fence on
// each side), so a barrier costs one L2 atomic per CTA plus the polling latency.
struct GridBarrier {
  unsigned* count;
  unsigned nblocks;
  unsigned epoch;
  __device__ __forceinline__ GridBarrier(unsigned* c) : count(c), nblocks(gridDim.x), epoch(0) {}
  __device__ __forceinline__ GridBarrier(unsigned* c, unsigned nb) : count(c), nblocks(nb), epoch(0) {}
  // a counter that is not reset between launches: this launch's barriers continue at epoch0
  __device__ __forceinline__ GridBarrier(unsigned* c, unsigned nb, unsigned epoch0)
      : count(c), nblocks(nb), epoch(epoch0) {}
  __device__ __forceinline__ void sync() {
    __syncthreads();
    if (threadIdx.x == 0) {
      ++epoch;
      __threadfence();
      atomicAdd(count, 1u);
      const unsigned target = epoch * nblocks;
      unsigned cur;
      do {
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(count) : "memory");
      } while ((int)(cur - target) < 0);
      __threadfence();
    }
    __syncthreads();
  }
};

struct GraphView {
  int n;
  int n_layouts;
  const int* layout_off;  // [n_layouts+1]
  const int* ce_rp;
  const int* ce_col;
  const int* se_rp;
  const int* se_col;
};

constexpr int kScanTile = 8192;  // elements per block of the partition scan (1024 threads x 8)

// Estimated search cost of a component of n vertices for the cost-balanced
// shard partition (north_star: size x k^n), capped at 2^32 so that the prefix
// sum over any n < 2^31 vertices stays below 2^63 (no wrap-around).
constexpr unsigned long long kEstimateCap = 1ull << 32;
__host__ __device__ __forceinline__ unsigned long long partition_estimate(int n, int k) {
  unsigned long long e = (unsigned long long)n;
  for (int i = 0; i < n && e < kEstimateCap; ++i) e *= (unsigned long long)k;
  return e < kEstimateCap ? e : kEstimateCap;
}

// Exact mode, spilled heavy searches (kernel_search.cu): a warp whose search
// of one component runs long hands its open work to all heavy warps as work
// items (node states); a slot per spilled component gathers the best key.
constexpr int kWQCap = 1 << 16;  // ring slots of spilled work items per word class
#ifndef MPLD_HELPERS_MIN_N
#define MPLD_HELPERS_MIN_N 12
#endif
constexpr int kHelpersMinN = MPLD_HELPERS_MIN_N;  // heavy components this large may run long enough to spill
constexpr int kSlots = 1024;     // spilled components per call
struct WorkItem {
  int slot, depth, cost, mu;
  unsigned long long pa, pb;  // path (2 bits per level, level 0 most significant)
  unsigned long long C[4], B[4], U;
  unsigned long long pad;
};
struct HeavySlot {
  int lock, pend;             // spin lock of the key; work units of the component not finished
  int cost, lcost;            // best key found, the light phase's key (their costs)
  int bcost, pad0;            // the best cost known (atomicMin, read without the lock: pruning)
  unsigned long long pa, pb, lpa, lpb;
  unsigned long long C[4];    // colour masks of the best leaf
  int ci, ncl;                // component (pool record); its clique partition (R7 bound) for the items:
  unsigned long long cl[16];  // computed once by the spilling unit instead of once per item
};

struct Workspace {
  int* deg;        // live conflict degree (simplification), then the recovery state of a hidden vertex:
                   // uncoloured hidden predecessors | popped-before bits << 8 (kernels_graph.cu kPackedPred)
  int* hround;     // -1 kept, else the round the vertex was hidden in
  unsigned long long* bmask;  // recovery, unpacked variant only (MPLD_PACKED_PRED=0): bit t = CE entry t of the
                              // row pops before the vertex (or is kept)
  unsigned* prio;  // lowbias32(layout-local id), recovery priority (R9)
  int* q0;         // frontier queues (double-buffered)
  int* q1;
  int* roots;      // component-search seeds (kept vertices without a smaller kept neighbour)
  unsigned long long* crec;   // component records: pool offset << 8 | size
  unsigned long long* pmask;  // component pool: adj, sadj word pairs in BFS column order
  int* porder;                // component pool: vertex ids in BFS column order
  int* hcomp;      // heavy components (exact mode): component index ...
  int* hcost;      // ... and the light phase's best cost
  int* wide;       // components of > 32 vertices (pool index), searched by the 64-bit lane kernel
  Control* ctl;
  WorkItem* wq;    // [2][kWQCap] spilled work items per word class (rings)
  unsigned long long* wq_flag;  // [2][kWQCap] == epoch << 32 | position once the item at that position is written
  HeavySlot* hslot;   // [kSlots]
  unsigned long long* est;   // [n] sharded search: estimated search cost of the component rooted at v, then
                             // its inclusive prefix sum over vertex ids (the balanced partition)
  unsigned long long* bsum;  // [n / kScanTile + 2] block sums of that scan
  unsigned epoch;     // this search call's tag for wq_flag
  unsigned spill_iters;  // a heavy unit's iterations before it may spill (multiple of 64; MPLD_HEAVY_SPILL)
  int tail_slots;        // cluster tails: frontier slots per CTA in use (MPLD_TAIL_SLOTS lowers it: tests)
  int* build_err;        // set when a CSR built on the device (upper-triangle upload) saw bad input; the
                         // simplification turns it into MPLD_ERR_GRAPH and clears it
  long long diag_cap;    // u64 entries of est usable by diagnostics (MPLD_DIAG_HEAVY builds)
  unsigned greedy_salt;  // heavy search: seed offset of the greedy starting colourings (MPLD_GREEDY_SALT)
  int greedy_rounds;     // heavy search: rounds of 32 greedy colourings (MPLD_GREEDY_ROUNDS, default 1)
  const int* gate;       // whole-graph kernels after the tile pipeline: run only if *gate != 0 (nullptr:
                         // always run)
  // the tile pipeline's piece order (kernel_tile.cu mpld_piece_order), [n] each
  int* t_par;   // union-find: parent - v (0 = root)
  int* t_cnt;   // piece size at its root (then the positions still to hand out)
  int* t_end;   // end position of the piece, at its root
  int* t_pos;   // vertex -> position (pieces contiguous)
  int* t_perm;  // position -> vertex
  int* t_pend;  // position -> end position of its piece
};

// The whole-graph kernels return at once when they follow the tile pipeline
// and it took the input (every thread of the grid reads the same word).
__device__ __forceinline__ bool gated_off(const Workspace& w) {
  return w.gate != nullptr && *(volatile const int*)w.gate == 0;
}

// Layout of vertex v: the l with layout_off[l] <= v < layout_off[l+1] (binary
// search; the offsets are tiny and stay in L1).
__device__ __forceinline__ int layout_of(const GraphView& g, int v) {
  int a = 0, b = g.n_layouts;
  while (b - a > 1) {
    const int m = (a + b) >> 1;
    if (__ldg(&g.layout_off[m]) <= v) a = m; else b = m;
  }
  return a;
}

// Eq. (1) outputs: per-layout (n_conflicts, n_stitches) accumulated by the
// search kernels (counts), the cost and the statistics written at the end of
// the recovery (enabled) or by the evaluation kernel.
struct Outputs {
  long long* counts;  // [2 * n_layouts]
  double* cost;       // [n_layouts]
  long long* stats;   // [MPLD_STAT_LEN] or null
  double alpha;
  int launches;
  int enabled;
  int cluster_tail;  // the last levels run on mpld_recover_tail (set by launch_recover)
};

// 32-bit counter-based mix (a bijection), recovery priority of DESIGN.md R9.
__host__ __device__ __forceinline__ uint32_t lowbias32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

// Programmatic dependent launch (PDL): a kernel launched with the attribute
// may be scheduled while its predecessor in the stream drains; it triggers
// its own dependents and waits for its predecessor's memory at its first
// statement (both no-ops without the attribute).
__device__ __forceinline__ void pdl_begin() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

bool pdl_enabled();         // MPLD_PDL=0 disables it (A/B measurements)
void set_pdl(bool enable);

template <typename... KArgs, typename... Args>
cudaError_t launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl,
                      bool coop, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  unsigned na = 0;
  if (pdl && pdl_enabled()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (coop) {
    at[na].id = cudaLaunchAttributeCooperative;
    at[na].val.cooperative = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

__host__ __device__ __forceinline__ unsigned long long wq_tag(unsigned epoch, int pos) {
  return ((unsigned long long)epoch << 32) | (unsigned)pos;
}

// launch wrappers (kernels_graph.cu, kernel_search.cu); each returns the
// cudaError_t of its launch.  `pdl`: the stream's previous operation is one
// of these kernels.
cudaError_t launch_simplify_components(const GraphView& g, Workspace ws, int k, int* colors,
                                       long long* counts, int validate, cudaStream_t s, int blocks, int threads,
                                       int separate_prep);
// the recovery's share of the final pass (separate_prep above), on a second stream
cudaError_t launch_recover_prep(const GraphView& g, Workspace ws, cudaStream_t s, int blocks, int threads);
cudaError_t launch_discover(const GraphView& g, Workspace ws, int k, int sharded, cudaStream_t s, int blocks, bool pdl);
cudaError_t launch_partition_scan(const GraphView& g, Workspace ws, cudaStream_t s);  // inclusive scan of ws.est
cudaError_t launch_search(const GraphView& g, Workspace ws, int k, int w_stitch, long long max_steps, int* colors,
                          unsigned light_steps, long long* counts, int shard_index, int shard_count, cudaStream_t s,
                          int blocks, bool pdl);
constexpr unsigned kLightStepsDefault = 48;  // exact mode: one-lane budget before a component turns heavy
// the components of > 32 vertices the light kernel listed, one per lane on 64-bit words
cudaError_t launch_search_wide(const GraphView& g, Workspace ws, int k, int w_stitch, long long max_steps,
                               int* colors, unsigned light_steps, long long* counts, cudaStream_t s, int blocks);
cudaError_t configure_search_wide(int num_sms, int* blocks);
cudaError_t launch_search_heavy(const GraphView& g, Workspace ws, int k, int w_stitch, int* colors, long long* counts,
                                cudaStream_t s, const int* blocks, bool pdl);
cudaError_t configure_search_heavy(int num_sms, int* blocks);  // blocks[3]: resident grids of the heavy kernels (k = 2..4)
cudaError_t launch_recover(const GraphView& g, Workspace ws, int k, int* colors, Outputs out, cudaStream_t s,
                           int blocks, int threads, bool pdl);
// One cooperative launch building on the device the symmetric CE CSR from its
// upper triangle (deg_up != NULL) and / or the SE CSR from stitch pairs
// (m_se >= 0): see kernels_graph.cu mpld_graph_build.
struct GraphBuild {
  int n;
  int m_up;                    // upper-triangle entries (deg_up != NULL)
  const unsigned char* deg_up;
  const int* col_up;
  int* ce_rp;                  // [n+1] out
  int* ce_col;                 // [2 m_up] out
  int m_se;                    // stitch pairs (-1: no SE build)
  const int* se_pairs;
  int* se_rp;                  // [n+1] out
  int* se_col;                 // [2 m_se] out
  int* rp_up;                  // [n+1] scratch
  int* cnt_ce;                 // [n] scratch: row lengths, CE | SE << 24
  int* fill_ce;                // [n] scratch: entries placed, CE | SE << 24
  int* tot;                    // [3 * blocks] scratch: per-CTA sums
  int* err;                    // set on invalid input (Workspace::build_err)
  unsigned* bar;               // grid-barrier counter (zeroed before the launch)
  unsigned epoch0;             // barriers already counted on it (0)
};
constexpr unsigned kBuildBarriers = 5;  // grid barriers per mpld_graph_build launch
cudaError_t launch_graph_build(const GraphBuild& b, cudaStream_t s, int blocks);
int coop_blocks_build(int num_sms);

// The fused tile pipeline (kernel_tile.cu).  finish = 0: every tile
// (simplification, sub-graphs, light search, recovery); finish = 1: the
// recovery of the sub-tiles whose components went to the heavy / wide search,
// then the Eq. (1a) costs and statistics (last CTA).  `launches` is the call's
// kernel count for MPLD_STAT_LAUNCHES.
struct TileLaunch {
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
  int finish;
};
cudaError_t configure_tile();
int coop_blocks_piece(int num_sms);
// the piece order of the tile pipeline (cooperative; see kernel_tile.cu)
cudaError_t launch_piece_order(const GraphView& g, const Workspace& w, cudaStream_t s, int blocks);
int resident_blocks_tile(int num_sms);
cudaError_t launch_tile(const GraphView& g, const Workspace& w, int k, const TileLaunch& t, cudaStream_t s,
                        int blocks, bool pdl);
bool recover_tail_available();  // the cluster tail kernel can be launched (cluster size support)
int simplify_launches();        // kernels launch_simplify_components enqueues (1, or 3 with the cluster tail)
cudaError_t configure_recover_tail();
cudaError_t launch_evaluate(const GraphView& g, Workspace ws, const int* colors, double alpha,
                            long long* counts, double* cost, long long* stats, int launches,
                            cudaStream_t s, int blocks);

// sharded runs: compact (vertex, colour) list of the colours a shard's search wrote, and its scatter
cudaError_t launch_shard_export(int n, const int* colors, int* pairs, unsigned long long* count, cudaStream_t s,
                                int blocks);
cudaError_t launch_shard_import(long long m, const int* pairs, int n, int* colors, cudaStream_t s, int blocks);

// occupancy helpers for the cooperative (persistent) kernels
int coop_blocks_simplify(int threads, int num_sms);
int coop_blocks_recover(int threads, int num_sms);
int resident_blocks_search(int threads, int num_sms);
int resident_blocks_discover(int num_sms);
int resident_blocks_evaluate(int num_sms);

}  // namespace mpld
