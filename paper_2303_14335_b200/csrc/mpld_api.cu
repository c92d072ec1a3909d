// C ABI of include/mpld.h: contexts, device workspace, host entry points and
// the launch sequence of the hot path.
//
// Launch sequence of one call (all on one stream, no host synchronisation):
//   mpld_simplify_components   cooperative: validation, simplification rounds, seeds,
//                              recovery pop keys and level 0
//   mpld_component_discover    one warp per seed: components -> pool of bit-packed matrices
//   mpld_exact_cover_search<K> one component of <= 32 vertices per lane (32-bit words)
//   mpld_exact_cover_search_wide<K> one component of > 32 vertices per lane (64-bit words)
//   mpld_exact_cover_search_heavy<K,W> (exact mode) one warp per heavy component, one launch
//                              per word class (32-bit: n <= 32, 64-bit: n > 32)
//   mpld_recover_prep          (second stream, beside discovery and search) recovery
//                              predecessor counts and level 0
//   mpld_recover               cooperative: LIFO recovery of hidden vertices (large levels)
//   mpld_recover_tail          one thread-block cluster: the last levels, Eq. (1a) costs, stats
//   mpld_evaluate              only after a sharded search: Eq. (1) per layout + stats
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "mpld_internal.cuh"

using namespace mpld;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(MPLD_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

enum KernelId { K_SIMPLIFY = 0, K_DISCOVER, K_SEARCH, K_SEARCH_HEAVY, K_RECOVER, K_EVALUATE, K_PREP, K_SEARCH_WIDE,
                K_BUILD, K_TILE, K_TILE_FINISH, K_PIECES, K_COUNT };
const char* kKernelNames[K_COUNT] = {"mpld_simplify_components", "mpld_component_discover",
                                     "mpld_exact_cover_search", "mpld_exact_cover_search_heavy", "mpld_recover",
                                     "mpld_evaluate", "mpld_recover_prep", "mpld_exact_cover_search_wide",
                                     "mpld_graph_build", "mpld_tile_decompose", "mpld_tile_finish",
                                     "mpld_piece_order"};

constexpr int kCoopThreads = 1024;
#ifndef MPLD_SEPARATE_PREP
#define MPLD_SEPARATE_PREP 1
#endif

}  // namespace

// One staging slot of the asynchronous host entry point: device copies of a
// batch's inputs and outputs, pinned host copies of the outputs that need
// post-processing, and the events that order upload -> compute -> download.
// Three staging slots: the upload of submit t+1 never waits for the download
// of submit t-1 (with two, the slot reuse chained upload, compute and download
// of consecutive submits).
constexpr int kAsyncSlots = 3;

struct AsyncSlot {
  int* lo = nullptr;
  int* ce_rp = nullptr;
  int* ce_col = nullptr;
  int* se_rp = nullptr;
  int* se_col = nullptr;
  int* se_pairs = nullptr;  // stitch edges as pairs (the pairs entry point)
  unsigned char* up_deg = nullptr;  // conflict edges as the upper triangle (the upper entry point)
  int* up_col = nullptr;
  int64_t cap_up = -1, cap_up_n = -1;
  int* colors = nullptr;
  long long* counts = nullptr;
  double* cost = nullptr;
  long long* stats = nullptr;
  int64_t cap_n = -1, cap_ce = -1, cap_se = -1, cap_pairs = -1;
  int32_t cap_l = -1;
  long long* h_counts = nullptr;  // pinned
  long long* h_stats = nullptr;   // pinned [MPLD_STAT_LEN]
  cudaEvent_t ev_h2d = nullptr, ev_comp = nullptr, ev_d2h = nullptr;
  int64_t ticket = -1;      // submit in flight (or last submitted)
  bool pending = false;     // its results still need post-processing
  int64_t fin_ticket = -1;  // last post-processed submit and its return code
  int fin_rc = MPLD_OK;
  int32_t n_layouts = 0;    // user outputs of the submit in flight
  int64_t* u_nc = nullptr;
  int64_t* u_ns = nullptr;
  int64_t* u_stats = nullptr;
};

struct mpld_context {
  int device = 0;
  int num_sms = 0;
  int64_t cap_n = 0;
  int32_t cap_layouts = 0;
  // workspace
  int* deg = nullptr;
  int* hround = nullptr;
  unsigned* prio = nullptr;
  unsigned long long* bmask = nullptr;
  int* q0 = nullptr;
  int* q1 = nullptr;
  int* roots = nullptr;
  unsigned long long* crec = nullptr;
  unsigned long long* pmask = nullptr;
  int* porder = nullptr;
  int* hcomp = nullptr;
  int* hcost = nullptr;
  int* wide = nullptr;
  int* t_par = nullptr;  // the tile pipeline's piece order (Workspace::t_*)
  int* t_cnt = nullptr;
  int* t_end = nullptr;
  int* t_pos = nullptr;
  int* t_perm = nullptr;
  int* t_pend = nullptr;
  int blocks_piece = 0;
  unsigned greedy_salt = 0;  // MPLD_GREEDY_SALT (experiments)
  int greedy_rounds = 1;     // MPLD_GREEDY_ROUNDS
  WorkItem* wq = nullptr;     // spilled heavy-search work (fixed size)
  unsigned long long* wq_flag = nullptr;
  HeavySlot* hslot = nullptr;
  unsigned long long* est = nullptr;   // sharded search: cost-balanced partition (cap_n)
  unsigned long long* bsum = nullptr;
  unsigned epoch = 0;         // search calls so far (tags wq_flag)
  unsigned spill_iters = 256; // heavy-search spill threshold; MPLD_HEAVY_SPILL overrides (tests of the spill path)
  int tail_slots = 1 << 30;   // cluster-tail frontier slots per CTA (capped at the kernel's); MPLD_TAIL_SLOTS lowers it
  Control* ctl = nullptr;       // the whole-graph pipeline's control block (ctl[0])
  Control* ctl_tile = nullptr;  // the tile pipeline's (ctl[1]; one allocation, one reset per call)
  int blocks_tile = 0;
  bool gate_active = false;  // enqueuing the whole-graph kernels behind the tile pipeline (Workspace::gate)
  bool last_tiles = false;   // the last call ran the tile pipeline (diagnostics read its control block)
  // phase-split calls: the prepared graph
  GraphView g{};
  int k = 0;
  bool prepared = false;
  int call_launches = 0;
  unsigned light_steps = kLightStepsDefault;  // MPLD_LIGHT_STEPS overrides (tuning)
  int blocks_simplify = 0, blocks_recover = 0, blocks_search = 0, blocks_stream = 0, blocks_discover = 0;
  int blocks_heavy[3] = {0, 0, 0};  // per k = 2..4
  int blocks_wide = 0;                        // the 64-bit lane kernel
  long long* counts = nullptr;  // the prepare phase's d_counts (zeroed by the simplification kernel)
  bool search_counted = false;  // the search accumulated the counts (one shard)
  int searches_since_prepare = 0;
  // cross-stream ordering: calls share the workspace and control block, so a
  // call enqueued on a stream other than the previous call's waits for that
  // call's last operation (ev_last, recorded at the end of every entry point)
  int* build_err = nullptr;  // device flag of the CSR builds from compact uploads (Workspace::build_err)
  unsigned* build_bar = nullptr;  // grid-barrier counter of mpld_graph_build (zeroed before every build)
  int* build_tot = nullptr;       // [3 * blocks_build] per-CTA sums
  int blocks_build = 0;
  cudaEvent_t ev_last = nullptr;
  cudaStream_t last_stream = nullptr;
  bool has_last = false;
  // the recovery's share of the final pass runs on `aux` beside the search
  // (forked after the simplification, joined before the recovery)
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int blocks_prep = 0;
  bool prep_forked = false;
  // host-API staging (device copies of host inputs / outputs)
  int64_t cap_ce = 0, cap_se = 0, cap_stage_n = 0;
  int32_t cap_stage_layouts = 0;  // own capacity: ensure_workspace() grows cap_layouts first
  int* h_lo = nullptr;
  int* h_ce_rp = nullptr;
  int* h_ce_col = nullptr;
  int* h_se_rp = nullptr;
  int* h_se_col = nullptr;
  int* h_colors = nullptr;
  long long* h_counts = nullptr;
  double* h_cost = nullptr;
  long long* h_stats = nullptr;
  cudaStream_t stream = nullptr;  // compute stream of the host entry points
  // asynchronous host entry points: kAsyncSlots staging slots, upload / download streams
  AsyncSlot slot[kAsyncSlots];
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  int64_t next_ticket = 0;
  // timing
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
  double acc_ms[K_COUNT] = {0};
  int64_t launches[K_COUNT] = {0};
  std::mutex mu;
};

namespace {

template <typename T>
cudaError_t grow(T** p, int64_t count) {
  if (*p) cudaFree(*p);
  *p = nullptr;
  return cudaMalloc((void**)p, sizeof(T) * (size_t)(count > 0 ? count : 1));
}

int ensure_workspace(mpld_context* ctx, int64_t n, int32_t n_layouts) {
  if (n > ctx->cap_n) {
    int64_t cap = std::max<int64_t>(n, ctx->cap_n * 3 / 2);
    cudaError_t e = cudaSuccess;
    for (int** p : {&ctx->deg, &ctx->hround, &ctx->q0, &ctx->q1, &ctx->roots, &ctx->porder, &ctx->hcomp, &ctx->hcost,
                    &ctx->wide, &ctx->t_par, &ctx->t_cnt, &ctx->t_end, &ctx->t_pos, &ctx->t_perm, &ctx->t_pend}) {
      e = grow(p, cap + 1);  // + 1: q1 is the graph build's [n+1] row-pointer scratch
      if (e != cudaSuccess) return fail(MPLD_ERR_NOMEM, "workspace allocation failed");
    }
    if (grow(&ctx->est, cap) != cudaSuccess || grow(&ctx->bsum, cap / kScanTile + 2) != cudaSuccess)
      return fail(MPLD_ERR_NOMEM, "workspace allocation failed");
    if (grow(&ctx->prio, cap) != cudaSuccess || grow(&ctx->bmask, cap) != cudaSuccess ||
        grow(&ctx->crec, cap) != cudaSuccess || grow(&ctx->pmask, 2 * cap) != cudaSuccess)
      return fail(MPLD_ERR_NOMEM, "workspace allocation failed");
    ctx->cap_n = cap;
  }
  if (n_layouts > ctx->cap_layouts) {
    int32_t cap = std::max<int32_t>(n_layouts, 16);
    ctx->cap_layouts = cap;
  }
  return MPLD_OK;
}

cudaEvent_t take_event(mpld_context* ctx) {
  if (ctx->ev_pool.empty()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  cudaEvent_t e = ctx->ev_pool.back();
  ctx->ev_pool.pop_back();
  return e;
}

struct TimedLaunch {
  mpld_context* ctx;
  int id;
  cudaStream_t s;
  cudaEvent_t a = nullptr, b = nullptr;
  TimedLaunch(mpld_context* c, int i, cudaStream_t st) : ctx(c), id(i), s(st) {
    if (ctx->timing) {
      a = take_event(ctx);
      b = take_event(ctx);
      cudaEventRecord(a, s);
    }
  }
  void done() {
    if (ctx->timing) {
      cudaEventRecord(b, s);
      ctx->pending.push_back({id, {a, b}});
    }
    ctx->launches[id] += 1;
  }
};

int check_scalars(int32_t n, int32_t k, double alpha, int* w_stitch) {
  if (n < 0) return fail(MPLD_ERR_ARG, "n < 0");
  if (k < 2 || k > MPLD_MAX_K) return fail(MPLD_ERR_ARG, "k must be in [2, 4]");
  if (!(alpha >= 0.0 && alpha <= 1000.0)) return fail(MPLD_ERR_ARG, "alpha must be in [0, 1000]");
  double a = alpha * MPLD_COST_UNITS;
  double r = std::nearbyint(a);
  if (std::fabs(a - r) > 1e-6) return fail(MPLD_ERR_ARG, "alpha must be a multiple of 0.001");
  *w_stitch = (int)r;
  return MPLD_OK;
}

// A call on a stream other than the previous call's waits for the previous
// call's last operation (same stream: stream order suffices, and programmatic
// dependent launch between the call's kernels is kept).
int order_after_last(mpld_context* ctx, cudaStream_t s) {
  if (!ctx->has_last || s == ctx->last_stream) return MPLD_OK;
  const cudaError_t e = cudaStreamWaitEvent(s, ctx->ev_last, 0);
  return e == cudaSuccess ? MPLD_OK : cuda_fail(e, "cross-stream ordering");
}

int mark_last(mpld_context* ctx, cudaStream_t s) {
  const cudaError_t e = cudaEventRecord(ctx->ev_last, s);
  if (e != cudaSuccess) return cuda_fail(e, "cross-stream ordering");
  ctx->last_stream = s;
  ctx->has_last = true;
  return MPLD_OK;
}

Workspace workspace(mpld_context* ctx) {
  return Workspace{ctx->deg,   ctx->hround, ctx->bmask,  ctx->prio,  ctx->q0,    ctx->q1,    ctx->roots,
                   ctx->crec,  ctx->pmask,  ctx->porder, ctx->hcomp, ctx->hcost, ctx->wide,  ctx->ctl,   ctx->wq,
                   ctx->wq_flag, ctx->hslot, ctx->est,  ctx->bsum,  ctx->epoch, ctx->spill_iters, ctx->tail_slots,
                   ctx->build_err, ctx->cap_n, ctx->greedy_salt, ctx->greedy_rounds,
                   ctx->gate_active ? &ctx->ctl_tile->gate : nullptr,
                   ctx->t_par, ctx->t_cnt, ctx->t_end, ctx->t_pos, ctx->t_perm, ctx->t_pend};
}

// phase 1: validate?, simplification, components (colours initialised to -1)
int phase_prepare(mpld_context* ctx, cudaStream_t s, const GraphView& g, int k, uint32_t flags, int* colors,
                  long long* counts, bool reset = true) {
  Workspace ws = workspace(ctx);
  ctx->g = g;
  ctx->k = k;
  ctx->counts = counts;
  ctx->search_counted = false;
  ctx->searches_since_prepare = 0;
  ctx->prepared = true;
  ctx->call_launches = 0;
  // the control block (counters, barrier arrivals, error bits) starts every call at zero
  // (behind the tile pipeline: zeroed with its control block at the start of the call)
  cudaError_t e = reset ? cudaMemsetAsync(ctx->ctl, 0, sizeof(Control), s) : cudaSuccess;
  if (e != cudaSuccess) return cuda_fail(e, "control reset");
  TimedLaunch t(ctx, K_SIMPLIFY, s);
  // behind the tile pipeline the recovery's prep runs inside the simplification (no stream fork)
  const int separate_prep = MPLD_SEPARATE_PREP && !ctx->gate_active ? 1 : 0;
  e = launch_simplify_components(g, ws, k, colors, counts, (flags & MPLD_FLAG_VALIDATE) ? 1 : 0, s,
                                 ctx->blocks_simplify, kCoopThreads, separate_prep);
  if (e != cudaSuccess) return cuda_fail(e, "mpld_simplify_components");
  t.done();
  ctx->call_launches += simplify_launches();
  ctx->prep_forked = false;
  if (separate_prep) {  // the recovery's prep beside the search: fork onto the second stream
    e = cudaEventRecord(ctx->ev_fork, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->aux, ctx->ev_fork, 0);
    if (e != cudaSuccess) return cuda_fail(e, "prep fork");
    TimedLaunch tp(ctx, K_PREP, ctx->aux);
    e = launch_recover_prep(g, ws, ctx->aux, ctx->blocks_prep, kCoopThreads);
    if (e != cudaSuccess) return cuda_fail(e, "mpld_recover_prep");
    tp.done();
    e = cudaEventRecord(ctx->ev_join, ctx->aux);
    if (e != cudaSuccess) return cuda_fail(e, "prep join");
    ++ctx->call_launches;
    ctx->prep_forked = true;
  }
  return MPLD_OK;
}

// phase 2: the exact-cover search of this shard's components
int phase_search(mpld_context* ctx, cudaStream_t s, int w_stitch, long long max_steps, int shard_index,
                 int shard_count, int* colors) {
  Workspace ws = workspace(ctx);
  const GraphView& g = ctx->g;
  // the component pool and the heavy queue belong to this search call (several
  // shards may share a context); the first search after prepare finds them zeroed
  // by the call's control reset, so the kernels follow each other directly (PDL)
  const bool pdl = ctx->searches_since_prepare++ == 0;
  if (!pdl) {
    cudaError_t e0 = cudaMemsetAsync(&ctx->ctl->n_heavy, 0,
                                     offsetof(Control, comp_pool) + sizeof(unsigned long long) -
                                         offsetof(Control, n_heavy), s);
    if (e0 != cudaSuccess) return cuda_fail(e0, "search counters reset");
  }
  // one shard: the search kernels accumulate the Eq. (1) counts of the final
  // colourings (the recovery adds no conflict, R9), so the finish
  // phase needs no evaluation pass
  ++ctx->epoch;  // fresh tag for the spilled-work flags of this call
  ws.epoch = ctx->epoch;
  ctx->search_counted = shard_count == 1;
  long long* count = ctx->search_counted ? ctx->counts : nullptr;
  // sharded: every shard discovers all components; a scan of their estimated
  // costs in vertex-id order gives the cost-balanced partition
  const int sharded = shard_count > 1 ? 1 : 0;
  if (sharded) {
    cudaError_t e = cudaMemsetAsync(ws.est, 0, sizeof(unsigned long long) * (size_t)g.n, s);
    if (e != cudaSuccess) return cuda_fail(e, "partition reset");
  }
  {
    TimedLaunch t(ctx, K_DISCOVER, s);
    cudaError_t e = launch_discover(g, ws, ctx->k, sharded, s, ctx->blocks_discover, pdl && !sharded);
    if (e != cudaSuccess) return cuda_fail(e, "mpld_component_discover");
    t.done();
    ++ctx->call_launches;
  }
  if (sharded) {
    cudaError_t e = launch_partition_scan(g, ws, s);
    if (e != cudaSuccess) return cuda_fail(e, "partition scan");
    ctx->call_launches += 3;
  }
  {
    TimedLaunch t(ctx, K_SEARCH, s);
    cudaError_t e = launch_search(g, ws, ctx->k, w_stitch, max_steps, colors, ctx->light_steps, count, shard_index,
                                  shard_count, s, ctx->blocks_search, !sharded);
    if (e != cudaSuccess) return cuda_fail(e, "mpld_exact_cover_search");
    t.done();
    ++ctx->call_launches;
  }
  if (max_steps > 0) {  // budgeted mode: the components of > 32 vertices, one per lane on 64-bit words
                        // (exact mode hands them to the warp-parallel search directly)
    TimedLaunch t(ctx, K_SEARCH_WIDE, s);
    cudaError_t e = launch_search_wide(g, ws, ctx->k, w_stitch, max_steps, colors, ctx->light_steps, count, s,
                                       ctx->blocks_wide);
    if (e != cudaSuccess) return cuda_fail(e, "mpld_exact_cover_search_wide");
    t.done();
    ++ctx->call_launches;
  }
  if (max_steps <= 0) {  // exact mode: heavy components on the warp-parallel search
    TimedLaunch t(ctx, K_SEARCH_HEAVY, s);
    cudaError_t e = launch_search_heavy(g, ws, ctx->k, w_stitch, colors, count, s, ctx->blocks_heavy, true);
    if (e != cudaSuccess) return cuda_fail(e, "mpld_exact_cover_search_heavy");
    t.done();
    ++ctx->call_launches;
  }
  return MPLD_OK;
}

// phase 3: recovery of the hidden vertices and Eq. (1)
int phase_finish(mpld_context* ctx, cudaStream_t s, double alpha, int* colors, long long* counts, double* cost,
                 long long* stats) {
  Workspace ws = workspace(ctx);
  const GraphView& g = ctx->g;
  Outputs out;
  out.counts = counts;
  out.cost = cost;
  out.stats = stats;
  out.alpha = alpha;
  out.enabled = ctx->search_counted && counts == ctx->counts;
  out.cluster_tail = 0;  // set by launch_recover
  if (ctx->prep_forked) {  // join the recovery's prep (second stream)
    cudaError_t e = cudaStreamWaitEvent(s, ctx->ev_join, 0);
    if (e != cudaSuccess) return cuda_fail(e, "prep join");
  }
  if (!out.enabled) {  // the evaluation pass accumulates into counts: start it at zero
    cudaError_t e = cudaMemsetAsync(counts, 0, sizeof(long long) * 2 * (size_t)g.n_layouts, s);
    if (e != cudaSuccess) return cuda_fail(e, "counts reset");
  }
  {
    TimedLaunch t(ctx, K_RECOVER, s);
    ctx->call_launches += recover_tail_available() ? 2 : 1;  // + the cluster tail of the last levels
    out.launches = ctx->call_launches;
    // PDL after the search kernels of the same thread of calls (a sharded run
    // puts an all-reduce between the search and this call)
    cudaError_t e = launch_recover(g, ws, ctx->k, colors, out, s, ctx->blocks_recover, kCoopThreads,
                                   ctx->search_counted && !ctx->prep_forked);
    if (e != cudaSuccess) return cuda_fail(e, "mpld_recover");
    t.done();
  }
  if (!out.enabled) {  // sharded search: the counts come from one pass over the combined colours
    TimedLaunch t(ctx, K_EVALUATE, s);
    cudaError_t e = launch_evaluate(g, ws, colors, alpha, counts, cost, stats, ctx->call_launches + 1, s,
                                    ctx->blocks_stream);
    if (e != cudaSuccess) return cuda_fail(e, "mpld_evaluate");
    t.done();
  }
  ctx->prepared = false;
  return MPLD_OK;
}

// kernels the whole-graph pipeline enqueues for one call
int whole_graph_launches(long long max_steps) {
  (void)max_steps;  // one search kernel after the light one: wide (budgeted) or heavy (exact)
  return simplify_launches() + 3 + (recover_tail_available() ? 2 : 1);
}

// The fused tile pipeline (kernel_tile.cu): tiles -> heavy / wide search ->
// recovery of the pending sub-tiles and the outputs; then the whole-graph
// pipeline, gated: its kernels return at once unless the tiles could not take
// the input, in which case they recompute every output (identical results).
int run_tiles(mpld_context* ctx, cudaStream_t s, const GraphView& g, int k, int w_stitch, double alpha,
              long long max_steps, uint32_t flags, int* colors, long long* counts, double* cost, long long* stats) {
  cudaError_t e = cudaMemsetAsync(ctx->ctl, 0, 2 * sizeof(Control), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(counts, 0, sizeof(long long) * 2 * (size_t)g.n_layouts, s);
  if (e != cudaSuccess) return cuda_fail(e, "control reset");
  ctx->gate_active = false;
  Workspace wt = workspace(ctx);
  wt.ctl = ctx->ctl_tile;
  wt.epoch = ++ctx->epoch;  // fresh tag for the spilled-work flags of this search
  TileLaunch tl{w_stitch, max_steps, ctx->light_steps, colors, counts, cost, stats, alpha,
                5 + whole_graph_launches(max_steps), (flags & MPLD_FLAG_VALIDATE) ? 1 : 0, 0};
  {
    TimedLaunch t(ctx, K_PIECES, s);
    e = launch_piece_order(g, wt, s, ctx->blocks_piece);
    if (e != cudaSuccess) return cuda_fail(e, "mpld_piece_order");
    t.done();
  }
  {
    TimedLaunch t(ctx, K_TILE, s);
    e = launch_tile(g, wt, k, tl, s, ctx->blocks_tile, false);
    if (e != cudaSuccess) return cuda_fail(e, "mpld_tile_decompose");
    t.done();
  }
  {  // the components of windows with more than one lane batch (deferred by the tiles)
    TimedLaunch t(ctx, K_SEARCH, s);
    e = launch_search(g, wt, k, w_stitch, max_steps, colors, ctx->light_steps, counts, 0, 1, s, ctx->blocks_search,
                      true);
    if (e != cudaSuccess) return cuda_fail(e, "mpld_exact_cover_search");
    t.done();
  }
  if (max_steps > 0) {
    TimedLaunch t(ctx, K_SEARCH_WIDE, s);
    e = launch_search_wide(g, wt, k, w_stitch, max_steps, colors, ctx->light_steps, counts, s, ctx->blocks_wide);
    if (e != cudaSuccess) return cuda_fail(e, "mpld_exact_cover_search_wide");
    t.done();
  } else {
    TimedLaunch t(ctx, K_SEARCH_HEAVY, s);
    e = launch_search_heavy(g, wt, k, w_stitch, colors, counts, s, ctx->blocks_heavy, true);
    if (e != cudaSuccess) return cuda_fail(e, "mpld_exact_cover_search_heavy");
    t.done();
  }
  tl.finish = 1;
  {
    TimedLaunch t(ctx, K_TILE_FINISH, s);
    e = launch_tile(g, wt, k, tl, s, ctx->blocks_tile, true);
    if (e != cudaSuccess) return cuda_fail(e, "mpld_tile_finish");
    t.done();
  }
  ctx->gate_active = true;
  int rc = phase_prepare(ctx, s, g, k, flags, colors, counts, false);
  if (rc == MPLD_OK) rc = phase_search(ctx, s, w_stitch, max_steps, 0, 1, colors);
  if (rc == MPLD_OK) rc = phase_finish(ctx, s, alpha, colors, counts, cost, stats);
  ctx->gate_active = false;
  if (rc == MPLD_OK) rc = mark_last(ctx, s);
  ctx->last_tiles = true;
  return rc;
}

int run_pipeline(mpld_context* ctx, cudaStream_t s, const GraphView& g, int k, int w_stitch, double alpha,
                 long long max_steps, uint32_t flags, int* colors, long long* counts, double* cost,
                 long long* stats) {
  if (flags & MPLD_FLAG_TILES)
    return run_tiles(ctx, s, g, k, w_stitch, alpha, max_steps, flags, colors, counts, cost, stats);
  ctx->last_tiles = false;
  int rc = phase_prepare(ctx, s, g, k, flags, colors, counts);
  if (rc == MPLD_OK) rc = phase_search(ctx, s, w_stitch, max_steps, 0, 1, colors);
  if (rc == MPLD_OK) rc = phase_finish(ctx, s, alpha, colors, counts, cost, stats);
  if (rc == MPLD_OK) rc = mark_last(ctx, s);
  return rc;
}

std::mutex g_ctx_mu;
std::vector<mpld_context*> g_host_ctx;  // one per device for the host entry points

mpld_context* host_context(int* err) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) {
    *err = cuda_fail(e, "cudaGetDevice");
    return nullptr;
  }
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  if ((int)g_host_ctx.size() <= dev) g_host_ctx.resize(dev + 1, nullptr);
  if (!g_host_ctx[dev]) {
    mpld_context* c = nullptr;
    int rc = mpld_context_create(dev, 1 << 16, 16, &c);
    if (rc != MPLD_OK) {
      *err = rc;
      return nullptr;
    }
    g_host_ctx[dev] = c;
  }
  *err = MPLD_OK;
  return g_host_ctx[dev];
}


// ---- asynchronous host entry point -------------------------------------------

int slot_reserve(AsyncSlot& a, int64_t n, int64_t m_ce, int64_t m_se, int32_t L) {
  if (!a.ev_h2d) {
    if (cudaEventCreateWithFlags(&a.ev_h2d, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&a.ev_comp, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&a.ev_d2h, cudaEventDisableTiming) != cudaSuccess ||
        cudaMallocHost((void**)&a.h_stats, sizeof(long long) * MPLD_STAT_LEN) != cudaSuccess)
      return fail(MPLD_ERR_NOMEM, "async slot allocation failed");
  }
  if (n > a.cap_n) {
    a.cap_n = std::max<int64_t>(n, a.cap_n * 3 / 2);
    if (grow(&a.ce_rp, a.cap_n + 1) != cudaSuccess || grow(&a.se_rp, a.cap_n + 1) != cudaSuccess ||
        grow(&a.colors, a.cap_n) != cudaSuccess)
      return fail(MPLD_ERR_NOMEM, "async staging allocation failed");
  }
  if (m_ce > a.cap_ce) {
    a.cap_ce = std::max<int64_t>(m_ce, a.cap_ce * 3 / 2);
    if (grow(&a.ce_col, a.cap_ce) != cudaSuccess) return fail(MPLD_ERR_NOMEM, "async staging allocation failed");
  }
  if (m_se > a.cap_se) {
    a.cap_se = std::max<int64_t>(m_se, a.cap_se * 3 / 2);
    if (grow(&a.se_col, a.cap_se) != cudaSuccess) return fail(MPLD_ERR_NOMEM, "async staging allocation failed");
  }
  if (L > a.cap_l) {
    a.cap_l = std::max<int32_t>(L, 16);
    if (a.h_counts) cudaFreeHost(a.h_counts);
    a.h_counts = nullptr;
    if (grow(&a.lo, a.cap_l + 1) != cudaSuccess || grow(&a.counts, 2 * (int64_t)a.cap_l) != cudaSuccess ||
        grow(&a.cost, a.cap_l) != cudaSuccess || grow(&a.stats, MPLD_STAT_LEN) != cudaSuccess ||
        cudaMallocHost((void**)&a.h_counts, sizeof(long long) * 2 * a.cap_l) != cudaSuccess)
      return fail(MPLD_ERR_NOMEM, "async staging allocation failed");
  }
  return MPLD_OK;
}

// wait for the slot's submit, then split the counts and check the error bits
int slot_finish(AsyncSlot& a) {
  if (!a.pending) return a.fin_rc;
  a.pending = false;
  a.fin_ticket = a.ticket;
  cudaError_t e = cudaEventSynchronize(a.ev_d2h);
  if (e != cudaSuccess) return a.fin_rc = cuda_fail(e, "async pipeline / D2H copy");
  for (int l = 0; l < a.n_layouts; ++l) {
    a.u_nc[l] = a.h_counts[2 * l];
    a.u_ns[l] = a.h_counts[2 * l + 1];
  }
  if (a.u_stats) std::memcpy(a.u_stats, a.h_stats, sizeof(long long) * MPLD_STAT_LEN);
  const long long err = a.h_stats[MPLD_STAT_ERROR];
  if (err & kErrGraph) return a.fin_rc = fail(MPLD_ERR_GRAPH, "graph violates the CSR invariants of mpld.h");
  if (err & kErrComponent) return a.fin_rc = fail(MPLD_ERR_COMPONENT, "a component exceeds MPLD_MAX_COMPONENT vertices");
  return a.fin_rc = MPLD_OK;
}

}  // namespace

extern "C" {

const char* mpld_last_error(void) { return g_last_error.c_str(); }
const char* mpld_version(void) { return MPLD_VERSION; }

int mpld_context_create(int device, int64_t max_vertices, int32_t max_layouts, mpld_context** out) {
  if (!out) return fail(MPLD_ERR_ARG, "out is NULL");
  *out = nullptr;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  mpld_context* ctx = new mpld_context();
  ctx->device = device;
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
  int coop = 0;
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device);
  if (!coop) {
    delete ctx;
    return fail(MPLD_ERR_CUDA, "device does not support cooperative launch");
  }
  if (cudaMalloc((void**)&ctx->ctl, 2 * sizeof(Control)) != cudaSuccess) {
    mpld_context_destroy(ctx);
    return fail(MPLD_ERR_NOMEM, "control block allocation failed");
  }
  ctx->ctl_tile = ctx->ctl + 1;
  cudaMemset(ctx->ctl, 0, 2 * sizeof(Control));
  ctx->blocks_build = coop_blocks_build(ctx->num_sms);
  if (ctx->blocks_build <= 0 || cudaMalloc((void**)&ctx->build_err, sizeof(int)) != cudaSuccess ||
      cudaMalloc((void**)&ctx->build_bar, sizeof(unsigned)) != cudaSuccess ||
      cudaMalloc((void**)&ctx->build_tot, sizeof(int) * 3 * (size_t)ctx->blocks_build) != cudaSuccess) {
    mpld_context_destroy(ctx);
    return fail(MPLD_ERR_NOMEM, "control block allocation failed");
  }
  cudaMemset(ctx->build_err, 0, sizeof(int));
  cudaMemset(ctx->build_bar, 0, sizeof(unsigned));
  if (cudaMalloc((void**)&ctx->wq, sizeof(WorkItem) * 2 * kWQCap) != cudaSuccess ||
      cudaMalloc((void**)&ctx->wq_flag, sizeof(unsigned long long) * 2 * kWQCap) != cudaSuccess ||
      cudaMalloc((void**)&ctx->hslot, sizeof(HeavySlot) * kSlots) != cudaSuccess) {
    mpld_context_destroy(ctx);
    return fail(MPLD_ERR_NOMEM, "heavy-search work queue allocation failed");
  }
  cudaMemset(ctx->wq_flag, 0, sizeof(unsigned long long) * 2 * kWQCap);  // epochs start at 1
  ctx->blocks_simplify = coop_blocks_simplify(kCoopThreads, ctx->num_sms);
  ctx->blocks_recover = coop_blocks_recover(kCoopThreads, ctx->num_sms);
  ctx->blocks_search = resident_blocks_search(32, ctx->num_sms);
  ctx->blocks_discover = resident_blocks_discover(ctx->num_sms);
  ctx->blocks_stream = resident_blocks_evaluate(ctx->num_sms);
  if (const char* pd = std::getenv("MPLD_PDL")) set_pdl(std::strtol(pd, nullptr, 10) != 0);
  if (const char* ts = std::getenv("MPLD_TAIL_SLOTS")) ctx->tail_slots = (int)std::strtol(ts, nullptr, 10);
  if (const char* hs = std::getenv("MPLD_HEAVY_SPILL")) {
    const long v = std::strtol(hs, nullptr, 10);
    if (v >= 64) ctx->spill_iters = (unsigned)std::min<long>(v & ~63L, 1L << 30);
  }
  if (const char* gs = std::getenv("MPLD_GREEDY_SALT")) ctx->greedy_salt = (unsigned)std::strtoul(gs, nullptr, 10);
  if (const char* gr = std::getenv("MPLD_GREEDY_ROUNDS")) {
    const long v = std::strtol(gr, nullptr, 10);
    if (v >= 1 && v <= 64) ctx->greedy_rounds = (int)v;
  }
  if (const char* ls = std::getenv("MPLD_LIGHT_STEPS")) {
    const long v = std::strtol(ls, nullptr, 10);
    if (v >= 1 && v <= (1L << 24)) ctx->light_steps = (unsigned)v;
  }
  e = configure_recover_tail();
  if (e != cudaSuccess) {
    mpld_context_destroy(ctx);
    return cuda_fail(e, "configure recovery tail");
  }
  e = configure_tile();
  if (e != cudaSuccess) {
    mpld_context_destroy(ctx);
    return cuda_fail(e, "configure tile pipeline");
  }
  ctx->blocks_tile = resident_blocks_tile(ctx->num_sms);
  ctx->blocks_piece = coop_blocks_piece(ctx->num_sms);
  e = configure_search_heavy(ctx->num_sms, ctx->blocks_heavy);
  if (e == cudaSuccess) e = configure_search_wide(ctx->num_sms, &ctx->blocks_wide);
  if (e != cudaSuccess || ctx->blocks_wide <= 0) {
    mpld_context_destroy(ctx);
    return cuda_fail(e, "configure heavy search");
  }
  int min_heavy = ctx->blocks_heavy[0];
  for (int b : ctx->blocks_heavy) min_heavy = std::min(min_heavy, b);
  if (ctx->blocks_simplify <= 0 || ctx->blocks_recover <= 0 || ctx->blocks_search <= 0 || min_heavy <= 0 ||
      ctx->blocks_discover <= 0 || ctx->blocks_tile <= 0 || ctx->blocks_piece <= 0) {
    mpld_context_destroy(ctx);
    return fail(MPLD_ERR_CUDA, "occupancy query failed (kernel image missing for this device?)");
  }
  int rc = ensure_workspace(ctx, max_vertices, max_layouts);
  if (rc != MPLD_OK) {
    mpld_context_destroy(ctx);
    return rc;
  }
  e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_last, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    mpld_context_destroy(ctx);
    return cuda_fail(e, "cudaStreamCreate");
  }
  ctx->blocks_prep = ctx->num_sms;  // one CTA per SM on the second stream, beside the search kernels
  if (const char* pb = std::getenv("MPLD_PREP_BLOCKS")) {  // experiments: fewer SMs for the prep
    const long v = std::strtol(pb, nullptr, 10);
    if (v >= 1 && v <= ctx->num_sms) ctx->blocks_prep = (int)v;
  }
  *out = ctx;
  return MPLD_OK;
}

void mpld_context_destroy(mpld_context* ctx) {
  if (!ctx) return;
  for (void* p : {(void*)ctx->deg, (void*)ctx->hround, (void*)ctx->bmask, (void*)ctx->prio, (void*)ctx->q0, (void*)ctx->q1,
                  (void*)ctx->roots, (void*)ctx->crec, (void*)ctx->pmask, (void*)ctx->porder, (void*)ctx->hcomp,
                  (void*)ctx->hcost, (void*)ctx->wide, (void*)ctx->t_par, (void*)ctx->t_cnt, (void*)ctx->t_end,
                  (void*)ctx->t_pos, (void*)ctx->t_perm, (void*)ctx->t_pend, (void*)ctx->build_err, (void*)ctx->build_bar,
                  (void*)ctx->build_tot, (void*)ctx->ctl, (void*)ctx->wq, (void*)ctx->wq_flag, (void*)ctx->hslot,
                  (void*)ctx->est, (void*)ctx->bsum,
                  (void*)ctx->h_lo,
                  (void*)ctx->h_ce_rp, (void*)ctx->h_ce_col, (void*)ctx->h_se_rp, (void*)ctx->h_se_col,
                  (void*)ctx->h_colors, (void*)ctx->h_counts, (void*)ctx->h_cost, (void*)ctx->h_stats})
    if (p) cudaFree(p);
  for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
  for (auto& p : ctx->pending) {
    cudaEventDestroy(p.second.first);
    cudaEventDestroy(p.second.second);
  }
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->aux) cudaStreamDestroy(ctx->aux);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  if (ctx->ev_last) cudaEventDestroy(ctx->ev_last);
  for (AsyncSlot& a : ctx->slot) {
    for (void* p : {(void*)a.lo, (void*)a.ce_rp, (void*)a.ce_col, (void*)a.se_rp, (void*)a.se_col, (void*)a.se_pairs,
                    (void*)a.up_deg, (void*)a.up_col, (void*)a.colors,
                    (void*)a.counts, (void*)a.cost, (void*)a.stats})
      if (p) cudaFree(p);
    if (a.h_counts) cudaFreeHost(a.h_counts);
    if (a.h_stats) cudaFreeHost(a.h_stats);
    for (cudaEvent_t e : {a.ev_h2d, a.ev_comp, a.ev_d2h})
      if (e) cudaEventDestroy(e);
  }
  if (ctx->s_h2d) cudaStreamDestroy(ctx->s_h2d);
  if (ctx->s_d2h) cudaStreamDestroy(ctx->s_d2h);
  delete ctx;
}

int mpld_decompose_device(mpld_context* ctx, void* stream, int32_t n_layouts, const int32_t* d_layout_offsets,
                          int32_t n, const int32_t* d_ce_rowptr, const int32_t* d_ce_col,
                          const int32_t* d_se_rowptr, const int32_t* d_se_col, int32_t k, double alpha,
                          int64_t max_steps, uint32_t flags, int32_t* d_colors, int64_t* d_counts, double* d_cost,
                          int64_t* d_stats) {
  if (!ctx) return fail(MPLD_ERR_ARG, "ctx is NULL");
  int w_stitch = 0;
  int rc = check_scalars(n, k, alpha, &w_stitch);
  if (rc != MPLD_OK) return rc;
  if (n_layouts < 1) return fail(MPLD_ERR_ARG, "n_layouts < 1");
  if (!d_layout_offsets || !d_ce_rowptr || !d_se_rowptr || !d_colors || !d_counts || !d_cost)
    return fail(MPLD_ERR_ARG, "NULL device pointer");
  std::lock_guard<std::mutex> lk(ctx->mu);
  cudaSetDevice(ctx->device);
  rc = ensure_workspace(ctx, n, n_layouts);
  if (rc != MPLD_OK) return rc;
  GraphView g{n, n_layouts, d_layout_offsets, d_ce_rowptr, d_ce_col, d_se_rowptr, d_se_col};
  rc = order_after_last(ctx, (cudaStream_t)stream);
  if (rc != MPLD_OK) return rc;
  return run_pipeline(ctx, (cudaStream_t)stream, g, k, w_stitch, alpha, (long long)max_steps, flags, d_colors,
                      (long long*)d_counts, d_cost, (long long*)d_stats);
}

int mpld_prepare_device(mpld_context* ctx, void* stream, int32_t n_layouts, const int32_t* d_layout_offsets,
                        int32_t n, const int32_t* d_ce_rowptr, const int32_t* d_ce_col,
                        const int32_t* d_se_rowptr, const int32_t* d_se_col, int32_t k, uint32_t flags,
                        int32_t* d_colors, int64_t* d_counts) {
  if (!ctx) return fail(MPLD_ERR_ARG, "ctx is NULL");
  int w_stitch = 0;
  int rc = check_scalars(n, k, 0.0, &w_stitch);
  if (rc != MPLD_OK) return rc;
  if (n_layouts < 1 || !d_layout_offsets || !d_ce_rowptr || !d_se_rowptr || !d_colors || !d_counts)
    return fail(MPLD_ERR_ARG, "bad argument (NULL device pointer or n_layouts < 1)");
  std::lock_guard<std::mutex> lk(ctx->mu);
  cudaSetDevice(ctx->device);
  rc = ensure_workspace(ctx, n, n_layouts);
  if (rc != MPLD_OK) return rc;
  GraphView g{n, n_layouts, d_layout_offsets, d_ce_rowptr, d_ce_col, d_se_rowptr, d_se_col};
  rc = order_after_last(ctx, (cudaStream_t)stream);
  if (rc == MPLD_OK) rc = phase_prepare(ctx, (cudaStream_t)stream, g, k, flags, d_colors, (long long*)d_counts);
  if (rc == MPLD_OK) rc = mark_last(ctx, (cudaStream_t)stream);
  return rc;
}

int mpld_search_device(mpld_context* ctx, void* stream, double alpha, int64_t max_steps, int32_t shard_index,
                       int32_t shard_count, int32_t* d_colors) {
  if (!ctx || !d_colors) return fail(MPLD_ERR_ARG, "ctx or d_colors is NULL");
  if (shard_count < 1 || shard_index < 0 || shard_index >= shard_count)
    return fail(MPLD_ERR_ARG, "shard_index must be in [0, shard_count)");
  std::lock_guard<std::mutex> lk(ctx->mu);
  if (!ctx->prepared) return fail(MPLD_ERR_ARG, "mpld_prepare_device must be called first");
  int w_stitch = 0;
  int rc = check_scalars(ctx->g.n, ctx->k, alpha, &w_stitch);
  if (rc != MPLD_OK) return rc;
  cudaSetDevice(ctx->device);
  rc = order_after_last(ctx, (cudaStream_t)stream);
  if (rc == MPLD_OK)
    rc = phase_search(ctx, (cudaStream_t)stream, w_stitch, (long long)max_steps, shard_index, shard_count, d_colors);
  if (rc == MPLD_OK) rc = mark_last(ctx, (cudaStream_t)stream);
  return rc;
}

int mpld_finish_device(mpld_context* ctx, void* stream, double alpha, int32_t* d_colors, int64_t* d_counts,
                       double* d_cost, int64_t* d_stats) {
  if (!ctx || !d_colors || !d_counts || !d_cost) return fail(MPLD_ERR_ARG, "NULL argument");
  std::lock_guard<std::mutex> lk(ctx->mu);
  if (!ctx->prepared) return fail(MPLD_ERR_ARG, "mpld_prepare_device must be called first");
  int w_stitch = 0;
  int rc = check_scalars(ctx->g.n, ctx->k, alpha, &w_stitch);
  if (rc != MPLD_OK) return rc;
  cudaSetDevice(ctx->device);
  rc = order_after_last(ctx, (cudaStream_t)stream);
  if (rc == MPLD_OK)
    rc = phase_finish(ctx, (cudaStream_t)stream, alpha, d_colors, (long long*)d_counts, d_cost, (long long*)d_stats);
  if (rc == MPLD_OK) rc = mark_last(ctx, (cudaStream_t)stream);
  return rc;
}

int mpld_shard_export(mpld_context* ctx, void* stream, const int32_t* d_colors, int32_t* d_pairs, int64_t* d_count) {
  if (!ctx || !d_colors || !d_pairs || !d_count) return fail(MPLD_ERR_ARG, "NULL argument");
  std::lock_guard<std::mutex> lk(ctx->mu);
  if (!ctx->prepared) return fail(MPLD_ERR_ARG, "mpld_prepare_device must be called first");
  cudaSetDevice(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  int rc = order_after_last(ctx, s);
  if (rc != MPLD_OK) return rc;
  const cudaError_t e = launch_shard_export(ctx->g.n, d_colors, d_pairs, (unsigned long long*)d_count, s,
                                            ctx->blocks_stream);
  if (e != cudaSuccess) return cuda_fail(e, "mpld_shard_export");
  return mark_last(ctx, s);
}

int mpld_shard_import(mpld_context* ctx, void* stream, const int32_t* d_pairs, int64_t n_pairs, int32_t* d_colors) {
  if (!ctx || !d_colors || (n_pairs > 0 && !d_pairs) || n_pairs < 0) return fail(MPLD_ERR_ARG, "bad argument");
  std::lock_guard<std::mutex> lk(ctx->mu);
  if (!ctx->prepared) return fail(MPLD_ERR_ARG, "mpld_prepare_device must be called first");
  cudaSetDevice(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  int rc = order_after_last(ctx, s);
  if (rc != MPLD_OK) return rc;
  const cudaError_t e = launch_shard_import((long long)n_pairs, d_pairs, ctx->g.n, d_colors, s, ctx->blocks_stream);
  if (e != cudaSuccess) return cuda_fail(e, "mpld_shard_import");
  return mark_last(ctx, s);
}

int mpld_decompose_batch(int32_t n_layouts, const int32_t* layout_offsets, int32_t n, const int32_t* ce_rowptr,
                         const int32_t* ce_col, const int32_t* se_rowptr, const int32_t* se_col, int32_t k,
                         double alpha, int64_t max_steps, uint32_t flags, int32_t* colors, int64_t* n_conflicts,
                         int64_t* n_stitches, double* cost, int64_t* stats) {
  int w_stitch = 0;
  int rc = check_scalars(n, k, alpha, &w_stitch);
  if (rc != MPLD_OK) return rc;
  if (n_layouts < 1 || !layout_offsets || !ce_rowptr || !se_rowptr || (n > 0 && !colors) || !n_conflicts ||
      !n_stitches || !cost)
    return fail(MPLD_ERR_ARG, "bad argument (NULL pointer or n_layouts < 1)");
  if (layout_offsets[0] != 0 || layout_offsets[n_layouts] != n)
    return fail(MPLD_ERR_ARG, "layout_offsets must start at 0 and end at n");
  const int64_t m_ce = ce_rowptr[n], m_se = se_rowptr[n];
  if (m_ce < 0 || m_se < 0 || (m_ce > 0 && !ce_col) || (m_se > 0 && !se_col))
    return fail(MPLD_ERR_ARG, "bad CSR row pointer / column array");
  mpld_context* ctx = host_context(&rc);
  if (!ctx) return rc;
  std::lock_guard<std::mutex> lk(ctx->mu);
  cudaSetDevice(ctx->device);
  rc = ensure_workspace(ctx, n, n_layouts);
  if (rc != MPLD_OK) return rc;
  // staging buffers
  if (n > ctx->cap_stage_n || !ctx->h_ce_rp) {
    ctx->cap_stage_n = std::max<int64_t>(n, ctx->cap_n);
    if (grow(&ctx->h_ce_rp, ctx->cap_stage_n + 1) != cudaSuccess ||
        grow(&ctx->h_se_rp, ctx->cap_stage_n + 1) != cudaSuccess || grow(&ctx->h_colors, ctx->cap_stage_n) != cudaSuccess)
      return fail(MPLD_ERR_NOMEM, "staging allocation failed");
  }
  if (m_ce > ctx->cap_ce || !ctx->h_ce_col) {
    ctx->cap_ce = std::max<int64_t>(m_ce, ctx->cap_ce * 3 / 2);
    if (grow(&ctx->h_ce_col, ctx->cap_ce) != cudaSuccess) return fail(MPLD_ERR_NOMEM, "staging allocation failed");
  }
  if (m_se > ctx->cap_se || !ctx->h_se_col) {
    ctx->cap_se = std::max<int64_t>(m_se, ctx->cap_se * 3 / 2);
    if (grow(&ctx->h_se_col, ctx->cap_se) != cudaSuccess) return fail(MPLD_ERR_NOMEM, "staging allocation failed");
  }
  if (!ctx->h_lo || n_layouts > ctx->cap_stage_layouts || !ctx->h_counts) {
    ctx->cap_stage_layouts = std::max<int32_t>(n_layouts, ctx->cap_layouts);
    if (grow(&ctx->h_lo, ctx->cap_stage_layouts + 1) != cudaSuccess ||
        grow(&ctx->h_counts, 2 * (int64_t)ctx->cap_stage_layouts) != cudaSuccess ||
        grow(&ctx->h_cost, ctx->cap_stage_layouts) != cudaSuccess || grow(&ctx->h_stats, MPLD_STAT_LEN) != cudaSuccess)
      return fail(MPLD_ERR_NOMEM, "staging allocation failed");
  }
  cudaStream_t s = ctx->stream;
  rc = order_after_last(ctx, s);
  if (rc != MPLD_OK) return rc;
  cudaError_t e;
  e = cudaMemcpyAsync(ctx->h_lo, layout_offsets, sizeof(int) * (n_layouts + 1), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(ctx->h_ce_rp, ce_rowptr, sizeof(int) * (n + 1), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(ctx->h_se_rp, se_rowptr, sizeof(int) * (n + 1), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && m_ce)
    e = cudaMemcpyAsync(ctx->h_ce_col, ce_col, sizeof(int) * m_ce, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && m_se)
    e = cudaMemcpyAsync(ctx->h_se_col, se_col, sizeof(int) * m_se, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_fail(e, "H2D copy");
  GraphView g{n, n_layouts, ctx->h_lo, ctx->h_ce_rp, ctx->h_ce_col, ctx->h_se_rp, ctx->h_se_col};
  rc = run_pipeline(ctx, s, g, k, w_stitch, alpha, (long long)max_steps, flags, ctx->h_colors, ctx->h_counts,
                    ctx->h_cost, ctx->h_stats);
  if (rc != MPLD_OK) return rc;
  std::vector<long long> counts(2 * (size_t)n_layouts);
  long long st[MPLD_STAT_LEN];
  if (n > 0) e = cudaMemcpyAsync(colors, ctx->h_colors, sizeof(int) * n, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(counts.data(), ctx->h_counts, sizeof(long long) * 2 * n_layouts, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(cost, ctx->h_cost, sizeof(double) * n_layouts, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(st, ctx->h_stats, sizeof(st), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "pipeline / D2H copy");
  for (int l = 0; l < n_layouts; ++l) {
    n_conflicts[l] = counts[2 * l];
    n_stitches[l] = counts[2 * l + 1];
  }
  if (stats) std::memcpy(stats, st, sizeof(st));
  if (st[MPLD_STAT_ERROR] & kErrGraph) return fail(MPLD_ERR_GRAPH, "graph violates the CSR invariants of mpld.h");
  if (st[MPLD_STAT_ERROR] & kErrComponent)
    return fail(MPLD_ERR_COMPONENT, "a component exceeds MPLD_MAX_COMPONENT vertices");
  g_last_error.clear();
  return MPLD_OK;
}

namespace {
// The pipelined host submit; stitch edges either as CSR (se_rowptr, se_col) or
// as n_pairs (u, v) pairs (se_pairs, se_rowptr == NULL), built into CSR on the device.
// Conflict edges as CSR (ce_rowptr, ce_col) or as the upper triangle
// (ce_up_deg, ce_up_col with n_ce_up entries; ce_rowptr == NULL), built into
// the symmetric CSR on the device.
int submit_async(mpld_context* ctx, int32_t n_layouts, const int32_t* layout_offsets, int32_t n,
                 const int32_t* ce_rowptr, const int32_t* ce_col, const int32_t* se_rowptr, const int32_t* se_col,
                 const int32_t* se_pairs, int64_t n_pairs, int32_t k, double alpha, int64_t max_steps,
                 uint32_t flags, int32_t* colors, int64_t* n_conflicts, int64_t* n_stitches, double* cost,
                 int64_t* stats, int64_t* ticket, const unsigned char* ce_up_deg = nullptr,
                 const int32_t* ce_up_col = nullptr, int64_t n_ce_up = 0) {
  if (!ctx || !ticket) return fail(MPLD_ERR_ARG, "bad context / ticket pointer");
  int w_stitch = 0;
  int rc = check_scalars(n, k, alpha, &w_stitch);
  if (rc != MPLD_OK) return rc;
  const bool pairs = se_rowptr == nullptr;
  const bool upper = ce_rowptr == nullptr;
  if (upper && (n_ce_up < 0 || n_ce_up > (int64_t)INT32_MAX / 2 || (n > 0 && !ce_up_deg) || (n_ce_up > 0 && !ce_up_col)))
    return fail(MPLD_ERR_ARG, "bad upper-triangle conflict edges");
  if (n_layouts < 1 || !layout_offsets || (!upper && !ce_rowptr) || (n > 0 && !colors) || !n_conflicts ||
      !n_stitches || !cost)
    return fail(MPLD_ERR_ARG, "bad argument (NULL pointer or n_layouts < 1)");
  if (layout_offsets[0] != 0 || layout_offsets[n_layouts] != n)
    return fail(MPLD_ERR_ARG, "layout_offsets must start at 0 and end at n");
  if (pairs) {
    if (n_pairs < 0 || (n_pairs > 0 && !se_pairs) || 2 * n_pairs > (int64_t)INT32_MAX)
      return fail(MPLD_ERR_ARG, "bad stitch pairs");
    for (int64_t i = 0; i < 2 * n_pairs; i += 2) {  // ids and self loops; the rest is the device validation's
      const int32_t u = se_pairs[i], v = se_pairs[i + 1];
      if (u < 0 || u >= n || v < 0 || v >= n || u == v)
        return fail(MPLD_ERR_GRAPH, "stitch pair " + std::to_string(i / 2) + " out of range or a self loop");
    }
  }
  const int64_t m_ce = upper ? 2 * n_ce_up : ce_rowptr[n], m_se = pairs ? 2 * n_pairs : se_rowptr[n];
  if (m_ce < 0 || m_se < 0 || (!upper && m_ce > 0 && !ce_col) || (!pairs && m_se > 0 && !se_col))
    return fail(MPLD_ERR_ARG, "bad CSR row pointer / column array");
  std::lock_guard<std::mutex> lk(ctx->mu);
  cudaSetDevice(ctx->device);
  if (!ctx->s_h2d) {
    if (cudaStreamCreateWithFlags(&ctx->s_h2d, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->s_d2h, cudaStreamNonBlocking) != cudaSuccess)
      return fail(MPLD_ERR_CUDA, "async stream creation failed");
  }
  const int64_t t = ctx->next_ticket;
  AsyncSlot& a = ctx->slot[t % kAsyncSlots];
  slot_finish(a);  // the slot's previous submit (t - 3) is complete and post-processed before reuse
  if (n > ctx->cap_n) cudaStreamSynchronize(ctx->stream);  // the workspace grows: the other slot's compute must end
  rc = ensure_workspace(ctx, n, n_layouts);
  if (rc == MPLD_OK) rc = slot_reserve(a, n, m_ce, m_se, n_layouts);
  if (rc == MPLD_OK && pairs && m_se > a.cap_pairs) {
    a.cap_pairs = std::max<int64_t>(m_se, a.cap_pairs * 3 / 2);
    if (grow(&a.se_pairs, a.cap_pairs) != cudaSuccess) rc = fail(MPLD_ERR_NOMEM, "async staging allocation failed");
  }
  if (rc == MPLD_OK && upper && n_ce_up > a.cap_up) {
    a.cap_up = std::max<int64_t>(n_ce_up, a.cap_up * 3 / 2);
    if (grow(&a.up_col, a.cap_up) != cudaSuccess) rc = fail(MPLD_ERR_NOMEM, "async staging allocation failed");
  }
  if (rc == MPLD_OK && upper && n > a.cap_up_n) {
    a.cap_up_n = std::max<int64_t>(n, a.cap_up_n * 3 / 2);
    if (grow(&a.up_deg, a.cap_up_n) != cudaSuccess) rc = fail(MPLD_ERR_NOMEM, "async staging allocation failed");
  }
  if (rc != MPLD_OK) return rc;
  cudaStream_t up = ctx->s_h2d, ks = ctx->stream, down = ctx->s_d2h;
  cudaError_t e = cudaMemcpyAsync(a.lo, layout_offsets, sizeof(int) * (n_layouts + 1), cudaMemcpyHostToDevice, up);
  if (e == cudaSuccess && !upper)
    e = cudaMemcpyAsync(a.ce_rp, ce_rowptr, sizeof(int) * (n + 1), cudaMemcpyHostToDevice, up);
  if (e == cudaSuccess && !pairs)
    e = cudaMemcpyAsync(a.se_rp, se_rowptr, sizeof(int) * (n + 1), cudaMemcpyHostToDevice, up);
  if (e == cudaSuccess && !upper && m_ce)
    e = cudaMemcpyAsync(a.ce_col, ce_col, sizeof(int) * m_ce, cudaMemcpyHostToDevice, up);
  if (e == cudaSuccess && upper && n > 0) e = cudaMemcpyAsync(a.up_deg, ce_up_deg, n, cudaMemcpyHostToDevice, up);
  if (e == cudaSuccess && upper && n_ce_up)
    e = cudaMemcpyAsync(a.up_col, ce_up_col, sizeof(int) * n_ce_up, cudaMemcpyHostToDevice, up);
  if (e == cudaSuccess && m_se)
    e = pairs ? cudaMemcpyAsync(a.se_pairs, se_pairs, sizeof(int) * m_se, cudaMemcpyHostToDevice, up)
              : cudaMemcpyAsync(a.se_col, se_col, sizeof(int) * m_se, cudaMemcpyHostToDevice, up);
  if (e == cudaSuccess) e = cudaEventRecord(a.ev_h2d, up);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(ks, a.ev_h2d, 0);
  if (e != cudaSuccess) return cuda_fail(e, "async H2D copy");
  rc = order_after_last(ctx, ks);
  if (rc != MPLD_OK) return rc;
  if (upper || pairs) {  // the CE CSR from its upper triangle and / or the SE CSR from pairs, on the device
    // (one cooperative launch; scratch: the workspace arrays, rewritten by the hot path later)
    GraphBuild gb{};
    gb.n = n;
    gb.m_up = upper ? (int)n_ce_up : 0;
    gb.deg_up = upper ? a.up_deg : nullptr;
    gb.col_up = a.up_col;
    gb.ce_rp = a.ce_rp;
    gb.ce_col = a.ce_col;
    gb.m_se = pairs ? (int)n_pairs : -1;
    gb.se_pairs = a.se_pairs;
    gb.se_rp = a.se_rp;
    gb.se_col = a.se_col;
    gb.rp_up = ctx->q1;
    gb.cnt_ce = ctx->deg;
    gb.fill_ce = ctx->roots;
    gb.tot = ctx->build_tot;
    gb.err = ctx->build_err;
    gb.bar = ctx->build_bar;
    gb.epoch0 = 0;
    // the barrier counter starts every build at zero (a build that never
    // finished cannot leave later ones waiting)
    e = cudaMemsetAsync(ctx->build_bar, 0, sizeof(unsigned), ks);
    if (e != cudaSuccess) return cuda_fail(e, "graph build");
    TimedLaunch tb(ctx, K_BUILD, ks);
    e = launch_graph_build(gb, ks, ctx->blocks_build);
    if (e != cudaSuccess) return cuda_fail(e, "graph build");
    tb.done();
  }
  GraphView g{n, n_layouts, a.lo, a.ce_rp, a.ce_col, a.se_rp, a.se_col};
  rc = run_pipeline(ctx, ks, g, k, w_stitch, alpha, (long long)max_steps, flags, a.colors, a.counts, a.cost,
                    a.stats);
  if (rc != MPLD_OK) return rc;
  e = cudaEventRecord(a.ev_comp, ks);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(down, a.ev_comp, 0);
  if (e == cudaSuccess && n > 0) e = cudaMemcpyAsync(colors, a.colors, sizeof(int) * n, cudaMemcpyDeviceToHost, down);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(a.h_counts, a.counts, sizeof(long long) * 2 * n_layouts, cudaMemcpyDeviceToHost, down);
  if (e == cudaSuccess) e = cudaMemcpyAsync(cost, a.cost, sizeof(double) * n_layouts, cudaMemcpyDeviceToHost, down);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(a.h_stats, a.stats, sizeof(long long) * MPLD_STAT_LEN, cudaMemcpyDeviceToHost, down);
  if (e == cudaSuccess) e = cudaEventRecord(a.ev_d2h, down);
  // the next upload into this slot must not overwrite inputs the compute still reads
  if (e != cudaSuccess) return cuda_fail(e, "async D2H copy");
  a.ticket = t;
  a.pending = true;
  a.n_layouts = n_layouts;
  a.u_nc = n_conflicts;
  a.u_ns = n_stitches;
  a.u_stats = stats;
  ctx->next_ticket = t + 1;
  *ticket = t;
  g_last_error.clear();
  return MPLD_OK;
}
}  // namespace

int mpld_decompose_batch_async(mpld_context* ctx, int32_t n_layouts, const int32_t* layout_offsets, int32_t n,
                               const int32_t* ce_rowptr, const int32_t* ce_col, const int32_t* se_rowptr,
                               const int32_t* se_col, int32_t k, double alpha, int64_t max_steps, uint32_t flags,
                               int32_t* colors, int64_t* n_conflicts, int64_t* n_stitches, double* cost,
                               int64_t* stats, int64_t* ticket) {
  if (!se_rowptr) return fail(MPLD_ERR_ARG, "bad argument (NULL se_rowptr)");
  return submit_async(ctx, n_layouts, layout_offsets, n, ce_rowptr, ce_col, se_rowptr, se_col, nullptr, 0, k, alpha,
                      max_steps, flags, colors, n_conflicts, n_stitches, cost, stats, ticket);
}

int mpld_decompose_batch_pairs_async(mpld_context* ctx, int32_t n_layouts, const int32_t* layout_offsets, int32_t n,
                                     const int32_t* ce_rowptr, const int32_t* ce_col, int64_t n_stitch_pairs,
                                     const int32_t* stitch_pairs, int32_t k, double alpha, int64_t max_steps,
                                     uint32_t flags, int32_t* colors, int64_t* n_conflicts, int64_t* n_stitches,
                                     double* cost, int64_t* stats, int64_t* ticket) {
  return submit_async(ctx, n_layouts, layout_offsets, n, ce_rowptr, ce_col, nullptr, nullptr, stitch_pairs,
                      n_stitch_pairs, k, alpha, max_steps, flags, colors, n_conflicts, n_stitches, cost, stats,
                      ticket);
}

int mpld_decompose_batch_upper_async(mpld_context* ctx, int32_t n_layouts, const int32_t* layout_offsets, int32_t n,
                                     const uint8_t* ce_up_deg, int64_t n_ce_edges, const int32_t* ce_up_col,
                                     int64_t n_stitch_pairs, const int32_t* stitch_pairs, int32_t k, double alpha,
                                     int64_t max_steps, uint32_t flags, int32_t* colors, int64_t* n_conflicts,
                                     int64_t* n_stitches, double* cost, int64_t* stats, int64_t* ticket) {
  return submit_async(ctx, n_layouts, layout_offsets, n, nullptr, nullptr, nullptr, nullptr, stitch_pairs,
                      n_stitch_pairs, k, alpha, max_steps, flags, colors, n_conflicts, n_stitches, cost, stats,
                      ticket, ce_up_deg, ce_up_col, n_ce_edges);
}

int mpld_wait(mpld_context* ctx, int64_t ticket) {
  if (!ctx || ticket < 0 || ticket >= ctx->next_ticket) return fail(MPLD_ERR_ARG, "bad context / unknown ticket");
  std::lock_guard<std::mutex> lk(ctx->mu);
  AsyncSlot& a = ctx->slot[ticket % kAsyncSlots];
  if (a.pending && a.ticket == ticket) return slot_finish(a);
  if (a.fin_ticket == ticket) return a.fin_rc;
  return MPLD_OK;  // an older submit of this slot: completed before the slot was reused
}

int mpld_decompose(int32_t n, const int32_t* ce_rowptr, const int32_t* ce_col, const int32_t* se_rowptr,
                   const int32_t* se_col, int32_t k, double alpha, int64_t max_steps, int32_t* colors,
                   int64_t* n_conflicts, int64_t* n_stitches, double* cost) {
  int32_t lo[2] = {0, n};
  return mpld_decompose_batch(1, lo, n, ce_rowptr, ce_col, se_rowptr, se_col, k, alpha, max_steps, 0u, colors,
                              n_conflicts, n_stitches, cost, nullptr);
}

int mpld_context_set_timing(mpld_context* ctx, int enable) {
  if (!ctx) return fail(MPLD_ERR_ARG, "ctx is NULL");
  ctx->timing = enable != 0;
  return MPLD_OK;
}

static void drain_timing(mpld_context* ctx) {
  for (auto& p : ctx->pending) {
    cudaEventSynchronize(p.second.second);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.second.first, p.second.second);
    ctx->acc_ms[p.first] += ms;
    ctx->ev_pool.push_back(p.second.first);
    ctx->ev_pool.push_back(p.second.second);
  }
  ctx->pending.clear();
}

int mpld_context_reset_timing(mpld_context* ctx) {
  if (!ctx) return fail(MPLD_ERR_ARG, "ctx is NULL");
  std::lock_guard<std::mutex> lk(ctx->mu);
  drain_timing(ctx);
  for (int i = 0; i < K_COUNT; ++i) {
    ctx->acc_ms[i] = 0.0;
    ctx->launches[i] = 0;
  }
  return MPLD_OK;
}

int mpld_kernel_count(void) { return K_COUNT; }

int mpld_context_debug(mpld_context* ctx, int64_t* out, int n) {
  if (!ctx || !out || n < 0) return fail(MPLD_ERR_ARG, "bad argument");
  Control c;
  cudaError_t e = cudaMemcpy(&c, ctx->ctl_tile, sizeof(Control), cudaMemcpyDeviceToHost);
  const int64_t gate = ctx->last_tiles ? c.gate : -1;
  if (e == cudaSuccess && (!ctx->last_tiles || c.gate))  // whole-graph pipeline (alone, or behind a gated tile pass)
    e = cudaMemcpy(&c, ctx->ctl, sizeof(Control), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "debug copy");
  int64_t v[96];
  for (int i = 0; i < 16; ++i) v[i] = (int64_t)c.t[i];
  for (int i = 0; i < 32; ++i) {
    v[20 + i] = (int64_t)c.tr[i];
    v[52 + i] = c.nr[i];
  }
  v[16] = c.n_levels;
  v[17] = c.n_hidden;
  v[18] = c.n_rounds;
  v[19] = c.max_steps_comp;
  for (int i = 0; i < 8; ++i) v[84 + i] = (int64_t)c.dbg[i];
  v[85] = (int64_t)c.steps_heavy;
  v[87] = (int64_t)c.steps;
  v[92] = c.n_seed;
  v[93] = c.n_heavy[0] + c.n_heavy[1];
  v[94] = c.n_comp;
  v[95] = c.truncated;
  v[88] = gate;
  for (int i = 0; i < n && i < 96; ++i) out[i] = v[i];
  if (n > 96 && ctx->est) {  // MPLD_DIAG_HEAVY builds: the heavy-search trace (4 words per unit)
    const int64_t m = std::min<int64_t>(n - 96, std::min<int64_t>(4 * (int64_t)c.dbg[7], ctx->cap_n));
    if (m > 0) {
      e = cudaMemcpy(out + 96, ctx->est, sizeof(int64_t) * (size_t)m, cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) return cuda_fail(e, "debug copy");
    }
  }
  return MPLD_OK;
}

const char* mpld_kernel_name(int i) { return (i >= 0 && i < K_COUNT) ? kKernelNames[i] : ""; }

int mpld_context_kernel_time(mpld_context* ctx, int i, double* ms, int64_t* launches) {
  if (!ctx || i < 0 || i >= K_COUNT) return fail(MPLD_ERR_ARG, "bad context / kernel index");
  std::lock_guard<std::mutex> lk(ctx->mu);
  drain_timing(ctx);
  if (ms) *ms = ctx->acc_ms[i];
  if (launches) *launches = ctx->launches[i];
  return MPLD_OK;
}

}  // extern "C"
