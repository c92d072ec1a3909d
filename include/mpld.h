/*
 * mpld.h — C ABI of the B200 multiple-patterning layout decomposition (MPLD)
 * hot path (arxiv 2303.14335, "GPU-accelerated matrix cover algorithm for
 * multiple patterning layout decomposition").
 *
 * The library decomposes a decomposed graph DG = (V, CE ∪ SE) into k masks,
 * minimising PAPER.md Eq. (1):
 *
 *     min_x  sum_{e_ij in CE} c_ij + alpha * sum_{e_ij in SE} s_ij
 *     c_ij = (x_i == x_j),  s_ij = (x_i != x_j),  x_i in {0, ..., k-1}      (§2.1, Eq. 1a-1d)
 *
 * following the flow of PAPER.md §2.2 / Fig. 2 ("simplify the layout graph ...
 * call the graph coloring solver ... recover the nodes removed in
 * simplification step") with the solver replaced by an exact-cover search
 * (§2.3, Alg. 1).  All steps run in CUDA kernels for sm_100a; see DESIGN.md
 * §1 for the step list and §2 for the readings R1..R10 of the paper that fix
 * the exact result (every result is bit-identical to the CPU oracle in
 * oracle/, which shares no code with this library).
 *
 * Graph layout (all int32, shared by every entry point):
 *   n            number of vertices (polygon features or stitch segments, §2.1
 *                "every node v_i in V corresponds to one feature"), 0 <= n < 2^31.
 *   ce_rowptr    [n+1] CSR row pointer of the conflict edges CE, ce_rowptr[0] = 0.
 *   ce_col       [ce_rowptr[n]] neighbour ids; each undirected edge appears in
 *                both rows; every row strictly ascending; no self loops.
 *   se_rowptr,   the same for the stitch edges SE (Fig. 1(c) "stitch insertion";
 *   se_col       an SE edge joins two segments of one feature).  CE ∩ SE = ∅.
 *   A batch of independent layouts is their disjoint union: vertex ids of
 *   layout l are [layout_offsets[l], layout_offsets[l+1]) and no edge crosses
 *   a layout boundary.
 *
 * Parameters:
 *   k            number of masks, 2 <= k <= MPLD_MAX_K (DPLD, TPLD, QPLD).
 *   alpha        stitch weight of Eq. (1a) (§2.1 "set as 0.1 by default"); must
 *                be a multiple of 0.001 in [0, 1000] (R2: the search
 *                compares costs exactly in integer units of 1/1000).
 *   max_steps    search budget per component (R7): once a complete
 *                colouring exists and a component's search has entered more
 *                than max_steps nodes, its search stops with the best colouring
 *                found so far (counted in MPLD_STAT_TRUNCATED); the node order is
 *                the sequential one of R5-R7, so truncated results are still
 *                reproducible.  <= 0: exact mode — no budget; components whose
 *                sequential search needs more than 48 nodes are finished by a
 *                warp-parallel search that returns the same first optimal leaf
 *                (R7).  A safety cap of 2^22 nodes per lane bounds exact mode;
 *                components hitting it are counted in MPLD_STAT_TRUNCATED.
 *
 * Outputs:
 *   colors       [n] mask of every vertex, in [0, k).
 *   n_conflicts  #{e_ij in CE : x_i == x_j}    (Table 1 "cn#")
 *   n_stitches   #{e_ij in SE : x_i != x_j}    (Table 1 "st#")
 *   cost         n_conflicts + alpha * n_stitches, IEEE double, computed as
 *                fl(fl(alpha * n_stitches) + n_conflicts).
 *   stats        optional [MPLD_STAT_LEN] int64 (NULL to skip), see enum.
 *
 * Errors: every entry point returns MPLD_OK (0) or an MPLD_ERR_* code and
 * leaves a one-line description in mpld_last_error() (thread-local).  On error
 * the output buffers are unspecified.  Components (after simplification) with
 * more than MPLD_MAX_COMPONENT vertices are rejected with MPLD_ERR_COMPONENT.
 *
 * Ownership: the library never takes ownership of caller buffers.  Host entry
 * points copy inputs to device memory owned by an internal per-device context
 * and block until the result is on the host.  Device entry points take device
 * pointers, enqueue everything on the given stream and return without host
 * synchronisation; the caller keeps buffers alive until the stream passes.
 */
#ifndef MPLD_H_
#define MPLD_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPLD_VERSION "0.1.0"
#define MPLD_MAX_K 4
#define MPLD_MAX_COMPONENT 64
#define MPLD_COST_UNITS 1000 /* cost units per conflict (R2) */

enum mpld_status {
  MPLD_OK = 0,
  MPLD_ERR_ARG = 1,       /* bad scalar argument or NULL pointer */
  MPLD_ERR_GRAPH = 2,     /* CSR not symmetric / not strictly ascending / self loop / CE ∩ SE != ∅ */
  MPLD_ERR_COMPONENT = 3, /* a component exceeds MPLD_MAX_COMPONENT vertices */
  MPLD_ERR_CUDA = 4,      /* CUDA runtime error (message in mpld_last_error) */
  MPLD_ERR_NOMEM = 5      /* device allocation failed */
};

/* flags */
#define MPLD_FLAG_VALIDATE 1u /* check the CSR invariants on the device first (MPLD_ERR_GRAPH): row
                               * pointers, ascending rows, id range, self loops and CE ∩ SE exactly;
                               * symmetry by two 64-bit multiset hashes (sum H(v,u) == sum H(u,v);
                               * an asymmetric graph passes with probability ~2^-64) */

#define MPLD_FLAG_TILES 2u /* run the tile pipeline (kernel_tile.cu: piece order, then simplification,
                            * search and recovery of whole pieces per CTA in shared memory) with the
                            * whole-graph pipeline gated behind it as the fallback; results are
                            * identical.  Off by default: measured slower on the
                            * synthetic configs */

/* stats[] layout */
enum mpld_stat {
  MPLD_STAT_COMPONENTS = 0, /* components solved by the exact-cover search (Alg. 1 line 4) */
  MPLD_STAT_HIDDEN = 1,     /* vertices hidden by simplification (§2.2) */
  MPLD_STAT_ROUNDS = 2,     /* simplification rounds (R8) */
  MPLD_STAT_MAX_COMP = 3,   /* largest component size */
  MPLD_STAT_STEPS = 4,      /* search nodes entered, summed over components */
  MPLD_STAT_TRUNCATED = 5,  /* components whose search hit max_steps */
  MPLD_STAT_ERROR = 6,      /* device-side error bits (1 = graph, 2 = component too large) */
  MPLD_STAT_LAUNCHES = 7,   /* kernels launched by the call */
  MPLD_STAT_MAX_STEPS = 8,  /* largest per-component step count */
  MPLD_STAT_SPILL_REFUSED = 9, /* exact mode: spills of open search work refused (work ring full or no
                                * component slot left; the unit went on alone — a slowdown, not an error) */
  MPLD_STAT_LEN = 10
};

/* Last error message of the calling thread ("" if none). */
const char* mpld_last_error(void);
const char* mpld_version(void);

/* One layout, host buffers (end-to-end call: H2D copy, all kernels, D2H copy).
 * The north_star signature: PAPER.md §2.1 Eq. (1) is the objective, §2.2 /
 * Fig. 2 the flow (simplify -> colouring solver -> recover), §2.3 / Alg. 1 the
 * solver; colors [n], *n_conflicts (Eq. 1b), *n_stitches (Eq. 1c), *cost
 * (Eq. 1a) are written on MPLD_OK.  No validation (see mpld_decompose_batch). */
int mpld_decompose(int32_t n, const int32_t* ce_rowptr, const int32_t* ce_col,
                   const int32_t* se_rowptr, const int32_t* se_col, int32_t k,
                   double alpha, int64_t max_steps, int32_t* colors,
                   int64_t* n_conflicts, int64_t* n_stitches, double* cost);

/* A batch of n_layouts layouts (disjoint union), host buffers.
 * layout_offsets [n_layouts+1]; n_conflicts, n_stitches, cost: [n_layouts].
 * Alg. 1 lines 1-4 ("the original DG will be decomposed into sub-graphs ...
 * parallelly executed on different blocks"): every component of every layout
 * of the batch is searched in the same launches; a batched layout decomposes
 * exactly as alone (R10).  flags: MPLD_FLAG_VALIDATE.  Blocks until
 * the results are on the host. */
int mpld_decompose_batch(int32_t n_layouts, const int32_t* layout_offsets, int32_t n,
                         const int32_t* ce_rowptr, const int32_t* ce_col,
                         const int32_t* se_rowptr, const int32_t* se_col, int32_t k,
                         double alpha, int64_t max_steps, uint32_t flags, int32_t* colors,
                         int64_t* n_conflicts, int64_t* n_stitches, double* cost,
                         int64_t* stats);

/* ---- device-resident interface (inputs already in HBM) ---------------------- */
typedef struct mpld_context mpld_context;

/* Create a context on `device` with workspace for up to max_vertices vertices
 * and max_layouts layouts (grown on demand by later calls).  A context owns
 * its device workspace and control block; calls of one context may be
 * enqueued on different streams (a call on a stream other than the previous
 * call's waits for that call's last operation through an event), but the
 * context must not be used from several host threads at once. */
int mpld_context_create(int device, int64_t max_vertices, int32_t max_layouts, mpld_context** out);
void mpld_context_destroy(mpld_context* ctx);

/* Enqueue the whole hot path on `stream` (a cudaStream_t; NULL = legacy default):
 * the same computation as mpld_decompose_batch (§2.2 flow, §2.3
 * Alg. 1 solver, Eq. (1) outputs) on inputs already resident in HBM.
 * The recovery's preparation runs on the context's own second stream, forked
 * from `stream` by an event after the simplification and joined back before
 * the recovery, so all work stays ordered with respect to `stream`.
 * All pointers are device pointers.  d_counts [2*n_layouts] int64 receives
 * (n_conflicts, n_stitches) per layout, d_cost [n_layouts] the Eq. (1a) cost,
 * d_stats [MPLD_STAT_LEN] the statistics (MPLD_STAT_ERROR != 0 means the
 * result is invalid: check it after the stream synchronises).  Host-side
 * argument errors are returned immediately. */
int mpld_decompose_device(mpld_context* ctx, void* stream, int32_t n_layouts,
                          const int32_t* d_layout_offsets, int32_t n,
                          const int32_t* d_ce_rowptr, const int32_t* d_ce_col,
                          const int32_t* d_se_rowptr, const int32_t* d_se_col, int32_t k,
                          double alpha, int64_t max_steps, uint32_t flags, int32_t* d_colors,
                          int64_t* d_counts, double* d_cost, int64_t* d_stats);

/* ---- asynchronous host-buffer entry point (pipelined batches) ---------------
 * mpld_decompose_batch_async: the host batch call of mpld_decompose_batch
 * (same arguments and outputs, same results) on an explicit context, returning
 * before the result is ready.  It enqueues the upload of the inputs into one of
 * the context's three device staging slots (its own copy stream), the hot path
 * after the upload (the context's compute stream) and the download of colors /
 * counts / cost / stats after the compute (a third stream), then writes a
 * ticket.  Consecutive submits rotate through the slots, so submit t+1's upload
 * overlaps submit t's compute and t's download overlaps t+1's compute.
 * Ownership: the host buffers of a submit must stay valid and unmodified until
 * mpld_wait(ctx, ticket) returns; the outputs are complete only then (counts
 * are split into n_conflicts / n_stitches by mpld_wait).  Page-locked
 * (pinned) host memory makes the copies asynchronous; pageable memory is
 * correct but serialises them.  A submit reusing a slot first waits for and
 * finishes the submit that used it three calls before.
 * Errors: argument errors are returned by the submit; device-side results
 * (MPLD_ERR_GRAPH / MPLD_ERR_COMPONENT from the error bits, CUDA errors) by
 * mpld_wait.  The context must not be used from several threads at once. */
int mpld_decompose_batch_async(mpld_context* ctx, int32_t n_layouts, const int32_t* layout_offsets, int32_t n,
                               const int32_t* ce_rowptr, const int32_t* ce_col, const int32_t* se_rowptr,
                               const int32_t* se_col, int32_t k, double alpha, int64_t max_steps,
                               uint32_t flags, int32_t* colors, int64_t* n_conflicts, int64_t* n_stitches,
                               double* cost, int64_t* stats, int64_t* ticket);

/* The same submit with the stitch edges given as n_stitch_pairs (u, v) pairs
 * (stitch_pairs [2 * n_stitch_pairs], each SE edge once, in either direction)
 * instead of CSR: the H2D copy carries 8 B per stitch edge instead of the
 * (n+1)-entry SE row-pointer array, and the SE CSR is built on the device
 * (degrees, scan, scatter, rows sorted) before the hot path.  Pairs with an id
 * outside [0, n) or u == v are rejected on the host (MPLD_ERR_GRAPH); duplicate
 * pairs and CE ∩ SE are caught by MPLD_FLAG_VALIDATE on the built CSR.  A
 * vertex with 128 or more stitch pairs is reported as MPLD_ERR_GRAPH (the
 * device build counts them in 8 bits).  Results are identical to
 * mpld_decompose_batch_async on the same graph. */
int mpld_decompose_batch_pairs_async(mpld_context* ctx, int32_t n_layouts, const int32_t* layout_offsets, int32_t n,
                                     const int32_t* ce_rowptr, const int32_t* ce_col, int64_t n_stitch_pairs,
                                     const int32_t* stitch_pairs, int32_t k, double alpha, int64_t max_steps,
                                     uint32_t flags, int32_t* colors, int64_t* n_conflicts, int64_t* n_stitches,
                                     double* cost, int64_t* stats, int64_t* ticket);

/* The same submit with the conflict edges given as the upper triangle of
 * their CSR: ce_up_deg [n] uint8 = the number of CE neighbours u > v of each
 * vertex v (< 256 per vertex), ce_up_col [n_ce_edges] = those neighbours,
 * rows in vertex order, each row strictly ascending (every undirected CE edge
 * once, in the row of its smaller end); stitch candidates as pairs.  The
 * upload carries n + 4|CE| + 8|SE| bytes instead of 4(n+1) + 8|CE| + 8|SE|
 * and the symmetric CE CSR (rows ascending) is built on the device before the
 * hot path (§2.1: E = {CE ∪ SE} is undirected, so the triangle holds
 * the whole graph).  Entries outside (v, n), rows not strictly ascending or
 * degrees not summing to n_ce_edges are reported by mpld_wait as
 * MPLD_ERR_GRAPH (whatever the flags); results are identical to
 * mpld_decompose_batch_pairs_async on the same graph. */
int mpld_decompose_batch_upper_async(mpld_context* ctx, int32_t n_layouts, const int32_t* layout_offsets, int32_t n,
                                     const uint8_t* ce_up_deg, int64_t n_ce_edges, const int32_t* ce_up_col,
                                     int64_t n_stitch_pairs, const int32_t* stitch_pairs, int32_t k, double alpha,
                                     int64_t max_steps, uint32_t flags, int32_t* colors, int64_t* n_conflicts,
                                     int64_t* n_stitches, double* cost, int64_t* stats, int64_t* ticket);

/* Block until submit `ticket` of ctx has completed; returns its result code
 * (MPLD_OK or the error of that submit).  Waiting on an older ticket whose slot
 * has been reused returns its stored result. */
int mpld_wait(mpld_context* ctx, int64_t ticket);

/* ---- one batch sharded over several processes ----------------
 * The same hot path split in three phases so that the components of ONE
 * layout batch can be searched by shard_count processes (one per GPU):
 *   1. every process: mpld_prepare_device   (validate?, simplification, components)
 *   2. every process: mpld_search_device     with its shard_index: discovers every
 *      component, estimates its search cost as n * k^n (capped at 2^32; the
 *      north_star's "size x k^n"), takes the inclusive prefix sum of the
 *      estimates in order of the components' roots (smallest vertex ids), and
 *      searches the components whose cost interval starts in the shard_index-th
 *      of shard_count equal parts of the total (contiguous root ranges of
 *      equal estimated cost, computed identically by every process); writes
 *      their colours into d_colors and leaves -1 on every other vertex;
 *   3. the caller combines d_colors across the processes — the only exchange:
 *      an element-wise maximum (an NCCL all-reduce MAX of n int32), or the
 *      compact lists of mpld_shard_export / mpld_shard_import (all-gather);
 *   4. every process: mpld_finish_device     (recovery of the hidden vertices, Eq. 1).
 * The graph pointers and k of phase 1 are remembered by the context and must
 * stay valid until phase 4 is enqueued.  With shard_count == 1 the phases
 * compute exactly mpld_decompose_device.  All calls are stream-ordered. */
/* Phase 1 — PAPER.md §2.2 "simplify the layout graph" and Alg. 1 lines 1-3
 * (components).  d_counts is zeroed here. */
int mpld_prepare_device(mpld_context* ctx, void* stream, int32_t n_layouts, const int32_t* d_layout_offsets,
                        int32_t n, const int32_t* d_ce_rowptr, const int32_t* d_ce_col,
                        const int32_t* d_se_rowptr, const int32_t* d_se_col, int32_t k, uint32_t flags,
                        int32_t* d_colors, int64_t* d_counts);
/* Phase 2 — Alg. 1 lines 4-19 (the exact-cover search) over this shard's
 * components; d_colors of the other kept vertices stay -1. */
int mpld_search_device(mpld_context* ctx, void* stream, double alpha, int64_t max_steps, int32_t shard_index,
                       int32_t shard_count, int32_t* d_colors);
/* Phase 3, compact form — instead of combining the full d_colors
 * arrays, each process exports the colours its search wrote as a compact list
 * and scatters the lists of all processes (after an all-gather):
 *   mpld_shard_export: d_pairs [2 * n] int32 receives (vertex, colour) pairs,
 *     one per vertex with d_colors >= 0 (the vertices of this shard's
 *     components; order unspecified); *d_count (device int64) their number.
 *   mpld_shard_import: for each of n_pairs pairs with vertex in [0, n),
 *     d_colors[vertex] = colour (pairs with vertex < 0 are padding, skipped).
 * Both are stream-ordered device calls between phases 2 and 4 (the colours of
 * §2.2's coloring solver, Fig. 2, gathered before the recovery). */
int mpld_shard_export(mpld_context* ctx, void* stream, const int32_t* d_colors, int32_t* d_pairs,
                      int64_t* d_count);
int mpld_shard_import(mpld_context* ctx, void* stream, const int32_t* d_pairs, int64_t n_pairs,
                      int32_t* d_colors);

/* Phase 4 — §2.2 "recover the nodes removed in simplification step" and
 * Eq. (1).  d_counts may be any [2*n_layouts] int64 buffer: when it is not
 * the one of phase 1, or the search was sharded, it is reset and recomputed
 * from the combined colours (mpld_evaluate). */
int mpld_finish_device(mpld_context* ctx, void* stream, double alpha, int32_t* d_colors, int64_t* d_counts,
                       double* d_cost, int64_t* d_stats);

/* Kernel timing inside the context (for bench.py's roofline): when enabled,
 * every launch is bracketed by CUDA events on the launch stream and its
 * duration accumulated per kernel.  mpld_kernel_count() kernels, indexed
 * 0..count-1: name, accumulated milliseconds and launches since the last reset.
 * Reading the times synchronises the context's events. */
int mpld_context_set_timing(mpld_context* ctx, int enable);
int mpld_context_reset_timing(mpld_context* ctx);
int mpld_kernel_count(void);
const char* mpld_kernel_name(int i);
int mpld_context_kernel_time(mpld_context* ctx, int i, double* ms, int64_t* launches);

/* Diagnostics of the last call (synchronous copy): out[0..15] device
 * %globaltimer stamps (ns) at phase boundaries, out[16] recovery levels
 * (depth of the pop-order DAG + 1), out[17] hidden vertices, out[18] rounds,
 * out[19] largest per-component step count, out[20..51] per round (0..15) / recovery
 * level (16..31) start stamps, out[52..83] their frontier sizes,
 * out[84] slowest discovery (cycles << 16 | n), out[86] slowest light search
 * (cycles << 24 | steps << 8 | n), out[85] search nodes of the warp-parallel
 * (heavy) search, out[87] search nodes in total, out[88] the tile pipeline's gate
 * (0: the tiles took the input; else the reasons the whole-graph pipeline
 * recomputed it, bits: 1 row pointer / id out of range, 2 a piece larger than a
 * window, 4 a neighbour outside its piece's window, 8 / 16 / 128 validation
 * (rows, symmetry, layout offsets), 32 a component > 64 vertices, 64 invalid
 * compact upload; -1: the last call ran without MPLD_FLAG_TILES), out[89] the slowest
 * heavy component (cycles), out[90] the slowest heavy warp (cycles over all its
 * components), out[91] the slowest heavy component's size, out[92] component-search seeds,
 * out[93] heavy components, out[94] components, out[95] truncated searches.
 * Copies min(n, 96); out[96..n) receives the heavy-search trace of MPLD_DIAG_HEAVY
 * builds (4 words per search unit: ci | n << 32 | item << 48, nodes, start and end
 * %globaltimer ns), unspecified otherwise. */
int mpld_context_debug(mpld_context* ctx, int64_t* out, int n);

#ifdef __cplusplus
}
#endif
#endif /* MPLD_H_ */
