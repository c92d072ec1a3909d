// Internal declarations of the MPLD CUDA library (not part of the C ABI).
//
// Data layout in HBM:
//   graph   : caller's CSR arrays (int32), read-only.
//   per-vertex workspace (int32 [n] each): deg, hround, hid, parent, loc
//   per-round : rcnt[n+2] (vertices hidden in round r), roff[n+2] (their offset in hid)
//   per-component : roots[n]
//   Control : one Control block (counters, error bits) per context.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "mpld.h"

namespace mpld {

constexpr int kMaxComp = MPLD_MAX_COMPONENT;  // one 64-bit word per mask
constexpr int kCostUnits = MPLD_COST_UNITS;

enum ErrBits : int { kErrGraph = 1, kErrComponent = 2 };

// Device-resident control block, zeroed at the start of every call by the
// simplification kernel (phase A) except `err`, which the validation kernel may
// set first (the host zeroes it with the graph upload / a memset node).
struct Control {
  int n_rounds;     // simplification rounds R (R8)
  int n_hidden;     // |hidden vertices|
  int n_comp;       // components found
  int next_comp;    // dynamic work counter of the search kernel
  int max_comp;     // largest component
  int truncated;    // components whose search hit max_steps
  int err;          // ErrBits
  int done_blocks;  // last-block detection of the evaluation kernel
  int left[3];      // recovery: uncoloured vertices per iteration (rotating)
  int pad;
  unsigned long long steps;  // search nodes entered
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

struct Workspace {
  int* deg;
  int* hround;  // -1 kept, else the round the vertex was hidden in
  int* hid;     // hidden vertices, grouped by round
  int* rcnt;    // [n+2]
  int* roff;    // [n+2]
  int* parent;  // union-find
  int* loc;     // local index of a kept vertex inside its component
  int* roots;   // component roots (min vertex id of the component)
  Control* ctl;
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

// launch wrappers (kernels_graph.cu, kernel_search.cu); each returns the
// cudaError_t of its launch.
cudaError_t launch_validate(const GraphView& g, Workspace ws, cudaStream_t s, int blocks);
cudaError_t launch_simplify_components(const GraphView& g, Workspace ws, int k, int* colors,
                                       long long* counts, cudaStream_t s, int blocks, int threads);
cudaError_t launch_search(const GraphView& g, Workspace ws, int k, int w_stitch, long long max_steps,
                          int* colors, cudaStream_t s, int blocks, int threads);
cudaError_t launch_recover(const GraphView& g, Workspace ws, int k, int* colors, cudaStream_t s,
                           int blocks, int threads);
cudaError_t launch_evaluate(const GraphView& g, Workspace ws, const int* colors, double alpha,
                            long long* counts, double* cost, long long* stats, int launches,
                            cudaStream_t s, int blocks);

// occupancy helpers for the cooperative (persistent) kernels
int coop_blocks_simplify(int threads, int num_sms);
int coop_blocks_recover(int threads, int num_sms);
int resident_blocks_search(int threads, int num_sms);

}  // namespace mpld
