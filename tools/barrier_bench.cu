// Micro-benchmark of grid-wide barrier variants for the persistent kernels.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/barrier_bench tools/barrier_bench.cu
#include <cooperative_groups.h>
#include <cstdio>

namespace cg = cooperative_groups;

__device__ unsigned g_count;

template <int V>
__device__ __forceinline__ void bar(unsigned& epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    ++epoch;
    const unsigned target = epoch * gridDim.x;
    unsigned cur;
    if (V == 0) {  // fence + atomic + relaxed poll + fence
      __threadfence();
      atomicAdd(&g_count, 1u);
      do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(&g_count) : "memory"); } while ((int)(cur - target) < 0);
      __threadfence();
    } else if (V == 1) {  // release-add + acquire poll
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&g_count) : "memory");
      do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(&g_count) : "memory"); } while ((int)(cur - target) < 0);
    } else {  // release-add + relaxed poll + acquire fence
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&g_count) : "memory");
      do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(&g_count) : "memory"); } while ((int)(cur - target) < 0);
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
  }
  __syncthreads();
}

template <int V>
__global__ void k_bar(int iters, int* sink) {
  unsigned epoch = 0;
  int acc = 0;
  for (int i = 0; i < iters; ++i) {
    bar<V>(epoch);
    acc += sink[(blockIdx.x + i) & 1023];
  }
  if (acc == 0x7fffffff) sink[0] = acc;
}

__global__ void k_cg(int iters, int* sink) {
  cg::grid_group g = cg::this_grid();
  int acc = 0;
  for (int i = 0; i < iters; ++i) {
    g.sync();
    acc += sink[(blockIdx.x + i) & 1023];
  }
  if (acc == 0x7fffffff) sink[0] = acc;
}

template <typename K>
float run(K kern, int blocks, int threads, int iters, int* sink) {
  unsigned zero = 0;
  cudaMemcpyToSymbol(g_count, &zero, 4);
  void* args[] = {&iters, &sink};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaLaunchCooperativeKernel((void*)kern, blocks, threads, args, 0, 0);
  cudaMemcpyToSymbol(g_count, &zero, 4);
  cudaEventRecord(a);
  cudaLaunchCooperativeKernel((void*)kern, blocks, threads, args, 0, 0);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
  return 1e3f * ms / iters;
}

int main() {
  int* sink;
  cudaMalloc(&sink, 4096 * 4);
  cudaMemset(sink, 0, 4096 * 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 2000;
  for (int bps : {1, 2}) {
    for (int threads : {256, 1024}) {
      if (bps * threads > 2048) continue;
      int blocks = sms * bps;
      printf("blocks %4d x %4d: fence/relaxed %.2f us  release/acquire %.2f us  release/relaxed+fence %.2f us  cg %.2f us\n",
             blocks, threads, run(k_bar<0>, blocks, threads, iters, sink), run(k_bar<1>, blocks, threads, iters, sink),
             run(k_bar<2>, blocks, threads, iters, sink), run(k_cg, blocks, threads, iters, sink));
    }
  }
  printf("blocks %4d x %4d: fence/relaxed %.2f us\n", sms * 8, 256, run(k_bar<0>, sms * 8, 256, iters, sink));
  return 0;
}
