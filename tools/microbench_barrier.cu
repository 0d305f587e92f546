// microbench_barrier.cu -- cost of one grid-wide barrier on B200 (the
// persistent SSSP loop pays two per superstep).
//   flat     : one arrival counter + generation word
//   two-level: 16-CTA group counters, then a top counter (bsp.cuh grid_sync)
//   cg       : cooperative_groups::this_grid().sync()
//   cluster  : barrier.cluster (8 CTAs, hardware) -- for scale
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_barrier tools/microbench_barrier.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

namespace cg = cooperative_groups;

__device__ __forceinline__ void flat_sync(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vb = bar;
    const unsigned gen = vb[1];
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      vb[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (vb[1] == gen) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ void two_sync(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vb = bar;
    const unsigned gen = vb[0];
    const unsigned G = gridDim.x, grp = blockIdx.x / 16;
    const unsigned gsize = min(16u, G - grp * 16);
    const unsigned ngroups = (G + 15) / 16;
    __threadfence();
    if (atomicAdd(bar + 2 + grp, 1u) == gsize - 1) {
      vb[2 + grp] = 0;
      __threadfence();
      if (atomicAdd(bar + 1, 1u) == ngroups - 1) {
        vb[1] = 0;
        __threadfence();
        atomicAdd(bar, 1u);
      }
    }
    while (vb[0] == gen) __nanosleep(20);
    __threadfence();
  }
  __syncthreads();
}

// acquire/release flavour without full fences
__device__ __forceinline__ void ar_sync(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned gen;
    asm volatile("ld.relaxed.gpu.u32 %0, [%1];" : "=r"(gen) : "l"(bar));
    const unsigned G = gridDim.x, grp = blockIdx.x / 16;
    const unsigned gsize = min(16u, G - grp * 16);
    const unsigned ngroups = (G + 15) / 16;
    unsigned old;
    asm volatile("atom.acq_rel.gpu.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar + 2 + grp));
    if (old == gsize - 1) {
      asm volatile("st.relaxed.gpu.u32 [%0], 0;" ::"l"(bar + 2 + grp));
      asm volatile("atom.acq_rel.gpu.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar + 1));
      if (old == ngroups - 1) {
        asm volatile("st.relaxed.gpu.u32 [%0], 0;" ::"l"(bar + 1));
        asm volatile("red.release.gpu.add.u32 [%0], 1;" ::"l"(bar));
      }
    }
    unsigned g2;
    do {
      asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(g2) : "l"(bar));
    } while (g2 == gen);
  }
  __syncthreads();
}

template <int KIND>
__global__ void k_bar(unsigned* bar, int iters, unsigned* out) {
  unsigned acc = 0;
  for (int i = 0; i < iters; ++i) {
    if (KIND == 0) flat_sync(bar);
    else if (KIND == 1) two_sync(bar);
    else if (KIND == 2) cg::this_grid().sync();
    else if (KIND == 3) ar_sync(bar);
    acc += threadIdx.x;
  }
  if (acc == 0xdeadbeef) *out = acc;
}

int main() {
  unsigned *bar, *out;
  cudaMalloc(&bar, 1024);
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2000;
  const char* names[] = {"flat", "two-level", "cg", "acq/rel"};
  for (int threads : {256, 1024}) {
    for (int per_sm : {1, 2, 4, 8}) {
      if (threads * per_sm > 2048) continue;
      int G = 148 * per_sm;
      printf("grid %4d x %4d:", G, threads);
      for (int kind = 0; kind < 4; ++kind) {
        cudaMemset(bar, 0, 1024);
        void* k = kind == 0 ? (void*)k_bar<0> : kind == 1 ? (void*)k_bar<1>
                : kind == 2 ? (void*)k_bar<2> : (void*)k_bar<3>;
        int it = iters;
        void* args[] = {&bar, &it, &out};
        cudaLaunchCooperativeKernel(k, G, threads, args, 0, 0);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel(k, G, threads, args, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("  %s %.2f us", names[kind], ms * 1e3 / iters);
      }
      printf("   (%s)\n", cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
