// microbench_red.cu -- does a sparse stream of reductions (the SSSP advance's
// RED.MIN / RED.OR on ~3% of edges) throttle the dist gathers around it?
// Each element: one streamed record + one gather; every 32nd element also
// issues a write-like op to the gathered address.  Variants:
//   none      gathers only
//   red       RED.MIN.u32 (atomicMin, result unused)
//   atom      ATOM.MIN with the result consumed
//   st        plain st.global
//   red-nc    RED.MIN, gathers through ld.global.nc
//   red-cg    RED.MIN, gathers through ld.global.cg (L2 only)
// Index distributions: uniform, rmat (bits 1 w.p. 0.24).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_red tools/microbench_red.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ull; x ^= x >> 27; x *= 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

__global__ void k_fill(uint2* a, uint64_t n, int scale, int kind) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t v = 0;
    if (kind == 0) {
      v = (uint32_t)mix64(i * 0x9E3779B97F4A7C15ull + 1) & ((1u << scale) - 1);
    } else {
      uint64_t h = mix64(i + 77);
      for (int b = 0; b < scale; ++b) {
        if (b % 5 == 0 && b) h = mix64(h + b);
        uint32_t r = (uint32_t)(h & 4095);
        h >>= 12;
        if (r < (uint32_t)(0.24 * 4096)) v |= 1u << b;
      }
    }
    a[i] = make_uint2(v, (uint32_t)mix64(i) & 31);
  }
}

template <int MODE>
__device__ __forceinline__ uint32_t gat(const uint32_t* p) {
  if (MODE == 4) return __ldg(p);
  if (MODE == 5) return __ldcg(p);
  return *p;
}

// MODE 0 none, 1 red, 2 atom, 3 st, 4 red-nc, 5 red-cg
template <int VT, int MODE>
__global__ void __launch_bounds__(256, 8) k_mix(const uint2* __restrict__ a, uint32_t* d,
                                                uint64_t n, uint32_t* out) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride * VT) {
    uint2 v[VT];
#pragma unroll
    for (int r = 0; r < VT; ++r)
      v[r] = i + r * stride < n ? __ldcs(a + i + r * stride) : make_uint2(0, 1);
    uint32_t g[VT];
#pragma unroll
    for (int r = 0; r < VT; ++r) g[r] = gat<MODE>(d + v[r].x);
#pragma unroll
    for (int r = 0; r < VT; ++r) {
      acc += g[r];
      if (v[r].y == 0 && g[r] != 0x12345u) {
        if (MODE == 1 || MODE == 4 || MODE == 5) atomicMin(d + v[r].x, 7u);
        else if (MODE == 2) acc += atomicMin(d + v[r].x, 7u);
        else if (MODE == 3) d[v[r].x] = 7u;
      }
    }
  }
  if (acc == 0xdeadbeef) *out = acc;
}

int main() {
  const uint64_t n = 1ull << 27;
  const int scale = 24;
  uint2* a;
  uint32_t *d, *out;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&d, (4ull << scale));
  cudaMalloc(&out, 4);
  cudaMemset(d, 0x3f, 4ull << scale);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = 148 * 8;
  auto timeit = [&](auto launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int it = 0; it < 5; ++it) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return n / (ms / 5 * 1e6);
  };
  printf("G elements/s, 64 MB target, 1/32 of elements write\n");
  printf("%-8s %8s %8s %8s %8s %8s %8s\n", "dist", "none", "red", "atom", "st", "red-nc", "red-cg");
  for (int kind = 0; kind < 2; ++kind) {
    k_fill<<<blocks, 256>>>(a, n, scale, kind);
    double r0 = timeit([&] { k_mix<2, 0><<<blocks, 256>>>(a, d, n, out); });
    double r1 = timeit([&] { k_mix<2, 1><<<blocks, 256>>>(a, d, n, out); });
    double r2 = timeit([&] { k_mix<2, 2><<<blocks, 256>>>(a, d, n, out); });
    double r3 = timeit([&] { k_mix<2, 3><<<blocks, 256>>>(a, d, n, out); });
    double r4 = timeit([&] { k_mix<2, 4><<<blocks, 256>>>(a, d, n, out); });
    double r5 = timeit([&] { k_mix<2, 5><<<blocks, 256>>>(a, d, n, out); });
    printf("%-8s %8.1f %8.1f %8.1f %8.1f %8.1f %8.1f\n", kind ? "rmat" : "uniform", r0, r1, r2,
           r3, r4, r5);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
