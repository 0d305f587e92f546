// microbench_gather.cu -- how the dist-gather ceiling of the SSSP advance
// depends on the gathered footprint and on the index distribution.
//   uniform  : indices uniform over an array of 2^k floats
//   rmat     : indices drawn like RMAT destinations (each of the `scale` bits
//              is 1 with probability C+D = 0.24; unpermuted ids: hot vertices
//              scattered over the whole array)
//   rmat-rl  : the same draws after a popcount-major relabel (hot vertices
//              packed into a prefix: expected in-degree depends only on the
//              popcount of the id)
// Each element: one streamed 8-byte record holding the index + one gather.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_gather tools/microbench_gather.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ull; x ^= x >> 27; x *= 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// kind 0: uniform, 1: rmat dst, 2: rmat dst relabelled through perm
__global__ void k_fill(uint2* a, uint64_t n, int scale, int kind, const uint32_t* perm) {
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
      if (kind == 2) v = perm[v];
    }
    a[i] = make_uint2(v, (uint32_t)i);
  }
}

template <int VT, int MODE>
__global__ void __launch_bounds__(256) k_both(const uint2* __restrict__ a, float* d, uint64_t n,
                                              uint32_t* out) {
  float acc = 0;
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride * VT) {
    uint2 v[VT];
#pragma unroll
    for (int r = 0; r < VT; ++r) v[r] = i + r * stride < n ? __ldcs(a + i + r * stride) : make_uint2(0, 0);
    float g[VT];
#pragma unroll
    for (int r = 0; r < VT; ++r) {
      if (MODE == 0) g[r] = d[v[r].x];
      else if (MODE == 1) g[r] = __ldcg(d + v[r].x);
      else g[r] = __ldg(d + v[r].x);
    }
#pragma unroll
    for (int r = 0; r < VT; ++r) acc += g[r];
  }
  if (acc == 1234.5f) *out = 1;
}

// gather + RED.MIN on 3% of elements (the test-before-atomic mix)
template <int VT>
__global__ void __launch_bounds__(256) k_mix(const uint2* __restrict__ a, float* d, uint64_t n) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride * VT) {
    uint2 v[VT];
#pragma unroll
    for (int r = 0; r < VT; ++r) v[r] = i + r * stride < n ? __ldcs(a + i + r * stride) : make_uint2(0, 0);
    float g[VT];
#pragma unroll
    for (int r = 0; r < VT; ++r) g[r] = d[v[r].x];
#pragma unroll
    for (int r = 0; r < VT; ++r)
      if ((v[r].y & 31) == 0 && g[r] >= 0.f) atomicMin(reinterpret_cast<unsigned*>(d + v[r].x), 0u);
  }
}

int main() {
  const uint64_t n = 1ull << 27;  // 134M records = 1 GB
  uint2* a;
  float* d;
  uint32_t *out, *perm;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&d, (1ull << 26) * 4);
  cudaMalloc(&out, 4);
  cudaMalloc(&perm, (1ull << 26) * 4);
  cudaMemset(d, 0, (1ull << 26) * 4);
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
    return ms / 5;
  };
  printf("%-8s %5s %8s | %10s %10s %10s %10s  (G elements/s)\n", "dist", "scale", "MB", "ld",
         "ld.cg", "ld.nc", "ld+3%min");
  for (int kind = 0; kind < 3; ++kind) {
    for (int scale : {18, 20, 22, 23, 24, 25, 26}) {
      if (kind == 2) {  // popcount-major relabel
        std::vector<uint32_t> ids(1u << scale), p(1u << scale);
        for (uint32_t i = 0; i < ids.size(); ++i) ids[i] = i;
        std::stable_sort(ids.begin(), ids.end(), [](uint32_t x, uint32_t y) {
          return __builtin_popcount(x) < __builtin_popcount(y);
        });
        for (uint32_t r = 0; r < ids.size(); ++r) p[ids[r]] = r;
        cudaMemcpy(perm, p.data(), p.size() * 4, cudaMemcpyHostToDevice);
      }
      k_fill<<<blocks, 256>>>(a, n, scale, kind, perm);
      float t0 = timeit([&] { k_both<8, 0><<<blocks, 256>>>(a, d, n, out); });
      float t1 = timeit([&] { k_both<8, 1><<<blocks, 256>>>(a, d, n, out); });
      float t2 = timeit([&] { k_both<8, 2><<<blocks, 256>>>(a, d, n, out); });
      float t3 = timeit([&] { k_mix<8><<<blocks, 256>>>(a, d, n); });
      printf("%-8s %5d %8.1f | %10.1f %10.1f %10.1f %10.1f\n",
             kind == 0 ? "uniform" : kind == 1 ? "rmat" : "rmat-rl", scale,
             (4ull << scale) / 1048576.0, n / (t0 * 1e6), n / (t1 * 1e6), n / (t2 * 1e6),
             n / (t3 * 1e6));
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
