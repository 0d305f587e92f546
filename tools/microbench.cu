// microbench.cu -- ceilings for the SSSP advance's access pattern on B200.
//   stream : coalesced 8-byte record stream (DRAM)
//   gather : random 4-byte gathers into an L2-resident array (64 MB = the
//            fp32 distance array at RMAT scale 24)
//   both   : one stream record + one dependent gather per element
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16;
  return x;
}

template <int VT>
__global__ void k_stream(const uint2* __restrict__ a, uint64_t n, uint32_t* out) {
  uint32_t acc = 0;
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride * VT) {
    uint2 v[VT];
#pragma unroll
    for (int r = 0; r < VT; ++r) v[r] = i + r * stride < n ? __ldcs(a + i + r * stride) : make_uint2(0, 0);
#pragma unroll
    for (int r = 0; r < VT; ++r) acc += v[r].x ^ v[r].y;
  }
  if (acc == 0x12345678) *out = acc;
}

template <int VT>
__global__ void k_gather(const float* __restrict__ d, uint32_t mask, uint64_t n, uint32_t* out) {
  float acc = 0;
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride * VT) {
    float v[VT];
#pragma unroll
    for (int r = 0; r < VT; ++r) v[r] = d[hash32((uint32_t)(i + r * stride)) & mask];
#pragma unroll
    for (int r = 0; r < VT; ++r) acc += v[r];
  }
  if (acc == 1234.5f) *out = 1;
}

template <int VT>
__global__ void k_both(const uint2* __restrict__ a, const float* __restrict__ d, uint32_t mask,
                       uint64_t n, uint32_t* out) {
  float acc = 0;
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride * VT) {
    uint2 v[VT];
#pragma unroll
    for (int r = 0; r < VT; ++r) v[r] = i + r * stride < n ? __ldcs(a + i + r * stride) : make_uint2(0, 0);
    float g[VT];
#pragma unroll
    for (int r = 0; r < VT; ++r) g[r] = d[v[r].x & mask];
#pragma unroll
    for (int r = 0; r < VT; ++r) acc += g[r];
  }
  if (acc == 1234.5f) *out = 1;
}

__global__ void k_fill(uint2* a, uint64_t n, uint32_t mask) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    a[i] = make_uint2(hash32((uint32_t)i * 2654435761u) & mask, (uint32_t)i);
}

int main() {
  const uint64_t n = 1ull << 28;  // 268M records = 2 GB
  const uint32_t nd = 1u << 24;   // 16M floats = 64 MB
  uint2* a; float* d; uint32_t* out;
  cudaMalloc(&a, n * 8); cudaMalloc(&d, nd * 4); cudaMalloc(&out, 4);
  cudaMemset(d, 0, nd * 4);
  k_fill<<<148 * 8, 256>>>(a, n, nd - 1);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = 148;
  auto run = [&](const char* name, auto launch, double units, const char* unit) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int it = 0; it < 5; ++it) launch();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("%-28s %8.3f ms  %8.1f %s\n", name, ms, units / (ms * 1e-3) / 1e9, unit);
  };
  for (int blocks : {sms * 4, sms * 8}) {
    printf("grid %d x 256\n", blocks);
    run("stream VT4", [&] { k_stream<4><<<blocks, 256>>>(a, n, out); }, n * 8.0, "GB/s");
    run("stream VT8", [&] { k_stream<8><<<blocks, 256>>>(a, n, out); }, n * 8.0, "GB/s");
    run("gather VT1", [&] { k_gather<1><<<blocks, 256>>>(d, nd - 1, n, out); }, n, "G gathers/s");
    run("gather VT4", [&] { k_gather<4><<<blocks, 256>>>(d, nd - 1, n, out); }, n, "G gathers/s");
    run("gather VT8", [&] { k_gather<8><<<blocks, 256>>>(d, nd - 1, n, out); }, n, "G gathers/s");
    run("stream+gather VT4", [&] { k_both<4><<<blocks, 256>>>(a, d, nd - 1, n, out); }, n, "G edges/s");
    run("stream+gather VT8", [&] { k_both<8><<<blocks, 256>>>(a, d, nd - 1, n, out); }, n, "G edges/s");
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
