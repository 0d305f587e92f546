// rmat.cuh -- counter-based synthetic graph generators (host + device).
//
// Not in the reference (it ships only the G(n,p) test corpus,
// tests/random_graphs.hpp:15-30); BASELINE.md §2 defines the workloads.
// Edge i is a pure function of (seed, i): splitmix64 of a per-edge counter,
// two 32-bit RMAT level draws per hash, Graph500 A/B/C/D = .57/.19/.19/.05,
// labels unpermuted (vertex 0 is the hub), duplicates and self-loops kept.
// Weights: U{0..255} (u32) or U[0,1) on a 2^-24 grid (f32, exact in f32 and
// f64).  oracle/graflow_oracle.c restates this independently.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define GFB_HD __host__ __device__ __forceinline__
#else
#define GFB_HD inline
#endif

namespace gfb {

GFB_HD uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

GFB_HD uint64_t edge_hash(uint64_t seed, uint64_t i, uint32_t j) {
  return splitmix64(seed * 0xD1B54A32D192ED03ULL + i * 64ULL + j);
}

GFB_HD uint32_t f32_unit_bits(uint64_t h) {
  float f = (float)(h >> 40) * (1.0f / 16777216.0f);  // exact: 24-bit integer * 2^-24
  union {
    float f;
    uint32_t u;
  } c;
  c.f = f;
  return c.u;
}

// wkind 0: u32 U{0..255}; 1: f32 U[0,1)
GFB_HD void rmat_edge(int scale, uint64_t seed, int wkind, uint64_t i, uint32_t* src,
                      uint32_t* dst, uint32_t* wbits) {
  const uint32_t t1 = 0x91eb851eu, t2 = 0xc28f5c28u, t3 = 0xf3333333u;  // .57 .76 .95
  uint32_t s = 0, d = 0;
  uint64_t word = 0;
  for (int l = 0; l < scale; ++l) {
    if ((l & 1) == 0) word = edge_hash(seed, i, (uint32_t)(l >> 1));
    uint32_t r = (l & 1) ? (uint32_t)(word >> 32) : (uint32_t)word;
    uint32_t sb = r >= t2;
    uint32_t db = (r >= t1 && r < t2) || r >= t3;
    s = (s << 1) | sb;
    d = (d << 1) | db;
  }
  uint64_t wk = edge_hash(seed, i, 31);
  *src = s;
  *dst = d;
  *wbits = wkind == 0 ? (uint32_t)(wk >> 56) : f32_unit_bits(wk);
}

// grid edge u -> neighbour k (0 up, 1 left, 2 right, 3 down)
GFB_HD uint32_t grid_weight_bits(uint64_t seed, uint64_t u, int k) {
  return f32_unit_bits(splitmix64(seed * 0xD1B54A32D192ED03ULL + u * 4ULL + (uint64_t)k));
}

}  // namespace gfb
