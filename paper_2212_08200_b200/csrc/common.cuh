// common.cuh -- shared types, error plumbing and device helpers of libgfb.
//
// Layout in HBM:
//   ro    u32[n+1]          CSR row offsets (graph.hpp:116 csr_row_offsets_)
//   adj   EdgeRec<W>[m]     CSR {dst, weight} interleaved: one 8-byte record
//                           per edge for u32/f32 weights (16 B for f64), so a
//                           warp streams 256 contiguous bytes per load and a
//                           short row costs one sector run instead of two
//                           (graph.hpp:117-118 keep col/values as SoA).
//   co    u32[n+1]          CSC offsets           (graph.hpp:121)
//   cadj  EdgeRec<W>[m]     CSC {src, weight}     (graph.hpp:122-123)
//   ceid  u32[m]            CSC -> CSR edge id    (graph.hpp:124)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/gfb.h"

namespace gfb {

struct Error {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg);
void check_cuda(cudaError_t e, const char* what);
#define GFB_CUDA(x) ::gfb::check_cuda((x), #x)

constexpr uint32_t NIL = 0xFFFFFFFFu;

// ---------------------------------------------------------------------------
// Edge records and distance arithmetic per weight type.
// ---------------------------------------------------------------------------
template <class W> struct EdgeRec;
template <> struct alignas(8) EdgeRec<uint32_t> { uint32_t v; uint32_t w; };
template <> struct alignas(8) EdgeRec<float> { uint32_t v; float w; };
template <> struct alignas(16) EdgeRec<double> { uint32_t v; uint32_t pad; double w; };

// Distances are stored in the weight's type.  For non-negative values the
// IEEE bit pattern orders like the unsigned integer of the same width, so
// atomicMin on the bits is an exact min (-0.0 is canonicalised at upload).
template <class W> struct DT;
template <> struct DT<uint32_t> {
  using D = uint32_t;
  using Bits = unsigned int;
  static constexpr uint32_t INF_BITS = 0xFFFFFFFFu;
};
template <> struct DT<float> {
  using D = float;
  using Bits = unsigned int;
  static constexpr uint32_t INF_BITS = 0x7F800000u;
};
template <> struct DT<double> {
  using D = double;
  using Bits = unsigned long long;
  static constexpr unsigned long long INF_BITS = 0x7FF0000000000000ull;
};

template <class W>
__device__ __forceinline__ typename DT<W>::D dinf() {
  typename DT<W>::Bits b = DT<W>::INF_BITS;
  return *reinterpret_cast<typename DT<W>::D*>(&b);
}

// nd = d + w with one IEEE round-to-nearest (no FMA contraction possible:
// a plain add).  u32: exact integer sum; overflow past 2^32-2 flags an error
// (the reference's double would still be exact there).
__device__ __forceinline__ float dadd(float d, float w, unsigned*) { return __fadd_rn(d, w); }
__device__ __forceinline__ double dadd(double d, double w, unsigned*) { return __dadd_rn(d, w); }
__device__ __forceinline__ uint32_t dadd(uint32_t d, uint32_t w, unsigned* err) {
  uint64_t s = (uint64_t)d + w;
  if (s >= 0xFFFFFFFFull) {
    if (err && d != 0xFFFFFFFFu) atomicOr(err, 1u);
    return 0xFFFFFFFFu;
  }
  return (uint32_t)s;
}

__device__ __forceinline__ uint32_t atomic_min_d(uint32_t* p, uint32_t v) { return atomicMin(p, v); }
__device__ __forceinline__ float atomic_min_d(float* p, float v) {
  return __uint_as_float(atomicMin(reinterpret_cast<unsigned*>(p), __float_as_uint(v)));
}
__device__ __forceinline__ double atomic_min_d(double* p, double v) {
  return __longlong_as_double((long long)atomicMin(reinterpret_cast<unsigned long long*>(p),
                                                   (unsigned long long)__double_as_longlong(v)));
}
// Fire-and-forget min (RED.MIN): used where the prior value is not needed.
__device__ __forceinline__ void red_min_d(uint32_t* p, uint32_t v) { atomicMin(p, v); }
__device__ __forceinline__ void red_min_d(float* p, float v) {
  atomicMin(reinterpret_cast<unsigned*>(p), __float_as_uint(v));
}
__device__ __forceinline__ void red_min_d(double* p, double v) {
  atomicMin(reinterpret_cast<unsigned long long*>(p), (unsigned long long)__double_as_longlong(v));
}

// Streaming, read-only CSR/CSC record loads: non-coherent path, no L1
// allocation, L2 evict-first so the record stream does not push the
// distance array out of L2.
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ EdgeRec<uint32_t> ld_rec(const EdgeRec<uint32_t>* p) {
  uint32_t a, b;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
               : "=r"(a), "=r"(b) : "l"(p), "l"(evict_first_policy()));
  return {a, b};
}
__device__ __forceinline__ EdgeRec<float> ld_rec(const EdgeRec<float>* p) {
  uint32_t a, b;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
               : "=r"(a), "=r"(b) : "l"(p), "l"(evict_first_policy()));
  return {a, __uint_as_float(b)};
}
__device__ __forceinline__ EdgeRec<double> ld_rec(const EdgeRec<double>* p) {
  uint32_t a, b, c, d;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(p), "l"(evict_first_policy()));
  EdgeRec<double> r;
  r.v = a;
  r.pad = b;
  r.w = __hiloint2double((int)d, (int)c);
  return r;
}

// Distance loads during an advance: relaxed loads that may be served by L1.
// A stale (larger) value only costs a redundant atomic; it never loses an
// update because every lowering goes through an L2 atomic.
template <class D>
__device__ __forceinline__ D ld_dist(const D* p) { return *p; }

// Explicit fire-and-forget reductions (PTX red.*) with an optional L2
// eviction-priority hint.
__device__ __forceinline__ uint64_t evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void red_min_u32(unsigned* p, unsigned v) {
  asm volatile("red.global.min.u32 [%0], %1;" ::"l"(p), "r"(v));
}
__device__ __forceinline__ void red_min_u32_hint(unsigned* p, unsigned v, uint64_t pol) {
  asm volatile("red.global.L2::cache_hint.min.u32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol)
              );
}
__device__ __forceinline__ void red_min_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.global.min.u64 [%0], %1;" ::"l"(p), "l"(v));
}
__device__ __forceinline__ void red_min_u64_hint(unsigned long long* p, unsigned long long v,
                                                 uint64_t pol) {
  asm volatile("red.global.L2::cache_hint.min.u64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(pol)
              );
}
__device__ __forceinline__ void red_or_u32(unsigned* p, unsigned v) {
  asm volatile("red.global.or.b32 [%0], %1;" ::"l"(p), "r"(v));
}
__device__ __forceinline__ uint32_t ld_u32_hint(const void* p, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}

// float bits of a distance (u32 distances as float): log-scale bucket key
__device__ __forceinline__ uint32_t fkey(float d) { return __float_as_uint(d); }
__device__ __forceinline__ uint32_t fkey(uint32_t d) { return __float_as_uint((float)d); }
__device__ __forceinline__ uint32_t fkey(double d) { return __float_as_uint((float)d); }

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

// ---------------------------------------------------------------------------
// Decoupled look-back (single-pass chained scan) over (count, edges) pairs.
// Status word: flag(2) | count(31) | edges(31).  The device path therefore
// requires n < 2^31 and m < 2^31 (RMAT scale 26 EF16 has m = 1.07e9).
// ---------------------------------------------------------------------------
__device__ constexpr unsigned long long LB_FLAG_AGG = 1ull << 62;
__device__ constexpr unsigned long long LB_FLAG_INC = 2ull << 62;
__device__ constexpr unsigned long long LB_MASK31 = (1ull << 31) - 1;

__device__ __forceinline__ unsigned long long lb_pack(unsigned long long flag, uint32_t c,
                                                      uint32_t e) {
  return flag | ((unsigned long long)c << 31) | (unsigned long long)e;
}

// Called by ONE thread of tile `tile`; returns the exclusive prefix.
__device__ inline void lb_lookback(unsigned long long* status, uint32_t tile, uint32_t agg_c,
                                   uint32_t agg_e, uint32_t* pre_c, uint32_t* pre_e) {
  volatile unsigned long long* st = status;
  if (tile == 0) {
    st[0] = lb_pack(LB_FLAG_INC, agg_c, agg_e);
    *pre_c = 0;
    *pre_e = 0;
    return;
  }
  st[tile] = lb_pack(LB_FLAG_AGG, agg_c, agg_e);
  __threadfence();
  uint32_t c = 0, e = 0;
  int64_t j = (int64_t)tile - 1;
  while (j >= 0) {
    unsigned long long s = st[j];
    unsigned long long flag = s & (3ull << 62);
    if (flag == 0) continue;  // predecessor not published yet: spin
    c += (uint32_t)((s >> 31) & LB_MASK31);
    e += (uint32_t)(s & LB_MASK31);
    if (flag == LB_FLAG_INC) break;
    --j;
  }
  __threadfence();
  st[tile] = lb_pack(LB_FLAG_INC, c + agg_c, e + agg_e);
  *pre_c = c;
  *pre_e = e;
}

// Warp-parallel variant (called by all 32 lanes of one warp; agg_* must be
// valid in every lane): inspects 32 predecessors per step, so a chain of
// aggregate-only predecessors costs one L2 round trip per 32 tiles.
__device__ inline void lb_lookback_warp(unsigned long long* status, uint32_t tile, uint32_t agg_c,
                                        uint32_t agg_e, uint32_t* pre_c, uint32_t* pre_e) {
  volatile unsigned long long* st = status;
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) st[0] = lb_pack(LB_FLAG_INC, agg_c, agg_e);
    *pre_c = 0;
    *pre_e = 0;
    return;
  }
  if (lane == 0) {
    st[tile] = lb_pack(LB_FLAG_AGG, agg_c, agg_e);
    __threadfence();
  }
  __syncwarp();
  uint32_t c = 0, e = 0;
  int64_t base = (int64_t)tile - 1;
  for (;;) {
    int64_t j = base - lane;
    unsigned long long sv = j >= 0 ? st[j] : LB_FLAG_INC;
    unsigned long long flag = sv & (3ull << 62);
    if (__any_sync(0xffffffffu, flag == 0)) continue;  // someone not published: re-read
    unsigned inc = __ballot_sync(0xffffffffu, flag == LB_FLAG_INC);
    int last = inc ? __ffs(inc) - 1 : 31;  // lanes 0..last contribute
    uint32_t vc = lane <= last ? (uint32_t)((sv >> 31) & LB_MASK31) : 0u;
    uint32_t ve = lane <= last ? (uint32_t)(sv & LB_MASK31) : 0u;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      vc += __shfl_xor_sync(0xffffffffu, vc, d);
      ve += __shfl_xor_sync(0xffffffffu, ve, d);
    }
    c += vc;
    e += ve;
    if (inc) break;
    base -= 32;
  }
  if (lane == 0) {
    __threadfence();
    st[tile] = lb_pack(LB_FLAG_INC, c + agg_c, e + agg_e);
  }
  *pre_c = c;
  *pre_e = e;
}

}  // namespace gfb
