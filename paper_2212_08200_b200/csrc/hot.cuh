// hot.cuh -- the specialised hot-path advance kernels of gfb_sssp.
//
// Same edge-tile load balancing as k_advance_push/k_advance_pull
// (kernels.cuh), specialised for the SSSP relax condition
// (algorithms.hpp:586-593) with bitmap output, and restructured so every
// thread keeps H_VT independent memory operations in flight per phase:
//   A: H_VT streaming record loads  (8-byte {dst, w}, L1 no-allocate,
//      L2 evict-first)
//   B: H_VT distance gathers        (test-before-atomic)
//   C: H_VT atomicMin on improving candidates (returns consumed in D)
//   D: predecessor records + next-frontier bitmap (RED.OR)
// The generic kernels issue these one edge at a time (load -> gather ->
// atomic chained per edge, MLP ~ 1); ncu showed long-scoreboard stalls on
// exactly that chain (profiles/r01_push_v1.md).
#pragma once

#include "kernels.cuh"

namespace gfb {

constexpr int H_BLOCK = 256;
// edges per thread per tile: 8 for 4-byte weights (2048-edge tiles), 4 for
// f64 (keeps the f64 kernels under the 48 KB static shared-memory limit)
template <class W> struct HotCfg {
  static constexpr int VT = sizeof(W) == 8 ? 4 : 8;
  static constexpr int TILE = H_BLOCK * VT;
  static constexpr int RATIO = TILE / A_TILE;
  static_assert(TILE % A_TILE == 0, "hot tile must be a multiple of the plan tile");
};

// Stage the plan segments of hot tile t and build the edge->segment map.
// Returns the number of edges in the tile.
template <int H_VT, class D>
__device__ __forceinline__ uint32_t hot_stage(const Plan& plan, const D* dist, uint32_t t,
                                              uint32_t ntiles, uint32_t total, uint32_t k,
                                              uint32_t* s_off, uint32_t* s_start, uint32_t* s_u,
                                              D* s_du, uint16_t* s_seg, bool load_du) {
  constexpr int H_TILE = H_BLOCK * H_VT, H_RATIO = H_TILE / A_TILE;
  const int tid = threadIdx.x;
  const uint32_t e0 = t * H_TILE;
  const uint32_t cnt = min((uint32_t)H_TILE, total - e0);
  const uint32_t s0 = plan.tseg[t * H_RATIO];
  const uint32_t s1 = (t + 1 < ntiles) ? plan.tseg[(t + 1) * H_RATIO] : k - 1;
  const uint32_t nseg = s1 - s0 + 1;
  for (uint32_t j = tid; j < nseg; j += H_BLOCK) {
    uint32_t g = s0 + j;
    uint32_t off = plan.off[g];
    uint32_t u = plan.v[g];
    s_off[j] = off > e0 ? off - e0 : 0u;
    s_start[j] = plan.start[g] + (off < e0 ? e0 - off : 0u);
    s_u[j] = u;
    if (load_du) s_du[j] = dist[u];
  }
  __syncthreads();
  uint32_t le0 = tid * H_VT;
  if (le0 < cnt) {
    uint32_t lo = 0, hi = nseg - 1;  // largest j with s_off[j] <= le0
    while (lo < hi) {
      uint32_t mid = (lo + hi + 1) >> 1;
      if (s_off[mid] <= le0) lo = mid;
      else hi = mid - 1;
    }
    uint32_t j = lo;
#pragma unroll
    for (int r = 0; r < H_VT; ++r) {
      uint32_t le = le0 + r;
      if (le < cnt) {
        while (j + 1 < nseg && s_off[j + 1] <= le) ++j;
        s_seg[le] = (uint16_t)j;
      }
    }
  }
  __syncthreads();
  return cnt;
}

template <class W, int H_VT = HotCfg<W>::VT, int MINB = 4>
__global__ void __launch_bounds__(H_BLOCK, MINB) k_push_relax(AdvArgs<W> a) {
  using D = typename DT<W>::D;
  constexpr int H_TILE = H_BLOCK * H_VT;
  __shared__ uint32_t s_off[H_TILE + 2];
  __shared__ uint32_t s_start[H_TILE + 2];
  __shared__ uint32_t s_u[H_TILE + 2];
  __shared__ D s_du[H_TILE + 2];
  __shared__ uint16_t s_seg[H_TILE];

  for (uint32_t i = blockIdx.x * H_BLOCK + threadIdx.x; i < a.status_len; i += gridDim.x * H_BLOCK)
    a.status[i] = 0;
  const uint32_t total = a.ctl->total;
  const uint32_t k = a.ctl->k;
  const uint32_t ntiles = (total + H_TILE - 1) / H_TILE;
  const int tid = threadIdx.x;
  unsigned* err = &a.ctl->err;
  if (blockIdx.x == 0 && tid == 0) {
    a.ctl->relax += total;
    a.ctl->supersteps += 1;
    a.ctl->push_steps += 1;
  }
  for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint32_t cnt = hot_stage<H_VT, D>(a.plan, a.dist, t, ntiles, total, k, s_off, s_start,
                                            s_u, s_du, s_seg, true);
    uint32_t dst[H_VT];
    D nd[H_VT], cur[H_VT];
#pragma unroll
    for (int r = 0; r < H_VT; ++r) {  // A: record stream (+ candidate distance)
      uint32_t le = r * H_BLOCK + tid;
      dst[r] = NIL;
      if (le < cnt) {
        uint32_t j = s_seg[le];
        EdgeRec<W> rec = ld_rec(a.adj + (s_start[j] + (le - s_off[j])));
        dst[r] = rec.v;
        nd[r] = dadd(s_du[j], rec.w, err);
      }
    }
#pragma unroll
    for (int r = 0; r < H_VT; ++r)  // B: distance gathers (test before atomic)
      if (dst[r] != NIL) cur[r] = ld_dist(a.dist + dst[r]);
#pragma unroll
    for (int r = 0; r < H_VT; ++r) {  // C: atomics on candidates
      if (dst[r] != NIL && nd[r] < cur[r]) cur[r] = atomic_min_d(a.dist + dst[r], nd[r]);
      else dst[r] = NIL;
    }
#pragma unroll
    for (int r = 0; r < H_VT; ++r) {  // D: winners
      if (dst[r] != NIL && nd[r] < cur[r]) {
        uint32_t le = r * H_BLOCK + tid;
        uint32_t j = s_seg[le];
        a.predrec[dst[r]] = make_uint2(s_u[j], s_start[j] + (le - s_off[j]));
        atomicOr(a.bm_out + (dst[r] >> 5), 1u << (dst[r] & 31));
      }
    }
    __syncthreads();
  }
}

template <class W>
__global__ void __launch_bounds__(H_BLOCK, 4) k_pull_relax(AdvArgs<W> a, uint32_t total, uint32_t k) {
  using D = typename DT<W>::D;
  using Bits = typename DT<W>::Bits;
  constexpr int H_VT = HotCfg<W>::VT, H_TILE = HotCfg<W>::TILE, H_RATIO = HotCfg<W>::RATIO;
  __shared__ uint32_t s_off[H_TILE + 2];
  __shared__ uint32_t s_start[H_TILE + 2];
  __shared__ uint32_t s_u[H_TILE + 2];
  __shared__ Bits s_best[H_TILE + 2];
  __shared__ uint32_t s_slot[H_TILE + 2];
  __shared__ uint16_t s_seg[H_TILE];
  for (uint32_t i = blockIdx.x * H_BLOCK + threadIdx.x; i < a.status_len; i += gridDim.x * H_BLOCK)
    a.status[i] = 0;
  const uint32_t ntiles = (total + H_TILE - 1) / H_TILE;
  const int tid = threadIdx.x;
  unsigned* err = &a.ctl->err;
  if (blockIdx.x == 0 && tid == 0) {
    a.ctl->supersteps += 1;
    a.ctl->pull_steps += 1;
  }
  uint32_t n_elig = 0;
  for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    // s_best doubles as the (unused) s_du staging slot: initialise after
    const uint32_t cnt = hot_stage<H_VT, Bits>(a.plan, nullptr, t, ntiles, total, k, s_off, s_start,
                                         s_u, s_best, s_seg, false);
    const uint32_t nseg_max = min(cnt + 2, (uint32_t)H_TILE + 2);
    for (uint32_t j = tid; j < nseg_max; j += H_BLOCK) {
      s_best[j] = (Bits)DT<W>::INF_BITS;
      s_slot[j] = NIL;
    }
    uint32_t src[H_VT];
    W w[H_VT];
#pragma unroll
    for (int r = 0; r < H_VT; ++r) {  // A: CSC record stream
      uint32_t le = r * H_BLOCK + tid;
      src[r] = NIL;
      if (le < cnt) {
        uint32_t j = s_seg[le];
        EdgeRec<W> rec = ld_rec(a.adj + (s_start[j] + (le - s_off[j])));
        src[r] = rec.v;
        w[r] = rec.w;
      }
    }
    uint32_t word[H_VT];
#pragma unroll
    for (int r = 0; r < H_VT; ++r)  // B: frontier-bitmap gathers
      word[r] = src[r] != NIL ? a.bm_in[src[r] >> 5] : 0u;
    D nd[H_VT];
#pragma unroll
    for (int r = 0; r < H_VT; ++r) {  // C: distance gathers of active sources
      if ((word[r] >> (src[r] & 31)) & 1u) {
        ++n_elig;
        nd[r] = dadd(ld_dist(a.dist + src[r]), w[r], err);
      } else {
        src[r] = NIL;
      }
    }
    __syncthreads();  // s_best initialised
#pragma unroll
    for (int r = 0; r < H_VT; ++r)
      if (src[r] != NIL)
        atomicMin(&s_best[s_seg[r * H_BLOCK + tid]], *reinterpret_cast<Bits*>(&nd[r]));
    __syncthreads();
#pragma unroll
    for (int r = 0; r < H_VT; ++r) {
      if (src[r] == NIL) continue;
      uint32_t le = r * H_BLOCK + tid;
      uint32_t j = s_seg[le];
      if (*reinterpret_cast<Bits*>(&nd[r]) == s_best[j]) s_slot[j] = s_start[j] + (le - s_off[j]);
    }
    __syncthreads();
    const uint32_t nseg = (t + 1 < ntiles ? a.plan.tseg[(t + 1) * H_RATIO] : k - 1) -
                          a.plan.tseg[t * H_RATIO] + 1;
    for (uint32_t j = tid; j < nseg; j += H_BLOCK) {
      uint32_t sl = s_slot[j];
      if (sl == NIL) continue;
      Bits b = s_best[j];
      D best = *reinterpret_cast<D*>(&b);
      uint32_t u = s_u[j];
      if (best < ld_dist(a.dist + u)) {
        D old = atomic_min_d(a.dist + u, best);
        if (best < old) {
          a.predrec[u] = make_uint2(ld_rec(a.adj + sl).v, a.ceid[sl]);
          atomicOr(a.bm_out + (u >> 5), 1u << (u & 31));
        }
      }
    }
    __syncthreads();
  }
  n_elig = warp_sum(n_elig);
  if ((tid & 31) == 0 && n_elig) atomicAdd(&a.ctl->relax, (unsigned long long)n_elig);
}

}  // namespace gfb
