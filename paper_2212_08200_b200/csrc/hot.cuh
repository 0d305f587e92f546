// hot.cuh -- the advance kernels of gfb_sssp (neighbors_expand /
// neighbors_expand_pull with the SSSP relax, operators.hpp:35-68 / :76-114,
// algorithms.hpp:150-158).
//
//   k_push_range  push advance: warps claim TILE-edge tiles of the plan
//                 round-robin (merge-path style segment search by shuffles
//                 over a 32-segment window); record stream -> distance gather
//                 (test before atomic) -> fire-and-forget red.* of the
//                 distance, the packed (dist, pred) key and the frontier bit.
//                 Shapes (sssp.cu Runner::push): 32-bit distances one edge
//                 per lane, 6 CTAs per SM, the next 32-edge chunk's records
//                 in flight while the current chunk gathers (OPT 16),
//                 128-edge tiles for m <= 2^27, 256 above (opts.advance_tile
//                 overrides); REC (f64): returning 64-bit mins and {u, edge}
//                 records, same pipelined shape, 256-edge tiles; PEER
//                 (peer.cu): same shape, owner-addressed reductions.  range_expand<ENQ> is the tail
//                 kernel's variant (tail.cuh).
//   k_push_warp   warp-tile kernel with atomicMin-with-return; only the
//                 host-driven partitioned advance of mg.cu (PART) uses it.
//   k_pull_relax  pull over the CSC plan (CTA tiles in shared memory).
// Each step of the design is a measurement: profiles/r01_variants_s24.txt.
#pragma once

#include "kernels.cuh"

namespace gfb {

constexpr int H_BLOCK = 256;

// Packed predecessor key for 32-bit distances: (dist_bits << 32 | u).  One
// RED.MIN.64 keeps the pair jointly atomic (see k_push_range).
__device__ __forceinline__ unsigned long long pred_key(float d, uint32_t u) {
  return ((unsigned long long)__float_as_uint(d) << 32) | u;
}
__device__ __forceinline__ unsigned long long pred_key(uint32_t d, uint32_t u) {
  return ((unsigned long long)d << 32) | u;
}
// edges per thread per tile: 8 for 4-byte weights (2048-edge tiles), 4 for
// f64 (keeps the f64 kernels under the 48 KB static shared-memory limit)
template <class W> struct HotCfg {
  static constexpr int VT = sizeof(W) == 8 ? 4 : 8;
  static constexpr int TILE = H_BLOCK * VT;
  static constexpr int RATIO = TILE / PLAN_GRAIN;
  static_assert(TILE % PLAN_GRAIN == 0, "hot tile must be a multiple of the plan grain");
};

// Stage the plan segments of hot tile t and build the edge->segment map.
// Returns the number of edges in the tile.
template <int H_VT, class D>
__device__ __forceinline__ uint32_t hot_stage(const Plan& plan, const D* dist, uint32_t t,
                                              uint32_t ntiles, uint32_t total, uint32_t k,
                                              uint32_t* s_off, uint32_t* s_start, uint32_t* s_u,
                                              D* s_du, uint16_t* s_seg, bool load_du) {
  constexpr int H_TILE = H_BLOCK * H_VT, H_RATIO = H_TILE / PLAN_GRAIN;
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

template <class W, bool KEY = false>
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
        if constexpr (KEY) {  // fire-and-forget, as in k_push_range
          red_min_d(a.dist + u, best);
          atomicMin(reinterpret_cast<unsigned long long*>(a.predrec) + u,
                    pred_key(best, ld_rec(a.adj + sl).v));
          atomicOr(a.bm_out + (u >> 5), 1u << (u & 31));
          continue;
        }
        D old = atomic_min_d(a.dist + u, best);
        if (best < old) {
          a.predrec[u] = make_uint2(ld_rec(a.adj + sl).v, sl | PRED_CSC_SLOT);
          atomicOr(a.bm_out + (u >> 5), 1u << (u & 31));
        }
      }
    }
    __syncthreads();
  }
  n_elig = warp_sum(n_elig);
  if ((tid & 31) == 0 && n_elig) atomicAdd(&a.ctl->relax, (unsigned long long)n_elig);
}

// ---------------------------------------------------------------------------
// Warp-tile push advance (the default hot kernel).
//
// Every warp independently claims warp tiles of WT = 32*VT plan edges
// (persistent grid, no __syncthreads anywhere).  The plan segments (frontier
// vertices) intersecting the tile are processed in chunks of <= 32: lane j
// holds segment j's {first plan edge, row start, vertex, dist} in registers
// and every lane finds the segment of each of its edges with a 5-step
// shuffle search.  Edges are mapped lane-fastest, so each warp-wide record
// load is a contiguous run of 32 x 8 bytes; each lane keeps VT record loads,
// then VT distance gathers, then VT atomics in flight.
// ---------------------------------------------------------------------------
template <class D>
__device__ __forceinline__ D shfl_d(D x, int src) {
  return __shfl_sync(0xffffffffu, x, src);
}

template <class W, int VT, int MINB, bool PART = false>
__global__ void __launch_bounds__(256, MINB) k_push_warp(AdvArgs<W> a) {
  using D = typename DT<W>::D;
  constexpr int WT = 32 * VT;
  static_assert(WT % PLAN_GRAIN == 0 || PLAN_GRAIN % WT == 0, "warp tile vs plan grain");
  const int lane = threadIdx.x & 31;
  const uint32_t gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < a.status_len;
       i += gridDim.x * blockDim.x)
    a.status[i] = 0;
  const uint32_t total = a.ctl->total;
  const uint32_t k = a.ctl->k;
  unsigned* err = &a.ctl->err;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.ctl->relax += total;
    a.ctl->supersteps += 1;
    a.ctl->push_steps += 1;
  }
  const uint32_t ntiles = (total + WT - 1) / WT;
  for (uint32_t t = gwarp; t < ntiles; t += nwarps) {
    const uint32_t e0 = t * WT;
    const uint32_t e1 = min(e0 + WT, total);
    // first segment: the one holding edge e0 (tile map at PLAN_GRAIN)
    uint32_t sfirst;
    if (WT >= PLAN_GRAIN) {
      sfirst = a.plan.tseg[e0 / PLAN_GRAIN];
    } else {
      // finer tile than the map: search forward from the map entry
      uint32_t sj = a.plan.tseg[e0 / PLAN_GRAIN];
      for (;;) {  // warp-cooperative forward scan (segments are contiguous)
        uint32_t cand = sj + lane;
        uint32_t off = cand < k ? a.plan.off[cand + 1] : 0xFFFFFFFFu;  // end of cand
        unsigned m = __ballot_sync(0xffffffffu, cand < k && off > e0);
        if (m) {
          sfirst = sj + __ffs(m) - 1;
          break;
        }
        sj += 32;
      }
    }
    for (uint32_t cs = sfirst;; cs += 32) {  // chunks of <= 32 segments
      const uint32_t j = cs + lane;
      uint32_t off = 0xFFFFFFFFu, start = 0, u = 0;
      D du = D(0);
      if (j < k) {
        off = a.plan.off[j];
        start = a.plan.start[j];
        u = a.plan.v[j];
      }
      const uint32_t c0 = max(__shfl_sync(0xffffffffu, off, 0), e0);
      if (c0 >= e1) break;  // chunk starts past the tile
      if (j < k && off < e1) du = ld_dist(a.dist + u);
      // chunk end: first edge of segment cs+32 (or the tile end)
      uint32_t nxt = (cs + 32 < k) ? a.plan.off[cs + 32] : total;
      const uint32_t c1 = min(nxt, e1);
      for (uint32_t x = c0; x < c1; x += 32 * VT) {
        uint32_t dst[VT], eid[VT], srcl[VT];
        D nd[VT], cur[VT];
        unsigned long long rcur[PART ? VT : 1];
#pragma unroll
        for (int r = 0; r < VT; ++r) {  // A: segment search + record stream
          const uint32_t le = x + r * 32 + lane;
          dst[r] = NIL;
          int lo = 0;
#pragma unroll
          for (int step = 16; step >= 1; step >>= 1) {
            uint32_t o = __shfl_sync(0xffffffffu, off, lo + step);
            if (o <= le) lo += step;
          }
          uint32_t so = __shfl_sync(0xffffffffu, off, lo);
          uint32_t ss = __shfl_sync(0xffffffffu, start, lo);
          D sd = shfl_d(du, lo);
          srcl[r] = lo;
          if (le < c1) {
            eid[r] = ss + (le - so);
            EdgeRec<W> rec = ld_rec(a.adj + eid[r]);
            dst[r] = rec.v;
            nd[r] = dadd(sd, rec.w, err);
          }
        }
        if constexpr (!PART) {
#pragma unroll
          for (int r = 0; r < VT; ++r)  // B: distance gathers (test before atomic)
            if (dst[r] != NIL) cur[r] = ld_dist(a.dist + dst[r]);
#pragma unroll
          for (int r = 0; r < VT; ++r) {  // C: atomics on candidates
            if (dst[r] != NIL && nd[r] < cur[r]) cur[r] = atomic_min_d(a.dist + dst[r], nd[r]);
            else dst[r] = NIL;
          }
#pragma unroll
          for (int r = 0; r < VT; ++r) {  // D: winners
            uint32_t uu = __shfl_sync(0xffffffffu, u, srcl[r]);
            if (dst[r] != NIL && nd[r] < cur[r]) {
              a.predrec[dst[r]] = make_uint2(uu, eid[r]);
              atomicOr(a.bm_out + (dst[r] >> 5), 1u << (dst[r] & 31));
            }
          }
        } else {
          static_assert(sizeof(D) == 4, "partitioned mode packs 32-bit distances");
          const uint32_t span = a.hi - a.lo;
#pragma unroll
          for (int r = 0; r < VT; ++r) {  // B: local dist / remote staging gathers
            if (dst[r] == NIL) continue;
            if (dst[r] - a.lo < span) cur[r] = ld_dist(a.dist + (dst[r] - a.lo));
            else rcur[r] = a.rbest[dst[r]];
          }
#pragma unroll
          for (int r = 0; r < VT; ++r) {  // C + D
            const uint32_t uu = __shfl_sync(0xffffffffu, u, srcl[r]) + a.lo;  // global id
            if (dst[r] == NIL) continue;
            if (dst[r] - a.lo < span) {
              const uint32_t dl = dst[r] - a.lo;
              if (nd[r] < cur[r] && nd[r] < atomic_min_d(a.dist + dl, nd[r])) {
                a.predrec[dl] = make_uint2(uu, eid[r]);
                atomicOr(a.bm_out + (dl >> 5), 1u << (dl & 31));
              }
            } else {
              unsigned long long key =
                  ((unsigned long long)(*reinterpret_cast<uint32_t*>(&nd[r])) << 32) | uu;
              if (key < rcur[r] && key < atomicMin(a.rbest + dst[r], key))
                atomicOr(a.rbm + (dst[r] >> 5), 1u << (dst[r] & 31));
            }
          }
        }
      }
      if (c1 >= e1) break;
    }
  }
}


// ---------------------------------------------------------------------------
// Range push advance (the default hot kernel for 4-byte distances).
//
// Differences from k_push_warp, each removing a dependent memory round trip
// from the per-warp critical path (ncu of the dense s24 superstep: 66% of
// warp samples in long-scoreboard stalls, 49% occupancy, profiles/):
//  1. each warp owns ONE contiguous, equal share of the plan's edges instead
//     of strided 256-edge tiles, so the tile-map lookup and the segment
//     window setup (plan loads -> source-distance gather) happen once per 32
//     segments instead of once per 256 edges, and the next window's plan
//     entries are prefetched while the current one is expanded;
//  2. no atomic return values are waited on: a candidate that passes the
//     test-before-atomic (nd < dist[v]) proves dist[v] drops this superstep,
//     so it sets v's next-frontier bit itself (RED.OR) and lowers dist[v]
//     with RED.MIN.  The predecessor is a packed 64-bit key
//     (dist_bits << 32 | u) lowered with RED.MIN.64: after convergence the
//     key's high half equals dist[v] and its low half names an in-neighbour
//     whose final distance makes the edge tight (k_pred_verify<KEY>).
// ---------------------------------------------------------------------------

// Expand plan edges [e0, e1) with one warp (all lanes converged).
// COH: every load of data written earlier in the SAME launch (plan, source
// distances) goes through L2 (ld.cg) -- the persistent k_bsp crosses
// supersteps inside one kernel and L1 is not coherent across SMs.  The
// test-before-atomic gather may stay in L1: a stale (larger) value only
// costs a redundant reduction.
template <bool COH, class T>
__device__ __forceinline__ T ldc(const T* p) {
  if constexpr (COH) return __ldcg(p);
  else return *p;
}

// OPT bits (measured alternatives, tools/variants.py):
//   1: explicit PTX red.* (the compiler emits ATOMG ... RZ for unused atomics)
//   2: L2 evict_first hint on the predecessor-key reductions (128 MB at s24
//      that otherwise compete with the 64 MB distance array for L2)
//   4: L2 evict_last hint on the distance gathers and reductions
//   8: distance gathers through ld.global.nc
//  16: software-pipelined record loads (one edge per lane, no PEER / REC)
template <int OPT, class D>
__device__ __forceinline__ D test_gather(const D* p) {
  if constexpr ((OPT & 8) != 0) return __ldg(p);
  else if constexpr ((OPT & 4) != 0) {
    uint32_t v = ld_u32_hint(p, evict_last_policy());
    return *reinterpret_cast<D*>(&v);
  } else return ld_dist(p);
}

template <int OPT, class D>
__device__ __forceinline__ void relax_reds(D* dist, unsigned long long* pkey, uint32_t* bm,
                                           uint32_t v, D nd, uint32_t u) {
  if constexpr ((OPT & 1) != 0) {
    const uint32_t bits = *reinterpret_cast<uint32_t*>(&nd);
    if constexpr ((OPT & 4) != 0)
      red_min_u32_hint(reinterpret_cast<unsigned*>(dist + v), bits, evict_last_policy());
    else red_min_u32(reinterpret_cast<unsigned*>(dist + v), bits);
    if constexpr ((OPT & 2) != 0) red_min_u64_hint(pkey + v, pred_key(nd, u), evict_first_policy());
    else red_min_u64(pkey + v, pred_key(nd, u));
    red_or_u32(bm + (v >> 5), 1u << (v & 31));
  } else {
    red_min_d(dist + v, nd);
    atomicMin(pkey + v, pred_key(nd, u));
    atomicOr(bm + (v >> 5), 1u << (v & 31));
  }
}

// PEER: destinations are global ids owned by the ranks of the peer table
// (shared-memory copy `pt`): the test gather and the reductions go to the
// owner's slab (NVLink peer memory for remote owners), the packed key names
// the source by its global id.
// REC (f64 distances: no room for a packed key): the distance goes down with
// a returning 64-bit integer min on its bits (non-negative doubles order like
// their bit patterns); the relaxation that saw the old value above its own
// stores {u, csr edge} into predrec and sets the frontier bit.  A later,
// smaller relaxation may land its record first: k_pred_verify checks every
// record's tightness and the repair rounds fix the rest.
template <class W, int VT, bool COH = false, int OPT = 0, bool PEER = false, bool REC = false,
          bool ENQ = false>
__device__ __forceinline__ void range_expand(const AdvArgs<W>& a, uint32_t e0, uint32_t e1,
                                             uint32_t k, uint32_t total, unsigned* err,
                                             uint32_t* fmin = nullptr,
                                             const PeerTab* pt = nullptr) {
  using D = typename DT<W>::D;
  unsigned long long* pkey = reinterpret_cast<unsigned long long*>(a.predrec);
  const int lane = threadIdx.x & 31;
  // segment holding e0: tile-map entry, then a warp-cooperative forward scan
  uint32_t cs = ldc<COH>(a.plan.tseg + e0 / PLAN_GRAIN);
  for (;;) {
    uint32_t cand = cs + lane;
    // (the last segment ends at total: plans built in-kernel carry no off[k] sentinel)
    uint32_t end = cand + 1 < k ? ldc<COH>(a.plan.off + cand + 1) : total;
    unsigned msk = __ballot_sync(0xffffffffu, cand < k && end > e0);
    if (msk) {
      cs += __ffs(msk) - 1;
      break;
    }
    cs += 32;
  }
  // window = segments [cs, cs+32): lane j holds segment cs+j
  uint32_t off = 0xFFFFFFFFu, start = 0, u = 0;
  if (cs + lane < k) {
    off = ldc<COH>(a.plan.off + cs + lane);
    start = ldc<COH>(a.plan.start + cs + lane);
    u = ldc<COH>(a.plan.v + cs + lane);
  }
  D du = (cs + lane < k && off < e1) ? ldc<COH>(a.dist + u) : D(0);
  for (;;) {
    // prefetch the next window's plan entries (consumed after this window)
    const uint32_t nj = cs + 32 + lane;
    uint32_t noff = 0xFFFFFFFFu, nstart = 0, nu = 0;
    const bool more = __shfl_sync(0xffffffffu, off, 31) < e1 && cs + 32 < k;
    if (more && nj < k) {
      noff = ldc<COH>(a.plan.off + nj);
      nstart = ldc<COH>(a.plan.start + nj);
      nu = ldc<COH>(a.plan.v + nj);
    }
    const uint32_t nxt = cs + 32 < k ? (more ? __shfl_sync(0xffffffffu, noff, 0)
                                             : ldc<COH>(a.plan.off + cs + 32))
                                     : total;
    const uint32_t c0 = max(__shfl_sync(0xffffffffu, off, 0), e0);
    const uint32_t c1 = min(nxt, e1);
    if constexpr ((OPT & 16) != 0 && VT == 1) {
      // software-pipelined: the record of chunk x + 32 is in flight while
      // chunk x gathers and reduces (s24: 3.72 -> 3.55 ms together with 6
      // CTAs per SM; 8 CTAs per SM spill; two edges per lane or 4 CTAs per
      // SM are slower, profiles/r02_advance_variants.txt)
      // segment of each lane's edge by one OR-reduction of the window's
      // segment starts that fall in the chunk (bit p: a segment starts at
      // x + p) and a popcount, instead of a 5-step shuffle search: 3 SHFL per
      // 32 edges instead of 9 (they share the L1 data pipe with the gathers;
      // 3.49 -> 3.42 ms at s24)
      const uint32_t sbase = start - off;  // record index = sbase + plan edge
      int bj = __shfl_sync(0xffffffffu, off, 0) >= c0 ? -1 : 0;  // segment of edge c0 - 1
      auto fetch = [&](uint32_t x, EdgeRec<W>& rec, D& sd, uint32_t& su, uint32_t& se) {
        const uint32_t le = x + lane;
        const uint32_t p = off - x;  // (off >= x: unsigned wrap otherwise)
        const uint32_t mk = __reduce_or_sync(0xffffffffu, off >= x && p < 32u ? 1u << p : 0u);
        const int lo = bj + __popc(mk & (0xFFFFFFFFu >> (31 - lane)));
        bj += __popc(mk);
        const uint32_t sb = __shfl_sync(0xffffffffu, sbase, lo);
        sd = shfl_d(du, lo);
        su = __shfl_sync(0xffffffffu, u, lo);
        se = sb + le;  // the CSR edge (record mode)
        rec.v = NIL;
        if (le < c1) rec = ld_rec(a.adj + se);
      };
      EdgeRec<W> rec;
      D sd;
      uint32_t su, se;
      fetch(c0, rec, sd, su, se);
      for (uint32_t x = c0; x < c1; x += 32) {
        const uint32_t v = rec.v;
        // (only a loaded record: a lane past the chunk end holds no weight, and a
        // u32 sum with a stale register would raise the overflow flag)
        const D nd = v != NIL ? dadd(sd, rec.w, err) : D(0);
        const uint32_t uv = su, ev = se;
        if (x + 32 < c1) fetch(x + 32, rec, sd, su, se);
        if (v == NIL) continue;
        if constexpr (REC) {  // f64: returning min, the winner records {u, edge}
          const D cur = test_gather<OPT>(a.dist + v);
          if (nd < cur && nd < atomic_min_d(a.dist + v, nd)) {
            a.predrec[v] = make_uint2(uv, ev);
            red_or_u32(a.bm_out + (v >> 5), 1u << (v & 31));
            if (fmin) *fmin = min(*fmin, fkey(nd));
          }
        } else if constexpr (PEER) {  // owner-addressed (see the VT loop below)
          const uint32_t q = v >> PEER_VBITS;
          const uint32_t vl = v & PEER_VMASK;
          const uint32_t* tp = q == pt->self ? pt->dist[q] : pt->rc;
          const D cur = test_gather<OPT>(reinterpret_cast<const D*>(tp) + vl);
          if (nd < cur) {
            if (q != pt->self) red_min_u32(reinterpret_cast<unsigned*>(pt->rc + vl), dbits(nd));
            relax_reds<OPT>(reinterpret_cast<D*>(pt->dist[q]), pt->pkey[q], pt->bm[q], vl, nd,
                            uv + pt->self_lo);
            if (fmin) *fmin = min(*fmin, fkey(nd));
          }
        } else {
          const D cur = test_gather<OPT>(a.dist + v);
          if (nd < cur) {
            relax_reds<OPT>(a.dist, pkey, a.bm_out, v, nd, uv);
            if (fmin) *fmin = min(*fmin, fkey(nd));
          }
        }
      }
    } else
    for (uint32_t x = c0; x < c1; x += 32 * VT) {
      uint32_t dst[VT], uu[VT];
      uint32_t eid[REC ? VT : 1];
      D nd[VT], cur[VT];
#pragma unroll
      for (int r = 0; r < VT; ++r) {  // A: segment search + record stream
        const uint32_t le = x + r * 32 + lane;
        int lo = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
          uint32_t o = __shfl_sync(0xffffffffu, off, lo + step);
          if (o <= le) lo += step;
        }
        const uint32_t so = __shfl_sync(0xffffffffu, off, lo);
        const uint32_t ss = __shfl_sync(0xffffffffu, start, lo);
        const D sd = shfl_d(du, lo);
        uu[r] = __shfl_sync(0xffffffffu, u, lo);
        dst[r] = NIL;
        if (le < c1) {
          EdgeRec<W> rec = ld_rec(a.adj + (ss + (le - so)));
          dst[r] = rec.v;
          nd[r] = dadd(sd, rec.w, err);
          if constexpr (REC) eid[r] = ss + (le - so);
        }
      }
      if constexpr (REC) {
#pragma unroll
        for (int r = 0; r < VT; ++r)  // B: distance gathers (test before atomic)
          if (dst[r] != NIL) cur[r] = test_gather<OPT>(a.dist + dst[r]);
#pragma unroll
        for (int r = 0; r < VT; ++r) {  // C: returning mins, all in flight
          if (dst[r] != NIL && nd[r] < cur[r]) cur[r] = atomic_min_d(a.dist + dst[r], nd[r]);
          else dst[r] = NIL;
        }
#pragma unroll
        for (int r = 0; r < VT; ++r) {  // D: winners record themselves
          if constexpr (ENQ) {  // tail (tail.cuh): returning-OR dedup, warp-aggregated append
            bool fresh = false;
            if (dst[r] != NIL && nd[r] < cur[r]) {
              a.predrec[dst[r]] = make_uint2(uu[r], eid[r]);
              const uint32_t bit = 1u << (dst[r] & 31);
              fresh = (atomicOr(a.tq_bm + (dst[r] >> 5), bit) & bit) == 0;
            }
            const unsigned m = __ballot_sync(0xffffffffu, fresh);
            if (m) {
              const int leader = __ffs(m) - 1;
              uint32_t base = 0;
              if (lane == leader) base = atomicAdd(a.tq_cnt, (uint32_t)__popc(m));
              base = __shfl_sync(0xffffffffu, base, leader);
              if (fresh) a.tq_out[base + __popc(m & lanemask_lt())] = dst[r];
            }
          } else if (dst[r] != NIL && nd[r] < cur[r]) {
            a.predrec[dst[r]] = make_uint2(uu[r], eid[r]);
            red_or_u32(a.bm_out + (dst[r] >> 5), 1u << (dst[r] & 31));
            if (fmin) *fmin = min(*fmin, fkey(nd[r]));
          }
        }
      } else if constexpr (PEER) {
        uint32_t q[VT];
#pragma unroll
        for (int r = 0; r < VT; ++r) {  // B: owner; local test (own dist or proposal cache)
          if (dst[r] == NIL) continue;
          q[r] = dst[r] >> PEER_VBITS;  // owner-encoded id (k_peer_encode)
          dst[r] &= PEER_VMASK;
          const uint32_t* tp = q[r] == pt->self ? pt->dist[q[r]] : pt->rc;
          cur[r] = test_gather<OPT>(reinterpret_cast<const D*>(tp) + dst[r]);
        }
#pragma unroll
        for (int r = 0; r < VT; ++r) {  // C: reductions into the owner's slab
          if (dst[r] != NIL && nd[r] < cur[r]) {
            if (q[r] != pt->self)
              red_min_u32(reinterpret_cast<unsigned*>(pt->rc + dst[r]), dbits(nd[r]));
            relax_reds<OPT>(reinterpret_cast<D*>(pt->dist[q[r]]), pt->pkey[q[r]], pt->bm[q[r]],
                            dst[r], nd[r], uu[r] + pt->self_lo);
            if (fmin) *fmin = min(*fmin, fkey(nd[r]));
          }
        }
      } else {
#pragma unroll
      for (int r = 0; r < VT; ++r)  // B: distance gathers (test before atomic)
        if (dst[r] != NIL) cur[r] = test_gather<OPT>(a.dist + dst[r]);
#pragma unroll
      for (int r = 0; r < VT; ++r) {  // C: fire-and-forget reductions
        if constexpr (ENQ) {  // tail: dedup with a returning OR, warp-aggregated append
          bool fresh = false;
          if (dst[r] != NIL && nd[r] < cur[r]) {
            red_min_u32(reinterpret_cast<unsigned*>(a.dist + dst[r]), dbits(nd[r]));
            red_min_u64(pkey + dst[r], pred_key(nd[r], uu[r]));
            const uint32_t bit = 1u << (dst[r] & 31);
            fresh = (atomicOr(a.tq_bm + (dst[r] >> 5), bit) & bit) == 0;
          }
          const unsigned m = __ballot_sync(0xffffffffu, fresh);
          if (m) {
            const int leader = __ffs(m) - 1;
            uint32_t base = 0;
            if (lane == leader) base = atomicAdd(a.tq_cnt, (uint32_t)__popc(m));
            base = __shfl_sync(0xffffffffu, base, leader);
            if (fresh) a.tq_out[base + __popc(m & lanemask_lt())] = dst[r];
          }
        } else if (dst[r] != NIL && nd[r] < cur[r]) {
          relax_reds<OPT>(a.dist, pkey, a.bm_out, dst[r], nd[r], uu[r]);
          if (fmin) *fmin = min(*fmin, fkey(nd[r]));  // for the distance-ordered plan
        }
      }
      }
    }
    if (c1 >= e1) break;
    cs += 32;
    off = noff;
    start = nstart;
    u = nu;
    du = (nj < k && noff < e1) ? ldc<COH>(a.dist + nu) : D(0);
  }
}

// TILE == 0: one contiguous equal share of the plan per warp.  TILE > 0:
// warps claim TILE-edge tiles round-robin, so the whole grid sweeps the plan
// in ascending vertex order.  On unpermuted RMAT the low ids are the hubs
// with the smallest distances: relaxing them first lets their improvements
// reach later edges of the SAME superstep (measured: contiguous shares do
// 4.4 relaxations per reached edge at s24, the sweep 3.5).
template <class W, int VT, int MINB, int TILE, int OPT = 0, bool PEER = false, bool REC = false>
__global__ void __launch_bounds__(256, MINB) k_push_range(AdvArgs<W> a) {
  using D = typename DT<W>::D;
  static_assert(REC || sizeof(D) == 4, "packed predecessor keys need 32-bit distances");
  static_assert(TILE % 32 == 0, "tiles are whole warp rows");
  __shared__ PeerTab s_pt[1];  // (eliminated when !PEER)
  if constexpr (PEER) {  // the peer table in shared memory (indexed per edge)
    constexpr int WORDS = sizeof(PeerTab) / 4;
    for (int i = threadIdx.x; i < WORDS; i += blockDim.x)
      reinterpret_cast<uint32_t*>(s_pt)[i] = reinterpret_cast<const uint32_t*>(a.peers)[i];
    __syncthreads();
  }
  const uint32_t gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const uint32_t total = a.ctl->total;
  const uint32_t k = a.ctl->k;
  unsigned* err = &a.ctl->err;
  if (blockIdx.x == 0 && threadIdx.x == 0 && total) {  // (empty after a tail hand-back)
    a.ctl->relax += total;
    a.ctl->supersteps += 1;
    a.ctl->push_steps += 1;
  }
  uint32_t fmin = 0xFFFFFFFFu;
  if constexpr (TILE == 0) {
    const uint32_t per = (uint32_t)((((uint64_t)total + nwarps - 1) / nwarps + 31) & ~31ull);
    const uint32_t e0 = (uint32_t)min((uint64_t)gwarp * per, (uint64_t)total);
    const uint32_t e1 = min(e0 + per, total);
    if (e0 < e1) range_expand<W, VT, false, OPT, PEER, REC>(a, e0, e1, k, total, err, &fmin, s_pt);
  } else {
    for (uint64_t e0 = (uint64_t)gwarp * TILE; e0 < total; e0 += (uint64_t)nwarps * TILE)
      range_expand<W, VT, false, OPT, PEER, REC>(a, (uint32_t)e0,
                                             (uint32_t)min(e0 + TILE, (uint64_t)total), k, total,
                                             err, &fmin, s_pt);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) fmin = min(fmin, __shfl_xor_sync(0xffffffffu, fmin, d));
  if ((threadIdx.x & 31) == 0 && fmin != 0xFFFFFFFFu) atomicMin(&a.ctl->fmin, fmin);
}

}  // namespace gfb
