// frontier.cuh -- next-frontier bitmap -> expansion plan for the SSSP loop
// (the filter/uniquify step, operators.hpp:191-200 + frontier.hpp:147-165:
// bitmap dedup, ascending order) as three launches with static tiles:
//
//   k_fcount  per 2048-vertex tile: warp-ballot count of set bits with
//             out-degree > 0 and their degree sum -> agg[tile]
//   k_fscan   one CTA: exclusive scan of agg -> tile prefixes; plan totals,
//             relaxation/superstep bookkeeping and the loop condition
//   k_fwrite  per tile: recount, place each kept vertex at its global
//             position (ascending), edge offsets, tile-map entries; copy the
//             word to the current-frontier bitmap and clear it
//
// No global atomics and no look-back chain: the single-pass k_compact
// (kernels.cuh) serialised 8192 CTAs on one tile counter (~50-100 us per
// superstep at scale 24, profiles/r01_launches.md).
#pragma once

#include "kernels.cuh"

namespace gfb {

// (measured: 4 x 16, 8 x 16 and 16 x 4 warps x words are 3-17% slower at s24)
constexpr int F_WARPS = 8;
constexpr int F_WPW = 8;                     // bitmap words per warp
constexpr int F_WORDS = F_WARPS * F_WPW;     // 64 words = 2048 vertices per tile
constexpr int F_SCAN_THREADS = 1024;

// The 8 words of this warp -> per-word (mask of kept bits, row start, degree)
// (plain compaction of bfs.cu; the ordered filter below loads in halves).
struct WarpWords {
  uint32_t keep[F_WPW];
  uint32_t st[F_WPW];
  uint32_t deg[F_WPW];
};

template <bool COH = false>
__device__ __forceinline__ void load_warp_words(const uint32_t* __restrict__ ro,
                                                const uint32_t* bm, uint32_t nwords,
                                                uint32_t wbase, WarpWords& w, uint32_t* raw_word) {
  const int lane = threadIdx.x & 31;
  uint32_t my = 0;
  if (lane < F_WPW && wbase + lane < nwords) my = COH ? __ldcg(bm + wbase + lane) : bm[wbase + lane];
  *raw_word = my;
  uint32_t words[F_WPW];
#pragma unroll
  for (int j = 0; j < F_WPW; ++j) words[j] = __shfl_sync(0xffffffffu, my, j);
  // issue every row-offset load before consuming any (F_WPW x 2 in flight)
#pragma unroll
  for (int j = 0; j < F_WPW; ++j) {
    bool bit = (words[j] >> lane) & 1u;
    uint32_t v = (wbase + j) * 32 + lane;
    w.st[j] = bit ? ro[v] : 0u;
    w.deg[j] = bit ? ro[v + 1] : 0u;
  }
#pragma unroll
  for (int j = 0; j < F_WPW; ++j) {
    bool bit = (words[j] >> lane) & 1u;
    w.deg[j] = bit ? w.deg[j] - w.st[j] : 0u;
    w.keep[j] = __ballot_sync(0xffffffffu, w.deg[j] > 0);
  }
}

// Tile-map entries tseg[b] = gi for every b*PLAN_GRAIN in [eoff, eoff+deg)
// of each lane's segment, written by the whole warp: a hub owns thousands of
// entries, and one lane looping over them serialises the warp (used by the
// persistent k_bsp, whose hub CTA owns most of them).
__device__ __forceinline__ void warp_tile_map(const Plan& plan, uint32_t gi, uint32_t eoff,
                                              uint32_t deg) {
  const int lane = threadIdx.x & 31;
  const uint32_t b0 = (eoff + PLAN_GRAIN - 1) / PLAN_GRAIN;
  const uint32_t b1 = deg ? (eoff + deg + PLAN_GRAIN - 1) / PLAN_GRAIN : b0;
  const uint32_t cnt = b1 - b0;
  const uint32_t cincl = warp_incl_scan(cnt, lane);
  const uint32_t ctot = __shfl_sync(0xffffffffu, cincl, 31);
  if (ctot == 0) return;  // warp-uniform
  const uint32_t cpre = cincl - cnt;
  for (uint32_t x = lane; x - lane < ctot; x += 32) {
    int lo = 0;  // owner lane: the first whose inclusive count exceeds x
#pragma unroll
    for (int step = 16; step >= 1; step >>= 1) {
      const uint32_t p = __shfl_sync(0xffffffffu, cincl, lo + step - 1);
      if (p <= x) lo += step;
    }
    const uint32_t ob0 = __shfl_sync(0xffffffffu, b0, lo);
    const uint32_t opre = __shfl_sync(0xffffffffu, cpre, lo);
    const uint32_t ogi = __shfl_sync(0xffffffffu, gi, lo);
    const uint32_t bb = ob0 + (x - opre);
    if (x < ctot && bb < plan.tseg_cap) plan.tseg[bb] = ogi;
  }
}

static __global__ void __launch_bounds__(F_WARPS * 32)
k_fcount(const uint32_t* __restrict__ ro, const uint32_t* __restrict__ bm, uint32_t nwords,
         uint2* agg) {
  __shared__ uint32_t s_c[F_WARPS], s_e[F_WARPS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpWords w;
  uint32_t raw;
  load_warp_words(ro, bm, nwords, blockIdx.x * F_WORDS + warp * F_WPW, w, &raw);
  uint32_t c = 0, e = 0;
#pragma unroll
  for (int j = 0; j < F_WPW; ++j) {
    c += __popc(w.keep[j]);
    e += w.deg[j];
  }
  e = warp_sum(e);
  if (lane == 0) {
    s_c[warp] = c;
    s_e[warp] = e;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t tc = 0, te = 0;
    for (int i = 0; i < F_WARPS; ++i) {
      tc += s_c[i];
      te += s_e[i];
    }
    agg[blockIdx.x] = make_uint2(tc, te);
  }
}

// Plan totals K (vertices) / T (edges) -> sentinels, bookkeeping, the
// push/pull decision and the device loop's conditionals (one thread).
__device__ __forceinline__ void plan_totals(uint32_t K, uint32_t T, Plan plan, Ctl* ctl,
                                            uint32_t m, float alpha, int can_pull, int force_pull,
                                            cudaGraphConditionalHandle loop_handle,
                                            cudaGraphConditionalHandle mode_handle, int set_loop,
                                            int set_mode) {
  ctl->k = K;
  ctl->total = T;
  plan.off[K] = T;
  const uint32_t sb = (T + PLAN_GRAIN - 1) / PLAN_GRAIN;
  if (sb < plan.tseg_cap) plan.tseg[sb] = K;
  const uint32_t mode = (force_pull || (can_pull && (float)T > (float)m / alpha)) ? 1u : 0u;
  ctl->mode = mode;
  // distance-ordered plan: freeze this frontier's minimum for k_fwrite_o and
  // open the next advance's
  ctl->blo = ctl->fmin;
  ctl->fmin = 0xFFFFFFFFu;
  // device loop: WHILE(K > 0) and the IF(pull) of the next body iteration
  if (set_loop) cudaGraphSetConditional(loop_handle, K > 0 ? 1u : 0u);
  if (set_mode) cudaGraphSetConditional(mode_handle, mode);
}

// One CTA.  agg -> exclusive prefixes (in place), plan totals, bookkeeping.
// ctl->mode: direction of the next superstep (1 = pull when the plan's edges
// exceed m / alpha and a CSC exists -- the push<->pull switch).
static __global__ void __launch_bounds__(F_SCAN_THREADS)
k_fscan(uint2* agg, uint32_t tiles, Plan plan, Ctl* ctl, uint32_t m, float alpha, int can_pull,
        int force_pull, cudaGraphConditionalHandle loop_handle,
        cudaGraphConditionalHandle mode_handle, int set_loop, int set_mode) {
  __shared__ uint32_t s_c[F_SCAN_THREADS / 32], s_e[F_SCAN_THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t per = (tiles + F_SCAN_THREADS - 1) / F_SCAN_THREADS;
  const uint32_t lo = tid * per, hi = min(lo + per, tiles);
  uint32_t c = 0, e = 0;
  for (uint32_t i = lo; i < hi; ++i) {
    uint2 a = agg[i];
    c += a.x;
    e += a.y;
  }
  uint32_t ic = warp_incl_scan(c, lane), ie = warp_incl_scan(e, lane);
  if (lane == 31) {
    s_c[warp] = ic;
    s_e[warp] = ie;
  }
  __syncthreads();
  if (warp == 0) {
    uint32_t wc = s_c[lane], we = s_e[lane];
    uint32_t xc = warp_incl_scan(wc, lane), xe = warp_incl_scan(we, lane);
    s_c[lane] = xc - wc;
    s_e[lane] = xe - we;
  }
  __syncthreads();
  uint32_t pc = s_c[warp] + ic - c, pe = s_e[warp] + ie - e;
  for (uint32_t i = lo; i < hi; ++i) {
    uint2 a = agg[i];
    agg[i] = make_uint2(pc, pe);
    pc += a.x;
    pe += a.y;
  }
  if (tid == F_SCAN_THREADS - 1)  // pc/pe are now the grand totals
    plan_totals(pc, pe, plan, ctl, m, alpha, can_pull, force_pull, loop_handle, mode_handle,
                set_loop, set_mode);
}

static __global__ void __launch_bounds__(F_WARPS * 32)
k_fwrite(const uint32_t* __restrict__ ro, uint32_t* bm_next, uint32_t* bm_cur, uint32_t nwords,
         const uint2* __restrict__ prefix, Plan plan) {
  __shared__ uint32_t s_c[F_WARPS], s_e[F_WARPS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t wbase = blockIdx.x * F_WORDS + warp * F_WPW;
  WarpWords w;
  uint32_t raw;
  load_warp_words(ro, bm_next, nwords, wbase, w, &raw);
  if (lane < F_WPW && wbase + lane < nwords) {
    if (bm_cur) bm_cur[wbase + lane] = raw;
    bm_next[wbase + lane] = 0;
  }
  uint32_t c = 0, e = 0;
#pragma unroll
  for (int j = 0; j < F_WPW; ++j) {
    c += __popc(w.keep[j]);
    e += w.deg[j];
  }
  e = warp_sum(e);
  if (lane == 0) {
    s_c[warp] = c;
    s_e[warp] = e;
  }
  __syncthreads();
  const uint2 tp = prefix[blockIdx.x];
  uint32_t gc = tp.x, ge = tp.y;
  for (int i = 0; i < warp; ++i) {
    gc += s_c[i];
    ge += s_e[i];
  }
#pragma unroll
  for (int j = 0; j < F_WPW; ++j) {
    const uint32_t keep = w.keep[j];
    if (keep == 0) continue;  // warp-uniform
    const bool mine = (keep >> lane) & 1u;
    const uint32_t incl = warp_incl_scan(w.deg[j], lane);
    if (mine) {  // per-lane tile map: cheaper here than warp_tile_map (8192 small CTAs)
      const uint32_t gi = gc + __popc(keep & lanemask_lt());
      const uint32_t eoff = ge + incl - w.deg[j];
      plan.v[gi] = (wbase + j) * 32 + lane;
      plan.start[gi] = w.st[j];
      plan.off[gi] = eoff;
      tile_map_entries(plan, gi, eoff, w.deg[j]);
    }
    gc += __popc(keep);
    ge += __shfl_sync(0xffffffffu, incl, 31);
  }
}

// ---------------------------------------------------------------------------
// Distance-ordered compaction (the default for 32-bit distances).
//
// The plan is laid out bucket-major: OB_N log-scale distance buckets above
// the frontier's smallest activation distance; inside a bucket, cells of
// 2048-vertex tiles in reservation order, arbitrary order inside a cell.  The push advance sweeps the plan roughly in order across the
// grid, so the closest vertices relax first and their improvements reach the
// rest of the same superstep (Gauss-Seidel within BSP).  Measured at RMAT s24
// with an exact sort (tools/order_exp.py): 3.53 -> 2.78 relaxations per
// reached edge; quarter-octave keys 2.82, whole octaves 2.96; descending
// distance 4.93.  Equal-width buckets over [min, max] gained nothing: the
// interesting spread is logarithmic.
// Each tile reserves its (slot, edge) range per bucket with one global 64-bit
// atomic per nonzero cell; inside the tile one shared 64-bit cursor per
// bucket hands out consistent (slot, edge offset) pairs.  Half-octave
// buckets, 32 of them = 16 octaves above the frontier minimum.
// ---------------------------------------------------------------------------
constexpr int OB_N = 32;          // buckets: 16 octaves above the minimum
constexpr int OB_SHIFT = 22;      // float bits >> 22 = exponent + 1 mantissa bit (half octaves)

// Default deferral cut: in a superstep whose frontier has >= m/4 edges only
// the closest distance buckets up to DEFER_PCT% of its edges are expanded.
// Re-swept on the final loop (RMAT s24 / s22, ms): 3% 3.82 / 1.38, 5% 3.85 /
// 1.36, 10% 3.92 / 1.42, 15% 3.99, 20% 4.50, 30% 4.72 (tools/variants.py).
constexpr uint32_t DEFER_PCT = 5;

__device__ __forceinline__ uint32_t obucket_k(uint32_t fk, uint32_t base) {
  const uint32_t k = fk >> OB_SHIFT;
  return k <= base ? 0u : min(k - base, (uint32_t)OB_N - 1);
}

// Partitioned loop (peer.cu): remote relaxations set the owner's remote
// frontier bitmap (rbm) without knowing whether they lowered its distance
// (the sender tested against its own proposal cache).  dexp[v] = distance
// bits v was last expanded with; in the count and write passes below a bit
// set ONLY remotely whose distance is unchanged is dropped.  Local bits come
// from relaxations that lowered v and need no check (one rank: none of the
// dexp reads).  DEXP = false: single GPU.

// Count: per tile (the F_WORDS-word tiles of k_fcount) and bucket -> agg,
// and the bucket totals accumulated in btot[OB_N] (64-bit: count << 32 | edges).
// Native 32-bit shared atomics (a 64-bit shared atomicAdd is a CAS loop).
template <class D, bool DEXP = false>
// (8 CTAs per SM: 32 registers, full occupancy -- 1% faster at s24 than 40)
__global__ void __launch_bounds__(F_WARPS * 32, 8)
k_fcount_o(const uint32_t* __restrict__ ro, const uint32_t* __restrict__ bm, uint32_t nwords,
           const D* __restrict__ dist, const Ctl* __restrict__ ctl,
           unsigned long long* agg, unsigned long long* btot, uint32_t* tflag,
           const uint32_t* dexp = nullptr, const uint32_t* rbm = nullptr) {
  __shared__ uint32_t s_c[OB_N], s_e[OB_N];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < OB_N) s_c[threadIdx.x] = s_e[threadIdx.x] = 0;
  const uint32_t base = ctl->fmin >> OB_SHIFT;
  const uint32_t wbase = blockIdx.x * F_WORDS + warp * F_WPW;
  // the tile's words in two halves of F_WPW / 2: 12 loads in flight per
  // lane and no register spills at the 32-register cap (one batch of 8
  // words spilled: s24 3.36 -> 3.26 ms with the halves); the bitmap words
  // are loaded before the barrier that publishes the cleared counters
  uint32_t raw, chk = 0;
  {
    uint32_t my = 0;
    if (lane < F_WPW && wbase + lane < nwords) {
      my = bm[wbase + lane];
      if (DEXP && rbm) {  // peers' bits: checked against dexp below
        const uint32_t r = rbm[wbase + lane];
        chk = r & ~my;
        my |= r;
      }
    }
    raw = my;
    __syncthreads();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      constexpr int HW = F_WPW / 2;
      uint32_t st[HW], en[HW];
      D dv[HW];
#pragma unroll
      for (int q = 0; q < HW; ++q) {
        const int j = h * HW + q;
        const bool bit = (__shfl_sync(0xffffffffu, my, j) >> lane) & 1u;
        const uint32_t v = (wbase + j) * 32 + lane;
        st[q] = bit ? ro[v] : 0u;
        en[q] = bit ? ro[v + 1] : 0u;
        dv[q] = bit ? dist[v] : D(0);
      }
#pragma unroll
      for (int q = 0; q < HW; ++q) {
        const int j = h * HW + q;
        const uint32_t deg = en[q] - st[q];
        bool kept = deg > 0;
        if constexpr (DEXP) {  // a bit set only by peers: did the distance move?
          const uint32_t cw = __shfl_sync(0xffffffffu, chk, j);
          if (kept && ((cw >> lane) & 1u)) kept = dbits(dv[q]) != dexp[(wbase + j) * 32 + lane];
        }
        if (kept) {
          const uint32_t b = obucket_k(fkey(dv[q]), base);
          atomicAdd(&s_c[b], 1u);
          atomicAdd(&s_e[b], deg);
        }
      }
    }
  }
  // any bit in this tile at all: k_fwrite_o skips tiles without one
  // (+2: remotely set bits to merge -- no all-deferred shortcut)
  const int any = __syncthreads_or(raw != 0);
  const int anyr = DEXP ? __syncthreads_or(chk != 0) : 0;
  if (threadIdx.x == 0) tflag[blockIdx.x] = any | (anyr << 1);
  if (threadIdx.x < OB_N) {
    const unsigned long long x = ((unsigned long long)s_c[threadIdx.x] << 32) | s_e[threadIdx.x];
    agg[(size_t)blockIdx.x * OB_N + threadIdx.x] = x;
    if (x) atomicAdd(btot + threadIdx.x, x);
  }
}

// Bucket totals -> bucket cursors (exclusive scan), plan totals, bookkeeping.
// One warp.  btot is cleared for the next superstep.
// defer_pct < 100: buckets past the one where the cumulative frontier edges
// reach defer_pct% stay pending in the bitmap for the next superstep (a soft
// near-far split inside BSP), when the frontier has >= defer_min edges.
static __global__ void k_fscan_o(unsigned long long* btot, unsigned long long* bcur, Plan plan,
                                 Ctl* ctl, uint32_t m, float alpha, int can_pull, int force_pull,
                                 cudaGraphConditionalHandle loop_handle,
                                 cudaGraphConditionalHandle mode_handle, int set_loop,
                                 int set_mode, uint32_t defer_pct = 100,
                                 uint32_t defer_min = 0,
                                 cudaGraphConditionalHandle tail_handle = {}, int set_tail = 0,
                                 uint32_t tail_edges = 0) {
  const int lane = threadIdx.x;
  static_assert(OB_N <= 32, "one warp scans the bucket totals");
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (PDL launch: the count's totals)
  const unsigned long long x = lane < OB_N ? btot[lane] : 0ull;
  unsigned long long incl = x;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += y;
  }
  const unsigned long long all = __shfl_sync(0xffffffffu, incl, 31);
  const uint32_t T_all = (uint32_t)all;
  uint32_t cut = OB_N - 1;
  if (defer_pct < 100 && T_all >= defer_min) {
    // first bucket whose inclusive edge count reaches defer_pct% of all
    const uint64_t need = (uint64_t)T_all * defer_pct;
    const bool reach = (uint64_t)(uint32_t)incl * 100 >= need;
    const unsigned bal = __ballot_sync(0xffffffffu, reach && lane < OB_N);
    if (bal) cut = __ffs(bal) - 1;
  }
  const unsigned long long upto = __shfl_sync(0xffffffffu, incl, cut);
  if (lane < OB_N) {
    bcur[lane] = incl - x;
    btot[lane] = 0;
  }
  if (lane == 31) {
    ctl->bcut = cut;
    ctl->k_all = (uint32_t)(all >> 32);
    ctl->t_all = T_all;
    plan_totals((uint32_t)(upto >> 32), (uint32_t)upto, plan, ctl, m, alpha, can_pull,
                force_pull, loop_handle, mode_handle, set_loop, set_mode);
    // small plan, nothing deferred: the next superstep starts the tail kernel
    // (not from the source's plan: its output is unknown -- the hub phase of
    // a skewed graph must keep the deferral)
    const uint32_t tail = tail_edges && ctl->supersteps > 0 && (upto >> 32) > 0 &&
                          upto == all && (uint32_t)upto < tail_edges ? 1u : 0u;
    ctl->tail = tail;
    if (set_tail) cudaGraphSetConditional(tail_handle, tail);
  }
}

// Write: each tile reserves its cell in every bucket up to the cut (one
// global atomic per nonzero cell); a lane's rank in its cell comes from a
// native 32-bit shared atomic, v/start go straight to their slots, and the
// edge offsets come from one block scan over the tile's degrees staged
// bucket-major in shared memory.  Deferred vertices keep their bitmap bit.
// (Measured alternatives: per-lane 64-bit shared cursors -- a CAS loop --
// 1-5% slower; full staging of v/start/deg 1.2x; a warp-aggregated atomic per
// distinct bucket of a word 2.1x.)
// (__launch_bounds__ minimum 7 CTAs/SM: 32 registers instead of 56 -- s24
// 3.38 -> 3.33 ms; 6 / 8: 3.36 / 3.36, r02_rejected_filter_variants.txt)
template <class D, bool DEXP = false>
__global__ void __launch_bounds__(F_WARPS * 32, 7)
k_fwrite_o(const uint32_t* __restrict__ ro, uint32_t* bm_next, uint32_t* bm_cur, uint32_t nwords,
            const D* __restrict__ dist, const Ctl* __restrict__ ctl,
            const unsigned long long* __restrict__ agg, unsigned long long* bcur, Plan plan,
            const uint32_t* __restrict__ tflag, uint32_t* dexp = nullptr,
            uint32_t* rbm = nullptr) {
  constexpr int TV = F_WORDS * 32, NT = F_WARPS * 32, VT = TV / NT;
  __shared__ uint32_t s_cb[OB_N], s_ce[OB_N], s_lb[OB_N], s_rank[OB_N];
  __shared__ uint32_t s_deg[TV], s_pre[TV];
  __shared__ uint8_t s_bk[TV];
  __shared__ uint32_t s_ws[F_WARPS + 1];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (PDL launch: the scan's cursors)
  const uint32_t tf = tflag[blockIdx.x];
  if (!tf) return;  // empty tile: nothing to place or clear
  const uint32_t cut = ctl->bcut;
  if (warp == 0) {
    const unsigned long long x =
        lane < OB_N && (uint32_t)lane <= cut ? agg[(size_t)blockIdx.x * OB_N + lane] : 0ull;
    const uint32_t cnt = (uint32_t)(x >> 32);
    const uint32_t incl = warp_incl_scan(cnt, lane);
    if (lane < OB_N) {
      const unsigned long long g = x ? atomicAdd(bcur + lane, x) : 0ull;
      s_cb[lane] = (uint32_t)(g >> 32);
      s_ce[lane] = (uint32_t)g;
      s_lb[lane] = incl - cnt;
      s_rank[lane] = 0;
    }
    if (lane == 31) s_ws[F_WARPS] = incl;  // placed vertices of this tile
  }
  const uint32_t base = ctl->blo >> OB_SHIFT;
  const uint32_t wbase = blockIdx.x * F_WORDS + warp * F_WPW;
  // this warp's bitmap words, loaded while warp 0 reserves the cells
  uint32_t my = 0, chk = 0;
  if (lane < F_WPW && wbase + lane < nwords) {
    my = bm_next[wbase + lane];
    if (DEXP && rbm && (tf & 2u)) {
      const uint32_t r = rbm[wbase + lane];
      chk = r & ~my;
      my |= r;
    }
  }
  // a tile whose set bits are all deferred: no row offsets / distances to
  // load, its bitmap words stay (degree-0 bits included: the count pass
  // ignores them), only the placed-set bitmap is cleared (s24: 3.43 -> 3.39 ms)
  __syncthreads();
  if (s_ws[F_WARPS] == 0 && (tf & 2u) == 0) {
    if (bm_cur && lane < F_WPW && wbase + lane < nwords) bm_cur[wbase + lane] = 0;
    return;
  }
  uint32_t raw, pend = 0;
  // place one word's vertices (b: bucket of kept lanes)
  auto place_word = [&](int j, bool kept, uint32_t b, uint32_t st, uint32_t deg) {
    const uint32_t v = (wbase + j) * 32 + lane;
    const bool place = kept && b <= cut;
    const unsigned dm = __ballot_sync(0xffffffffu, kept && !place);
    if (lane == j) pend = dm;
    if (place) {
      const uint32_t r = atomicAdd(&s_rank[b], 1u);
      const uint32_t p = s_lb[b] + r;
      const uint32_t gi = s_cb[b] + r;
      s_deg[p] = deg;
      s_bk[p] = (uint8_t)b;
      plan.v[gi] = v;
      plan.start[gi] = st;
      if constexpr (DEXP) {
        if (dexp) dexp[v] = dbits(dist[v]);
      }
    }
  };
  // two halves of F_WPW / 2 words, loads then placements (no spills at the
  // 32-register cap, like k_fcount_o: s24 3.26 -> 3.20 ms)
  {
    raw = my;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      constexpr int HW = F_WPW / 2;
      uint32_t st[HW], en[HW];
      D dv[HW];
#pragma unroll
      for (int q = 0; q < HW; ++q) {
        const int j = h * HW + q;
        const bool bit = (__shfl_sync(0xffffffffu, my, j) >> lane) & 1u;
        const uint32_t v = (wbase + j) * 32 + lane;
        st[q] = bit ? ro[v] : 0u;
        en[q] = bit ? ro[v + 1] : 0u;
        dv[q] = bit ? dist[v] : D(0);
      }
#pragma unroll
      for (int q = 0; q < HW; ++q) {
        const int j = h * HW + q;
        const uint32_t deg = en[q] - st[q];
        bool kept = deg > 0;
        if constexpr (DEXP) {
          const uint32_t cw = __shfl_sync(0xffffffffu, chk, j);
          if (kept && ((cw >> lane) & 1u)) kept = dbits(dv[q]) != dexp[(wbase + j) * 32 + lane];
        }
        place_word(j, kept, kept ? obucket_k(fkey(dv[q]), base) : 0u, st[q], deg);
      }
    }
  }
  if (lane < F_WPW && wbase + lane < nwords) {
    if (bm_cur) bm_cur[wbase + lane] = raw & ~pend;
    bm_next[wbase + lane] = pend;
    if (DEXP && rbm && (tf & 2u)) rbm[wbase + lane] = 0;  // merged (or dropped)
  }
  __syncthreads();
  const uint32_t placed = s_ws[F_WARPS];
  if (placed == 0) return;  // block-uniform
  // exclusive scan of the staged degrees (VT consecutive positions per thread)
  uint32_t d[VT], tsum = 0;
#pragma unroll
  for (int r = 0; r < VT; ++r) {
    const uint32_t p = tid * VT + r;
    d[r] = p < placed ? s_deg[p] : 0u;
    tsum += d[r];
  }
  const uint32_t incl = warp_incl_scan(tsum, lane);
  if (lane == 31) s_ws[warp] = incl;
  __syncthreads();
  uint32_t run = incl - tsum;
  for (int i = 0; i < warp; ++i) run += s_ws[i];
#pragma unroll
  for (int r = 0; r < VT; ++r) {
    s_pre[tid * VT + r] = run;
    run += d[r];
  }
  __syncthreads();
  for (uint32_t p = tid; p < placed; p += NT) {  // cells are contiguous slots
    const uint32_t b = s_bk[p];
    const uint32_t r = p - s_lb[b];
    const uint32_t gi = s_cb[b] + r;
    const uint32_t eoff = s_ce[b] + (s_pre[p] - s_pre[s_lb[b]]);
    plan.off[gi] = eoff;
    tile_map_entries(plan, gi, eoff, s_deg[p]);
  }
}

}  // namespace gfb
