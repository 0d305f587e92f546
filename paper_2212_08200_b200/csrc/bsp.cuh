// bsp.cuh -- the whole BSP loop of sssp() (algorithms.hpp:569-623) as ONE
// persistent cooperative kernel for 32-bit distances.
//
//   init (algorithms.hpp:579-583)                                  | sync
//   loop:  count   frontier bitmap -> per-CTA (vertices, edges)    | sync
//          write   CTA prefix -> ascending plan + tile map; the    | sync
//                  while (f.size() != 0) test (:602) and the push/
//                  pull decision are computed redundantly by every
//                  CTA from the per-CTA totals (no host round trip)
//          advance push (range_expand, hot.cuh) or warp-level pull | sync
//
// Every CTA is resident (cudaLaunchCooperativeKernel, grid = SMs x
// resident CTAs per SM), so a superstep costs three grid barriers instead of
// four kernel launches (count / scan / write / advance: 40-60 us per
// superstep at scale 24 in profiles/r01_launches_v20.txt, ~30% of the
// device time once the advance ran at ~200 G edges/s).
#pragma once

#include <cooperative_groups.h>

#include "frontier.cuh"
#include "hot.cuh"

namespace cg = cooperative_groups;

namespace gfb {

constexpr int B_THREADS = 1024;            // 2 resident CTAs per SM (64 warps)
constexpr int B_WARPS = B_THREADS / 32;
constexpr int B_MAX_GROUPS = 2 * B_THREADS;  // 8-word groups per CTA (n <= 155M at 296 CTAs)
constexpr int BAR_GROUP = 16;              // CTAs per first-level barrier counter
constexpr int BAR_WORDS = 2 + 64;          // [0] generation, [1] top count, [2..] groups

template <class W>
struct BspArgs {
  AdvArgs<W> push, pull;  // push: CSR + workspace plan; pull: CSC + static pull plan
  const uint32_t* ro;
  const uint32_t* nz;     // bit v: out-degree(v) > 0 (static per graph)
  uint32_t* bm_cur;       // = pull.bm_in (writable alias)
  uint32_t n, nwords, m;
  uint32_t pull_total, pull_k;
  uint2* agg;             // per-CTA (vertices, edges) of the frontier
  unsigned* agg_flag;     // per-CTA epoch: agg[i] of superstep `epoch` is published
  uint2* totals;          // (K, T) of the current plan, written by the last CTA
  unsigned* bar;          // BAR_WORDS barrier state
  const uint32_t* src_ptr;
  float alpha;
  int can_pull, force_pull;
  unsigned long long* trace;  // optional: %globaltimer after every phase (CTA 0)
  uint32_t trace_cap;
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Grid-wide barrier of the cooperative launch.  cooperative_groups'
// grid.sync() measured 1.3 us at 296 x 1024 threads on B200, vs 2.6 us for a
// flat atomic-counter barrier and 5.8 us for a two-level one
// (tools/microbench_barrier.cu, profiles/r01_microbench_barrier.txt).
__device__ __forceinline__ void grid_sync(unsigned*) { cg::this_grid().sync(); }

// Block-wide exclusive scan of (c, e) pairs; returns the block totals.
__device__ __forceinline__ uint2 block_excl_scan2(uint32_t& c, uint32_t& e, uint2* s) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t ic = warp_incl_scan(c, lane), ie = warp_incl_scan(e, lane);
  __syncthreads();
  if (lane == 31) s[warp] = make_uint2(ic, ie);
  __syncthreads();
  if (warp == 0) {
    uint2 x = s[lane];
    uint32_t xc = warp_incl_scan(x.x, lane), xe = warp_incl_scan(x.y, lane);
    s[lane] = make_uint2(xc - x.x, xe - x.y);
    if (lane == 31) s[32] = make_uint2(xc, xe);
  }
  __syncthreads();
  const uint2 wp = s[warp];
  c = wp.x + ic - c;
  e = wp.y + ie - e;
  return s[32];
}

__device__ __forceinline__ uint2 block_sum2(uint32_t c, uint32_t e, uint2* s) {
  uint32_t a = c, b = e;
  return block_excl_scan2(a, b, s);
}

// Frontier statistics of one bitmap word: vertices with out-degree > 0 and
// their edges.  Edges telescope over runs of consecutive set bits:
// sum deg(v) over [v0, v1) = ro[v1] - ro[v0] (2 loads per run, L1-cached).
__device__ __forceinline__ uint2 word_stats(const uint32_t* __restrict__ ro, uint32_t word,
                                            uint32_t kept, uint32_t wi) {
  uint32_t e = 0, x = word;
  while (x) {
    const int s0 = __ffs(x) - 1;
    const uint32_t t = ~(x >> s0);
    const int len = t ? __ffs(t) - 1 : 32 - s0;
    const uint32_t v0 = wi * 32 + s0;
    e += ro[v0 + len] - ro[v0];
    x = len + s0 >= 32 ? 0u : x & ~(((1u << len) - 1u) << s0);
  }
  return make_uint2(__popc(kept), e);
}

// Warp-level pull over CSC plan edges [e0, e1) (neighbors_expand_pull,
// operators.hpp:296-334, with the SSSP relax): each lane tests its in-edge's
// source against the current-frontier bitmap, forms the packed key
// (dist[src] + w, src), and a segmented shuffle-min leaves each destination's
// best candidate of the row in its first lane, which applies it.
template <class W, int VT>
__device__ __forceinline__ uint32_t pull_expand(const AdvArgs<W>& a, uint32_t e0, uint32_t e1,
                                                uint32_t k, uint32_t total, unsigned* err) {
  using D = typename DT<W>::D;
  unsigned long long* pkey = reinterpret_cast<unsigned long long*>(a.predrec);
  const int lane = threadIdx.x & 31;
  uint32_t n_elig = 0;
  uint32_t cs = __ldcg(a.plan.tseg + e0 / PLAN_GRAIN);
  for (;;) {
    uint32_t cand = cs + lane;
    uint32_t end = cand < k ? __ldcg(a.plan.off + cand + 1) : 0xFFFFFFFFu;
    unsigned msk = __ballot_sync(0xffffffffu, cand < k && end > e0);
    if (msk) {
      cs += __ffs(msk) - 1;
      break;
    }
    cs += 32;
  }
  for (;;) {
    uint32_t off = 0xFFFFFFFFu, u = 0;
    if (cs + lane < k) {
      off = __ldcg(a.plan.off + cs + lane);
      u = __ldcg(a.plan.v + cs + lane);
    }
    const uint32_t nxt = cs + 32 < k ? __ldcg(a.plan.off + cs + 32) : total;
    const uint32_t c0 = max(__shfl_sync(0xffffffffu, off, 0), e0);
    const uint32_t c1 = min(nxt, e1);
    for (uint32_t x = c0; x < c1; x += 32 * VT) {
      uint32_t src[VT], lo_[VT];
      W w[VT];
#pragma unroll
      for (int r = 0; r < VT; ++r) {  // A: CSC records (slot == plan edge)
        const uint32_t le = x + r * 32 + lane;
        int lo = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
          uint32_t o = __shfl_sync(0xffffffffu, off, lo + step);
          if (o <= le) lo += step;
        }
        lo_[r] = lo;
        src[r] = NIL;
        if (le < c1) {
          EdgeRec<W> rec = ld_rec(a.adj + le);
          src[r] = rec.v;
          w[r] = rec.w;
        }
      }
      uint32_t word[VT];
#pragma unroll
      for (int r = 0; r < VT; ++r)  // B: frontier-bitmap gathers
        word[r] = src[r] != NIL ? __ldcg(a.bm_in + (src[r] >> 5)) : 0u;
#pragma unroll
      for (int r = 0; r < VT; ++r) {  // C: candidates, segmented min, apply
        unsigned long long key = ~0ull;
        if (src[r] != NIL && ((word[r] >> (src[r] & 31)) & 1u)) {
          ++n_elig;
          key = pred_key(dadd(__ldcg(a.dist + src[r]), w[r], err), src[r]);
        }
        const uint32_t lo = lo_[r];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          unsigned long long o = __shfl_down_sync(0xffffffffu, key, d);
          uint32_t olo = __shfl_down_sync(0xffffffffu, lo, d);
          if (lane + d < 32 && olo == lo && o < key) key = o;
        }
        const uint32_t plo = __shfl_up_sync(0xffffffffu, lo, 1);
        const uint32_t dst = __shfl_sync(0xffffffffu, u, lo);
        if ((lane == 0 || plo != lo) && key != ~0ull) {
          const uint32_t kb = (uint32_t)(key >> 32);
          const D nd = *reinterpret_cast<const D*>(&kb);
          if (nd < ld_dist(a.dist + dst)) {
            red_min_d(a.dist + dst, nd);
            atomicMin(pkey + dst, key);
            atomicOr(a.bm_out + (dst >> 5), 1u << (dst & 31));
          }
        }
      }
    }
    if (c1 >= e1) break;
    cs += 32;
  }
  return n_elig;
}

template <class W, int VT, int TILE, int OPT = 0>
__global__ void __launch_bounds__(B_THREADS, 2) k_bsp(BspArgs<W> b) {
  using D = typename DT<W>::D;
  static_assert(sizeof(D) == 4, "packed predecessor keys need 32-bit distances");
  __shared__ uint2 s_scan[33];
  __shared__ uint2 s_pre[B_MAX_GROUPS];  // per 8-word group: (vertices, edges), then prefix
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t G = gridDim.x, bid = blockIdx.x;
  const uint32_t gtid = bid * B_THREADS + tid, gthreads = G * B_THREADS;
  Ctl* ctl = b.push.ctl;
  unsigned* err = &ctl->err;
  const Plan plan = b.push.plan;
  uint32_t* bm_next = b.push.bm_out;

  // ---- init (algorithms.hpp:579-583) ----
  {
    const uint32_t source = *b.src_ptr;
    D* dist = b.push.dist;
    unsigned long long* pkey = reinterpret_cast<unsigned long long*>(b.push.predrec);
    for (uint32_t i = gtid; i < b.n; i += gthreads) {
      dist[i] = i == source ? D(0) : dinf<W>();
      pkey[i] = ~0ull;
    }
    for (uint32_t i = gtid; i < b.nwords; i += gthreads) {
      bm_next[i] = (source >> 5) == i ? (1u << (source & 31)) : 0u;
      b.bm_cur[i] = 0;
    }
    for (uint32_t i = gtid; i < G; i += gthreads) b.agg_flag[i] = 0;
    if (gtid == 0) {
      Ctl c0 = {};
      *ctl = c0;
    }
  }
  uint32_t tr = 0;
  auto stamp = [&](uint32_t tag) {
    if (b.trace && bid == 0 && tid == 0 && tr < b.trace_cap) b.trace[tr++] = gtimer() << 2 | tag;
  };
  grid_sync(b.bar);
  stamp(0);

  // this CTA's contiguous bitmap words
  const uint32_t wpc = (b.nwords + G - 1) / G;
  const uint32_t w0 = min(bid * wpc, b.nwords), w1 = min(w0 + wpc, b.nwords);
  uint32_t n_elig = 0;
  for (uint32_t epoch = 1;; ++epoch) {
    // ---- compaction pass 1: per-group (vertices, edges) -> smem; publish ----
    // group = 8 consecutive bitmap words handled by one warp with all its
    // row-offset loads in flight (load_warp_words); groups of this CTA's
    // word range go round-robin over its 32 warps.
    const uint32_t ngroups = (w1 - w0 + F_WPW - 1) / F_WPW;
    uint32_t c = 0, e = 0;
    for (uint32_t gidx = warp; gidx < ngroups; gidx += B_WARPS) {
      WarpWords w;
      uint32_t raw;
      load_warp_words<true>(b.ro, bm_next, w1, w0 + gidx * F_WPW, w, &raw);
      uint32_t gc_ = 0, ge_ = 0;
#pragma unroll
      for (int j = 0; j < F_WPW; ++j) {
        gc_ += __popc(w.keep[j]);
        ge_ += w.deg[j];
      }
      ge_ = warp_sum(ge_);
      if (lane == 0) s_pre[gidx] = make_uint2(gc_, ge_);
      c += gc_;
      e += ge_;
    }
    const uint2 mine = block_sum2(lane == 0 ? c : 0u, lane == 0 ? e : 0u, s_scan);
    if (tid == 0) {
      b.agg[bid] = mine;
      __threadfence();
      atomicExch(b.agg_flag + bid, epoch);
    }
    // ---- look-back: sum of every earlier CTA's aggregate ----
    uint32_t pc = 0, pe = 0;
    for (uint32_t i = tid; i < bid; i += B_THREADS) {
      volatile unsigned* f = b.agg_flag + i;
      while (*f != epoch) __nanosleep(20);
      __threadfence();
      const uint2 x = __ldcg(b.agg + i);
      pc += x.x;
      pe += x.y;
    }
    const uint2 base = block_sum2(pc, pe, s_scan);
    if (bid == G - 1 && tid == 0) {  // grand totals: the last CTA's inclusive prefix
      const uint32_t K = base.x + mine.x, T = base.y + mine.y;
      *b.totals = make_uint2(K, T);
      plan.off[K] = T;
      const uint32_t sb = (T + PLAN_GRAIN - 1) / PLAN_GRAIN;
      if (sb < plan.tseg_cap) plan.tseg[sb] = K;
    }
    // ---- exclusive group prefixes (2 groups per thread) ----
    {
      uint2 g0 = 2 * tid < ngroups ? s_pre[2 * tid] : make_uint2(0, 0);
      uint2 g1 = 2 * tid + 1 < ngroups ? s_pre[2 * tid + 1] : make_uint2(0, 0);
      uint32_t xc = g0.x + g1.x, xe = g0.y + g1.y;
      block_excl_scan2(xc, xe, s_scan);  // syncs before any s_pre overwrite below
      if (2 * tid < ngroups) s_pre[2 * tid] = make_uint2(base.x + xc, base.y + xe);
      if (2 * tid + 1 < ngroups)
        s_pre[2 * tid + 1] = make_uint2(base.x + xc + g0.x, base.y + xe + g0.y);
      __syncthreads();
    }
    // ---- compaction pass 2: ascending plan + tile map, bm_cur = bm_next, clear ----
    for (uint32_t gidx = warp; gidx < ngroups; gidx += B_WARPS) {
      const uint32_t wbase = w0 + gidx * F_WPW;
      WarpWords w;
      uint32_t raw;
      load_warp_words<true>(b.ro, bm_next, w1, wbase, w, &raw);
      if (lane < F_WPW && wbase + lane < w1) {
        b.bm_cur[wbase + lane] = raw;
        if (raw) bm_next[wbase + lane] = 0;
      }
      const uint2 pre = s_pre[gidx];
      uint32_t gc = pre.x, ge = pre.y;
#pragma unroll
      for (int j = 0; j < F_WPW; ++j) {
        const uint32_t keep = w.keep[j];
        if (keep == 0) continue;  // warp-uniform
        const bool on = (keep >> lane) & 1u;
        const uint32_t deg = w.deg[j];
        const uint32_t incl = warp_incl_scan(deg, lane);
        const uint32_t gi = gc + __popc(keep & lanemask_lt());
        const uint32_t eoff = ge + incl - deg;
        if (on) {
          plan.v[gi] = (wbase + j) * 32 + lane;
          plan.start[gi] = w.st[j];
          plan.off[gi] = eoff;
        }
        warp_tile_map(plan, gi, eoff, on ? deg : 0u);
        gc += __popc(keep);
        ge += __shfl_sync(0xffffffffu, incl, 31);
      }
    }
    grid_sync(b.bar);
    stamp(1);
    const uint2 tot = __ldcg(b.totals);
    const uint32_t K = tot.x, T = tot.y;
    if (K == 0) break;  // the while (f.size() != 0) test, identical in every CTA
    const uint32_t mode =
        (b.force_pull || (b.can_pull && (float)T > (float)b.m / b.alpha)) ? 1u : 0u;
    if (gtid == 0) {
      ctl->k = K;
      ctl->total = T;
      ctl->mode = mode;
      ctl->supersteps += 1;
      if (mode) {
        ctl->pull_steps += 1;
      } else {
        ctl->push_steps += 1;
        ctl->relax += T;
      }
    }

    // ---- advance ----
    const uint32_t gwarp = gtid >> 5, nwarps = gthreads >> 5;
    if (mode == 0) {
      for (uint64_t e0 = (uint64_t)gwarp * TILE; e0 < T; e0 += (uint64_t)nwarps * TILE)
        range_expand<W, VT, true, OPT>(b.push, (uint32_t)e0, (uint32_t)min(e0 + TILE, (uint64_t)T), K,
                                  T, err);
    } else {
      for (uint64_t e0 = (uint64_t)gwarp * TILE; e0 < b.pull_total; e0 += (uint64_t)nwarps * TILE)
        n_elig += pull_expand<W, VT>(b.pull, (uint32_t)e0,
                                     (uint32_t)min(e0 + TILE, (uint64_t)b.pull_total), b.pull_k,
                                     b.pull_total, err);
    }
    grid_sync(b.bar);
    stamp(3);
  }
  if (gtid == 0) {
    ctl->k = 0;
    ctl->total = 0;
  }
  n_elig = warp_sum(n_elig);
  if (lane == 0 && n_elig) atomicAdd(&ctl->relax, (unsigned long long)n_elig);
}

}  // namespace gfb
