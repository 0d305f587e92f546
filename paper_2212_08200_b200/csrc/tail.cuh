// tail.cuh -- the small-frontier tail of the BSP loop as ONE persistent
// cooperative launch (push loops; any arithmetic).
//
// After the big supersteps an RMAT SSSP still runs 6-8 supersteps whose
// frontiers hold a few thousand edges; each costs the bitmap filter's three
// launches over all n/32 words (~30-40 us) for ~10 us of advance.  When the
// filter finds a plan below tail_edges edges with nothing deferred
// (k_fscan_o: ctl->tail), the loop hands over to k_tail, which keeps the same
// operators -- advance + relax over the frontier, uniquify, loop until empty
// (algorithms.hpp:151-167) -- but carries the frontier in vertex queues:
//
//   expand   the plan's edges (range_expand<ENQ>: edge-balanced tiles); a
//            relaxation that lowers v ORs v's bit into this superstep's dedup
//            bitmap with a returning atomic, and the first such lane appends
//            v to the next queue (warp-aggregated)               | grid sync
//   build    queue -> plan: per warp one 64-bit reservation of (slots, edges),
//            start / edge offsets / tile map; the dedup bits of the queued
//            vertices are cleared for the superstep after next    | grid sync
//
// The result is the same fixpoint (a label-correcting order change only);
// predecessors use the packed (dist, u) keys of k_push_range.  A rebuilt plan
// above tmax edges goes back to the bitmap filter: its vertices are marked in
// bm_next (bm[0] holds no dedup bits after a build), the plan is emptied and
// the loop continues (ctl->tail = 2).
#pragma once

#include <cooperative_groups.h>

#include "hot.cuh"

namespace gfb {

constexpr int TL_THREADS = 512;
constexpr uint32_t TL_TILE = 128;  // plan edges per warp tile

template <class W>
struct TailArgs {
  AdvArgs<W> a;               // plan = the workspace plan (built by the filter first)
  const uint32_t* ro;
  uint32_t* q[2];             // vertex queues (n entries each), by superstep parity
  uint32_t* qcnt;             // [3] rotating queue counts
  unsigned long long* cell;   // [3] rotating (slots << 32 | edges) reservation cursors
  uint32_t* bm[2];            // dedup bitmaps: [0] bm_next, [1] bm_cur
  uint32_t nwords;
  uint32_t tmax;              // a rebuilt plan above this many edges goes back to the filter
  cudaGraphConditionalHandle hloop;
  int set_loop;
};

template <class W>
__global__ void __launch_bounds__(TL_THREADS, 2) k_tail(TailArgs<W> t) {
  // 4-byte distances: packed (dist, pred) keys; f64: returning mins and {u, edge} records
  constexpr bool REC = sizeof(typename DT<W>::D) == 8;
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  AdvArgs<W> a = t.a;
  const int lane = threadIdx.x & 31;
  const uint32_t gtid = blockIdx.x * TL_THREADS + threadIdx.x;
  const uint32_t gthreads = gridDim.x * TL_THREADS;
  const uint32_t gwarp = gtid >> 5, nwarps = gthreads >> 5;
  unsigned* err = &a.ctl->err;
  // bm_cur may hold stale bits (the filter only rewrites tiles with bits)
  for (uint32_t i = gtid; i < t.nwords; i += gthreads) t.bm[1][i] = 0;
  uint32_t K = a.ctl->k, T = a.ctl->total;  // the filter's plan
  if (gtid == 0) {
    for (int i = 0; i < 3; ++i) {
      t.qcnt[i] = 0;
      t.cell[i] = 0;
    }
  }
  grid.sync();
  unsigned long long relax = 0;
  uint32_t steps = 0;
  uint32_t escaped = 0;
  for (uint32_t s = 0;; ++s) {
    // ---- expand the plan: improved vertices -> q[s & 1] ----
    a.tq_out = t.q[s & 1];
    a.tq_cnt = t.qcnt + s % 3;
    a.tq_bm = t.bm[s & 1];
    relax += T;
    ++steps;
    for (uint64_t e0 = (uint64_t)gwarp * TL_TILE; e0 < T; e0 += (uint64_t)nwarps * TL_TILE)
      range_expand<W, 1, true, 1, false, REC, true>(a, (uint32_t)e0,
                                                      (uint32_t)min(e0 + TL_TILE, (uint64_t)T),
                                                      K, T, err);
    if (gtid == 0) {  // the counters of superstep s + 1 (last read two barriers ago)
      t.qcnt[(s + 1) % 3] = 0;
      t.cell[(s + 1) % 3] = 0;
    }
    grid.sync();
    // ---- build the next plan from the queue ----
    const uint32_t Q = __ldcg(t.qcnt + s % 3);
    if (Q == 0) break;
    const uint32_t* qin = t.q[s & 1];
    unsigned long long* cell = t.cell + s % 3;
    for (uint32_t b0 = gwarp * 32; b0 < Q; b0 += nwarps * 32) {
      const uint32_t i = b0 + lane;
      uint32_t v = 0, st = 0, deg = 0;
      if (i < Q) {
        v = __ldcg(qin + i);
        st = t.ro[v];
        deg = t.ro[v + 1] - st;
        atomicAnd(t.bm[s & 1] + (v >> 5), ~(1u << (v & 31)));  // clean for superstep s + 2
      }
      const bool keep = deg > 0;
      const unsigned km = __ballot_sync(0xffffffffu, keep);
      if (km == 0) continue;
      const uint32_t incl = warp_incl_scan(keep ? deg : 0u, lane);
      const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(cell, ((unsigned long long)__popc(km) << 32) | tot);
      base = __shfl_sync(0xffffffffu, base, 0);
      if (keep) {
        const uint32_t gi = (uint32_t)(base >> 32) + __popc(km & lanemask_lt());
        const uint32_t eoff = (uint32_t)base + incl - deg;
        a.plan.v[gi] = v;
        a.plan.start[gi] = st;
        a.plan.off[gi] = eoff;
        tile_map_entries(a.plan, gi, eoff, deg);
      }
    }
    grid.sync();
    const unsigned long long tot = __ldcg(cell);
    K = (uint32_t)(tot >> 32);
    T = (uint32_t)tot;
    if (K == 0) break;  // only sinks were improved
    if (T > t.tmax) {  // grown past the tail: back to the bitmap filter (its
      // deferral and distance order), the plan's vertices marked in bm_next and
      // their smallest distance in ctl->fmin (the filter's bucket base)
      uint32_t fm = 0xFFFFFFFFu;
      for (uint32_t b0 = gwarp * 32; b0 < K; b0 += nwarps * 32) {
        const uint32_t i = b0 + lane;
        if (i < K) {
          const uint32_t v = __ldcg(a.plan.v + i);
          fm = min(fm, fkey(__ldcg(a.dist + v)));
          atomicOr(t.bm[0] + (v >> 5), 1u << (v & 31));
        }
      }
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) fm = min(fm, __shfl_xor_sync(0xffffffffu, fm, d));
      if (lane == 0 && fm != 0xFFFFFFFFu) atomicMin(&a.ctl->fmin, fm);
      escaped = 1;
      break;
    }
  }
  if (gtid == 0) {
    a.ctl->relax += relax;
    a.ctl->supersteps += steps;
    a.ctl->push_steps += steps;
    a.ctl->k = 0;  // (after an escape: the next push is empty, the filter rebuilds)
    a.ctl->total = 0;
    a.ctl->tail = escaped ? 2u : 0u;
    if (t.set_loop && !escaped) cudaGraphSetConditional(t.hloop, 0u);
  }
}

}  // namespace gfb
