// nearfar.cuh -- SSSP with a near-far filter (delta > 0) as ONE persistent
// cooperative kernel with queue frontiers: the high-diameter path (BASELINE
// configs[3], the 4096^2 grid: 8.5K BSP supersteps at ~215 relaxations per
// edge).
//
// Same operators as the BSP loop (algorithms.hpp:151-167): advance + relax
// over the frontier, a filter on the output, loop until empty.  The filter
// splits the improved vertices at a distance threshold (the
// near-far work-efficient variant of Davidson et al.):
//
//   near phase   expand the near queue; an improved v goes to the next near
//                queue when its new distance < thr, else to the far pile
//                (warp-aggregated appends of (v, dist) entries)  | grid sync
//   split phase  (near queue empty) min over the live far pile   | grid sync
//                thr = min + delta; far entries below thr move to the near
//                queue, the rest are compacted; stale entries    | grid sync
//                (vertex lowered again since) are dropped
//
// The fixpoint is the same as the BSP loop's (a label-correcting order
// change only), so distances are bit-identical; predecessors use the packed
// (dist, u) keys of k_push_range.  A queue overflow (more activations in one
// phase than the queue holds) flags ctl->err bit 1 and the host reruns the
// call on the BSP loop.  One launch; a phase costs one grid barrier
// (1.3 us, tools/microbench_barrier.cu) plus its work, instead of four
// kernel launches per superstep.
#pragma once

#include <cooperative_groups.h>

#include "hot.cuh"

namespace gfb {

namespace cgn = cooperative_groups;

constexpr int NF_THREADS = 1024;
// LH > 0: a warp chases up to LH rounds of its own near activations from a
// warp-local queue of NF_LQ entries before the grid barrier -- chaotic
// relaxation inside a phase (still the same fixpoint), fewer phases on
// high-diameter graphs.
constexpr uint32_t NF_LQ = 128;
constexpr uint32_t NF_CHASE = 128;

template <class W>
struct NfArgs {
  using D = typename DT<W>::D;
  const uint32_t* ro;
  const EdgeRec<W>* adj;
  D* dist;
  unsigned long long* pkey;
  uint2* nq[2];          // near queues: (v, dist bits at activation)
  uint2* fq[2];          // far piles, same entries
  uint32_t cap;          // entries per queue; overflow sets ctl->err bit 1
  uint32_t* cnt;         // [0..2] near counts (rotating), [3..4] far counts, [5..6] min-far bits
  Ctl* ctl;
  const uint32_t* src_ptr;
  uint32_t n, nwords;
  D delta;
  unsigned long long* trace;  // optional (GFB_TRACE=1): per phase (time << 24 | K)
  uint32_t trace_cap;
  // Heavy rows: an activated vertex with more than NF_HEAVY out-edges is not
  // expanded by the warp that dequeued it but listed here and expanded by
  // every warp (32-edge chunks) in the next phase -- one warp serialising a
  // hub's edges made the queue loop 50x slower than BSP on RMAT.
  uint2* hq[2];
  uint32_t hcap;
  unsigned long long* fmin64;  // [2] minimum live far distance (order key), by parity
};
constexpr uint32_t NF_HEAVY = 256;

// Queue entries are (v, tag of the distance that activated v).  4-byte
// distances: the tag is the distance's bits (exact stale test).  f64: the
// folded 64-bit pattern -- a collision only lets a stale entry expand again
// with v's CURRENT distance, which is correct, just redundant.
__device__ __forceinline__ uint32_t ntag(float d) { return __float_as_uint(d); }
__device__ __forceinline__ uint32_t ntag(uint32_t d) { return d; }
__device__ __forceinline__ uint32_t ntag(double d) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(d);
  return (uint32_t)(b ^ (b >> 32));
}
// order-preserving 64-bit key of a distance (non-negative)
__device__ __forceinline__ unsigned long long okey(float d) { return __float_as_uint(d); }
__device__ __forceinline__ unsigned long long okey(uint32_t d) { return d; }
__device__ __forceinline__ unsigned long long okey(double d) {
  return (unsigned long long)__double_as_longlong(d);
}
template <class D> __device__ __forceinline__ D dfrom_okey(unsigned long long k);
template <> __device__ __forceinline__ float dfrom_okey<float>(unsigned long long k) {
  return __uint_as_float((uint32_t)k);
}
template <> __device__ __forceinline__ uint32_t dfrom_okey<uint32_t>(unsigned long long k) {
  return (uint32_t)k;
}
template <> __device__ __forceinline__ double dfrom_okey<double>(unsigned long long k) {
  return __longlong_as_double((long long)k);
}

// One relaxation u -> v (edge eid) with candidate nd; true when it lowered
// dist[v] (as far as this thread can tell).  4-byte: fire-and-forget min and
// packed (dist, u) key (k_push_range); f64: returning 64-bit min and a
// {u, edge} record by the winner (k_push_range<REC>).
template <class D>
__device__ __forceinline__ bool nf_relax(D* dist, unsigned long long* pkey, uint32_t v, D nd,
                                         uint32_t u, uint32_t eid) {
  if (!(nd < __ldcg(dist + v))) return false;
  if constexpr (sizeof(D) == 8) {
    const D old = atomic_min_d(dist + v, nd);
    if (!(nd < old)) return false;
    reinterpret_cast<uint2*>(pkey)[v] = make_uint2(u, eid);
  } else {
    red_min_u32(reinterpret_cast<unsigned*>(dist + v), dbits(nd));
    red_min_u64(pkey + v, pred_key(nd, u));
  }
  return true;
}


// Append e to queue q (count *c) if this lane's flag is set: one atomicAdd per
// warp (ballot + popc), then each lane writes its own slot.
__device__ __forceinline__ void warp_append(bool flag, uint2 e, uint2* q, uint32_t* c,
                                            uint32_t cap, unsigned* err) {
  const unsigned m = __ballot_sync(0xffffffffu, flag);
  if (m == 0) return;
  const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
  uint32_t base = 0;
  if (lane == leader) base = atomicAdd(c, (uint32_t)__popc(m));
  base = __shfl_sync(0xffffffffu, base, leader);
  const uint32_t slot = base + __popc(m & lanemask_lt());
  if (flag) {
    if (slot < cap) q[slot] = e;
    else atomicOr(err, 2u);
  }
}

// Queue entries carry the distance that activated the vertex; an entry whose
// vertex has since been lowered again is stale (the lowering appended a newer
// entry) and is skipped -- dedup without a membership bitmap or a returning
// atomic on the critical path.
template <class W, int LH = 0, uint32_t CH = 32, bool HV = false>
__global__ void __launch_bounds__(NF_THREADS, 1) k_nearfar(NfArgs<W> a) {
  using D = typename DT<W>::D;
  cgn::grid_group grid = cgn::this_grid();
  const int lane = threadIdx.x & 31;
  const uint32_t gtid = blockIdx.x * NF_THREADS + threadIdx.x;
  const uint32_t gthreads = gridDim.x * NF_THREADS;
  const uint32_t gwarp = gtid >> 5, nwarps = gthreads >> 5;
  const int warp = threadIdx.x >> 5;
  unsigned* err = &a.ctl->err;
  __shared__ uint2 s_lq[NF_THREADS / 32][LH > 0 ? NF_LQ : 1];  // warp-local near queues

  // ---- init (algorithms.hpp:144-148) ----
  const uint32_t source = *a.src_ptr;
  for (uint32_t i = gtid; i < a.n; i += gthreads) {
    a.dist[i] = i == source ? D(0) : dinf<W>();
    a.pkey[i] = ~0ull;
  }
  if (gtid == 0) {
    Ctl c0 = {};
    *a.ctl = c0;
    a.nq[0][0] = make_uint2(source, 0u);  // dist bits of +0.0 / 0u
    a.cnt[0] = 1;
    a.cnt[1] = a.cnt[2] = a.cnt[3] = a.cnt[4] = 0;
    a.cnt[5] = a.cnt[6] = 0xFFFFFFFFu;  // (unused: the far minimum lives in fmin64)
    a.fmin64[0] = a.fmin64[1] = ~0ull;
    a.cnt[7] = a.cnt[8] = a.cnt[9] = 0;  // heavy-list counts (rotating like the near ones)
  }
  grid.sync();

  D thr = a.delta;  // near: dist < thr
  uint32_t fp = 0, mp = 0;
  unsigned long long relax = 0;
  uint32_t phases = 0;
  for (uint32_t ph = 0;; ++ph) {
    const uint32_t cur = ph & 1, nxt = cur ^ 1;
    const uint32_t K = min(__ldcg(a.cnt + ph % 3), a.cap);
    const uint2* qin = a.nq[cur];
    uint2* qout = a.nq[nxt];
    uint32_t* cout = a.cnt + (ph + 1) % 3;
    if (gtid == 0) a.cnt[(ph + 2) % 3] = 0;  // the count two phases ahead
    const uint32_t H = HV ? min(__ldcg(a.cnt + 7 + ph % 3), a.hcap) : 0u;  // heavy rows
    const uint2* hin = a.hq[ph & 1];
    uint2* hout = a.hq[(ph + 1) & 1];
    uint32_t* hcout = a.cnt + 7 + (ph + 1) % 3;
    if (gtid == 0) a.cnt[7 + (ph + 2) % 3] = 0;
    if (a.trace && gtid == 0 && ph < a.trace_cap) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.trace[ph] = (t << 24) | min(K, 0xFFFFFFu);
    }
    if (K > 0 || H > 0) {
      // ---------------- near phase: expand the near queue ----------------
      ++phases;
      uint32_t lq_n = 0;  // warp-local queue fill (warp-uniform)
      // Expand one queue entry per lane (valid lanes only); near activations go
      // to the warp-local queue while it has room (LH > 0), else global.
      auto expand = [&](bool valid, uint2 e) {
        uint32_t u = 0, st = 0, deg = 0;
        D du = D(0);
        if (valid) {
          u = e.x;
          st = a.ro[u];
          const uint32_t en = a.ro[u + 1];
          const D cu = __ldcg(a.dist + u);
          du = cu;
          deg = ntag(cu) == e.y ? en - st : 0u;  // stale entry: skip
        }
        // hubs go to the heavy list (whole-grid expansion next phase)
        if constexpr (HV) {
          const bool heavy = deg > NF_HEAVY;
          warp_append(heavy, e, hout, hcout, a.hcap, err);
          if (heavy) deg = 0;
        }
        const uint32_t incl = warp_incl_scan(deg, lane);
        const uint32_t off = incl - deg;  // first chunk edge of this lane's vertex
        const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
        relax += lane == 0 ? tot : 0;
        for (uint32_t x = 0; x < tot; x += 32) {
          const uint32_t le = x + lane;
          int lo = 0;  // owner lane: the first whose inclusive degree exceeds le
#pragma unroll
          for (int step = 16; step >= 1; step >>= 1) {
            const uint32_t p = __shfl_sync(0xffffffffu, incl, lo + step - 1);
            if (p <= le) lo += step;
          }
          const uint32_t ost = __shfl_sync(0xffffffffu, st, lo);
          const uint32_t ooff = __shfl_sync(0xffffffffu, off, lo);
          const uint32_t ou = __shfl_sync(0xffffffffu, u, lo);
          const D odu = shfl_d(du, lo);
          bool to_near = false, to_far = false;
          uint2 ent = make_uint2(0, 0);
          if (le < tot) {
            const EdgeRec<W> rec = ld_rec(a.adj + ost + (le - ooff));
            const D nd = dadd(odu, rec.w, err);
            if (nf_relax(a.dist, a.pkey, rec.v, nd, ou, ost + (le - ooff))) {
              ent = make_uint2(rec.v, ntag(nd));
              to_near = nd < thr;
              to_far = !to_near;
            }
          }
          if constexpr (LH > 0) {
            const unsigned m = __ballot_sync(0xffffffffu, to_near);
            const uint32_t room = NF_LQ - lq_n;
            const uint32_t rank = __popc(m & lanemask_lt());
            const bool loc = to_near && rank < room;
            if (loc) s_lq[warp][lq_n + rank] = ent;
            lq_n += min((uint32_t)__popc(m), room);
            __syncwarp();
            warp_append(to_near && !loc, ent, qout, cout, a.cap, err);
          } else {
            warp_append(to_near, ent, qout, cout, a.cap, err);
          }
          warp_append(to_far, ent, a.fq[fp], a.cnt + 3 + fp, a.cap, err);
        }
      };
      // heavy rows listed last phase: one CTA per row (rows strided over the
      // CTAs), its warps taking 32-edge chunks
      for (uint32_t hi = blockIdx.x; hi < H; hi += gridDim.x) {
        const uint2 e = __ldcg(hin + hi);
        const D cu = __ldcg(a.dist + e.x);
        if (ntag(cu) != e.y) continue;  // stale (block-uniform)
        const uint32_t st = a.ro[e.x], deg = a.ro[e.x + 1] - st;
        const D du = cu;
        if (threadIdx.x == 0) relax += deg;
        for (uint32_t base = warp * 32; base < deg; base += NF_THREADS) {
          const uint32_t le = base + lane;
          bool to_near = false, to_far = false;
          uint2 ent = make_uint2(0, 0);
          if (le < deg) {
            const EdgeRec<W> rec = ld_rec(a.adj + st + le);
            const D nd = dadd(du, rec.w, err);
            if (nf_relax(a.dist, a.pkey, rec.v, nd, e.x, st + le)) {
              ent = make_uint2(rec.v, ntag(nd));
              to_near = nd < thr;
              to_far = !to_near;
            }
          }
          warp_append(to_near, ent, qout, cout, a.cap, err);
          warp_append(to_far, ent, a.fq[fp], a.cnt + 3 + fp, a.cap, err);
        }
      }
      // CH queue entries per warp: fewer than 32 spreads a small near queue
      // (and the chasing of its activations) over more warps
      for (uint32_t base = gwarp * CH; base < K; base += nwarps * CH) {
        const uint32_t j = base + lane;
        const bool ok = (uint32_t)lane < CH && j < K;
        expand(ok, ok ? __ldcg(qin + j) : make_uint2(0, 0));
        if constexpr (LH > 0) {
          // chase this warp's own near activations without a grid barrier
          // at most NF_CHASE entries chased per queue chunk: bounds the
          // longest warp's chain, whose end every other warp waits for at the
          // grid barrier (78.7% of warp samples at barrier, 4096^2 grid,
          // profiles/r02_nearfar_grid4096_full.txt; budget 32 / 64 / 128 /
          // none: 41.2 / 32.7 / 31.1 / 31.9 ms)
          uint32_t chased = 0;
          for (int hop = 0; hop < LH && lq_n > 0 && chased < NF_CHASE; ++hop) {
            const uint32_t take = min(lq_n, 32u);
            chased += take;
            const bool v = (uint32_t)lane < take;
            const uint2 e = v ? s_lq[warp][lq_n - take + lane] : make_uint2(0, 0);
            lq_n -= take;
            __syncwarp();
            expand(v, e);
          }
        }
      }
      if constexpr (LH > 0) {  // hand the rest to the next phase
        for (uint32_t b0 = 0; b0 < lq_n; b0 += 32) {
          const bool v = b0 + lane < lq_n;
          warp_append(v, v ? s_lq[warp][b0 + lane] : make_uint2(0, 0), qout, cout, a.cap, err);
        }
        lq_n = 0;
        __syncwarp();
      }
      grid.sync();
      continue;
    }
    // ---------------- split phase: refill the near queue from the far pile ----
    const uint32_t F = min(__ldcg(a.cnt + 3 + fp), a.cap);
    const uint2* fin = a.fq[fp];
    // pass 1: minimum live far distance (64-bit order key for every type)
    unsigned long long mloc = ~0ull;
    for (uint32_t i = gtid; i < F; i += gthreads) {
      const uint2 e = __ldcg(fin + i);
      const D cd = __ldcg(a.dist + e.x);
      if (ntag(cd) == e.y) mloc = min(mloc, okey(cd));
    }
    for (int d = 16; d > 0; d >>= 1) mloc = min(mloc, __shfl_xor_sync(0xffffffffu, mloc, d));
    if (lane == 0 && mloc != ~0ull) atomicMin(a.fmin64 + mp, mloc);
    if (gtid == 0) {
      a.cnt[3 + (fp ^ 1)] = 0;
      a.fmin64[mp ^ 1] = ~0ull;
    }
    grid.sync();
    const unsigned long long mbits = __ldcg(a.fmin64 + mp);
    if (mbits == ~0ull) break;  // no live far entry: converged
    const D mfar = dfrom_okey<D>(mbits);
    thr = dadd(mfar, a.delta, nullptr);
    if (!(mfar < thr)) thr = dinf<W>();  // delta absorbed by rounding: take everything
    // pass 2: live entries below thr -> near queue, the rest stay far
    for (uint32_t b0 = gwarp * 32; b0 < F; b0 += nwarps * 32) {
      const uint32_t i = b0 + lane;
      uint2 e = make_uint2(0, 0);
      bool near = false, keep = false;
      if (i < F) {
        e = __ldcg(fin + i);
        const D cd = __ldcg(a.dist + e.x);
        if (ntag(cd) == e.y) {
          near = cd < thr;
          keep = !near;
        }
      }
      warp_append(near, e, qout, cout, a.cap, err);
      warp_append(keep, e, a.fq[fp ^ 1], a.cnt + 3 + (fp ^ 1), a.cap, err);
    }
    fp ^= 1;
    mp ^= 1;
    grid.sync();
  }
  if (relax) atomicAdd(&a.ctl->relax, relax);
  if (gtid == 0) {
    a.ctl->supersteps = phases;
    a.ctl->push_steps = phases;
  }
}

}  // namespace gfb
