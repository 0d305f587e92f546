// kernels.cuh -- the sm_100a kernels of the SSSP hot path.
//
//   k_compact        bitmap -> ascending frontier plan (filter/uniquify,
//                    operators.hpp:191-200 + frontier.hpp:147-165 convert):
//                    warp-ballot compaction, degree scan, decoupled look-back,
//                    edge-tile map for the load-balanced advance.
//   k_plan_list      sparse list (duplicates kept) -> frontier plan, order
//                    preserving (operators.hpp:17-24 active_vertices_of).
//   k_advance_push   push advance (operators.hpp:35-68 neighbors_expand +
//                    the relax lambda algorithms.hpp:151-158): merge-path
//                    edge tiles, coalesced 8-byte record stream,
//                    test-before-atomicMin, bitmap or ordered-queue output.
//   k_advance_pull   pull advance (operators.hpp:76-114): CSC edge tiles,
//                    frontier-bitmap test, shared-memory segmented min,
//                    one global atomic per (tile, destination).
//   k_init           algorithms.hpp:144-148 init (+ frontier seed).
//   k_pred_*         predecessor pass (algorithms.hpp:77-93 semantics:
//                    tight-edge tree, acyclic).
#pragma once

#include "common.cuh"

namespace gfb {

// ---------------------------------------------------------------------------
// Device control block (one per workspace / operator call).
// ---------------------------------------------------------------------------
struct Ctl {
  uint32_t k;          // segments in the current plan (frontier vertices, deg>0)
  uint32_t total;      // edges of the current plan
  uint32_t tile_ctr;   // dynamic tile counter for look-back kernels
  uint32_t err;        // bit 0: u32 distance overflow
  unsigned long long relax;  // sum of plan totals (cond invocations)
  uint32_t supersteps;
  uint32_t push_steps;
  uint32_t pull_steps;
  uint32_t out_count;  // ordered-queue output count
  uint32_t rec_count;  // RECORD op output count
  uint32_t unresolved; // predecessor pass
  uint32_t flag;       // generic
  uint32_t mode;       // 0 push, 1 pull (chosen by k_plan_direction)
  unsigned long long n_reach, m_reach;
  uint32_t resolved;   // predecessor repair: vertices resolved over all rounds
  // distance-ordered plan (frontier.cuh k_fcount_o): smallest activation
  // distance of the frontier being built (float bits, written by the push
  // advance) and the value frozen for the compaction in progress
  uint32_t fmin, blo;
  uint32_t bcut;       // ordered compaction: buckets above bcut stay pending
  // peer-memory partition (peer.cu): sums over all ranks from the last
  // cross-rank barrier (k_xbar) of k / flag / unresolved / resolved
  uint32_t gk, gflag, gunres, gresolved;
  // ordered compaction: vertices / edges in the bitmap (placed + deferred)
  uint32_t k_all, t_all;
  uint32_t tail;       // k_fscan_o: the next superstep starts the tail kernel (tail.cuh)
};

// Expansion plan: the frontier restricted to vertices with out-degree > 0.
struct Plan {
  uint32_t* v;       // vertex id
  uint32_t* start;   // first edge of the row
  uint32_t* off;     // exclusive prefix of degrees (off[k] = total)
  uint32_t* tseg;    // tseg[b] = segment holding edge b*PLAN_GRAIN
  uint32_t tseg_cap; // entries allocated in tseg
};

constexpr int A_BLOCK = 256;
constexpr int A_VT = 4;
constexpr int A_TILE = A_BLOCK * A_VT;  // edges per advance tile
constexpr int PLAN_GRAIN = 256;          // edge granularity of the plan's tile map
// predrec.y with this bit set holds a CSC slot (pull) instead of a CSR edge id
constexpr uint32_t PRED_CSC_SLOT = 0x80000000u;
constexpr int A_RATIO = A_TILE / PLAN_GRAIN;

constexpr int C_WARPS = 8;
constexpr int C_WPW = 8;                 // bitmap words per warp
constexpr int C_WORDS = C_WARPS * C_WPW; // words per compaction tile
constexpr int C_VERTS = C_WORDS * 32;    // vertices per compaction tile

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  return x;
}

__device__ __forceinline__ uint32_t warp_sum(uint32_t x) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) x += __shfl_xor_sync(0xffffffffu, x, d);
  return x;
}

// Write the tile map entries owned by segment `gi` = [eoff, eoff+deg).
__device__ __forceinline__ void tile_map_entries(const Plan& p, uint32_t gi, uint32_t eoff,
                                                 uint32_t deg) {
  uint32_t b = (eoff + PLAN_GRAIN - 1) / PLAN_GRAIN;
  for (uint64_t x = (uint64_t)b * PLAN_GRAIN; x < (uint64_t)eoff + deg && b < p.tseg_cap;
       x += PLAN_GRAIN, ++b)
    p.tseg[b] = gi;
}

// Finalise a plan from the inclusive totals (called by one thread).
__device__ __forceinline__ void plan_finish(Plan p, Ctl* ctl, uint32_t K, uint32_t T) {
  ctl->k = K;
  ctl->total = T;
  p.off[K] = T;
  uint32_t sb = (T + PLAN_GRAIN - 1) / PLAN_GRAIN;  // sentinel past the last tile
  if (sb < p.tseg_cap) p.tseg[sb] = K;
  ctl->tile_ctr = 0;
}

// ---------------------------------------------------------------------------
// k_compact: next-frontier bitmap -> plan.  One CTA per C_VERTS vertices,
// tiles claimed in launch order (dynamic counter) so the look-back always
// waits on a running predecessor.  Optionally copies the word into bm_cur
// (the frontier bitmap the pull kernel tests) and clears bm_next.
// ---------------------------------------------------------------------------
static __global__ void __launch_bounds__(C_WARPS * 32)
k_compact(const uint32_t* __restrict__ ro, uint32_t* bm_next, uint32_t* bm_cur,
          uint32_t nwords, uint32_t n, Plan plan, Ctl* ctl, unsigned long long* status,
          uint32_t ntiles, int clear) {
  __shared__ uint32_t s_v[C_VERTS];
  __shared__ uint32_t s_start[C_VERTS];
  __shared__ uint32_t s_deg[C_VERTS];
  __shared__ uint32_t s_wc[C_WARPS], s_we[C_WARPS];
  __shared__ uint32_t s_tile, s_pc, s_pe;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = atomicAdd(&ctl->tile_ctr, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;

  // ---- phase 1: warp-ballot compaction of this warp's words into smem ----
  const uint32_t wbase = tile * C_WORDS + warp * C_WPW;
  uint32_t my_word = 0;
  if (lane < C_WPW && wbase + lane < nwords) {
    my_word = bm_next[wbase + lane];
    if (bm_cur) bm_cur[wbase + lane] = my_word;
    if (clear) bm_next[wbase + lane] = 0;
  }
  uint32_t cnt = 0, edg = 0;
  uint32_t* sv = s_v + warp * (C_WPW * 32);
  uint32_t* ss = s_start + warp * (C_WPW * 32);
  uint32_t* sd = s_deg + warp * (C_WPW * 32);
#pragma unroll 1
  for (int j = 0; j < C_WPW; ++j) {
    uint32_t word = __shfl_sync(0xffffffffu, my_word, j);
    if (word == 0) continue;
    uint32_t v = (wbase + j) * 32 + lane;
    bool bit = (word >> lane) & 1u;
    uint32_t st = 0, deg = 0;
    if (bit && ro) {
      st = ro[v];
      deg = ro[v + 1] - st;
    }
    bool keep = bit && (deg > 0 || !ro);  // ro == nullptr: keep every set bit
    unsigned mask = __ballot_sync(0xffffffffu, keep);
    if (keep) {
      uint32_t pos = cnt + __popc(mask & lanemask_lt());
      sv[pos] = v;
      ss[pos] = st;
      sd[pos] = deg;
    }
    cnt += __popc(mask);
    edg += warp_sum(keep ? deg : 0u);
  }
  if (lane == 0) {
    s_wc[warp] = cnt;
    s_we[warp] = edg;
  }
  __syncthreads();

  // ---- phase 2: CTA totals, warp-parallel look-back for the global prefix ----
  if (warp == 0) {
    uint32_t tc = lane < C_WARPS ? s_wc[lane] : 0u, te = lane < C_WARPS ? s_we[lane] : 0u;
    uint32_t ic = warp_incl_scan(tc, lane), ie = warp_incl_scan(te, lane);
    uint32_t c = __shfl_sync(0xffffffffu, ic, 31), e = __shfl_sync(0xffffffffu, ie, 31);
    __syncwarp();
    if (lane < C_WARPS) {
      s_wc[lane] = ic - tc;
      s_we[lane] = ie - te;
    }
    uint32_t pc, pe;
    lb_lookback_warp(status, tile, c, e, &pc, &pe);
    if (lane == 0) {
      s_pc = pc;
      s_pe = pe;
      if (tile == ntiles - 1) {
        __threadfence();
        plan_finish(plan, ctl, pc + c, pe + e);
      }
    }
  }
  __syncthreads();

  // ---- phase 3: copy the stash out, ascending, with edge offsets ----
  uint32_t gbase = s_pc + s_wc[warp];
  uint32_t ebase = s_pe + s_we[warp];
  for (uint32_t i0 = 0; i0 < cnt; i0 += 32) {
    uint32_t i = i0 + lane;
    uint32_t deg = i < cnt ? sd[i] : 0u;
    uint32_t incl = warp_incl_scan(deg, lane);
    if (i < cnt) {
      uint32_t gi = gbase + i;
      uint32_t eoff = ebase + incl - deg;
      plan.v[gi] = sv[i];
      plan.start[gi] = ss[i];
      plan.off[gi] = eoff;
      tile_map_entries(plan, gi, eoff, deg);
    }
    ebase += __shfl_sync(0xffffffffu, incl, 31);
  }
}

// ---------------------------------------------------------------------------
// k_plan_list: sparse frontier list -> plan (duplicates and order kept,
// deg-0 entries dropped).  C_VERTS list entries per CTA.
// ---------------------------------------------------------------------------
static __global__ void __launch_bounds__(C_WARPS * 32)
k_plan_list(const uint32_t* __restrict__ ro, const uint32_t* __restrict__ list, uint32_t len,
            Plan plan, Ctl* ctl, unsigned long long* status, uint32_t ntiles) {
  __shared__ uint32_t s_v[C_VERTS];
  __shared__ uint32_t s_start[C_VERTS];
  __shared__ uint32_t s_deg[C_VERTS];
  __shared__ uint32_t s_wc[C_WARPS], s_we[C_WARPS];
  __shared__ uint32_t s_tile, s_pc, s_pe;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = atomicAdd(&ctl->tile_ctr, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t base = tile * C_VERTS + warp * (C_WPW * 32);
  uint32_t cnt = 0, edg = 0;
  uint32_t* sv = s_v + warp * (C_WPW * 32);
  uint32_t* ss = s_start + warp * (C_WPW * 32);
  uint32_t* sd = s_deg + warp * (C_WPW * 32);
  for (int j = 0; j < C_WPW; ++j) {
    uint32_t idx = base + j * 32 + lane;
    uint32_t v = 0, st = 0, deg = 0;
    if (idx < len) {
      v = list[idx];
      st = ro[v];
      deg = ro[v + 1] - st;
    }
    bool keep = idx < len && deg > 0;
    unsigned mask = __ballot_sync(0xffffffffu, keep);
    if (keep) {
      uint32_t pos = cnt + __popc(mask & lanemask_lt());
      sv[pos] = v;
      ss[pos] = st;
      sd[pos] = deg;
    }
    cnt += __popc(mask);
    edg += warp_sum(keep ? deg : 0u);
  }
  if (lane == 0) {
    s_wc[warp] = cnt;
    s_we[warp] = edg;
  }
  __syncthreads();
  // ---- phase 2: CTA totals, warp-parallel look-back for the global prefix ----
  if (warp == 0) {
    uint32_t tc = lane < C_WARPS ? s_wc[lane] : 0u, te = lane < C_WARPS ? s_we[lane] : 0u;
    uint32_t ic = warp_incl_scan(tc, lane), ie = warp_incl_scan(te, lane);
    uint32_t c = __shfl_sync(0xffffffffu, ic, 31), e = __shfl_sync(0xffffffffu, ie, 31);
    __syncwarp();
    if (lane < C_WARPS) {
      s_wc[lane] = ic - tc;
      s_we[lane] = ie - te;
    }
    uint32_t pc, pe;
    lb_lookback_warp(status, tile, c, e, &pc, &pe);
    if (lane == 0) {
      s_pc = pc;
      s_pe = pe;
      if (tile == ntiles - 1) {
        __threadfence();
        plan_finish(plan, ctl, pc + c, pe + e);
      }
    }
  }
  __syncthreads();
  uint32_t gbase = s_pc + s_wc[warp];
  uint32_t ebase = s_pe + s_we[warp];
  for (uint32_t i0 = 0; i0 < cnt; i0 += 32) {
    uint32_t i = i0 + lane;
    uint32_t deg = i < cnt ? sd[i] : 0u;
    uint32_t incl = warp_incl_scan(deg, lane);
    if (i < cnt) {
      uint32_t gi = gbase + i;
      uint32_t eoff = ebase + incl - deg;
      plan.v[gi] = sv[i];
      plan.start[gi] = ss[i];
      plan.off[gi] = eoff;
      tile_map_entries(plan, gi, eoff, deg);
    }
    ebase += __shfl_sync(0xffffffffu, incl, 31);
  }
}

// ---------------------------------------------------------------------------
// Advance operator arguments.
// ---------------------------------------------------------------------------
enum { OUT_BITMAP = 0, OUT_QUEUE = 1 };

// 4-byte distance <-> bits
__device__ __forceinline__ uint32_t dbits(float x) { return __float_as_uint(x); }
__device__ __forceinline__ uint32_t dbits(uint32_t x) { return x; }
template <class D> __device__ __forceinline__ D dfrom(uint32_t b);
template <> __device__ __forceinline__ float dfrom<float>(uint32_t b) { return __uint_as_float(b); }
template <> __device__ __forceinline__ uint32_t dfrom<uint32_t>(uint32_t b) { return b; }

// Peer-memory partition (peer.cu): owner q of global vertex v is the last q
// with start[q] <= v; its distance / packed key / next-frontier bitmap are
// reached through pointers into q's IPC-mapped slab, pre-offset so that
// dist[q][v], pkey[q][v] and bm[q][v >> 5] take the GLOBAL id (range starts
// are multiples of 32).  Local ranks use the same table (q == self).
constexpr int PEER_MAX = 8;
struct PeerTab {
  uint32_t start[PEER_MAX + 1];
  uint32_t* dist[PEER_MAX];
  unsigned long long* pkey[PEER_MAX];
  uint32_t* bm[PEER_MAX];
  uint32_t* res[PEER_MAX];
  uint32_t* cand[PEER_MAX];
  uint32_t* repair[PEER_MAX];
  // this rank's best proposal so far per REMOTE vertex (local memory, global
  // ids; null with one rank): the test-before-atomic for remote destinations
  // reads it instead of the owner's distance, so NVLink carries only
  // fire-and-forget reductions, once per improvement of this rank's own
  // proposal (the per-destination combining of a message exchange)
  uint32_t* rc;
  uint32_t nparts, self, self_lo, pad;
};

// The partitioned CSR stores each destination's owner in the top 3 bits of
// its id (n < 2^29, k_peer_encode): the advance decodes it with a shift.
constexpr uint32_t PEER_VBITS = 29, PEER_VMASK = (1u << PEER_VBITS) - 1;

__device__ __forceinline__ uint32_t peer_owner(const PeerTab& t, uint32_t v) {
  uint32_t q = 0;
#pragma unroll
  for (int i = 1; i < PEER_MAX; ++i) q += (i < (int)t.nparts && v >= t.start[i]) ? 1u : 0u;
  return q;
}

template <class W>
struct AdvArgs {
  using D = typename DT<W>::D;
  const EdgeRec<W>* adj;     // CSR records (push) / CSC records (pull)
  const uint32_t* ceid;      // CSC -> CSR edge id (pull only)
  D* dist;
  uint2* predrec;            // {u, csr edge} of the last improving relax
  Plan plan;
  Ctl* ctl;
  uint32_t* bm_out;          // OUT_BITMAP target (next frontier)
  const uint32_t* bm_in;     // pull: current frontier bitmap
  uint32_t* q_out;           // OUT_QUEUE target
  uint32_t* rec_src;         // RECORD op buffers
  uint32_t* rec_dst;
  uint32_t* rec_eid;
  uint64_t rec_cap;
  unsigned long long* status;  // zeroed here for the next look-back kernel
  uint32_t status_len;
  unsigned long long* qstatus; // OUT_QUEUE look-back state (zero at launch)
  // partitioned (multi-GPU) push: destinations in [lo, hi) are local (index
  // dst - lo); others are min-combined into rbest[dst] = (dist_bits << 32 |
  // src) and flagged in the remote bitmap rbm (mg.cu)
  uint32_t lo, hi;
  unsigned long long* rbest;
  uint32_t* rbm;
  int op;                    // gfb_op
  const PeerTab* peers;      // k_push_range<PEER>: owner-addressed destinations
  // tail queue (range_expand<ENQ>, tail.cuh): a relaxation that lowers v sets
  // v's bit in tq_bm with a returning OR; the first one appends v to tq_out
  uint32_t* tq_out;
  uint32_t* tq_cnt;
  uint32_t* tq_bm;
};

// Warp-aggregated append of `x` (one atomicAdd per warp).
__device__ __forceinline__ void warp_append(uint32_t* cnt, uint32_t* q, bool want, uint32_t x,
                                            uint64_t cap) {
  unsigned mask = __ballot_sync(0xffffffffu, want);
  if (!mask) return;
  int lane = threadIdx.x & 31;
  int leader = __ffs(mask) - 1;
  uint32_t base = 0;
  if (lane == leader) base = atomicAdd(cnt, (uint32_t)__popc(mask));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (want) {
    uint32_t pos = base + __popc(mask & lanemask_lt());
    if (pos < cap) q[pos] = x;
  }
}

__device__ __forceinline__ void warp_record(Ctl* ctl, uint32_t* rs, uint32_t* rd, uint32_t* re,
                                            uint64_t cap, bool want, uint32_t s, uint32_t d,
                                            uint32_t e) {
  unsigned mask = __ballot_sync(0xffffffffu, want);
  if (!mask) return;
  int lane = threadIdx.x & 31;
  int leader = __ffs(mask) - 1;
  uint32_t base = 0;
  if (lane == leader) base = atomicAdd(&ctl->rec_count, (uint32_t)__popc(mask));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (want) {
    uint64_t pos = (uint64_t)base + __popc(mask & lanemask_lt());
    if (pos < cap) {
      rs[pos] = s;
      rd[pos] = d;
      re[pos] = e;
    }
  }
}

// ---------------------------------------------------------------------------
// Push advance.  Persistent grid over A_TILE-edge tiles of the plan.
// Per tile: the segments intersecting it are staged in smem (vertex, row
// start, dist snapshot), every thread locates the segment of its first
// edge by binary search and walks A_VT edges to fill a local edge->segment
// map; then edges are processed thread-strided so that consecutive lanes
// stream consecutive records.
// OUT_QUEUE (operator API) keeps the reference's output order
// (frontier position, edge id): thread-contiguous edges + look-back.
// ---------------------------------------------------------------------------
template <class W, int OUT>
__global__ void __launch_bounds__(A_BLOCK)
k_advance_push(AdvArgs<W> a) {
  using D = typename DT<W>::D;
  __shared__ uint32_t s_off[A_TILE + 2];
  __shared__ uint32_t s_start[A_TILE + 2];
  __shared__ uint32_t s_u[A_TILE + 2];
  __shared__ D s_du[A_TILE + 2];
  __shared__ uint16_t s_seg[A_TILE];
  __shared__ uint32_t s_tile, s_base;
  __shared__ uint32_t s_wsum[A_BLOCK / 32];

  // Zero the look-back state for the next look-back kernel (stream order
  // guarantees the previous one has finished).
  for (uint32_t i = blockIdx.x * A_BLOCK + threadIdx.x; i < a.status_len;
       i += gridDim.x * A_BLOCK)
    a.status[i] = 0;

  const uint32_t total = a.ctl->total;
  const uint32_t k = a.ctl->k;
  const uint32_t ntiles = (total + A_TILE - 1) / A_TILE;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned* err = &a.ctl->err;
  if (blockIdx.x == 0 && tid == 0) {
    a.ctl->relax += total;  // one cond invocation per plan edge
    a.ctl->supersteps += 1;
    a.ctl->push_steps += 1;
  }

  for (uint32_t it = blockIdx.x;; it += gridDim.x) {
    uint32_t t;
    if (OUT == OUT_QUEUE) {
      // dynamic tile ids (launch order) so the look-back cannot deadlock
      if (tid == 0) s_tile = atomicAdd(&a.ctl->tile_ctr, 1u);
      __syncthreads();
      t = s_tile;
    } else {
      t = it;
    }
    if (t >= ntiles) break;
    const uint32_t e0 = t * A_TILE;
    const uint32_t cnt = min((uint32_t)A_TILE, total - e0);
    const uint32_t s0 = a.plan.tseg[t * A_RATIO];
    const uint32_t s1 = (t + 1 < ntiles) ? a.plan.tseg[(t + 1) * A_RATIO] : k - 1;
    const uint32_t nseg = s1 - s0 + 1;
    for (uint32_t j = tid; j < nseg; j += A_BLOCK) {
      uint32_t g = s0 + j;
      uint32_t off = a.plan.off[g];
      uint32_t u = a.plan.v[g];
      s_off[j] = off > e0 ? off - e0 : 0u;
      s_start[j] = a.plan.start[g] + (off < e0 ? e0 - off : 0u);
      s_u[j] = u;
      s_du[j] = a.dist ? a.dist[u] : D(0);
    }
    __syncthreads();
    // edge -> segment map
    {
      uint32_t le0 = tid * A_VT;
      if (le0 < cnt) {
        uint32_t lo = 0, hi = nseg - 1;  // largest j with s_off[j] <= le0
        while (lo < hi) {
          uint32_t mid = (lo + hi + 1) >> 1;
          if (s_off[mid] <= le0) lo = mid;
          else hi = mid - 1;
        }
        uint32_t j = lo;
#pragma unroll
        for (int r = 0; r < A_VT; ++r) {
          uint32_t le = le0 + r;
          if (le < cnt) {
            while (j + 1 < nseg && s_off[j + 1] <= le) ++j;
            s_seg[le] = (uint16_t)j;
          }
        }
      }
    }
    __syncthreads();

    if (OUT == OUT_BITMAP) {
#pragma unroll
      for (int r = 0; r < A_VT; ++r) {
        uint32_t le = r * A_BLOCK + tid;
        bool act = false, live = le < cnt;
        uint32_t e = 0, dst = 0, u = 0;
        if (live) {
          uint32_t j = s_seg[le];
          e = s_start[j] + (le - s_off[j]);
          EdgeRec<W> rec = ld_rec(a.adj + e);
          dst = rec.v;
          u = s_u[j];
          if (a.op == GFB_OP_RELAX_MIN) {
            D nd = dadd(s_du[j], rec.w, err);
            D cur = ld_dist(a.dist + dst);
            if (nd < cur) {
              D old = atomic_min_d(a.dist + dst, nd);
              if (nd < old) {
                act = true;
                a.predrec[dst] = make_uint2(u, e);
              }
            }
          } else if (a.op == GFB_OP_ALWAYS) {
            act = true;
          }
        }
        if (a.op == GFB_OP_RECORD)
          warp_record(a.ctl, a.rec_src, a.rec_dst, a.rec_eid, a.rec_cap, live, u, dst, e);
        if (act) atomicOr(a.bm_out + (dst >> 5), 1u << (dst & 31));
      }
    } else {
      // ordered queue output: thread owns edges [tid*A_VT, tid*A_VT + A_VT)
      uint32_t hits[A_VT];
      uint32_t nh = 0;
#pragma unroll
      for (int r = 0; r < A_VT; ++r) {
        uint32_t le = tid * A_VT + r;
        bool act = false, live = le < cnt;
        uint32_t e = 0, dst = 0, u = 0;
        if (live) {
          uint32_t j = s_seg[le];
          e = s_start[j] + (le - s_off[j]);
          EdgeRec<W> rec = ld_rec(a.adj + e);
          dst = rec.v;
          u = s_u[j];
          if (a.op == GFB_OP_RELAX_MIN) {
            D nd = dadd(s_du[j], rec.w, err);
            D cur = ld_dist(a.dist + dst);
            if (nd < cur) {
              D old = atomic_min_d(a.dist + dst, nd);
              if (nd < old) {
                act = true;
                a.predrec[dst] = make_uint2(u, e);
              }
            }
          } else if (a.op == GFB_OP_ALWAYS) {
            act = true;
          }
        }
        if (a.op == GFB_OP_RECORD)
          warp_record(a.ctl, a.rec_src, a.rec_dst, a.rec_eid, a.rec_cap, live, u, dst, e);
        if (act) hits[nh++] = dst;
      }
      // block-exclusive scan of per-thread hit counts
      uint32_t incl = warp_incl_scan(nh, lane);
      if (lane == 31) s_wsum[warp] = incl;
      __syncthreads();
      if (tid == 0) {
        uint32_t c = 0;
        for (int w = 0; w < A_BLOCK / 32; ++w) {
          uint32_t x = s_wsum[w];
          s_wsum[w] = c;
          c += x;
        }
        uint32_t pc, pe;
        lb_lookback(a.qstatus, t, c, 0u, &pc, &pe);
        s_base = pc;
        if (t == ntiles - 1) a.ctl->out_count = pc + c;
      }
      __syncthreads();
      uint32_t pos = s_base + s_wsum[warp] + incl - nh;
      for (uint32_t i = 0; i < nh; ++i) a.q_out[pos + i] = hits[i];
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Pull advance.  Segments = destination vertices with in-degree > 0 (a
// static plan over the CSC built at upload).  Every in-edge whose source is
// in the current frontier bitmap is a cond invocation; RELAX_MIN reduces
// the candidates per destination in smem (bit-pattern atomicMin) and does
// at most one global atomicMin per (tile, destination).
// ---------------------------------------------------------------------------
template <class W>
__global__ void __launch_bounds__(A_BLOCK)
k_advance_pull(AdvArgs<W> a, uint32_t total, uint32_t k) {
  using D = typename DT<W>::D;
  using Bits = typename DT<W>::Bits;
  __shared__ uint32_t s_off[A_TILE + 2];
  __shared__ uint32_t s_start[A_TILE + 2];
  __shared__ uint32_t s_u[A_TILE + 2];
  __shared__ Bits s_best[A_TILE + 2];
  __shared__ uint32_t s_slot[A_TILE + 2];
  __shared__ uint16_t s_seg[A_TILE];
  for (uint32_t i = blockIdx.x * A_BLOCK + threadIdx.x; i < a.status_len;
       i += gridDim.x * A_BLOCK)
    a.status[i] = 0;
  const uint32_t ntiles = (total + A_TILE - 1) / A_TILE;
  const int tid = threadIdx.x;
  unsigned* err = &a.ctl->err;
  if (blockIdx.x == 0 && tid == 0) {
    a.ctl->supersteps += 1;
    a.ctl->pull_steps += 1;
  }
  uint32_t n_elig = 0;
  for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint32_t e0 = t * A_TILE;
    const uint32_t cnt = min((uint32_t)A_TILE, total - e0);
    const uint32_t s0 = a.plan.tseg[t * A_RATIO];
    const uint32_t s1 = (t + 1 < ntiles) ? a.plan.tseg[(t + 1) * A_RATIO] : k - 1;
    const uint32_t nseg = s1 - s0 + 1;
    for (uint32_t j = tid; j < nseg; j += A_BLOCK) {
      uint32_t g = s0 + j;
      uint32_t off = a.plan.off[g];
      s_off[j] = off > e0 ? off - e0 : 0u;
      s_start[j] = a.plan.start[g] + (off < e0 ? e0 - off : 0u);
      s_u[j] = a.plan.v[g];
      s_best[j] = (Bits)DT<W>::INF_BITS;
      s_slot[j] = NIL;
    }
    __syncthreads();
    {
      uint32_t le0 = tid * A_VT;
      if (le0 < cnt) {
        uint32_t lo = 0, hi = nseg - 1;
        while (lo < hi) {
          uint32_t mid = (lo + hi + 1) >> 1;
          if (s_off[mid] <= le0) lo = mid;
          else hi = mid - 1;
        }
        uint32_t j = lo;
#pragma unroll
        for (int r = 0; r < A_VT; ++r) {
          uint32_t le = le0 + r;
          if (le < cnt) {
            while (j + 1 < nseg && s_off[j + 1] <= le) ++j;
            s_seg[le] = (uint16_t)j;
          }
        }
      }
    }
    __syncthreads();
    D cand[A_VT];
    uint32_t cslot[A_VT];
#pragma unroll
    for (int r = 0; r < A_VT; ++r) {
      uint32_t le = r * A_BLOCK + tid;
      cslot[r] = NIL;
      bool live = le < cnt;
      uint32_t slot = 0, src = 0, j = 0;
      bool elig = false;
      EdgeRec<W> rec;
      if (live) {
        j = s_seg[le];
        slot = s_start[j] + (le - s_off[j]);
        rec = ld_rec(a.adj + slot);
        src = rec.v;
        elig = (a.bm_in[src >> 5] >> (src & 31)) & 1u;
        n_elig += elig;
      }
      if (a.op == GFB_OP_RECORD) {
        uint32_t eid = elig ? a.ceid[slot] : 0u;
        warp_record(a.ctl, a.rec_src, a.rec_dst, a.rec_eid, a.rec_cap, elig, src,
                    live ? s_u[j] : 0u, eid);
      } else if (elig) {
        if (a.op == GFB_OP_RELAX_MIN) {
          D nd = dadd(ld_dist(a.dist + src), rec.w, err);
          cand[r] = nd;
          cslot[r] = slot;
          Bits b = *reinterpret_cast<Bits*>(&nd);
          atomicMin(&s_best[j], b);
        } else {  // ALWAYS: activation only
          s_slot[j] = slot;
        }
      }
    }
    __syncthreads();
    if (a.op == GFB_OP_RELAX_MIN) {
#pragma unroll
      for (int r = 0; r < A_VT; ++r) {
        if (cslot[r] != NIL) {
          uint32_t le = r * A_BLOCK + tid;
          uint32_t j = s_seg[le];
          D nd = cand[r];
          if (*reinterpret_cast<Bits*>(&nd) == s_best[j]) s_slot[j] = cslot[r];  // any tie
        }
      }
      __syncthreads();
    }
    for (uint32_t j = tid; j < nseg; j += A_BLOCK) {
      uint32_t slot = s_slot[j];
      if (slot == NIL) continue;
      uint32_t u = s_u[j];
      bool act = true;
      if (a.op == GFB_OP_RELAX_MIN) {
        Bits b = s_best[j];
        D best = *reinterpret_cast<D*>(&b);
        D cur = ld_dist(a.dist + u);
        act = false;
        if (best < cur) {
          D old = atomic_min_d(a.dist + u, best);
          if (best < old) {
            act = true;
            EdgeRec<W> rec = ld_rec(a.adj + slot);
            a.predrec[u] = make_uint2(rec.v, slot | PRED_CSC_SLOT);
          }
        }
      }
      if (act) atomicOr(a.bm_out + (u >> 5), 1u << (u & 31));
    }
    __syncthreads();
  }
  n_elig = warp_sum(n_elig);  // eligible in-edges = cond invocations
  if ((tid & 31) == 0 && n_elig) atomicAdd(&a.ctl->relax, (unsigned long long)n_elig);
}

// ---------------------------------------------------------------------------
// Init (algorithms.hpp:144-148): dist = +inf, pred = NIL, bitmaps clear,
// dist[source] = 0 and the source marked in the next-frontier bitmap.
// ---------------------------------------------------------------------------
template <class W>
__global__ void k_init(typename DT<W>::D* dist, uint2* predrec, uint32_t* bm_next,
                       uint32_t* bm_cur, uint32_t n, uint32_t nwords, const uint32_t* src_ptr,
                       Ctl* ctl) {
  using D = typename DT<W>::D;
  const uint32_t source = *src_ptr;  // device-resident: graph launches stay source-agnostic
  uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    dist[i] = i == source ? D(0) : dinf<W>();
    predrec[i] = make_uint2(NIL, NIL);
  }
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nwords; i += stride) {
    uint32_t w = (source >> 5) == i ? (1u << (source & 31)) : 0u;
    bm_next[i] = w;
    if (bm_cur) bm_cur[i] = 0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    Ctl c = {};
    *ctl = c;
  }
}

// ---------------------------------------------------------------------------
// Predecessor pass.
//  k_pred_verify: pred[v] = u of the recorded improving relax when that edge
//    is still tight and strictly decreasing (dist[u] < dist[v]); else v goes
//    to the repair set.  Strictly decreasing chains are acyclic.
//  repair rounds (k_pred_csc_block with a transpose, k_pred_list_round over
//    the collected in-edges without one): round r accepts a tight edge u->v
//    when u was resolved in an earlier round (round 1: dist[u] < dist[v];
//    later rounds: equal distances, the zero-weight tie classes that make a
//    plain argmin cycle, cf. algorithms.hpp:71-76).  Smallest u wins.
// Also accumulates n_reach / m_reach for the bench's GTEPS.
// ---------------------------------------------------------------------------
// PERM (relabelled loop, 32-bit keys): the loop's state lives in relabelled
// ids; the pass reads it through perm (dist_int / key_int), maps the key's
// source back through iperm and writes dist / predrec in the caller's ids --
// the unpermute pass fused into the verification.
template <class D>
struct PermView {
  const uint32_t* perm;
  const uint32_t* iperm;
  const D* dist_int;
  const unsigned long long* key_int;
  D* dist_out;
  unsigned long long* key_out;
  const void* adj_int;  // relabelled CSR records (record mode: {u', edge'} keys)
};

template <class W, bool KEY = false, bool PERM = false>
__global__ void __launch_bounds__(256)
k_pred_verify(const uint32_t* __restrict__ ro, const EdgeRec<W>* __restrict__ adj,
              const uint32_t* __restrict__ co, const EdgeRec<W>* __restrict__ cadj,
              const typename DT<W>::D* __restrict__ dist, const uint2* __restrict__ predrec,
              uint32_t* pred, uint32_t* res, uint32_t* repair_bm, uint32_t* unres_list,
              uint32_t n, uint32_t source, Ctl* ctl,
              PermView<typename DT<W>::D> pv = PermView<typename DT<W>::D>{}) {
  using D = typename DT<W>::D;
  constexpr int U = 4;  // vertices per thread per round, loads issued together
  __shared__ unsigned long long s_nr[8], s_mr[8];
  __shared__ uint32_t s_un[8];
  const uint32_t stride = gridDim.x * blockDim.x;
  unsigned long long nr = 0, mr = 0;
  uint32_t unres = 0;
  for (uint32_t v0 = blockIdx.x * blockDim.x + threadIdx.x; v0 < n; v0 += stride * U) {
    D dv[U];
    uint2 pr[U];
    uint32_t deg[U];
    uint32_t uint_[U];
#pragma unroll
    for (int r = 0; r < U; ++r) {
      uint32_t v = v0 + r * stride;
      if constexpr (PERM) {
        const uint32_t i = v < n ? pv.perm[v] : 0u;
        dv[r] = v < n ? pv.dist_int[i] : dinf<W>();
        const unsigned long long k = v < n ? pv.key_int[i] : ~0ull;
        pr[r] = make_uint2((uint32_t)k, (uint32_t)(k >> 32));  // .x: relabelled source
      } else {
        dv[r] = v < n ? dist[v] : dinf<W>();
        pr[r] = v < n ? predrec[v] : make_uint2(NIL, NIL);
      }
      deg[r] = v < n ? ro[v + 1] - ro[v] : 0u;
    }
    if constexpr (PERM) {  // the caller's ids of the key sources; write the results back
#pragma unroll
      for (int r = 0; r < U; ++r) {
        const uint32_t v = v0 + r * stride;
        uint_[r] = pr[r].x;
        if (pr[r].x != NIL) pr[r].x = pv.iperm[pr[r].x];
        if (v < n) {
          pv.dist_out[v] = dv[r];
          if (pv.key_out) pv.key_out[v] = ((unsigned long long)pr[r].y << 32) | pr[r].x;
        }
      }
    }
    EdgeRec<W> rec[U];
    D du[U];
#pragma unroll
    for (int r = 0; r < U; ++r) {
      uint32_t v = v0 + r * stride;
      bool look = v < n && v != source && !(dv[r] == dinf<W>()) && pr[r].x != NIL &&
                  pr[r].y != NIL;
      if (look && KEY) {
        // packed key (dist_bits << 32 | u), k_push_range: the edge u -> v
        // that proposed dist[v] is tight at the fixpoint (any later drop of
        // dist[u] re-expanded u and would have lowered the key)
        if constexpr (PERM) du[r] = pv.dist_int[uint_[r]];
        else du[r] = dist[pr[r].x];
        rec[r].v = pr[r].y == *reinterpret_cast<const uint32_t*>(&dv[r]) ? v : NIL;
      } else if (look && PERM) {
        // record mode on the relabelled loop: {u', edge'} index the relabelled
        // CSR; the edge must end at v's relabelled id
        rec[r] = reinterpret_cast<const EdgeRec<W>*>(pv.adj_int)[pr[r].y];
        rec[r].v = rec[r].v == pv.perm[v] ? v : NIL;
        du[r] = pv.dist_int[uint_[r]];
      } else if (look) {
        if (pr[r].y & PRED_CSC_SLOT) {  // recorded by a pull step: CSC slot of v
          const uint32_t sl = pr[r].y & ~PRED_CSC_SLOT;
          rec[r] = (cadj && sl >= co[v] && sl < co[v + 1]) ? cadj[sl] : EdgeRec<W>{};
          if (cadj && sl >= co[v] && sl < co[v + 1] && rec[r].v == pr[r].x) rec[r].v = v;
          else rec[r].v = NIL;
        } else {
          rec[r] = adj[pr[r].y];
        }
        du[r] = dist[pr[r].x];
      }
    }
#pragma unroll
    for (int r = 0; r < U; ++r) {
      uint32_t v = v0 + r * stride;
      if (v >= n) continue;
      uint32_t p = NIL, rr = 0;
      if (!(dv[r] == dinf<W>())) {
        ++nr;
        mr += deg[r];
        if (v == source) {
          rr = 1;
        } else {
          if (pr[r].x != NIL && pr[r].y != NIL && rec[r].v == v && du[r] < dv[r] &&
              (KEY || dadd(du[r], rec[r].w, nullptr) == dv[r])) {
            p = pr[r].x;
            rr = 1;
          }
          if (!rr) {
            ++unres;
            atomicOr(repair_bm + (v >> 5), 1u << (v & 31));
            unres_list[atomicAdd(&ctl->flag, 1u)] = v;  // rare: races and ties
          }
        }
      }
      pred[v] = p;
      res[v] = rr;
    }
  }
  // block reduction, then one atomic per counter per block
  for (int d = 16; d > 0; d >>= 1) {
    nr += __shfl_xor_sync(0xffffffffu, nr, d);
    mr += __shfl_xor_sync(0xffffffffu, mr, d);
    unres += __shfl_xor_sync(0xffffffffu, unres, d);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    s_nr[warp] = nr;
    s_mr[warp] = mr;
    s_un[warp] = unres;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    nr = mr = 0;
    unres = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      nr += s_nr[w];
      mr += s_mr[w];
      unres += s_un[w];
    }
    if (nr) atomicAdd(&ctl->n_reach, nr);
    if (mr) atomicAdd(&ctl->m_reach, mr);
    if (unres) atomicAdd(&ctl->unresolved, unres);
  }
}

// CSC repair round, one CTA per unresolved vertex (a hub's in-edge list is
// hundreds of thousands long: one warp scanning it took 80 us per round at
// s24).  The list length is read on the device (ctl->unresolved), so rounds
// can be queued without a host round trip.  Round 1 accepts strictly
// decreasing tight in-edges, round r > 1 equal-distance tight in-edges from
// vertices resolved in an earlier round.  Smallest acceptable CSC slot wins
// (= smallest source id: CSC slots are ascending by source).
template <class W>
__global__ void __launch_bounds__(256)
k_pred_csc_block(const uint32_t* __restrict__ co, const EdgeRec<W>* __restrict__ cadj,
                 const typename DT<W>::D* __restrict__ dist, uint32_t* pred, uint32_t* res,
                 const uint32_t* list, uint32_t round, Ctl* ctl, uint32_t base = 0) {
  using D = typename DT<W>::D;
  __shared__ uint32_t s_slot;
  const uint32_t count = ctl->unresolved;
  uint32_t done = 0;
  for (uint32_t i = blockIdx.x; i < count; i += gridDim.x) {
    const uint32_t v = list[i];
    if (res[v] != 0) continue;  // block-uniform
    const D dv = dist[v];
    const uint32_t lo = co[v], hi = co[v + 1];
    if (threadIdx.x == 0) s_slot = NIL;
    __syncthreads();
    for (uint32_t chunk = lo; chunk < hi; chunk += blockDim.x) {
      const uint32_t slot = chunk + threadIdx.x;
      if (slot < hi) {
        const EdgeRec<W> rec = cadj[slot];
        const D du = dist[rec.v];
        bool ok = false;
        if (!(du == dinf<W>()) && dadd(du, rec.w, nullptr) == dv) {
          if (round == 1) {
            ok = du < dv;
          } else {
            const uint32_t ru = res[rec.v];
            ok = du == dv && ru != 0 && ru <= base + round;
          }
        }
        if (ok) atomicMin(&s_slot, slot);
      }
      __syncthreads();
      if (s_slot != NIL) break;  // block-uniform: the first chunk with a hit holds the minimum
    }
    if (threadIdx.x == 0 && s_slot != NIL) {
      pred[v] = cadj[s_slot].v;
      res[v] = base + round + 1;
      ++done;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && done) {
    atomicAdd(&ctl->flag, done);
    atomicAdd(&ctl->resolved, done);
  }
}

// Key rounds (32-bit distances, before any in-edge scan): an unresolved v
// failed verification only because its key's source u0 has dist[u0] ==
// dist[v] (zero or absorbed weight) -- the edge is still tight.  Round k
// accepts u0 once u0 is resolved with res[u0] <= k (verify resolves with 1)
// and assigns k + 1, the equal-distance rule of the repair rounds, so chains
// stay acyclic.  Only keys that point around a zero-weight cycle are left
// for the in-edge rounds.
template <class W>
__global__ void k_pred_key_round(const uint32_t* __restrict__ list,
                                 const unsigned long long* __restrict__ key,
                                 const typename DT<W>::D* __restrict__ dist, uint32_t* pred,
                                 uint32_t* res, uint32_t* repair_bm, uint32_t k, Ctl* ctl,
                                 const uint32_t* __restrict__ perm = nullptr,
                                 const uint32_t* __restrict__ iperm = nullptr) {
  const uint32_t count = ctl->unresolved;
  uint32_t done = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
    const uint32_t v = list[i];
    if (res[v] != 0) continue;
    // relabelled loop: the keys stay in loop ids (k_pred_verify<PERM> does not
    // write them back for every vertex), mapped here for the few unresolved
    uint32_t u = perm ? (uint32_t)key[perm[v]] : (uint32_t)key[v];
    if (perm && u != NIL) u = iperm[u];
    if (u == NIL || !(dist[u] == dist[v])) continue;
    const uint32_t ru = res[u];
    if (ru != 0 && ru <= k) {
      pred[v] = u;
      res[v] = k + 1;
      atomicAnd(repair_bm + (v >> 5), ~(1u << (v & 31)));  // off the in-edge scan
      ++done;
    }
  }
  done = warp_sum(done);
  if ((threadIdx.x & 31) == 0 && done) atomicAdd(&ctl->resolved, done);
}

// Repair without a transpose: one pass over the CSR collects the in-edges of
// the (few) unresolved vertices into a list, then every round only scans the
// list.  Rows are walked warp-per-32-rows (shuffle search for the owning row)
// and rows longer than PR_BIG one CTA per row, so hubs do not serialise a
// warp.  Overflow of the list (cap entries) sets ctl->err bit 2.
constexpr uint32_t PR_BIG = 1024;
template <class W>
__device__ __forceinline__ void pr_emit(uint32_t u, const EdgeRec<W>& r, const uint32_t* repair_bm,
                                        uint4* list, uint32_t cap, Ctl* ctl) {
  if ((repair_bm[r.v >> 5] >> (r.v & 31)) & 1u) {
    const uint32_t i = atomicAdd(&ctl->out_count, 1u);
    if (i < cap) list[i] = make_uint4(u, r.v, *reinterpret_cast<const uint32_t*>(&r.w),
                                      sizeof(W) == 8 ? reinterpret_cast<const uint32_t*>(&r.w)[1] : 0u);
    else atomicOr(&ctl->err, 4u);
  }
}

template <class W>
__global__ void k_pred_inedges(const uint32_t* __restrict__ ro, const EdgeRec<W>* __restrict__ adj,
                               const uint32_t* __restrict__ repair_bm, uint32_t n, uint4* list,
                               uint32_t cap, uint32_t* big, Ctl* ctl) {
  const int lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t i0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; i0 < n;
       i0 += warps * 32) {
    const uint32_t u = i0 + lane;
    uint32_t s0 = 0, len = 0;
    if (u < n) {
      s0 = ro[u];
      len = ro[u + 1] - s0;
      if (len > PR_BIG) {
        big[atomicAdd(&ctl->rec_count, 1u)] = u;
        len = 0;
      }
    }
    const uint32_t incl = warp_incl_scan(len, lane);
    const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
    for (uint32_t x = lane; x - lane < tot; x += 32) {
      int lo = 0;
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const uint32_t q = __shfl_sync(0xffffffffu, incl, lo + step - 1);
        if (q <= x) lo += step;
      }
      const uint32_t os = __shfl_sync(0xffffffffu, s0, lo);
      const uint32_t opre = __shfl_sync(0xffffffffu, incl, lo) - __shfl_sync(0xffffffffu, len, lo);
      if (x < tot) pr_emit<W>(i0 + lo, adj[os + (x - opre)], repair_bm, list, cap, ctl);
    }
  }
}

template <class W>
__global__ void k_pred_inedges_big(const uint32_t* __restrict__ ro,
                                   const EdgeRec<W>* __restrict__ adj,
                                   const uint32_t* __restrict__ repair_bm, uint4* list,
                                   uint32_t cap, const uint32_t* big, Ctl* ctl) {
  const uint32_t cnt = ctl->rec_count;
  for (uint32_t k = blockIdx.x; k < cnt; k += gridDim.x) {
    const uint32_t u = big[k], s0 = ro[u], len = ro[u + 1] - s0;
    for (uint32_t x = threadIdx.x; x < len; x += blockDim.x)
      pr_emit<W>(u, adj[s0 + x], repair_bm, list, cap, ctl);
  }
}

// Few unresolved vertices (the usual case): one flat, coalesced pass over the
// edge records; a 64 Kbit shared-memory filter of the unresolved list
// (ctl->unresolved entries of `list`) screens destinations, and only filter
// hits read the repair bitmap and binary-search the source row.  The
// row-structured k_pred_inedges reads the same records but checks the global
// bitmap per edge (f64 s24: 5.0 ms for 357 unresolved vertices).
constexpr uint32_t PR_FILTER_BITS = 1u << 16;
constexpr uint32_t PR_FLAT_MAX = 8192;  // unresolved vertices the filter screens well
__device__ __forceinline__ uint32_t pr_hash(uint32_t v) { return (v * 2654435761u) >> 16; }

template <class W>
__global__ void __launch_bounds__(256)
k_pred_inedges_flat(const uint32_t* __restrict__ ro, const EdgeRec<W>* __restrict__ adj,
                    uint32_t n, uint64_t m, const uint32_t* __restrict__ repair_bm,
                    const uint32_t* __restrict__ list, uint4* out, uint32_t cap, Ctl* ctl) {
  __shared__ uint32_t s_f[PR_FILTER_BITS / 32];
  for (uint32_t i = threadIdx.x; i < PR_FILTER_BITS / 32; i += blockDim.x) s_f[i] = 0;
  __syncthreads();
  const uint32_t cnt = ctl->unresolved;
  for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) {
    const uint32_t h = pr_hash(list[i]);
    atomicOr(&s_f[h >> 5], 1u << (h & 31));
  }
  __syncthreads();
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const EdgeRec<W> r = ld_rec(adj + e);
    const uint32_t h = pr_hash(r.v);
    if (!((s_f[h >> 5] >> (h & 31)) & 1u)) continue;
    if (!((repair_bm[r.v >> 5] >> (r.v & 31)) & 1u)) continue;
    uint32_t lo = 0, hi = n;  // source row: the last u with ro[u] <= e
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if ((uint64_t)ro[mid] <= e) lo = mid;
      else hi = mid;
    }
    const uint32_t i = atomicAdd(&ctl->out_count, 1u);
    if (i < cap)
      out[i] = make_uint4(lo, r.v, *reinterpret_cast<const uint32_t*>(&r.w),
                          sizeof(W) == 8 ? reinterpret_cast<const uint32_t*>(&r.w)[1] : 0u);
    else atomicOr(&ctl->err, 4u);
  }
}

// One repair round over the collected in-edges (same acceptance rule as
// k_pred_csc_block; smallest source wins through atomicMin on cand[v]).
template <class W>
__global__ void k_pred_list_round(const uint4* __restrict__ list, const Ctl* __restrict__ ctl,
                                  uint32_t cap, const typename DT<W>::D* __restrict__ dist,
                                  const uint32_t* __restrict__ res, uint32_t* cand,
                                  uint32_t round, uint32_t base = 0) {
  using D = typename DT<W>::D;
  const uint32_t cnt = min(ctl->out_count, cap);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
    const uint4 e = list[i];
    if (res[e.y] != 0) continue;
    W w;
    if constexpr (sizeof(W) == 8) {
      const unsigned long long b = ((unsigned long long)e.w << 32) | e.z;
      w = *reinterpret_cast<const W*>(&b);
    } else {
      w = *reinterpret_cast<const W*>(&e.z);
    }
    const D du = dist[e.x], dv = dist[e.y];
    if (du == dinf<W>() || !(dadd(du, w, nullptr) == dv)) continue;
    bool ok;
    if (round == 1) {
      ok = du < dv;
    } else {
      const uint32_t ru = res[e.x];
      ok = du == dv && ru != 0 && ru <= base + round;
    }
    if (ok) atomicMin(cand + e.y, e.x);
  }
}

// Apply round `round`'s candidates; counts how many vertices were resolved.
static __global__ void k_pred_apply(uint32_t* cand, uint32_t* pred, uint32_t* res,
                             uint32_t* repair_bm, uint32_t n, uint32_t round, Ctl* ctl,
                             uint32_t base = 0) {
  uint32_t stride = gridDim.x * blockDim.x;
  uint32_t done = 0;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
    uint32_t c = cand[v];
    if (c != NIL && res[v] == 0) {
      pred[v] = c;
      res[v] = base + round + 1;
      cand[v] = NIL;
      atomicAnd(repair_bm + (v >> 5), ~(1u << (v & 31)));
      ++done;
    }
  }
  done = warp_sum(done);
  if ((threadIdx.x & 31) == 0 && done) atomicAdd(&ctl->flag, done);
}

}  // namespace gfb
