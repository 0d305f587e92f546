// mg.cu -- one rank's share of the 1-D partitioned SSSP.
//
// The global graph is split into contiguous vertex ranges [lo, hi) with
// edge-balanced cut points; a rank holds the CSR rows of its range (column
// ids stay global), the distances / frontier bitmaps of its vertices, and a
// per-destination staging array for remote candidates:
//   rbest[v] = min over this superstep's candidates of (dist_bits << 32 | src)
// (jointly atomic: the smallest distance, ties to the smallest source), with
// a bitmap rbm of touched remote v.  Per superstep (driver: mg.py):
//   gfb_part_advance  plan local frontier -> k_push_warp<PART> (local
//                     destinations relaxed in place, remote ones combined in
//                     rbest) -> messages {v, src, dist_bits, 0} in ascending v,
//                     i.e. grouped by owner, + per-owner counts
//   (driver)          all-to-all of counts and payload (NCCL over NVLink on
//                     GPUs, gloo in the CPU tests)
//   gfb_part_apply    owners atomicMin the received candidates, activate
//   gfb_part_pending  local next-frontier size -> allreduce -> convergence
// Only 4-byte distance modes (f32, u32) are partitioned.
#include <algorithm>
#include <cstring>

#include "frontier.cuh"
#include "hot.cuh"
#include "impl.hpp"

namespace gfb {

Graph* graph_upload(Ctx*, uint64_t, uint64_t, const uint32_t*, const uint32_t*, const void*, int,
                    int, int, uint64_t);



// ---- remote message compaction (ascending destination = grouped by owner)
__global__ void __launch_bounds__(256) k_rcount(const uint32_t* __restrict__ rbm, uint32_t nwords,
                                                uint32_t* agg) {
  __shared__ uint32_t s[8];
  uint32_t c = 0;
  for (uint32_t i = blockIdx.x * 2048 + threadIdx.x; i < min((blockIdx.x + 1) * 2048, nwords);
       i += 256)
    c += __popc(rbm[i]);
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < 8; ++w) t += s[w];
    agg[blockIdx.x] = t;
  }
}

// single CTA: exclusive scan of tile counts in place, total -> *tot
__global__ void __launch_bounds__(1024) k_rscan(uint32_t* agg, uint32_t tiles, uint32_t* tot) {
  __shared__ uint32_t s[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t per = (tiles + 1023) / 1024, lo = tid * per, hi = min(lo + per, tiles);
  uint32_t c = 0;
  for (uint32_t i = lo; i < hi; ++i) c += agg[i];
  uint32_t ic = warp_incl_scan(c, lane);
  if (lane == 31) s[warp] = ic;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = s[lane];
    s[lane] = warp_incl_scan(w, lane) - w;
  }
  __syncthreads();
  uint32_t p = s[warp] + ic - c;
  for (uint32_t i = lo; i < hi; ++i) {
    uint32_t a = agg[i];
    agg[i] = p;
    p += a;
  }
  if (tid == 1023) *tot = p;
}

// one warp per 64-word slice of the tile: messages in ascending v, staging reset
__global__ void __launch_bounds__(256) k_rwrite(uint32_t* rbm, unsigned long long* rbest,
                                                uint32_t nwords, const uint32_t* prefix,
                                                uint4* out, uint64_t cap) {
  __shared__ uint32_t s_w[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t base = blockIdx.x * 2048 + warp * 256;  // 256 words per warp
  uint32_t cnt = 0;
  for (uint32_t i = base + lane; i < min(base + 256, nwords); i += 32) cnt += __popc(rbm[i]);
  cnt = warp_sum(cnt);
  if (lane == 0) s_w[warp] = cnt;
  __syncthreads();
  uint32_t pos = prefix[blockIdx.x];
  for (int w = 0; w < warp; ++w) pos += s_w[w];
  const uint32_t end = min(base + 256, nwords);
  for (uint32_t c0 = base; c0 < end; c0 += 32) {
    const uint32_t my = c0 + lane < end ? rbm[c0 + lane] : 0u;  // 32 words per load
    if (!__any_sync(0xffffffffu, my != 0)) continue;
    for (int j = 0; j < 32; ++j) {
      const uint32_t word = __shfl_sync(0xffffffffu, my, j);
      if (!word) continue;  // warp-uniform
      if ((word >> lane) & 1u) {
        const uint32_t v = (c0 + j) * 32 + lane;
        const unsigned long long key = rbest[v];
        const uint64_t slot = (uint64_t)pos + __popc(word & lanemask_lt());
        if (slot < cap) out[slot] = make_uint4(v, (uint32_t)key, (uint32_t)(key >> 32), 0u);
        rbest[v] = ~0ull;
      }
      pos += __popc(word);
    }
    if (my) rbm[c0 + lane] = 0;
  }
}

__global__ void k_owner_counts(const uint4* msgs, const uint32_t* tot,
                               const uint32_t* range_starts, int nparts, uint32_t* counts) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nparts) return;
  const uint32_t total = *tot;
  auto lb = [&](uint32_t key) {
    uint32_t lo = 0, hi = total;
    while (lo < hi) {
      uint32_t mid = (lo + hi) >> 1;
      if (msgs[mid].x < key) lo = mid + 1;
      else hi = mid;
    }
    return lo;
  };
  counts[p] = lb(range_starts[p + 1]) - lb(range_starts[p]);
}

template <class W>
__global__ void k_apply(const uint4* __restrict__ msgs, uint64_t count, uint32_t lo,
                        typename DT<W>::D* dist, uint32_t* bm_next, uint2* predrec) {
  using D = typename DT<W>::D;
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    uint4 m = msgs[i];
    uint32_t v = m.x - lo;
    uint32_t bits = m.z;
    D nd = *reinterpret_cast<D*>(&bits);
    if (nd < ld_dist(dist + v) && nd < atomic_min_d(dist + v, nd)) {
      predrec[v] = make_uint2(m.y, NIL);
      atomicOr(bm_next + (v >> 5), 1u << (v & 31));
    }
  }
}

template <class W>
__global__ void k_part_init(typename DT<W>::D* dist, uint2* predrec, uint32_t* bm_next,
                            uint32_t* bm_cur, uint32_t n, uint32_t nwords, uint32_t lo,
                            uint32_t source, unsigned long long* rbest, uint32_t* rbm,
                            uint64_t n_global, uint32_t rwords) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (uint64_t i = t; i < n; i += stride) {
    dist[i] = (uint32_t)i + lo == source ? typename DT<W>::D(0) : dinf<W>();
    predrec[i] = make_uint2(NIL, NIL);
  }
  for (uint64_t i = t; i < nwords; i += stride) {
    uint32_t w = 0;
    if (source >= lo && source - lo < n && (source - lo) >> 5 == i) w = 1u << ((source - lo) & 31);
    bm_next[i] = w;
    bm_cur[i] = 0;
  }
  for (uint64_t i = t; i < n_global; i += stride) rbest[i] = ~0ull;
  for (uint64_t i = t; i < rwords; i += stride) rbm[i] = 0;
}

__global__ void k_count_bits(const uint32_t* bm, uint32_t nwords, unsigned long long* out) {
  uint32_t c = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nwords; i += gridDim.x * blockDim.x)
    c += __popc(bm[i]);
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (unsigned long long)c);
}

// Predecessor candidates over the local edges given the global distances:
// round 1 strict tight edges; round r > 1 equal-distance tight edges from
// sources resolved before round r (same rules as the single-GPU repair).
template <class W>
__global__ void k_part_pred(const uint32_t* __restrict__ ro, const EdgeRec<W>* __restrict__ adj,
                            uint32_t n, uint32_t lo, const typename DT<W>::D* __restrict__ gdist,
                            const uint32_t* __restrict__ res, uint32_t* cand, uint32_t round) {
  using D = typename DT<W>::D;
  const int lane = threadIdx.x & 31;
  uint32_t warps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t ul = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); ul < n; ul += warps) {
    uint32_t u = ul + lo;
    D du = gdist[u];
    if (du == dinf<W>()) continue;
    uint32_t ru = res[u];
    if (round > 1 && (ru == 0 || ru > round)) continue;
    for (uint32_t e = ro[ul] + lane; e < ro[ul + 1]; e += 32) {
      EdgeRec<W> rec = adj[e];
      uint32_t v = rec.v;
      if (res[v] != 0) continue;
      D dv = gdist[v];
      bool ok = round == 1 ? du < dv : du == dv;
      if (ok && dadd(du, rec.w, nullptr) == dv) atomicMin(cand + v, u);
    }
  }
}

template <class W>
static void part_init_t(Part* p, uint32_t source) {
  Ctx* c = p->ctx;
  const uint32_t n = (uint32_t)p->g->n, nwords = (n + 31) / 32;
  const uint32_t rwords = (uint32_t)((p->n_global + 31) / 32);
  k_part_init<W><<<stride_grid(c), 256, 0, c->stream>>>(
      p->dist.as<typename DT<W>::D>(), p->predrec.as<uint2>(), p->bm_next.as<uint32_t>(),
      p->bm_cur.as<uint32_t>(), n, nwords, p->lo, source, p->rbest.as<unsigned long long>(),
      p->rbm.as<uint32_t>(), p->n_global, rwords);
  GFB_CUDA(cudaMemsetAsync(p->ctl.p, 0, sizeof(Ctl), c->stream));
  GFB_CUDA(cudaGetLastError());
  c->sync();
  p->relax = 0;
  p->supersteps = 0;
}

template <class W>
static uint64_t part_advance_t(Part* p, void* out, uint64_t cap, const uint32_t* range_starts,
                               int nparts, uint32_t* counts_host) {
  using D = typename DT<W>::D;
  Ctx* c = p->ctx;
  cudaStream_t s = c->stream;
  Graph* g = p->g.get();
  const uint32_t n = (uint32_t)g->n, nwords = (n + 31) / 32;
  const uint32_t rwords = (uint32_t)((p->n_global + 31) / 32);
  Plan plan{p->pv.as<uint32_t>(), p->pstart.as<uint32_t>(), p->poff.as<uint32_t>(),
            p->ptseg.as<uint32_t>(), (uint32_t)(p->ptseg.bytes / 4)};
  // local frontier -> plan
  cudaGraphConditionalHandle none{};
  k_fcount<<<p->ftiles, F_WARPS * 32, 0, s>>>(g->ro.as<uint32_t>(), p->bm_next.as<uint32_t>(),
                                             nwords, p->agg.as<uint2>());
  k_fscan<<<1, F_SCAN_THREADS, 0, s>>>(p->agg.as<uint2>(), p->ftiles, plan, p->ctl.as<Ctl>(),
                                      (uint32_t)g->m, 1.0f, 0, 0, none, none, 0, 0);
  k_fwrite<<<p->ftiles, F_WARPS * 32, 0, s>>>(g->ro.as<uint32_t>(), p->bm_next.as<uint32_t>(),
                                             p->bm_cur.as<uint32_t>(), nwords, p->agg.as<uint2>(),
                                             plan);
  // partitioned push
  AdvArgs<W> a{};
  a.adj = g->adj.as<EdgeRec<W>>();
  a.dist = p->dist.as<D>();
  a.predrec = p->predrec.as<uint2>();
  a.plan = plan;
  a.ctl = p->ctl.as<Ctl>();
  a.bm_out = p->bm_next.as<uint32_t>();
  a.op = GFB_OP_RELAX_MIN;
  a.lo = p->lo;
  a.hi = p->hi;
  a.rbest = p->rbest.as<unsigned long long>();
  a.rbm = p->rbm.as<uint32_t>();
  k_push_warp<W, 8, 4, true><<<c->num_sms * 4, 256, 0, s>>>(a);
  // remote messages, grouped by owner
  k_rcount<<<p->rtiles, 256, 0, s>>>(p->rbm.as<uint32_t>(), rwords, p->ragg.as<uint32_t>());
  k_rscan<<<1, 1024, 0, s>>>(p->ragg.as<uint32_t>(), p->rtiles, p->rtot.as<uint32_t>());
  k_rwrite<<<p->rtiles, 256, 0, s>>>(p->rbm.as<uint32_t>(), p->rbest.as<unsigned long long>(),
                                     rwords, p->ragg.as<uint32_t>(), static_cast<uint4*>(out), cap);
  // range starts ride in the tail of the counts buffer (no per-call allocation)
  uint32_t* rs = p->counts.as<uint32_t>() + 4096;
  GFB_CUDA(cudaMemcpyAsync(rs, range_starts, (nparts + 1) * 4, cudaMemcpyHostToDevice, s));
  k_owner_counts<<<(nparts + 127) / 128, 128, 0, s>>>(static_cast<uint4*>(out),
                                                      p->rtot.as<uint32_t>(), rs, nparts,
                                                      p->counts.as<uint32_t>());
  GFB_CUDA(cudaGetLastError());
  uint32_t tot = 0;
  GFB_CUDA(cudaMemcpyAsync(&tot, p->rtot.p, 4, cudaMemcpyDeviceToHost, s));
  GFB_CUDA(cudaMemcpyAsync(counts_host, p->counts.p, nparts * 4, cudaMemcpyDeviceToHost, s));
  Ctl h = c->read_ctl(p->ctl.as<Ctl>());
  if (h.err & 1u) fail(GFB_ERANGE, "sssp: u32 distance overflow");
  if (tot > cap) fail(GFB_ERANGE, "part_advance: message buffer too small");
  p->relax = h.relax;
  p->supersteps = h.supersteps;
  return tot;
}

template <class W>
static void part_apply_t(Part* p, const void* in, uint64_t count) {
  Ctx* c = p->ctx;
  if (count)
    k_apply<W><<<std::min<uint64_t>((count + 255) / 256, (uint64_t)c->num_sms * 8), 256, 0,
                 c->stream>>>(static_cast<const uint4*>(in), count, p->lo,
                              p->dist.as<typename DT<W>::D>(), p->bm_next.as<uint32_t>(),
                              p->predrec.as<uint2>());
  GFB_CUDA(cudaGetLastError());
  c->sync();
}

Part* part_create(Ctx* c, uint64_t n_global, uint32_t lo, uint32_t hi, uint64_t m_local,
                  const uint32_t* ro, const uint32_t* col, const void* w, int htype, int wtype) {
  if (wtype == GFB_W_F64) fail(GFB_EINVAL, "partitioned sssp: f32 or u32 arithmetic only");
  if (hi < lo || hi > n_global) fail(GFB_EINVAL, "partitioned sssp: bad vertex range");
  auto p = std::make_unique<Part>();
  p->ctx = c;
  p->n_global = n_global;
  p->lo = lo;
  p->hi = hi;
  p->g.reset(graph_upload(c, hi - lo, m_local, ro, col, w, htype, wtype, 0, n_global));
  cudaStream_t s = c->stream;
  const uint64_t n = hi - lo, nwords = (n + 31) / 32;
  const uint64_t rwords = (n_global + 31) / 32;
  p->dist.alloc(n * 4, s);
  p->predrec.alloc(n * 8, s);
  p->bm_next.alloc(nwords * 4, s);
  p->bm_cur.alloc(nwords * 4, s);
  p->pv.alloc((n + 1) * 4, s);
  p->pstart.alloc((n + 1) * 4, s);
  p->poff.alloc((n + 1) * 4, s);
  p->ptseg.alloc((m_local / PLAN_GRAIN + 3) * 4, s);
  p->ftiles = (uint32_t)std::max<uint64_t>((nwords + F_WORDS - 1) / F_WORDS, 1);
  p->agg.alloc((size_t)p->ftiles * 8, s);
  p->ctl.alloc(sizeof(Ctl), s);
  p->rbest.alloc(n_global * 8, s);
  p->rbm.alloc(rwords * 4, s);
  p->rtiles = (uint32_t)std::max<uint64_t>((rwords + 2047) / 2048, 1);
  p->ragg.alloc((size_t)p->rtiles * 4, s);
  p->rtot.alloc(16, s);
  p->counts.alloc((4096 + 4097) * 4 + 16, s);  // counts | range starts | pending
  return p.release();
}

void part_init(Part* p, uint32_t source) {
  if (source >= p->n_global) fail(GFB_ERANGE, "sssp: source out of range");
  if (p->g->wtype == GFB_W_F32) part_init_t<float>(p, source);
  else part_init_t<uint32_t>(p, source);
}

uint64_t part_advance(Part* p, void* out, uint64_t cap, const uint32_t* range_starts, int nparts,
                      uint32_t* counts_host) {
  if (nparts < 1 || nparts > 4096) fail(GFB_EINVAL, "part_advance: bad part count");
  if (p->g->wtype == GFB_W_F32)
    return part_advance_t<float>(p, out, cap, range_starts, nparts, counts_host);
  return part_advance_t<uint32_t>(p, out, cap, range_starts, nparts, counts_host);
}

void part_apply(Part* p, const void* in, uint64_t count) {
  if (p->g->wtype == GFB_W_F32) part_apply_t<float>(p, in, count);
  else part_apply_t<uint32_t>(p, in, count);
}

uint64_t part_pending(Part* p) {
  Ctx* c = p->ctx;
  const uint32_t nwords = (uint32_t)((p->g->n + 31) / 32);
  unsigned long long* cnt =
      reinterpret_cast<unsigned long long*>(p->counts.as<uint32_t>() + 4096 + 4098);
  GFB_CUDA(cudaMemsetAsync(cnt, 0, 8, c->stream));
  k_count_bits<<<stride_grid(c), 256, 0, c->stream>>>(p->bm_next.as<uint32_t>(), nwords, cnt);
  GFB_CUDA(cudaGetLastError());
  unsigned long long h = 0;
  GFB_CUDA(cudaMemcpyAsync(&h, cnt, 8, cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  return h;
}

// part_pending without the host read: the device counter (for an allreduce)
unsigned long long* part_pending_launch(Part* p) {
  Ctx* c = p->ctx;
  const uint32_t nwords = (uint32_t)((p->g->n + 31) / 32);
  unsigned long long* cnt =
      reinterpret_cast<unsigned long long*>(p->counts.as<uint32_t>() + 4096 + 4098);
  GFB_CUDA(cudaMemsetAsync(cnt, 0, 8, c->stream));
  k_count_bits<<<stride_grid(c), 256, 0, c->stream>>>(p->bm_next.as<uint32_t>(), nwords, cnt);
  GFB_CUDA(cudaGetLastError());
  return cnt;
}

void part_read(Part* p, void* dist_native, uint64_t* relax, uint64_t* supersteps) {
  Ctx* c = p->ctx;
  if (dist_native)
    GFB_CUDA(cudaMemcpyAsync(dist_native, p->dist.p, p->g->n * 4, cudaMemcpyDeviceToHost,
                             c->stream));
  c->sync();
  if (relax) *relax = p->relax;
  if (supersteps) *supersteps = p->supersteps;
}

void part_pred(Part* p, const void* gdist, const uint32_t* res, uint32_t* cand, uint32_t round) {
  Ctx* c = p->ctx;
  Graph* g = p->g.get();
  if (g->wtype == GFB_W_F32)
    k_part_pred<float><<<stride_grid(c), 256, 0, c->stream>>>(
        g->ro.as<uint32_t>(), g->adj.as<EdgeRec<float>>(), (uint32_t)g->n, p->lo,
        static_cast<const float*>(gdist), res, cand, round);
  else
    k_part_pred<uint32_t><<<stride_grid(c), 256, 0, c->stream>>>(
        g->ro.as<uint32_t>(), g->adj.as<EdgeRec<uint32_t>>(), (uint32_t)g->n, p->lo,
        static_cast<const uint32_t*>(gdist), res, cand, round);
  GFB_CUDA(cudaGetLastError());
  c->sync();
}

}  // namespace gfb
