// ops.cu -- operator-level entry points (operators.hpp): push / pull advance
// with a recognised condition, uniquify, and the device frontier type.
// These let the reference's own composition (sssp() as a loop of
// neighbors_expand calls, algorithms.hpp:164-183) run on the device one
// operator call at a time; gfb_sssp (sssp.cu) is the fused fast path.
#include <algorithm>
#include <cmath>

#include "impl.hpp"

namespace gfb {

__global__ void k_set_bits(const uint32_t* list, uint64_t k, uint32_t* bits) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += stride) {
    uint32_t v = list[i];
    atomicOr(bits + (v >> 5), 1u << (v & 31));
  }
}

__global__ void k_popcount(const uint32_t* bits, uint64_t nwords, unsigned long long* out) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint32_t c = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nwords; i += stride)
    c += __popc(bits[i]);
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (unsigned long long)c);
}

__global__ void k_check_range(const uint32_t* list, uint64_t k, uint64_t n,
                              unsigned long long* bad) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += stride)
    if (list[i] >= n) atomicMin(bad, (unsigned long long)i);
}

static void ensure_ctx_ctl(Ctx* c) {
  if (!c->ctl.p) c->ctl.alloc(sizeof(Ctl), c->stream);
}

static uint32_t compact_tiles_for(uint64_t nwords) {
  uint32_t t = (uint32_t)((nwords + C_WORDS - 1) / C_WORDS);
  return t ? t : 1;
}

// Ascending list of the set bits of `bits` into `out` (len returned).
static uint64_t bitmap_to_list(Ctx* c, const uint32_t* bits, uint64_t n, DBuf& out_list,
                               uint64_t* cap) {
  const uint64_t nwords = (n + 31) / 32;
  const uint32_t tiles = compact_tiles_for(nwords);
  ensure_ctx_ctl(c);
  c->ensure_status(tiles + 1);
  cudaStream_t s = c->stream;
  TBuf start, off, tseg;
  if (*cap < n + 1) {
    out_list.alloc((n + 1) * 4, s);
    *cap = n + 1;
  }
  start.alloc((n + 1) * 4, s);
  off.alloc((n + 1) * 4, s);
  tseg.alloc(16, s);
  GFB_CUDA(cudaMemsetAsync(c->ctl.p, 0, sizeof(Ctl), s));
  GFB_CUDA(cudaMemsetAsync(c->status.p, 0, (size_t)(tiles + 1) * 8, s));
  Plan p{out_list.as<uint32_t>(), start.as<uint32_t>(), off.as<uint32_t>(), tseg.as<uint32_t>(), 4};
  k_compact<<<tiles, C_WARPS * 32, 0, s>>>(nullptr, const_cast<uint32_t*>(bits), nullptr,
                                           (uint32_t)nwords, (uint32_t)n, p, c->ctl.as<Ctl>(),
                                           c->status.as<unsigned long long>(), tiles, 0);
  GFB_CUDA(cudaGetLastError());
  return c->read_ctl(c->ctl.as<Ctl>()).k;
}

Frontier* frontier_create(Ctx* c, uint64_t n, int repr) {
  if (repr != GFB_SPARSE && repr != GFB_DENSE) fail(GFB_EINVAL, "frontier: bad representation");
  auto f = std::make_unique<Frontier>();
  f->ctx = c;
  f->n = n;
  f->repr = repr;
  if (repr == GFB_DENSE) {
    f->bits.alloc(f->nwords() * 4, c->stream);
    GFB_CUDA(cudaMemsetAsync(f->bits.p, 0, f->nwords() * 4, c->stream));
    c->sync();
  }
  return f.release();
}

void frontier_assign(Frontier* f, const uint32_t* list, uint64_t k) {
  Ctx* c = f->ctx;
  cudaStream_t s = c->stream;
  TBuf tmp, bad;
  tmp.alloc(k * 4, s);
  bad.alloc(8, s);
  if (k) GFB_CUDA(cudaMemcpyAsync(tmp.p, list, k * 4, cudaMemcpyHostToDevice, s));
  GFB_CUDA(cudaMemsetAsync(bad.p, 0xFF, 8, s));
  if (k) k_check_range<<<stride_grid(c), 256, 0, s>>>(tmp.as<uint32_t>(), k, f->n,
                                                      bad.as<unsigned long long>());
  unsigned long long hb = 0;
  GFB_CUDA(cudaMemcpyAsync(&hb, bad.p, 8, cudaMemcpyDeviceToHost, s));
  c->sync();
  if (hb != ~0ull)  // frontier.hpp:74-76
    fail(GFB_ERANGE, "add_vertex: vertex " + std::to_string(list[hb]) + " out of range");
  if (f->repr == GFB_SPARSE) {
    f->reserve(k);
    if (k) GFB_CUDA(cudaMemcpyAsync(f->list.p, tmp.p, k * 4, cudaMemcpyDeviceToDevice, s));
    f->len = k;
  } else {
    GFB_CUDA(cudaMemsetAsync(f->bits.p, 0, f->nwords() * 4, s));
    if (k) k_set_bits<<<stride_grid(c), 256, 0, s>>>(tmp.as<uint32_t>(), k, f->bits.as<uint32_t>());
    GFB_CUDA(cudaGetLastError());
  }
  c->sync();
}

uint64_t frontier_size(Frontier* f) {
  if (f->repr == GFB_SPARSE) return f->len;
  Ctx* c = f->ctx;
  TBuf cnt;
  cnt.alloc(8, c->stream);
  GFB_CUDA(cudaMemsetAsync(cnt.p, 0, 8, c->stream));
  k_popcount<<<stride_grid(c), 256, 0, c->stream>>>(f->bits.as<uint32_t>(), f->nwords(),
                                                    cnt.as<unsigned long long>());
  GFB_CUDA(cudaGetLastError());
  unsigned long long h = 0;
  GFB_CUDA(cudaMemcpyAsync(&h, cnt.p, 8, cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  return h;
}

void frontier_read(Frontier* f, uint32_t* out, uint64_t cap, uint64_t* k) {
  Ctx* c = f->ctx;
  if (f->repr == GFB_SPARSE) {
    *k = f->len;
    uint64_t cnt = std::min(cap, f->len);
    if (cnt) GFB_CUDA(cudaMemcpyAsync(out, f->list.p, cnt * 4, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    return;
  }
  TBuf lst;
  uint64_t lcap = 0;
  uint64_t len = bitmap_to_list(c, f->bits.as<uint32_t>(), f->n, lst, &lcap);
  *k = len;
  uint64_t cnt = std::min(cap, len);
  if (cnt) GFB_CUDA(cudaMemcpyAsync(out, lst.p, cnt * 4, cudaMemcpyDeviceToHost, c->stream));
  c->sync();
}

// ---------------------------------------------------------------------------
// Operator calls
// ---------------------------------------------------------------------------
struct OpPlan {
  TBuf v, start, off, tseg;
};

// Plan of the input frontier (vertices with out-degree > 0, order kept).
static Ctl build_plan(Ctx* c, const Graph* g, Frontier* in, OpPlan& p) {
  cudaStream_t s = c->stream;
  ensure_ctx_ctl(c);
  uint64_t len = in->repr == GFB_SPARSE ? in->len : g->n;
  p.v.alloc((len + 1) * 4, s);
  p.start.alloc((len + 1) * 4, s);
  p.off.alloc((len + 1) * 4, s);
  // tile map size bound: total edges <= len * max_deg; computed after the
  // plan in a second pass when larger than the first guess.
  uint64_t guess = std::max<uint64_t>(g->m / PLAN_GRAIN + 3, 16);
  p.tseg.alloc(guess * 4, s);
  for (int attempt = 0; attempt < 2; ++attempt) {
    GFB_CUDA(cudaMemsetAsync(c->ctl.p, 0, sizeof(Ctl), s));
    Plan pl{p.v.as<uint32_t>(), p.start.as<uint32_t>(), p.off.as<uint32_t>(), p.tseg.as<uint32_t>(),
            (uint32_t)guess};
    uint32_t tiles;
    if (in->repr == GFB_SPARSE) {
      tiles = (uint32_t)std::max<uint64_t>((len + C_VERTS - 1) / C_VERTS, 1);
      c->ensure_status(tiles + 1);
      GFB_CUDA(cudaMemsetAsync(c->status.p, 0, (size_t)(tiles + 1) * 8, s));
      k_plan_list<<<tiles, C_WARPS * 32, 0, s>>>(g->ro.as<uint32_t>(), in->list.as<uint32_t>(),
                                                 (uint32_t)len, pl, c->ctl.as<Ctl>(),
                                                 c->status.as<unsigned long long>(), tiles);
    } else {
      tiles = compact_tiles_for(in->nwords());
      c->ensure_status(tiles + 1);
      GFB_CUDA(cudaMemsetAsync(c->status.p, 0, (size_t)(tiles + 1) * 8, s));
      k_compact<<<tiles, C_WARPS * 32, 0, s>>>(g->ro.as<uint32_t>(), in->bits.as<uint32_t>(),
                                               nullptr, (uint32_t)in->nwords(), (uint32_t)g->n,
                                               pl, c->ctl.as<Ctl>(),
                                               c->status.as<unsigned long long>(), tiles, 0);
    }
    GFB_CUDA(cudaGetLastError());
    Ctl h = c->read_ctl(c->ctl.as<Ctl>());
    uint64_t need = (uint64_t)h.total / PLAN_GRAIN + 3;
    if (need <= guess) return h;
    guess = need;
    p.tseg.alloc(guess * 4, s);
  }
  return c->read_ctl(c->ctl.as<Ctl>());
}

static void check_op(const Graph* g, Frontier* in, Frontier* out, int op, void* state) {
  if (!g || !in || !out) fail(GFB_EINVAL, "advance: null handle");
  if (in->n != g->n || out->n != g->n) fail(GFB_EINVAL, "advance: frontier size != num_vertices");
  if (op < GFB_OP_RELAX_MIN || op > GFB_OP_ALWAYS) fail(GFB_EINVAL, "advance: unknown condition");
  if (op == GFB_OP_RELAX_MIN) {
    auto* d = static_cast<Dist*>(state);
    if (!d || d->g != g) fail(GFB_EINVAL, "advance: relax_min needs the graph's distance map");
  }
  if (op == GFB_OP_RECORD && !state) fail(GFB_EINVAL, "advance: record needs a recorder");
}

template <class W>
static void fill_state(AdvArgs<W>& a, int op, void* state) {
  a.op = op;
  if (op == GFB_OP_RELAX_MIN) {
    auto* d = static_cast<Dist*>(state);
    a.dist = d->dist.as<typename DT<W>::D>();
    a.predrec = d->predrec.as<uint2>();
  } else if (op == GFB_OP_RECORD) {
    auto* r = static_cast<Record*>(state);
    a.rec_src = r->src.as<uint32_t>();
    a.rec_dst = r->dst.as<uint32_t>();
    a.rec_eid = r->eid.as<uint32_t>();
    a.rec_cap = r->cap;
  }
}

// Recorders append across calls: seed the device counter with the count so far.
static void seed_record(Ctx* c, int op, void* state) {
  if (op != GFB_OP_RECORD) return;
  auto* r = static_cast<Record*>(state);
  uint32_t base = (uint32_t)std::min<uint64_t>(r->count, 0xFFFFFFFFu);
  GFB_CUDA(cudaMemcpyAsync(&c->ctl.as<Ctl>()->rec_count, &base, 4, cudaMemcpyHostToDevice,
                           c->stream));
  c->sync();
}

static void finish_state(Ctx* c, int op, void* state, uint64_t relax) {
  Ctl h = c->read_ctl(c->ctl.as<Ctl>());
  if (op == GFB_OP_RELAX_MIN) {
    if (h.err & 1u) fail(GFB_ERANGE, "advance: u32 distance overflow");
    static_cast<Dist*>(state)->relax += relax ? relax : h.relax;
  } else if (op == GFB_OP_RECORD) {
    static_cast<Record*>(state)->count = h.rec_count;
  }
}

template <class W>
static void push_impl(Ctx* c, const Graph* g, Frontier* in, Frontier* out, int op, void* state) {
  cudaStream_t s = c->stream;
  OpPlan p;
  Ctl h = build_plan(c, g, in, p);
  // prepare output
  if (out->repr == GFB_SPARSE) {
    out->reserve(std::max<uint64_t>(h.total, 1));
    out->len = 0;
  } else {
    GFB_CUDA(cudaMemsetAsync(out->bits.p, 0, out->nwords() * 4, s));
  }
  if (h.total == 0) {
    c->sync();
    return;
  }
  uint32_t ntiles = (h.total + A_TILE - 1) / A_TILE;
  c->ensure_status(ntiles + 1);
  GFB_CUDA(cudaMemsetAsync(c->qstatus.p, 0, (size_t)(ntiles + 1) * 8, s));
  AdvArgs<W> a{};
  a.adj = g->adj.as<EdgeRec<W>>();
  a.ceid = g->ceid.as<uint32_t>();
  a.plan = Plan{p.v.as<uint32_t>(), p.start.as<uint32_t>(), p.off.as<uint32_t>(), p.tseg.as<uint32_t>(),
                (uint32_t)(p.tseg.bytes / 4)};
  a.ctl = c->ctl.as<Ctl>();
  a.bm_out = out->repr == GFB_DENSE ? out->bits.as<uint32_t>() : nullptr;
  a.q_out = out->repr == GFB_SPARSE ? out->list.as<uint32_t>() : nullptr;
  a.status = c->status.as<unsigned long long>();
  a.status_len = 0;
  a.qstatus = c->qstatus.as<unsigned long long>();
  fill_state<W>(a, op, state);
  seed_record(c, op, state);
  uint32_t grid = std::min<uint32_t>(ntiles, c->num_sms * 8);
  if (out->repr == GFB_SPARSE)
    k_advance_push<W, OUT_QUEUE><<<grid, A_BLOCK, 0, s>>>(a);
  else
    k_advance_push<W, OUT_BITMAP><<<grid, A_BLOCK, 0, s>>>(a);
  GFB_CUDA(cudaGetLastError());
  finish_state(c, op, state, h.total);
  if (out->repr == GFB_SPARSE) out->len = c->read_ctl(c->ctl.as<Ctl>()).out_count;
}

template <class W>
static void pull_impl(Ctx* c, const Graph* g, Frontier* in, Frontier* out, int op, void* state) {
  cudaStream_t s = c->stream;
  ensure_ctx_ctl(c);
  GFB_CUDA(cudaMemsetAsync(c->ctl.p, 0, sizeof(Ctl), s));
  GFB_CUDA(cudaMemsetAsync(out->bits.p, 0, out->nwords() * 4, s));
  if (g->pull_total == 0) {
    c->sync();
    return;
  }
  AdvArgs<W> a{};
  a.adj = g->cadj.as<EdgeRec<W>>();
  a.ceid = g->ceid.as<uint32_t>();
  a.plan = Plan{g->pull_v.as<uint32_t>(), g->pull_off.as<uint32_t>(), g->pull_off.as<uint32_t>(),
                g->pull_tseg.as<uint32_t>(), (uint32_t)(g->pull_tseg.bytes / 4)};
  a.ctl = c->ctl.as<Ctl>();
  a.bm_out = out->bits.as<uint32_t>();
  a.bm_in = in->bits.as<uint32_t>();
  a.status = nullptr;
  a.status_len = 0;
  fill_state<W>(a, op, state);
  seed_record(c, op, state);
  uint32_t ntiles = (g->pull_total + A_TILE - 1) / A_TILE;
  uint32_t grid = std::min<uint32_t>(ntiles, c->num_sms * 8);
  k_advance_pull<W><<<grid, A_BLOCK, 0, s>>>(a, g->pull_total, g->pull_k);
  GFB_CUDA(cudaGetLastError());
  finish_state(c, op, state, 0);
}

void advance_push(Ctx* c, const Graph* g, Frontier* in, Frontier* out, int op, void* state) {
  check_op(g, in, out, op, state);
  if (g->wtype == GFB_W_F32) push_impl<float>(c, g, in, out, op, state);
  else if (g->wtype == GFB_W_F64) push_impl<double>(c, g, in, out, op, state);
  else push_impl<uint32_t>(c, g, in, out, op, state);
}

void advance_pull(Ctx* c, const Graph* g, Frontier* in, Frontier* out, int op, void* state) {
  check_op(g, in, out, op, state);
  if (!g->csc_wanted)  // operators.hpp:79-80
    fail(GFB_EINVAL, "neighbors_expand_pull: transpose not built");
  if (in->repr != GFB_DENSE || out->repr != GFB_DENSE)  // operators.hpp:81-82
    fail(GFB_EINVAL, "neighbors_expand_pull: dense frontier required");
  ensure_csc(const_cast<Graph*>(g));
  if (op == GFB_OP_RECORD) ensure_ceid(const_cast<Graph*>(g));  // CSR ids of CSC slots
  if (g->wtype == GFB_W_F32) pull_impl<float>(c, g, in, out, op, state);
  else if (g->wtype == GFB_W_F64) pull_impl<double>(c, g, in, out, op, state);
  else pull_impl<uint32_t>(c, g, in, out, op, state);
}

// uniquify (operators.hpp:191-200): bitmap dedup + warp-ballot compaction.
void filter_unique(Ctx* c, Frontier* in, Frontier* out) {
  if (in->repr != GFB_SPARSE || out->repr != GFB_SPARSE)
    fail(GFB_EINVAL, "uniquify: sparse frontier required");
  if (in->n != out->n) fail(GFB_EINVAL, "uniquify: frontier sizes differ");
  cudaStream_t s = c->stream;
  const uint64_t nwords = in->nwords();
  TBuf bits;
  bits.alloc(nwords * 4, s);
  GFB_CUDA(cudaMemsetAsync(bits.p, 0, nwords * 4, s));
  if (in->len)
    k_set_bits<<<stride_grid(c), 256, 0, s>>>(in->list.as<uint32_t>(), in->len, bits.as<uint32_t>());
  GFB_CUDA(cudaGetLastError());
  TBuf lst;
  uint64_t lcap = 0;
  uint64_t len = bitmap_to_list(c, bits.as<uint32_t>(), in->n, lst, &lcap);
  out->reserve(std::max<uint64_t>(len, 1));
  if (len) GFB_CUDA(cudaMemcpyAsync(out->list.p, lst.p, len * 4, cudaMemcpyDeviceToDevice, s));
  out->len = len;
  c->sync();
}

// ---------------------------------------------------------------------------
// filter (operators.hpp:163-188): keep exactly the frontier elements whose
// predicate holds, same representation; a sparse frontier keeps its order and
// duplicates (the reference's sequential order, :184-186).  Host predicates
// cannot cross the ABI: the recognised ones compare a device distance map
// with a threshold in the reference's double domain (every device arithmetic
// widens exactly) -- the near-far split of the SSSP loop (nearfar.cuh).
// Sparse: count per 2048-element tile -> one-CTA exclusive scan -> ordered
// write (warp ballots); dense: one pass over the bitmap words.
// ---------------------------------------------------------------------------
constexpr int FL_THREADS = 256, FL_VT = 8, FL_TILE = FL_THREADS * FL_VT;

template <class D>
__device__ __forceinline__ bool filter_pred(const D* dist, uint32_t v, int pred, double thr) {
  const D x = dist[v];  // widened exactly; the device's "unreachable" is +inf
  const double d = x == dinf<D>() ? __longlong_as_double(0x7FF0000000000000ll) : (double)x;
  if (pred == GFB_PRED_DIST_BELOW) return d < thr;
  if (pred == GFB_PRED_DIST_AT_LEAST) return d >= thr;
  return !isinf(d);  // GFB_PRED_REACHED (dist < +inf)
}

template <class D>
__global__ void __launch_bounds__(FL_THREADS)
k_filter_count(const uint32_t* __restrict__ list, uint64_t k, const D* __restrict__ dist, int pred,
               double thr, uint32_t* cnt) {
  __shared__ uint32_t s_w[FL_THREADS / 32];
  const uint64_t base = (uint64_t)blockIdx.x * FL_TILE;
  uint32_t c = 0;
#pragma unroll
  for (int r = 0; r < FL_VT; ++r) {
    const uint64_t i = base + r * FL_THREADS + threadIdx.x;
    if (i < k && filter_pred(dist, list[i], pred, thr)) ++c;
  }
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < FL_THREADS / 32; ++w) t += s_w[w];
    cnt[blockIdx.x] = t;
  }
}

// one CTA: exclusive scan of the tile counts in place; total -> cnt[tiles]
__global__ void __launch_bounds__(1024) k_filter_scan(uint32_t* cnt, uint32_t tiles) {
  __shared__ uint32_t s_w[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t carry = 0;
  for (uint32_t i0 = 0; i0 < tiles; i0 += 1024) {
    const uint32_t i = i0 + tid;
    const uint32_t x = i < tiles ? cnt[i] : 0u;
    const uint32_t incl = warp_incl_scan(x, lane);
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    if (warp == 0) s_w[lane] = warp_incl_scan(s_w[lane], lane);
    __syncthreads();
    const uint32_t pre = carry + (warp ? s_w[warp - 1] : 0u) + incl - x;
    if (i < tiles) cnt[i] = pre;
    carry += s_w[31];
    __syncthreads();
  }
  if (tid == 0) cnt[tiles] = carry;
}

template <class D>
__global__ void __launch_bounds__(FL_THREADS)
k_filter_write(const uint32_t* __restrict__ list, uint64_t k, const D* __restrict__ dist, int pred,
               double thr, const uint32_t* __restrict__ off, uint32_t* out) {
  __shared__ uint32_t s_w[FL_THREADS / 32];
  __shared__ uint32_t s_run;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t base = (uint64_t)blockIdx.x * FL_TILE;
  if (threadIdx.x == 0) s_run = off[blockIdx.x];
  __syncthreads();
  for (int r = 0; r < FL_VT; ++r) {  // rows of FL_THREADS consecutive elements, in order
    const uint64_t i = base + r * FL_THREADS + threadIdx.x;
    const uint32_t v = i < k ? list[i] : 0u;
    const bool keep = i < k && filter_pred(dist, v, pred, thr);
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) s_w[warp] = __popc(bal);
    __syncthreads();
    uint32_t pre = s_run;
    for (int w = 0; w < warp; ++w) pre += s_w[w];
    if (keep) out[pre + __popc(bal & lanemask_lt())] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t t = 0;
      for (int w = 0; w < FL_THREADS / 32; ++w) t += s_w[w];
      s_run += t;
    }
    __syncthreads();
  }
}

template <class D>
__global__ void k_filter_bits(const uint32_t* __restrict__ in, uint64_t nwords, uint64_t n,
                              const D* __restrict__ dist, int pred, double thr, uint32_t* out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t wi = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; wi < nwords; wi += stride) {
    uint32_t word = in[wi], keep = 0;
    while (word) {
      const int b = __ffs(word) - 1;
      word &= word - 1;
      const uint64_t v = wi * 32 + b;
      if (v < n && filter_pred(dist, (uint32_t)v, pred, thr)) keep |= 1u << b;
    }
    out[wi] = keep;
  }
}

template <class D>
static void filter_impl(Ctx* c, Frontier* in, Frontier* out, int pred, const D* dist, double thr) {
  cudaStream_t s = c->stream;
  if (in->repr == GFB_DENSE) {
    k_filter_bits<D><<<stride_grid(c), 256, 0, s>>>(in->bits.as<uint32_t>(), in->nwords(), in->n,
                                                    dist, pred, thr, out->bits.as<uint32_t>());
    GFB_CUDA(cudaGetLastError());
    c->sync();
    return;
  }
  const uint64_t k = in->len;
  if (k == 0) {
    out->len = 0;
    return;
  }
  const uint32_t tiles = (uint32_t)((k + FL_TILE - 1) / FL_TILE);
  TBuf cnt;
  cnt.alloc((size_t)(tiles + 1) * 4, s);
  k_filter_count<D><<<tiles, FL_THREADS, 0, s>>>(in->list.as<uint32_t>(), k, dist, pred, thr,
                                                 cnt.as<uint32_t>());
  k_filter_scan<<<1, 1024, 0, s>>>(cnt.as<uint32_t>(), tiles);
  uint32_t total = 0;
  GFB_CUDA(cudaMemcpyAsync(&total, cnt.as<uint32_t>() + tiles, 4, cudaMemcpyDeviceToHost, s));
  c->sync();
  out->reserve(std::max<uint64_t>(total, 1));
  k_filter_write<D><<<tiles, FL_THREADS, 0, s>>>(in->list.as<uint32_t>(), k, dist, pred, thr,
                                                 cnt.as<uint32_t>(), out->list.as<uint32_t>());
  GFB_CUDA(cudaGetLastError());
  out->len = total;
  c->sync();
}

void filter(Ctx* c, Frontier* in, Frontier* out, int pred, const Dist* d, double thr) {
  if (pred < GFB_PRED_DIST_BELOW || pred > GFB_PRED_REACHED)
    fail(GFB_EINVAL, "filter: unrecognised predicate (device policy: dist_below, "
                     "dist_at_least, reached)");
  if (!d) fail(GFB_EINVAL, "filter: the distance predicates need a distance map");
  if (in->repr != out->repr) fail(GFB_EINVAL, "filter: output representation must match input");
  if (in->n != out->n || in->n != d->g->n) fail(GFB_EINVAL, "filter: vertex counts differ");
  if (std::isnan(thr)) fail(GFB_EINVAL, "filter: threshold is NaN");
  const int wt = d->g->wtype;
  if (wt == GFB_W_F32) filter_impl<float>(c, in, out, pred, d->dist.as<float>(), thr);
  else if (wt == GFB_W_F64) filter_impl<double>(c, in, out, pred, d->dist.as<double>(), thr);
  else filter_impl<uint32_t>(c, in, out, pred, d->dist.as<uint32_t>(), thr);
}

// ---------------------------------------------------------------------------
template <class W>
__global__ void k_dist_init(typename DT<W>::D* dist, uint2* predrec, uint32_t n, uint32_t source) {
  uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    dist[i] = i == source ? typename DT<W>::D(0) : dinf<W>();
    predrec[i] = make_uint2(NIL, NIL);
  }
}

Dist* dist_create(Ctx* c, const Graph* g) {
  auto d = std::make_unique<Dist>();
  d->ctx = c;
  d->g = g;
  d->dist.alloc(g->n * (g->wtype == GFB_W_F64 ? 8 : 4), c->stream);
  d->predrec.alloc(g->n * 8, c->stream);
  return d.release();
}

void dist_init(Dist* d, uint32_t source) {
  const Graph* g = d->g;
  if (source >= g->n) fail(GFB_ERANGE, "sssp: source out of range");
  Ctx* c = d->ctx;
  uint32_t n = (uint32_t)g->n;
  if (g->wtype == GFB_W_F32) k_dist_init<float><<<stride_grid(c), 256, 0, c->stream>>>(d->dist.as<float>(), d->predrec.as<uint2>(), n, source);
  else if (g->wtype == GFB_W_F64) k_dist_init<double><<<stride_grid(c), 256, 0, c->stream>>>(d->dist.as<double>(), d->predrec.as<uint2>(), n, source);
  else k_dist_init<uint32_t><<<stride_grid(c), 256, 0, c->stream>>>(d->dist.as<uint32_t>(), d->predrec.as<uint2>(), n, source);
  GFB_CUDA(cudaGetLastError());
  d->relax = 0;
  c->sync();
}

template <class W>
__global__ void k_widen2(const typename DT<W>::D* d, double* out, uint32_t n) {
  uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    typename DT<W>::D x = d[i];
    out[i] = x == dinf<W>() ? __longlong_as_double(0x7FF0000000000000ll) : (double)x;
  }
}

void dist_read(Dist* d, double* out, uint64_t* relax) {
  Ctx* c = d->ctx;
  const Graph* g = d->g;
  uint32_t n = (uint32_t)g->n;
  if (out) {
    TBuf tmp;
    tmp.alloc((size_t)n * 8, c->stream);
    if (g->wtype == GFB_W_F32) k_widen2<float><<<stride_grid(c), 256, 0, c->stream>>>(d->dist.as<float>(), tmp.as<double>(), n);
    else if (g->wtype == GFB_W_F64) k_widen2<double><<<stride_grid(c), 256, 0, c->stream>>>(d->dist.as<double>(), tmp.as<double>(), n);
    else k_widen2<uint32_t><<<stride_grid(c), 256, 0, c->stream>>>(d->dist.as<uint32_t>(), tmp.as<double>(), n);
    GFB_CUDA(cudaGetLastError());
    GFB_CUDA(cudaMemcpyAsync(out, tmp.p, (size_t)n * 8, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
  }
  if (relax) *relax = d->relax;
}

Record* record_create(Ctx* c, uint64_t cap) {
  auto r = std::make_unique<Record>();
  r->ctx = c;
  r->cap = cap;
  r->src.alloc(cap * 4, c->stream);
  r->dst.alloc(cap * 4, c->stream);
  r->eid.alloc(cap * 4, c->stream);
  return r.release();
}

void record_read(Record* r, uint32_t* s, uint32_t* d, uint32_t* e, uint64_t cap, uint64_t* count) {
  Ctx* c = r->ctx;
  *count = r->count;
  uint64_t k = std::min(std::min(cap, r->count), r->cap);
  if (k) {
    if (s) GFB_CUDA(cudaMemcpyAsync(s, r->src.p, k * 4, cudaMemcpyDeviceToHost, c->stream));
    if (d) GFB_CUDA(cudaMemcpyAsync(d, r->dst.p, k * 4, cudaMemcpyDeviceToHost, c->stream));
    if (e) GFB_CUDA(cudaMemcpyAsync(e, r->eid.p, k * 4, cudaMemcpyDeviceToHost, c->stream));
  }
  c->sync();
}

}  // namespace gfb
